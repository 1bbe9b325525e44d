#!/bin/bash
# Round-end ncu --set full captures (run via gpurun): the dominant GEMMs (conv2
# dgrad / wgrad through tools/conv_layer_bench.py) and the memory-bound kernels
# of one AlexNet training step (the second step's 10 LRN / pool launches).
O=gpurun_out/ncu_round; mkdir -p $O
for P in d w; do
  python tools/conv_layer_bench.py --layers conv2 --passes $P --reps 1 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 2 -c 1 -o $O/conv2_$P -f \
    python tools/conv_layer_bench.py --layers conv2 --passes $P --reps 1 > $O/conv2_$P.log 2>&1
done
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1 && \
ncu --set full --clock-control none -k regex:"lrn_|pool_max" -s 10 -c 10 -o $O/mem -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > $O/mem.log 2>&1
for r in conv2_d conv2_w mem; do
  ncu -i $O/$r.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread > $O/$r.csv 2>&1
done
echo done
