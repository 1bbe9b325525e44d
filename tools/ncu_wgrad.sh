#!/bin/bash
# Launch list + one full capture of the conv3/conv1 wgrad pass (run via gpurun).
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed
for L in conv3 conv1; do
python tools/conv_layer_bench.py --layers $L --passes w --reps 1 > gpurun_out/w_$L.txt 2>&1 && \
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/w_${L}_launches.csv python tools/conv_layer_bench.py --layers $L --passes w --reps 1 > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 3 -c 1 -o gpurun_out/conv3_wgrad_full -f python tools/conv_layer_bench.py --layers conv3 --passes w --reps 1 > gpurun_out/ncu_full.log 2>&1
echo done
