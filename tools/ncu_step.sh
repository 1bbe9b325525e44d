# per-kernel time + DRAM/L2/SM utilisation for one training step of the bench
M=gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/plain.log 2>&1 && \
ncu --metrics $M --clock-control none -c 1500 --csv --log-file gpurun_out/step_kernels.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ncu_step.log 2>&1
echo done
