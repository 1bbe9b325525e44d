M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed
python tools/conv_layer_bench.py --layers conv2 --passes w --reps 1 > /dev/null && ncu --metrics $M --clock-control none --csv --log-file gpurun_out/w_launches.csv python tools/conv_layer_bench.py --layers conv2 --passes w --reps 1 > /dev/null 2>&1
python tools/conv_layer_bench.py --layers conv3 --passes f --reps 1 > /dev/null && ncu --metrics $M --clock-control none --csv --log-file gpurun_out/f3_launches.csv python tools/conv_layer_bench.py --layers conv3 --passes f --reps 1 > /dev/null 2>&1
echo done
