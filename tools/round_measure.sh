#!/bin/bash
# One measurement pass (run via gpurun): bench lines for every BASELINE config,
# per-layer profiles, the reference arm, and the ncu launch list of one step.
# Usage: tools/round_measure.sh TAG
T=${1:-v3}; O=gpurun_out/$T; mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --profile-layers --steps 20 --no-cpu-baseline --no-e2e 2> $O/layers.txt > /dev/null
for n in vgg16bn cifar lenet; do
  python bench.py --net $n > $O/bench_$n.json 2> $O/bench_$n.err
  python bench.py --net $n --profile-layers --steps 10 --no-cpu-baseline --no-e2e 2> $O/layers_$n.txt > /dev/null
done
python bench.py --math fp32 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_fp32.json 2> $O/bench_fp32.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
M=gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none -c 1500 --csv --log-file $O/step_kernels.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > $O/ncu_step.log 2>&1
python tools/show_step.py $O/step_kernels.csv 45 > $O/step_summary.txt
python tools/step_order.py $O/step_kernels.csv > $O/step_order.txt
for f in $O/bench*.json; do echo "$f $(python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d.get('value'),d.get('ms_per_step'),d.get('unit'))")"; done
