#!/bin/bash
M=gpu__time_duration.sum
for L in fc6 conv1 conv2; do
python tools/conv_layer_bench.py --layers $L --reps 1 > /dev/null 2>&1 && \
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/l_${L}_launches.csv python tools/conv_layer_bench.py --layers $L --reps 1 > /dev/null 2>&1
done
echo done
