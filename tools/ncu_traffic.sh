#!/bin/bash
# dram traffic per launch of a conv GEMM (run via gpurun): $1 layer, $2 pass (f/d/w)
L=${1:-conv2}; P=${2:-w}
python tools/conv_layer_bench.py --layers $L --passes $P --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/${L}_${P}_full -f \
  python tools/conv_layer_bench.py --layers $L --passes $P --reps 1 > gpurun_out/ncu_${L}_${P}.log 2>&1
echo done
