#!/bin/bash
# full ncu captures of the fc6 GEMM launches (fprop, dgrad, wgrad) of tools/conv_layer_bench.py
python tools/conv_layer_bench.py --layers fc6 --reps 1 > gpurun_out/fc6_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"tc_gemm|splitk" -s 6 -c 6 -o gpurun_out/fc6_full -f \
  python tools/conv_layer_bench.py --layers fc6 --reps 1 > gpurun_out/ncu_fc6.log 2>&1
echo done
