python tools/block_bench.py
python tools/block_bench.py --only "pool1 bwd" --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:pool_bwd -s 2 -c 1 -o gpurun_out/pool1_bwd_full -f python tools/block_bench.py --only "pool1 bwd" --reps 1 > gpurun_out/ncu_pool.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:lrn_bwd -s 2 -c 1 -o gpurun_out/norm1_bwd_full -f python tools/block_bench.py --only "norm1 bwd" --reps 1 > gpurun_out/ncu_lrn.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/fc6_wgrad_full -f python tools/conv_layer_bench.py --layers fc6 --passes w --reps 1 > gpurun_out/ncu_fc6.log 2>&1
echo done
