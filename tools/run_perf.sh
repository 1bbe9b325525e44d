timeout 300 python -m pytest tests/test_gpu_blocks.py -x -q -k "conv" 2>&1 | tail -2
python tools/conv_layer_bench.py --passes w
CK_TC_WGRID=0 python tools/conv_layer_bench.py --passes w
