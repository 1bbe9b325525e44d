timeout 600 python -m pytest tests/test_gpu_blocks.py -x -q -k "conv" 2>&1 | tail -3
python tools/conv_layer_bench.py --passes f,d
CK_TC_SHIFT=0 python tools/conv_layer_bench.py --passes f,d
