timeout 300 python -m pytest tests/test_gpu_blocks.py -x -q -k "conv" 2>&1 | tail -1
python tools/conv_layer_bench.py --passes w
CK_TC_WKS=32 python tools/conv_layer_bench.py --passes w --layers conv1,conv2,conv3
