timeout 600 python -m pytest tests/test_gpu_blocks.py -x -q 2>&1 | tail -5
python tools/conv_layer_bench.py
