python -m pytest tests/test_gpu_blocks.py -x -q -k "conv" 2>&1 | tail -3
python tools/conv_layer_bench.py
python tools/gemm_probe.py
