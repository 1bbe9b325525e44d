timeout 600 python -m pytest tests/test_gpu_blocks.py -x -q 2>&1 | tail -5
python tools/block_bench.py
python bench.py --profile-layers --no-cpu-baseline > gpurun_out/bench14.json 2> gpurun_out/bench14.err; cat gpurun_out/bench14.json gpurun_out/bench14.err
