timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-200
python bench.py --profile-layers --steps 5 2>&1 | grep -v "^{" | head -40 | grep "conv\|gemm"
