# scratch driver for gpurun experiments (edit freely): GPU tests, bench line, per-layer times
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py 2>/dev/null | tail -1 | cut -c1-250
python bench.py --profile-layers --steps 20 2>&1 | grep -v "^{" | head -50
