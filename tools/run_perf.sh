timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for bn in 0 256 0 256; do echo "== WBN=$bn"; CK_TC_WBN=$bn python tools/gemm_exp.py 2>&1 | grep "conv1\|conv2" | sed 's/fprop.*wgrad/wgrad/; s/dgrad.*//'; done
python bench.py --steps 50 --no-e2e --no-cpu-baseline 2>/dev/null | cut -c1-130
