python bench.py --profile-layers --steps 20 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep -E "^  conv[2-5]"
python bench.py --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | cut -c1-120
