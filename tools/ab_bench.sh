# A/B: $1 = env assignment for the B arm (e.g. CK_NO_PREPACK=1)
for e in "$1" "CK_AB_NONE=1"; do
  echo "$e"
  env $e python bench.py --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | cut -c1-120
done
env "$1" python bench.py --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | cut -c1-120
python bench.py --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | cut -c1-120
