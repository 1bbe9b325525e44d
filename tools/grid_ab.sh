# A/B of the grid transform's channel tiles per block (run via gpurun)
for t in 1 0; do
  echo "CK_GRID_TPB=$t"
  CK_GRID_TPB=$t python bench.py --profile-layers --steps 20 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep -E "^  conv[2-5]"
  CK_GRID_TPB=$t python bench.py --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | cut -c1-120
done
