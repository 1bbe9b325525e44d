# A/B the LRN backward prefetch distance / occupancy (run via gpurun)
for v in "8 5" "4 6" "4 7" "2 8"; do
  set -- $v
  touch paper_1412_4564_b200/csrc/kernels.cu
  CK_EXTRA_NVCC="-DCK_LRN_BWD_P=$1 -DCK_LRN_GRID_MINB=$2" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo build-fail
  echo "P=$1 minB=$2"
  python bench.py --profile-layers --steps 20 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep -E "norm|conv1 |conv2 "
  python bench.py --steps 30 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | cut -c1-140
done
