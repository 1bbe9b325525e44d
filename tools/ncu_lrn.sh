# full ncu captures of the LRN kernels inside one bench step (run via gpurun)
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:lrn_ -s 4 -c 4 -o gpurun_out/lrn_full -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ncu_lrn.log 2>&1
echo done
