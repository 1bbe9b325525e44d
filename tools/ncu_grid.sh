# full ncu captures of the grid transforms inside one bench step (run via gpurun)
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:to_grid_pm -s 7 -c 7 -o gpurun_out/grid_full -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ncu_grid.log 2>&1
echo done
