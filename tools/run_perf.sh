python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-200
python bench.py --profile-layers --steps 20 2> gpurun_out/layers.txt > /dev/null
