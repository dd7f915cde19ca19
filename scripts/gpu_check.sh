set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -15
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python bench.py --steps 50 --warmup 5 --cpu-seconds 10 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
