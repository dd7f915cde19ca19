# Quick GPU check: non-slow parity tests, smoke, short C4 bench.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/tests_fast.txt 2>&1; tail -5 gpurun_out/tests_fast.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-variants > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -3 gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
