mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-variants --no-exact-sample > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -2 gpurun_out/bench_q.err; cat gpurun_out/bench_q.json
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-exact-sample --no-variants --e2e-steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -3 gpurun_out/bench_c5.err; cat gpurun_out/bench_c5.json
