# Packed-key pass: parity tests, then C4 bench with and without it (VD_NO_PACK=1).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/tests_fast.txt 2>&1; tail -5 gpurun_out/tests_fast.txt
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-variants --no-exact-sample > gpurun_out/bench_pack.json 2> gpurun_out/bench_pack.err; tail -3 gpurun_out/bench_pack.err; cat gpurun_out/bench_pack.json
VD_NO_PACK=1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-variants --no-exact-sample > gpurun_out/bench_nopack.json 2> gpurun_out/bench_nopack.err; tail -3 gpurun_out/bench_nopack.err; cat gpurun_out/bench_nopack.json
