# Windowed (REL) fast path check: parity at N > 32768, then C5 and C4 bench lines.
set -x
mkdir -p gpurun_out
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -k "windowed or large_grid or large_n" -x -q -p no:cacheprovider > gpurun_out/tests_rel.txt 2>&1; tail -15 gpurun_out/tests_rel.txt
timeout 900 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline --no-exact-sample --no-variants --e2e-steps 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -3 gpurun_out/bench_c5.err; cat gpurun_out/bench_c5.json
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/tests_fast.txt 2>&1; tail -3 gpurun_out/tests_fast.txt
