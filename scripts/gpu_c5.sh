# Large-grid check: parity of the windowed / generic kernels, C5 per-launch list, C5 bench.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/tests_fast.txt 2>&1; tail -3 gpurun_out/tests_fast.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -k "windowed or large_grid or large_n" -q -p no:cacheprovider > gpurun_out/tests_rel.txt 2>&1; tail -5 gpurun_out/tests_rel.txt
VD_CFG=C5 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python scripts/jfa_passes.py > gpurun_out/c5_launches.log 2>&1
timeout 900 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline --no-exact-sample --no-variants --e2e-steps 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -3 gpurun_out/bench_c5.err; cat gpurun_out/bench_c5.json
