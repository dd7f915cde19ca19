mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q -p no:cacheprovider -k "packed or shard or peer or djfa" > gpurun_out/tests_pack2.txt 2>&1; tail -3 gpurun_out/tests_pack2.txt
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-variants --no-exact-sample > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -2 gpurun_out/bench_q.err; cat gpurun_out/bench_q.json
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python scripts/profile_pass.py > /dev/null 2>&1; python scripts/summarize_launches.py gpurun_out/launches_q.csv
