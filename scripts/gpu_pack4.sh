python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q -p no:cacheprovider -k "packed or shard or peer or variant or manhattan or djfa or stf" 2>&1 | tail -3
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-exact-sample > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -2 gpurun_out/bench_q.err; python -c "
import json; b=json.load(open('gpurun_out/bench_q.json')); print(b['value'], b['roofline']['avg_launch_ms'], b['djfam'], b['jfa']['value'])"
