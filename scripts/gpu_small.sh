set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for c in C2 C3; do
timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --no-variants > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; cat gpurun_out/bench_$c.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d['jfa']['value'], d['e2e']['value'], d['roofline']['avg_launch_ms'], d['gpu_launches'])"
done
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-variants > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print('C4', d['value'], d['e2e'])"
