# quick iteration: parity tests, kernel timings (ncu launch list), bench
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -iE "error" | head
timeout 600 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -4
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_iter.csv python scripts/profile_pass.py > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/launches_iter.csv
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; tail -3 gpurun_out/bench_iter.err
python -c "import json; d=json.load(open('gpurun_out/bench_iter.json')); print({k: d[k] for k in ('value','ms_per_step','gpix_pass_per_s','speedup_vs_jfa','similarity_vs_jfa_pct')}); print(d['jfa']); print(d['roofline']); print(d['e2e']); print(d['clocks'])"
