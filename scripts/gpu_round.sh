# Full measurement session: tests, smoke, bench, launch list, ncu full capture of one dJFA frame.
set -x
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -iE "error" | head
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tests_$TAG.txt 2>&1; tail -3 gpurun_out/tests_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_$TAG.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
kill $SMI
tail -2 gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python scripts/profile_pass.py > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-exact-sample --e2e-steps 3 > gpurun_out/bench_under_ncu_$TAG.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jump_pass -s 14 -c 6 -o /tmp/prof_pass_$TAG python scripts/profile_pass.py > /dev/null 2>&1
ncu -i /tmp/prof_pass_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_pass_${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/prof_pass_$TAG.ncu-rep --page source --csv --print-source sass -k regex:jump_pass -c 1 > gpurun_out/prof_pass_${TAG}_src.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:remap -c 1 -o /tmp/prof_remap_$TAG python scripts/profile_pass.py > /dev/null 2>&1
ncu -i /tmp/prof_remap_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_remap_${TAG}_raw.csv 2>/dev/null
ls gpurun_out
du -sh gpurun_out; ls -la gpurun_out
