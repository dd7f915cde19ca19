set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python bench.py --steps 50 --warmup 5 --cpu-seconds 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err; cat gpurun_out/bench2.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python scripts/profile_pass.py
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jump_pass -s 14 -c 6 -o gpurun_out/prof_pass_r01 python scripts/profile_pass.py
ls -la gpurun_out
