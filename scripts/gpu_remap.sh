python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q -p no:cacheprovider -k "djfa or packed or shard or c3" 2>&1 | tail -2
timeout 900 python scripts/time_variants.py
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python scripts/profile_pass.py > /dev/null 2>&1; python scripts/summarize_launches.py gpurun_out/launches_q.csv | grep remap
