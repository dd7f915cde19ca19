set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none -k regex:"label_hash|match_count" -c 2 -o gpurun_out/prof_reduce python scripts/prof_reduce.py > /dev/null 2>&1
ncu -i gpurun_out/prof_reduce.ncu-rep --page raw --csv > gpurun_out/prof_reduce_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_reduce.ncu-rep --page details --csv > gpurun_out/prof_reduce_details.csv 2>/dev/null
rm -f gpurun_out/prof_reduce.ncu-rep
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -k "windowed or large_grid" -q -p no:cacheprovider > gpurun_out/tests_rel.txt 2>&1; tail -3 gpurun_out/tests_rel.txt
