# C5: full-size windowed parity test + ncu --set full capture of the dJFA frame's passes.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -k "full_c5" -x -q -p no:cacheprovider > gpurun_out/tests_c5.txt 2>&1; tail -3 gpurun_out/tests_c5.txt
TAG=r01c5
VD_CFG=C5 VD_FRAMES=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:jump_pass -s 10 -c 6 -o gpurun_out/prof_pass_$TAG python scripts/profile_pass.py > gpurun_out/prof_$TAG.log 2>&1; tail -3 gpurun_out/prof_$TAG.log
ncu -i gpurun_out/prof_pass_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_pass_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_pass_$TAG.ncu-rep --page source --csv --print-source sass -k regex:jump_pass -c 1 > gpurun_out/prof_pass_${TAG}_src.csv 2>/dev/null
rm -f gpurun_out/prof_pass_$TAG.ncu-rep
ls -la gpurun_out | tail -5
