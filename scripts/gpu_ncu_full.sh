# one ncu --set full capture of the dJFA frame's jump passes (C4) + source page
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -iE "error" | head
TAG=${TAG:-r01}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jump_pass -s 14 -c 6 -o gpurun_out/prof_pass_$TAG python scripts/profile_pass.py > /dev/null 2>&1
ncu -i gpurun_out/prof_pass_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_pass_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_pass_$TAG.ncu-rep --page source --csv --print-source sass -k regex:jump_pass -c 1 > gpurun_out/prof_pass_${TAG}_src.csv 2>/dev/null
ls -la gpurun_out | tail -5
