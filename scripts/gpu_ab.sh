# A/B: frame/pass timings of build/variants/*.so vs the in-tree libvd.so, plus an ncu launch
# list (kernel durations, DRAM bytes) of each under scripts/profile_pass.py (C4)
mkdir -p gpurun_out
timeout 600 python scripts/time_variants.py
for lib in build/variants/*.so paper_2209_00117_b200/libvd.so; do
  n=$(basename $lib .so)
  VD_LIB=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ab_$n.csv python scripts/profile_pass.py > /dev/null 2>&1
  echo "== $n"; python scripts/summarize_launches.py gpurun_out/ab_$n.csv
done
