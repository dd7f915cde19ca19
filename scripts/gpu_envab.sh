# A/B one env knob (e.g. VD_FUSED_REMAP=0,1): parity tests, frame/pass timings, ncu launch lists
mkdir -p gpurun_out
VAR=${1%%=*}; VALS=${1#*=}
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python scripts/time_variants.py "$1"
for v in ${VALS//,/ }; do
  env $VAR=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/envab_$v.csv python scripts/profile_pass.py > /dev/null 2>&1
  echo "== $VAR=$v"; python scripts/summarize_launches.py gpurun_out/envab_$v.csv
done
