# One GPU session script, parameterised by task names (run under gpurun):
#   bash scripts/gpu.sh TASK [TASK ...]      TAG=r02 by default
# Tasks:
#   info      host CPU / RAM / GPU of the box
#   tests     pytest -m "gpu and not slow"      slowtests  pytest -m "gpu and slow"
#   alltests  pytest -m gpu (the driver's round-end set)
#   smoke     __graft_entry__.smoke()
#   bench     bench.py C4 (default flags)       benchq     bench.py C4, GPU legs only
#   bench5    bench.py --config C5, GPU legs only
#   ref       bench.py --impl reference
#   launches  ncu launch list of a short bench.py run
#   ncupass   ncu --set full of one dJFA frame's jump passes (C4) + source page
#   ncujfa    ncu --set full of one JFA frame's jump passes (C4)
#   ncuremap  ncu --set full of the remap kernel (C4)
#   c4launch  ncu launch list (durations + DRAM bytes) of C4 JFA + 3 dJFA frames
#   c5launch  ncu launch list (durations + DRAM bytes) of C5 JFA + dJFA frames
#   variants  scripts/time_variants.py (build/variants/*.so)
#   skab      A/B of the shared-term pass kernel (VD_NO_SK=1 vs 0), per-k pass times
#   sweeps    scripts/sweep.py radius + density at 4096^2 (BASELINE configs[2])
#   sanitize  (closed on this pool since r02b) compute-sanitizer on scripts/sanitize_small.py
set -x
TAG=${TAG:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -iE "error|warning" | head
for t in "$@"; do
case $t in
info) (lscpu | head -20; free -g; nproc; nvidia-smi) > gpurun_out/info_$TAG.txt 2>&1 ;;
tests) timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/tests_$TAG.txt 2>&1; tail -5 gpurun_out/tests_$TAG.txt ;;
slowtests) timeout 2400 python -m pytest tests -m "gpu and slow" -x -q -p no:cacheprovider --durations=0 > gpurun_out/slowtests_$TAG.txt 2>&1; tail -30 gpurun_out/slowtests_$TAG.txt ;;
alltests) timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/alltests_$TAG.txt 2>&1; tail -25 gpurun_out/alltests_$TAG.txt ;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 ;;
bench) timeout 1200 python bench.py --frames-csv gpurun_out/frames_$TAG.csv > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json ;;
benchq) timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-exact > gpurun_out/benchq_$TAG.json 2> gpurun_out/benchq_$TAG.err; tail -3 gpurun_out/benchq_$TAG.err; cat gpurun_out/benchq_$TAG.json ;;
bench5) timeout 1500 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-exact --no-variants --e2e-steps 3 > gpurun_out/bench5_$TAG.json 2> gpurun_out/bench5_$TAG.err; tail -3 gpurun_out/bench5_$TAG.err; cat gpurun_out/bench5_$TAG.json ;;
ref) timeout 1200 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_$TAG.json 2> gpurun_out/ref_$TAG.err; tail -3 gpurun_out/ref_$TAG.err; cat gpurun_out/ref_$TAG.json ;;
launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-exact --e2e-steps 3 > gpurun_out/bench_under_ncu_$TAG.json 2>&1 ;;
ncupass) timeout 900 ncu --set full --clock-control none --import-source on -k regex:jump_pass -s 14 -c 6 -o /tmp/prof_pass_$TAG python scripts/profile_pass.py > /dev/null 2>&1
  ncu -i /tmp/prof_pass_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_pass_${TAG}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_pass_$TAG.ncu-rep --page source --csv --print-source sass -k regex:jump_pass -c 1 > gpurun_out/prof_pass_${TAG}_src.csv 2>/dev/null ;;
ncujfa) VD_FRAMES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:jump_pass -c 14 -o /tmp/prof_jfa_$TAG python scripts/profile_pass.py > /dev/null 2>&1
  ncu -i /tmp/prof_jfa_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_jfa_${TAG}_raw.csv 2>/dev/null ;;
ncuremap) timeout 900 ncu --set full --clock-control none --import-source on -k regex:remap -c 1 -o /tmp/prof_remap_$TAG python scripts/profile_pass.py > /dev/null 2>&1
  ncu -i /tmp/prof_remap_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_remap_${TAG}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_remap_$TAG.ncu-rep --page source --csv --print-source sass -k regex:remap -c 1 > gpurun_out/prof_remap_${TAG}_src.csv 2>/dev/null ;;
c4launch) timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c4_launches_$TAG.csv python scripts/profile_pass.py > gpurun_out/c4_launches_$TAG.log 2>&1 ;;
c5launch) VD_CFG=C5 VD_FRAMES=2 timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c5_launches_$TAG.csv python scripts/profile_pass.py > gpurun_out/c5_launches_$TAG.log 2>&1 ;;
variants) timeout 1500 python scripts/time_variants.py 2>&1 | tee gpurun_out/variants_$TAG.txt ;;
skab) timeout 900 python scripts/time_variants.py VD_NO_SK=1,0 2>&1 | tee gpurun_out/skab_$TAG.txt ;;
envab) timeout 900 python scripts/time_variants.py $ENVAB 2>&1 | tee -a gpurun_out/envab_$TAG.txt ;;
sweeps) timeout 900 python scripts/sweep.py --kind radius > gpurun_out/sweep_radius_$TAG.jsonl 2> gpurun_out/sweep_radius_$TAG.err
  timeout 900 python scripts/sweep.py --kind density > gpurun_out/sweep_density_$TAG.jsonl 2> gpurun_out/sweep_density_$TAG.err ;;
sanitize) echo "compute-sanitizer is closed on this GPU pool (r02b); use the VD_CHECK debug build (scripts/check_wsk_variant.py)"; continue
  for tool in memcheck racecheck synccheck initcheck; do
    echo "# compute-sanitizer --tool $tool python scripts/sanitize_small.py ($TAG)" > gpurun_out/sanitizer_${tool}_$TAG.txt
    timeout 1200 compute-sanitizer --tool $tool python scripts/sanitize_small.py >> gpurun_out/sanitizer_${tool}_$TAG.txt 2>&1
    tail -3 gpurun_out/sanitizer_${tool}_$TAG.txt
  done ;;
*) echo "unknown task $t" ;;
esac
done
ls -la gpurun_out | tail -20
