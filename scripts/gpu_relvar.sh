# Compare REL kernel variants at C5 (pass time from bench.py's live pass timing).
for v in build/variants/*.so; do
  VD_LIB=$v timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-exact-sample --no-variants --e2e-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), round(d['roofline']['avg_launch_ms'],3), round(d['jfa']['ms_per_frame'],1))"
done
