mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i error
for t in memcheck racecheck synccheck; do
  echo "# compute-sanitizer --tool $t python scripts/sanitize_small.py (r01, packed-key walk)" > gpurun_out/sanitizer_$t.txt
  timeout 900 compute-sanitizer --tool $t python scripts/sanitize_small.py >> gpurun_out/sanitizer_$t.txt 2>&1
  tail -3 gpurun_out/sanitizer_$t.txt
done
timeout 900 python scripts/time_variants.py
