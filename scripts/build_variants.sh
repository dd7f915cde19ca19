# build libvd variants with different compile-time knobs into build/variants/
#   bash scripts/build_variants.sh "-DVD_SMEM_KB=48" "-DVD_MAX_WALK=20" ...
set -e
mkdir -p build/variants
for v in "$@"; do
  name=$(echo "$v" | tr ' =' '_-')
  python -c "import sys; sys.path.insert(0, '.'); from paper_2209_00117_b200 import build as b; b.compile_all('build/variants/libvd_${name}.so', extra=sys.argv[1].split())" "$v" &
done
wait
ls build/variants
