# build libvd variants with different compile-time knobs into build/variants/
set -e
mkdir -p build/variants
NCCL_INC=$(python -c "import nvidia.nccl, os; print(os.path.join(list(nvidia.nccl.__path__)[0], 'include'))")
for v in "$@"; do
  name=$(echo "$v" | tr ' =' '_-')
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared -cudart shared -Xlinker -rpath=/usr/local/cuda/lib64 \
    -I include -I $NCCL_INC $v -o build/variants/libvd_${name}.so paper_2209_00117_b200/csrc/vd.cu -ldl &
done
wait
ls build/variants
