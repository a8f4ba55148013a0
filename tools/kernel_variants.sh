# Build liboptfuse_b200.so variants under build/variants/ (run here, CPU):
# fp32 unroll x min-blocks, bf16 unroll x min-blocks, cache-streaming hints
set -e
cd "$(dirname "$0")/.."
rm -f build/variants/*.so
mkdir -p build/variants
for v in ${VARIANTS:-"4 1 2 4 0" "4 1 2 3 0" "4 1 4 2 0" "4 1 1 8 0" "4 1 4 3 0" "4 2 2 4 0" "8 1 4 2 0"}; do
  set -- $v
  /usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -std=c++17 \
    -Xcompiler -fPIC -shared -I include -DOF_UNROLL=$1 -DOF_MIN_BLOCKS=$2 -DOF_UNROLL_BF16=$3 \
    -DOF_MIN_BLOCKS_BF16=$4 -DOF_CS=$5 \
    -o build/variants/liboptfuse_u$1_b$2_bf$3x$4_cs$5.so paper_2104_00237_b200/csrc/optfuse_kernels.cu \
    paper_2104_00237_b200/csrc/optfuse_wgrad.cu &
done
wait
ls build/variants
