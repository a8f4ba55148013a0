# Build TMA-staged kernel variants (tile elements, stages, CTAs/SM) under build/variants/
set -e
cd "$(dirname "$0")/.."
rm -f build/variants/*.so
mkdir -p build/variants
for v in "2048 4 1" "1024 8 1" "1024 4 2" "4096 2 1" "1024 6 1"; do
  set -- $v
  /usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -std=c++17 \
    -Xcompiler -fPIC -shared -I include -DOF_TMA_TILE=$1 -DOF_TMA_STAGES=$2 -DOF_TMA_CTAS=$3 \
    -o build/variants/liboptfuse_tma_t$1_s$2_c$3.so paper_2104_00237_b200/csrc/optfuse_kernels.cu &
done
wait
ls build/variants
