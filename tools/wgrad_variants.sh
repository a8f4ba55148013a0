# Build wgrad-kernel probe variants under build/wv/ (run here, CPU)
set -e
cd "$(dirname "$0")/.."
mkdir -p build/wv
rm -f build/wv/*.so
NV="/usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -shared -I include"
SRC="paper_2104_00237_b200/csrc/optfuse_kernels.cu paper_2104_00237_b200/csrc/optfuse_wgrad.cu"
$NV -o build/wv/ring192.so $SRC &
$NV -DOFW_RING_BYTES=98304 -o build/wv/ring96.so $SRC &
$NV -DOFW_RING_BYTES=131072 -o build/wv/ring128.so $SRC &
$NV -DOFW_NO_UPDATE=1 -o build/wv/noupd.so $SRC &
$NV -DOFW_MAX_SPLIT=1 -o build/wv/split1.so $SRC &
$NV -DOFW_MAX_SPLIT=2 -o build/wv/split2.so $SRC &
wait
ls build/wv
