# Build the A/B libraries of the update kernel under build/ab/ (run here, CPU):
#   old.so    : the tile-per-tensor kernel of round 1 (git $OLD_REV, default 2812f47)
#   spt0.so   : slot-space kernel, always the U-vector build
#   spt1.so   : slot-space kernel, 1-vector build up to 1 slot per resident thread (default)
#   spt4.so   : slot-space kernel, 1-vector build up to 4 slots per resident thread
set -e
cd "$(dirname "$0")/.."
OLD_REV=${OLD_REV:-2812f47}
mkdir -p build/ab/src
git show $OLD_REV:paper_2104_00237_b200/csrc/optfuse_kernels.cu | sed 's#"../../include/optfuse_b200.h"#"optfuse_b200.h"#' > build/ab/src/old_kernels.cu
git show $OLD_REV:paper_2104_00237_b200/csrc/optfuse_ops.cuh | sed 's%"../../include/optfuse_b200.h"%"optfuse_b200.h"%' > build/ab/src/optfuse_ops.cuh
git show $OLD_REV:include/optfuse_b200.h > build/ab/src/optfuse_b200.h
NV="/usr/local/cuda/bin/nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -shared"
$NV -I build/ab/src -o build/ab/old.so build/ab/src/old_kernels.cu paper_2104_00237_b200/csrc/optfuse_wgrad.cu &
for s in 0 1 4; do
  $NV -I include -DOF_SMALL_SLOTS=$s -o build/ab/spt$s.so paper_2104_00237_b200/csrc/optfuse_kernels.cu paper_2104_00237_b200/csrc/optfuse_wgrad.cu &
done
wait
ls -la build/ab/*.so
