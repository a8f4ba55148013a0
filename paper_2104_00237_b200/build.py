"""In-tree build of the native libraries (sm_100a only).

    python -m paper_2104_00237_b200.build

Produces ``paper_2104_00237_b200/liboptfuse_b200.so`` (the C-ABI kernel
library).  Built files stay in the source tree so they travel to the GPU box
with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

KERNEL_SRC = PKG / "csrc" / "optfuse_kernels.cu"
KERNEL_LIB = PKG / "liboptfuse_b200.so"


def _stale(target: Path, sources) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(s).stat().st_mtime > t for s in sources)


def build_kernels(force: bool = False, verbose: bool = False) -> Path:
    deps = [KERNEL_SRC, ROOT / "include" / "optfuse_b200.h"]
    if not force and not _stale(KERNEL_LIB, deps):
        return KERNEL_LIB
    cmd = [NVCC, "-O3", *ARCH, "-lineinfo", "--fmad=false", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-I", str(ROOT / "include"),
           "-o", str(KERNEL_LIB), str(KERNEL_SRC)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return KERNEL_LIB


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_kernels(force=force, verbose=verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
