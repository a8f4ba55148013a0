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
KERNEL_SRCS = [KERNEL_SRC, PKG / "csrc" / "optfuse_wgrad.cu"]
KERNEL_LIB = PKG / "liboptfuse_b200.so"


def _stale(target: Path, sources) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(s).stat().st_mtime > t for s in sources)


def build_kernels(force: bool = False, verbose: bool = False) -> Path:
    deps = [*KERNEL_SRCS, PKG / "csrc" / "optfuse_ops.cuh", ROOT / "include" / "optfuse_b200.h"]
    if not force and not _stale(KERNEL_LIB, deps):
        return KERNEL_LIB
    cmd = [NVCC, "-O3", *ARCH, "-lineinfo", "--fmad=false", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-I", str(ROOT / "include"),
           "-o", str(KERNEL_LIB), *[str(x) for x in KERNEL_SRCS]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return KERNEL_LIB


ENGINE_SRC = PKG / "csrc" / "optfuse_engine.cpp"


def engine_lib_path() -> Path:
    import sysconfig
    return PKG / ("_optfuse_engine" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_engine(force: bool = False, verbose: bool = False) -> Path:
    """The native hook scheduler: a torch extension module linked against
    liboptfuse_b200.so (found next to it through an $ORIGIN rpath)."""
    import sysconfig

    import torch
    from torch.utils import cpp_extension as ce

    target = engine_lib_path()
    deps = [ENGINE_SRC, ROOT / "include" / "optfuse_b200.h", KERNEL_LIB]
    if not force and not _stale(target, deps):
        return target
    incs = ce.include_paths("cuda") + [sysconfig.get_paths()["include"], str(ROOT / "include")]
    libs = ce.library_paths("cuda")
    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-fPIC", "-shared",
           f"-D_GLIBCXX_USE_CXX11_ABI={abi}", "-DTORCH_EXTENSION_NAME=_optfuse_engine",
           "-DTORCH_API_INCLUDE_EXTENSION_H", "-fvisibility=hidden",
           *[f"-I{i}" for i in incs], str(ENGINE_SRC), "-o", str(target),
           *[f"-L{d}" for d in libs], f"-L{PKG}",
           "-loptfuse_b200", "-lc10", "-lc10_cuda", "-ltorch", "-ltorch_cpu", "-ltorch_cuda",
           "-ltorch_python", "-lcudart", "-Wl,-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return target


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_kernels(force=force, verbose=verbose)
    build_engine(force=force, verbose=verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
