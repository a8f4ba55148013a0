"""Run the streaming probe (tools/probe/stream_probe.cu) on the GPU box:
GB/s of pure copies with 1R1W, 2R2W, 3R2W (SGD-momentum's pattern) and 4R3W
(Adam's pattern) over 1 GiB per stream, grid sizes 1x/2x/8x the SM count."""

import ctypes
import json
import statistics
import subprocess
import sys
from pathlib import Path

import torch

HERE = Path(__file__).resolve().parent
SO = HERE / "libstream_probe.so"
if not SO.exists():
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-Xcompiler", "-fPIC", "-shared", "-o", str(SO), str(HERE / "stream_probe.cu")],
                   check=True)
lib = ctypes.CDLL(str(SO))
lib.probe_stream.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p] * 7 + [ctypes.c_int64, ctypes.c_void_p]
n = 1 << 28          # floats per stream (1 GiB)
bufs = [torch.ones(n, device="cuda") for _ in range(7)]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = {}
INPLACE = len(sys.argv) > 1 and sys.argv[1] == "inplace"
for r, w, unr in ((1, 1, 4), (3, 2, 4), (4, 3, 2), (4, 3, 4)):
    for mult in (2, 8):
        grid = sms * mult
        ts = []
        for i in range(5):
            flush.zero_()
            flush.sum()
            torch.cuda._sleep(2_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            # in place: the outputs are the first inputs (the update's theta, m, v)
            ptrs = [b.data_ptr() for b in bufs]
            if INPLACE:
                ptrs = ptrs[:4] + [ptrs[0], ptrs[2], ptrs[3]]
            st = lib.probe_stream(r, w, unr, grid, *ptrs, n // 4,
                                  torch.cuda.current_stream().cuda_stream)
            e1.record()
            torch.cuda.synchronize()
            assert st == 0, st
            if i:
                ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        out[f"{r}R{w}W_unr{unr}_grid{mult}x" + ("_inplace" if INPLACE else "")] = round((r + w) * n * 4 / ms / 1e6, 1)
print(json.dumps(out))
