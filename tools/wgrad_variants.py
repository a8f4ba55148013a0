"""Device time of the wgrad kernel per build variant (build/wv/*.so, one
process each via OPTFUSE_B200_LIB), 20 launches captured in a CUDA graph and
replayed (no host launch cost in the timing), BERT-base Linear shapes at 4096
tokens; the default library also times cuBLAS's GEMM and the unfused pair
(cuBLAS GEMM + of_policy_step_mt) the same way."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SHAPES = [(768, 768), (3072, 768), (768, 3072)]
T = 4096


def graph_us(fn, n=20, reps=5):
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) * 1e3 / n
        best = t if best is None else min(best, t)
    return best


def one(with_ref):
    sys.path.insert(0, str(ROOT))
    import torch
    from paper_2104_00237_b200 import _native as nat
    from paper_2104_00237_b200 import kernels
    torch.backends.cuda.matmul.allow_tf32 = False
    out = {}
    for M, N in SHAPES:
        dy = (torch.randn(T, M, device="cuda") * 0.1).to(torch.bfloat16)
        x = torch.randn(T, N, device="cuda").to(torch.bfloat16)
        th = torch.randn(M, N, device="cuda") * 0.02
        m, v = torch.zeros_like(th), torch.zeros_like(th)
        w16 = th.to(torch.bfloat16)
        hp = kernels.hparams("adamw", 1e-4, 0.9, 0.01, 1e-8, 0.9, 0.999, 0.9, 5)
        row = {"fused_us": round(graph_us(lambda: kernels.wgrad_step(dy, x, th, m, v, hp, shadow=w16)), 2)}
        if with_ref:
            gb = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            tl = kernels.TensorList(1)
            tl.set(0, th, gb, m, v, w16)
            tl.set_dtypes(torch.float32, torch.bfloat16)
            row["cublas_us"] = round(graph_us(lambda: torch.matmul(dy.t(), x, out=gb)), 2)

            def unfused():
                torch.matmul(dy.t(), x, out=gb)
                kernels.policy_step(tl, hp, None, nat.OF_FLAG_SHADOW_BF16, None)
            row["unfused_us"] = round(graph_us(unfused), 2)
        row["fused_tflops"] = round(2 * M * N * T / row["fused_us"] / 1e6, 1)
        out[f"{M}x{N}"] = row
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one(len(sys.argv) > 2)
        sys.exit(0)
    res = {}
    libs = sorted((ROOT / "build" / "wv").glob("*.so"))
    for so in libs:
        env = dict(os.environ, OPTFUSE_B200_LIB=str(so))
        cmd = [sys.executable, __file__, "--one"] + (["ref"] if so.stem == "ring192" else [])
        r = subprocess.run(cmd, env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-800:]
        print(so.stem, line, flush=True)
        try:
            res[so.stem] = json.loads(line)
        except ValueError:
            res[so.stem] = {"error": line}
    print(json.dumps(res))
