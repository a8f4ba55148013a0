"""wgrad kernel probe (GPU box): per-launch device time vs the token count
(fixed cost + cost per 64-token block) for one shape, and a single launch
for ncu.

    python tools/wgrad_probe.py sweep [M N]     # JSON: tokens -> us (CUDA events over 20 graph-captured launches)
    python tools/wgrad_probe.py one [M N T]     # one launch (for ncu -k regex:wgrad)
"""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2104_00237_b200 import kernels  # noqa: E402


def problem(M, N, T):
    dy = (torch.randn(T, M, device="cuda") * 0.1).to(torch.bfloat16)
    x = torch.randn(T, N, device="cuda").to(torch.bfloat16)
    th = torch.randn(M, N, device="cuda") * 0.02
    m, v = torch.zeros_like(th), torch.zeros_like(th)
    hp = kernels.hparams("adamw", 1e-4, 0.9, 0.01, 1e-8, 0.9, 0.999, 0.9, 5)
    return dy, x, th, m, v, hp


def main():
    mode = sys.argv[1]
    if mode == "one":
        M, N, T = (int(a) for a in sys.argv[2:5]) if len(sys.argv) > 4 else (3072, 768, 4096)
        dy, x, th, m, v, hp = problem(M, N, T)
        for _ in range(3):
            kernels.wgrad_step(dy, x, th, m, v, hp)
        torch.cuda.synchronize()
        return
    M, N = (int(a) for a in sys.argv[2:4]) if len(sys.argv) > 3 else (3072, 768)
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from wgrad_variants import graph_us   # 20 launches captured and replayed: device time only
    out = {"M": M, "N": N, "rows": []}
    for T in (256, 512, 1024, 2048, 4096, 8192):
        dy, x, th, m, v, hp = problem(M, N, T)
        us = graph_us(lambda: kernels.wgrad_step(dy, x, th, m, v, hp))
        g = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        cu = graph_us(lambda: torch.matmul(dy.t(), x, out=g))
        out["rows"].append({"T": T, "fused_us": round(us, 2), "cublas_us": round(cu, 2),
                            "fused_tflops": round(2 * M * N * T / us / 1e6, 1)})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
