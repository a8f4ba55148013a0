"""Consumer-fused backward fusion vs its unfused pair, per BERT-base Linear
shape (bf16 module, fp32 master + AdamW state), B200:

  fused    of_wgrad_step: tcgen05 dW = dY^T X, AdamW applied from TMEM to the
           fp32 master/m/v, bf16 weight written (no gradient in memory)
  unfused  cuBLAS bf16 GEMM (torch.matmul, fp32 accumulate, bf16 dW written)
           + of_policy_step_mt (bf16 gradient in, fp32 master/m/v, bf16 weight out)
  gemm     the cuBLAS GEMM alone (what the GEMM part of the fused kernel competes with)

L2 flushed before every repetition; CUDA events; median of 20.
    python tools/wgrad_bench.py > profiles/r02_wgrad_fused.json
"""

import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2104_00237_b200 import _native as nat  # noqa: E402
from paper_2104_00237_b200 import kernels  # noqa: E402

SHAPES = [("attn q/k/v/out 768x768", 768, 768), ("ffn up 3072x768", 3072, 768),
          ("ffn down 768x3072", 768, 3072)]
T = 4096   # tokens: batch 32 x seq 128


def timeit(fn, flush, reps=20):
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def main():
    torch.backends.cuda.matmul.allow_tf32 = False
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {"tokens": T, "rows": []}
    for name, M, N in SHAPES:
        g = torch.Generator(device="cpu").manual_seed(0)
        dy = (torch.randn(T, M, generator=g) * 0.1).to(torch.bfloat16).cuda()
        x = torch.randn(T, N, generator=g).to(torch.bfloat16).cuda()
        master = (torch.randn(M, N, generator=g) * 0.02).cuda()
        m, v = torch.zeros_like(master), torch.zeros_like(master)
        w16 = master.to(torch.bfloat16)
        hp = kernels.hparams("adamw", 1e-4, 0.9, 0.01, 1e-8, 0.9, 0.999, 0.9, 5)

        def fused():
            kernels.wgrad_step(dy, x, master, m, v, hp, shadow=w16)
        gbuf = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        tl = kernels.TensorList(1)
        tl.set(0, master, gbuf, m, v, w16)
        tl.set_dtypes(torch.float32, torch.bfloat16)

        def unfused():
            torch.matmul(dy.t(), x, out=gbuf)
            kernels.policy_step(tl, hp, None, nat.OF_FLAG_SHADOW_BF16, None)

        def gemm():
            torch.matmul(dy.t(), x, out=gbuf)
        n0 = nat.launch_count()
        fused()
        torch.cuda.synchronize()
        assert nat.launch_count() == n0 + 1
        tf, tu, tg = timeit(fused, flush), timeit(unfused, flush), timeit(gemm, flush)
        flops = 2.0 * M * N * T
        upd_bytes = M * N * (4 + 8 + 4 + 8 + 2)      # master + m/v read and written, bf16 weight out
        out["rows"].append({
            "layer": name, "M": M, "N": N, "T": T,
            "fused_us": round(tf, 2), "unfused_us": round(tu, 2), "cublas_gemm_us": round(tg, 2),
            "speedup_fused_vs_unfused": round(tu / tf, 3),
            "fused_tflops": round(flops / tf / 1e6, 1), "cublas_tflops": round(flops / tg / 1e6, 1),
            "update_bytes_fused": upd_bytes, "update_bytes_unfused": upd_bytes + M * N * (2 + 2),
            "gradient_bytes_saved": M * N * 4})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
