"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)
over every kernel of liboptfuse_b200.so, at shapes that hit the edge paths:
ragged tails (scalar loop), misaligned views (no 128-bit path), zero-element
tensors, the 1-vector small-launch tiles and the 4-vector large ones, f32 /
f64 / bf16-grad + fp32 master + bf16 shadow, the clip scale in f32 and f64,
the peer step at world 1, the multi-tensor copy and the sq-norm reduction.

    compute-sanitizer --tool memcheck python tools/sanitize_kernels.py

Exits non-zero if any result differs from a second, unsanitized-order run of
the same launches (a cheap determinism check).  Logs live in profiles/.
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2104_00237_b200 import _native as nat  # noqa: E402
from paper_2104_00237_b200 import kernels  # noqa: E402

DEV = "cuda"
SIZES = [0, 1, 3, 4, 5, 1023, 1024, 1025, 4097, 70001, 1 << 20]


def _tensors(dt, sizes, offset):
    """Views at an element offset into larger buffers (offset 1: misaligned)."""
    out = []
    for n in sizes:
        base = torch.randn(n + offset + 8, device=DEV).to(dt)
        out.append(base[offset:offset + n])
    return out


def policy_steps(seed: int) -> list:
    torch.manual_seed(seed)
    results = []
    for kind, slots in (("sgd", 0), ("sgd-momentum", 1), ("adagrad", 1), ("rmsprop", 1),
                        ("adadelta", 2), ("adam", 2), ("adamw", 2)):
        for pdt, gdt, shadow in ((torch.float32, torch.float32, False),
                                 (torch.float64, torch.float64, False),
                                 (torch.float32, torch.bfloat16, True)):
            for offset in (0, 1):
                p = _tensors(pdt, SIZES, offset)
                g = [x.to(gdt) * 0.01 for x in _tensors(torch.float32, SIZES, offset)]
                s0 = [x.abs() for x in _tensors(pdt, SIZES, offset)] if slots >= 1 else None
                s1 = [x.abs() for x in _tensors(pdt, SIZES, offset)] if slots >= 2 else None
                sh = [torch.empty(n, dtype=torch.bfloat16, device=DEV) for n in SIZES] if shadow else None
                tl = kernels.TensorList(len(SIZES))
                for i in range(len(SIZES)):
                    tl.set(i, p[i], g[i], s0[i] if s0 else None, s1[i] if s1 else None,
                           sh[i] if sh else None)
                tl.set_dtypes(pdt, gdt)
                hp = kernels.hparams(kind, 1e-3, 0.9, 1e-4, 1e-8, 0.9, 0.999, 0.9, 3)
                flags = nat.OF_FLAG_ZERO_GRAD | (nat.OF_FLAG_SHADOW_BF16 if shadow else 0)
                scale = torch.full((), 0.5, dtype=torch.float64 if pdt == torch.float64 else torch.float32,
                                   device=DEV)
                kernels.policy_step(tl, hp, scale, flags, None)
                results += [x.float().sum().item() for x in p]
    return results


def copies_norms_peer() -> list:
    out = []
    src = _tensors(torch.float32, SIZES, 1)
    dst = [torch.empty_like(s) for s in src]
    kernels.copy_mt(kernels.CopyList(dst, src))
    out += [float(d.double().sum()) for d in dst]
    tl = kernels.TensorList(len(src))
    for i, s in enumerate(src):
        tl.set(i, None, s)
    tl.set_dtypes(torch.float32, torch.float32)
    ws = torch.empty(kernels.sqnorm_workspace_len(), dtype=torch.float64, device=DEV)
    sq = torch.empty((), dtype=torch.float64, device=DEV)
    kernels.sqnorm(tl, ws, sq, accumulate=False, stream=None)
    coef = torch.empty((), dtype=torch.float32, device=DEV)
    fac = torch.empty((), dtype=torch.float64, device=DEV)
    kernels.clip_coef(sq, 1.0, coef, fac, None)
    out += [float(sq), float(coef), float(fac)]
    # peer step at world 1: this GPU's own buffers are the only "peer"
    n = 1 << 16
    for kind in ("sgd-momentum", "adam"):
        flat_p = torch.randn(n, device=DEV)
        flat_g = torch.randn(n, device=DEV) * 0.01
        s0, s1 = torch.zeros(n, device=DEV), torch.zeros(n, device=DEV)
        pb = kernels.PeerBucket(1, 0, torch.float32, torch.float32, [flat_g.data_ptr()],
                                [flat_p.data_ptr()], None, s0, s1 if kind == "adam" else None, 0, n)
        kernels.dp_step_peer(pb, kernels.hparams(kind, 1e-3, 0.9, 0.0, 1e-8, 0.9, 0.999, 0.9, 1),
                             None, 0, None)
        out.append(float(flat_p.double().sum()))
    a = torch.randn(33, 17, device=DEV)
    b = torch.randn(17, 29, device=DEV)
    from paper_2104_00237_b200.models import fixed_order_matmul
    out.append(float(fixed_order_matmul(a, b).double().sum()))
    return out


def main() -> int:
    n0 = nat.launch_count()
    r1 = policy_steps(0) + copies_norms_peer()
    torch.cuda.synchronize()
    r2 = policy_steps(0) + copies_norms_peer()
    torch.cuda.synchronize()
    launches = nat.launch_count() - n0
    same = r1 == r2
    print(f"sanitize workload: {launches} liboptfuse_b200 launches, repeat identical: {same}")
    return 0 if same else 1


if __name__ == "__main__":
    sys.exit(main())
