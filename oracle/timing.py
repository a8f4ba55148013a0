"""CPU baseline leg of bench.py (test/bench infrastructure, never the product).

Times the reference's CPU path for the benchmark workload on the host cores:
the reference update (optim.py:74-148, restated bit-exactly in
oracle.optim_ref -- numpy, single-threaded as in the reference) applied to a
real network's parameters, after a forward/backward pass on torch-CPU.  The
reference's own autodiff engine (graph.py) only supports its synthetic chains,
so torch-CPU stands in for it; that stage uses every host core allowed.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import optim_ref


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_training_sample(model_name: str, batch: int, iters: int, kind: str, hp: dict,
                        threads: int | None = None, seed: int = 0) -> dict:
    """``iters`` iterations of forward/backward (torch CPU) + the reference
    update (numpy oracle) on ``model_name``; returns timings and images/s."""
    import torch
    import torch.nn.functional as F

    from paper_2104_00237_b200.models import CLASSIFIERS, synthetic_batch

    threads = threads or host_cores()
    torch.set_num_threads(threads)
    torch.manual_seed(seed)
    net = CLASSIFIERS[model_name][0]()
    x, y = synthetic_batch(model_name, batch, device="cpu", seed=seed)
    params = [p for p in net.parameters() if p.requires_grad]
    h = optim_ref.Hyper(kind=kind, **hp)
    slots = [dict() for _ in params]
    fb, upd = [], []
    for t in range(1, iters + 1):
        t0 = time.perf_counter()
        loss = F.cross_entropy(net(x), y)
        loss.backward()
        t1 = time.perf_counter()
        for p, sl in zip(reversed(params), reversed(slots)):
            theta = p.detach().numpy().reshape(-1)   # shares storage with the torch parameter
            grad = p.grad.numpy().reshape(-1)
            optim_ref.step(kind, h, theta, grad, sl, t)
        t2 = time.perf_counter()
        fb.append(t1 - t0)
        upd.append(t2 - t1)
    n_elem = sum(p.numel() for p in params)
    per_iter = float(np.mean(fb) + np.mean(upd))
    return {"images_per_s": batch / per_iter, "ms_per_iter": per_iter * 1e3,
            "fwd_bwd_ms": float(np.mean(fb)) * 1e3, "update_ms": float(np.mean(upd)) * 1e3,
            "update_elems": n_elem, "threads": threads, "batch": batch, "iters": iters}


def reference_update_rate(kind: str, hp: dict, elems: int = 1 << 22, reps: int = 3) -> dict:
    """Throughput of the reference update alone (OptimizerPolicy.step restated
    in numpy, one thread as in the reference) on one ``elems``-element f32
    tensor: elements/s and algorithmic GB/s (same byte model as the kernels)."""
    rng = np.random.default_rng(0)
    theta = rng.standard_normal(elems).astype(np.float32)
    h = optim_ref.Hyper(kind=kind, **hp)
    slots: dict = {}
    ts = []
    for t in range(1, reps + 2):
        grad = (rng.standard_normal(elems) * 0.01).astype(np.float32)
        t0 = time.perf_counter()
        optim_ref.step(kind, h, theta, grad, slots, t)
        ts.append(time.perf_counter() - t0)
    sec = float(np.median(ts[1:]))
    bpe = 4 * (2 + 2 * len(optim_ref.SLOTS[kind])) + 4
    return {"elems_per_s": elems / sec, "gbs": elems * bpe / sec / 1e9, "threads": 1,
            "sample": f"{reps} steps of one {elems}-element f32 tensor"}


def reference_harness_breakdown(layers: int = 8, width: int = 32, batch: int = 32, iters: int = 30,
                                warmup: int = 5) -> dict:
    """The reference CLI's default workload (chain 8x32, adam 1e-3, batch 32)
    through the oracle port of its three schedules, numpy single-threaded as
    the reference runs: mean ms per iteration of each (the CPU side of the
    harness breakdown the GPU CLI reports)."""
    from . import chain_ref
    out = {}
    for name, run in (("baseline", chain_ref.run_baseline),
                      ("forward-fusion", chain_ref.run_forward_fusion),
                      ("backward-fusion", chain_ref.run_backward_fusion)):
        m = chain_ref.build("chain", layers=layers, width=width, seed=0)
        pol = chain_ref.Policy("adam", eta=1e-3)
        xs = chain_ref.iteration_inputs(m, batch, 0, warmup + iters)
        for x in xs[:warmup]:
            run(m, pol, x)
        t0 = time.perf_counter()
        for x in xs[warmup:]:
            run(m, pol, x)
        out[name] = (time.perf_counter() - t0) / iters * 1e3
    return {"ms_per_iter": {k: round(v, 3) for k, v in out.items()}, "threads": 1,
            "sample": f"chain {layers}x{width}, adam, batch {batch}, {iters} iterations each"}
