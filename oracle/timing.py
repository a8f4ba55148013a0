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


def _network(model_name: str):
    """The benchmark network, built here from torchvision (the reference arm
    must not touch the product package): CIFAR-shaped MobileNetV2 / ResNet-18."""
    import torch
    import torchvision
    if model_name == "mobilenet_v2_cifar":
        return torchvision.models.mobilenet_v2(num_classes=10), (3, 32, 32), 10
    if model_name == "resnet18_cifar":
        m = torchvision.models.resnet18(num_classes=10)
        m.conv1 = torch.nn.Conv2d(3, 64, kernel_size=3, stride=1, padding=1, bias=False)
        m.maxpool = torch.nn.Identity()
        return m, (3, 32, 32), 10
    raise ValueError(f"no CPU baseline for {model_name!r}")


def _batch(shape, classes: int, batch: int, seed: int):
    """x ~ N(0, 1), y ~ U{0..classes-1} from a CPU generator (the GPU arm's
    synthetic_batch draws the same way)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randn((batch,) + shape, generator=g), torch.randint(0, classes, (batch,), generator=g)


def cpu_training_sample(model_name: str, batch: int, iters: int, kind: str, hp: dict,
                        threads: int | None = None, seed: int = 0, warmup: int = 1) -> dict:
    """``warmup`` + ``iters`` iterations of forward/backward (torch CPU) + the
    reference update (numpy oracle, one thread) on ``model_name``, pinned to
    the first ``threads`` allowed cores (all of them by default); returns the
    timed iterations' means and images/s."""
    import torch
    import torch.nn.functional as F

    allowed = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None
    threads = threads or host_cores()
    if allowed is not None:
        os.sched_setaffinity(0, allowed[:threads])
    prev_threads = torch.get_num_threads()
    torch.set_num_threads(threads)
    try:
        torch.manual_seed(seed)
        net, shape, classes = _network(model_name)
        x, y = _batch(shape, classes, batch, seed)
        params = [p for p in net.parameters() if p.requires_grad]
        h = optim_ref.Hyper(kind=kind, **hp)
        slots = [dict() for _ in params]
        fb, upd = [], []
        for t in range(1, warmup + iters + 1):
            t0 = time.perf_counter()
            loss = F.cross_entropy(net(x), y)
            loss.backward()
            t1 = time.perf_counter()
            for p, sl in zip(reversed(params), reversed(slots)):
                theta = p.detach().numpy().reshape(-1)   # shares storage with the torch parameter
                grad = p.grad.numpy().reshape(-1)
                optim_ref.step(kind, h, theta, grad, sl, t)
            t2 = time.perf_counter()
            if t > warmup:
                fb.append(t1 - t0)
                upd.append(t2 - t1)
    finally:
        torch.set_num_threads(prev_threads)
        if allowed is not None:
            os.sched_setaffinity(0, allowed)
    n_elem = sum(p.numel() for p in params)
    per_iter = float(np.mean(fb) + np.mean(upd))
    return {"images_per_s": batch / per_iter, "ms_per_iter": per_iter * 1e3,
            "fwd_bwd_ms": float(np.mean(fb)) * 1e3, "update_ms": float(np.mean(upd)) * 1e3,
            "update_elems": n_elem, "threads": threads, "batch": batch, "iters": iters,
            "warmup": warmup}


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
