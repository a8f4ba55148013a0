"""Data-parallel plumbing (reduce-scatter -> sharded update -> all-gather) on
CPU with the gloo backend, world size 2.

The sharded update here is the numpy oracle (host stand-in for the sm_100a
kernel, which the GPU tests cover); what is under test is the host logic:
bucketing, padding, shard ownership, the collectives, bucket readiness from
the gradient hooks, forward-fusion deferral and the 1/W averaging.  The
result must equal a single process that averages both ranks' gradients and
applies the reference update -- bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

KIND, ETA, WD = "adam", 1e-2, 1e-3
ITERS = 4


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(rank):
    rng = np.random.default_rng(100 + rank)
    return [torch.from_numpy(rng.uniform(0.1, 1.0, (3, 6)).astype(np.float32)) for _ in range(ITERS)]


def _oracle_update(theta, grad, slots, t):
    from oracle import optim_ref
    hp = optim_ref.Hyper(kind=KIND, eta=ETA, weight_decay=WD)
    np_slots = {k: v.numpy() for k, v in slots.items()}
    optim_ref.step(KIND, hp, theta.numpy(), grad.numpy(), np_slots, t)


def _worker(rank, world, port, schedule, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2104_00237_b200 as of
        from paper_2104_00237_b200.dp import DataParallelFusion
        g = of.build_model("shared-chain", layers=4, width=6, device="cpu", exact=False,
                           track_input_grad=False)
        pol = of.OptimizerPolicy(KIND, eta=ETA, weight_decay=WD)
        dp = DataParallelFusion(g, pol, bucket_elems=40, update_fn=_oracle_update)
        assert len(dp.buckets) >= 2
        run = {"backward-fusion": dp.run_backward_fusion, "baseline": dp.run_baseline,
               "forward-fusion": dp.run_forward_fusion}[schedule]
        for x in _inputs(rank):
            run(x)
        dp.flush()
        flat = np.concatenate([p.value.detach().numpy().reshape(-1) for p in g.parameters])
        out[rank] = flat.tobytes()
    finally:
        dist.destroy_process_group()


def _single_process_reference():
    import paper_2104_00237_b200 as of
    from oracle import optim_ref
    g = of.build_model("shared-chain", layers=4, width=6, device="cpu", exact=False,
                       track_input_grad=False)
    hp = optim_ref.Hyper(kind=KIND, eta=ETA, weight_decay=WD)
    slots = [dict() for _ in g.parameters]
    xs = [_inputs(r) for r in range(2)]
    for it in range(ITERS):
        grads = []
        for r in range(2):
            for p in g.parameters:
                p.value.grad = None
            g.module(xs[r][it]).backward()
            grads.append([p.value.grad.numpy().reshape(-1).copy() for p in g.parameters])
        for k, p in enumerate(g.parameters):
            avg = (grads[0][k] + grads[1][k]) * np.float32(0.5)
            theta = p.value.detach().numpy().reshape(-1)
            optim_ref.step(KIND, hp, theta, avg, slots[k], it + 1)
    return np.concatenate([p.value.detach().numpy().reshape(-1) for p in g.parameters]).tobytes()


@pytest.mark.parametrize("schedule", ["backward-fusion", "baseline", "forward-fusion"])
def test_sharded_update_equals_single_process(schedule):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker, args=(2, _free_port(), schedule, out), nprocs=2, join=True,
                       start_method="spawn")
    assert out[0] == out[1], "ranks disagree after the all-gather"
    want = _single_process_reference()
    got = np.frombuffer(out[0], np.float32)
    ref = np.frombuffer(want, np.float32)
    assert got.tobytes() == ref.tobytes(), np.abs(got - ref).max()


# -- mixed precision (C4): bf16 module, fp32 master shards, bf16 all-gather --

def _worker_mixed(rank, world, port, schedule, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2104_00237_b200 as of
        from paper_2104_00237_b200.dp import DataParallelFusion
        g = of.build_model("shared-chain", layers=4, width=6, device="cpu", exact=False,
                           track_input_grad=False)
        g.use_master_weights()
        pol = of.OptimizerPolicy(KIND, eta=ETA, weight_decay=WD)
        dp = DataParallelFusion(g, pol, bucket_elems=40, update_fn=_oracle_update)
        assert dp.mixed and all(p.master is None for p in g.parameters)
        assert all(b.master.dtype == torch.float32 and b.flat_param.dtype == torch.bfloat16
                   for b in dp.buckets)
        run = {"backward-fusion": dp.run_backward_fusion, "baseline": dp.run_baseline,
               "forward-fusion": dp.run_forward_fusion}[schedule]
        for x in _inputs(rank):
            run(x.to(torch.bfloat16))
        dp.flush()
        flat = torch.cat([p.value.detach().reshape(-1) for p in g.parameters])
        shards = [(b.master.numpy().copy(), [p.id for p in b.params], list(b.offsets))
                  for b in dp.buckets]
        out[rank] = (flat.view(torch.int16).numpy().tobytes(), shards)
    finally:
        dist.destroy_process_group()


def _single_process_mixed():
    """One process, both ranks' bf16 gradients summed in bf16 (the reduce-
    scatter), averaged in fp32, fp32 master updated by the reference rule, bf16
    parameter = round(master)."""
    import paper_2104_00237_b200 as of
    from oracle import optim_ref
    g = of.build_model("shared-chain", layers=4, width=6, device="cpu", exact=False,
                       track_input_grad=False)
    masters = [p.value.detach().reshape(-1).clone().numpy() for p in g.parameters]
    g.module.to(torch.bfloat16)
    hp = optim_ref.Hyper(kind=KIND, eta=ETA, weight_decay=WD)
    slots = [dict() for _ in g.parameters]
    xs = [_inputs(r) for r in range(2)]
    for it in range(ITERS):
        grads = []
        for r in range(2):
            for p in g.parameters:
                p.value.grad = None
            g.module(xs[r][it].to(torch.bfloat16)).float().backward()
            grads.append([p.value.grad.reshape(-1).clone() for p in g.parameters])
        for k, p in enumerate(g.parameters):
            avg = ((grads[0][k] + grads[1][k]).float() * 0.5).numpy()
            optim_ref.step(KIND, hp, masters[k], avg, slots[k], it + 1)
            with torch.no_grad():
                p.value.copy_(torch.from_numpy(masters[k]).view_as(p.value))
    flat = torch.cat([p.value.detach().reshape(-1) for p in g.parameters])
    return flat.view(torch.int16).numpy().tobytes(), masters


@pytest.mark.parametrize("schedule", ["backward-fusion", "forward-fusion"])
def test_sharded_mixed_precision_equals_single_process(schedule):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker_mixed, args=(2, _free_port(), schedule, out), nprocs=2, join=True,
                       start_method="spawn")
    assert out[0][0] == out[1][0], "ranks disagree on the bf16 parameters after the all-gather"
    want_bf16, want_master = _single_process_mixed()
    assert out[0][0] == want_bf16
    # each rank owns one shard of every bucket's fp32 master: stitch rank 0 +
    # rank 1 per bucket and compare with the reference masters bit for bit
    for (s0, ids, offs), (s1, ids1, _) in zip(out[0][1], out[1][1]):
        assert ids == ids1
        full = np.concatenate([s0, s1])
        mask = np.ones(full.size, bool)
        for i, off in zip(ids, offs):
            w = want_master[i]
            assert full[off:off + w.size].tobytes() == w.tobytes()
            mask[off:off + w.size] = False
        assert not full[mask].any()     # alignment gaps and padding stay zero


# -- global-norm clipping under data parallel --------------

CLIP = 0.05


def _worker_clip(rank, world, port, schedule, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2104_00237_b200 as of
        from paper_2104_00237_b200.dp import DataParallelFusion
        g = of.build_model("shared-chain", layers=4, width=6, device="cpu", exact=False,
                           track_input_grad=False)
        pol = of.OptimizerPolicy(KIND, eta=ETA, weight_decay=WD, clip_norm=CLIP)
        dp = DataParallelFusion(g, pol, bucket_elems=40, update_fn=_oracle_update)
        if schedule == "backward-fusion":
            with pytest.raises(of.GlobalInfoRequired):
                dp.run_backward_fusion(_inputs(rank)[0])
            out[rank] = b""
            return
        run = {"baseline": dp.run_baseline, "forward-fusion": dp.run_forward_fusion}[schedule]
        for x in _inputs(rank):
            run(x)
        dp.flush()
        out[rank] = np.concatenate([p.value.detach().numpy().reshape(-1) for p in g.parameters]).tobytes()
    finally:
        dist.destroy_process_group()


def _single_process_clip():
    import paper_2104_00237_b200 as of
    from oracle import optim_ref
    g = of.build_model("shared-chain", layers=4, width=6, device="cpu", exact=False,
                       track_input_grad=False)
    hp = optim_ref.Hyper(kind=KIND, eta=ETA, weight_decay=WD)
    slots = [dict() for _ in g.parameters]
    xs = [_inputs(r) for r in range(2)]
    for it in range(ITERS):
        grads = []
        for r in range(2):
            for p in g.parameters:
                p.value.grad = None
            g.module(xs[r][it]).backward()
            grads.append([p.value.grad.numpy().reshape(-1).copy() for p in g.parameters])
        avg = [(grads[0][k] + grads[1][k]) * np.float32(0.5) for k in range(len(g.parameters))]
        optim_ref.clip_by_global_norm(avg, CLIP)
        for k, p in enumerate(g.parameters):
            theta = p.value.detach().numpy().reshape(-1)
            optim_ref.step(KIND, hp, theta, avg[k], slots[k], it + 1)
    return np.concatenate([p.value.detach().numpy().reshape(-1) for p in g.parameters])


@pytest.mark.parametrize("schedule", ["baseline", "forward-fusion", "backward-fusion"])
def test_sharded_clip_matches_single_process(schedule):
    """Baseline / forward fusion with a global-norm clip: one all-reduced f64
    scalar per iteration, the factor of the averaged gradient; equal to the
    single-process reference within the clip's own tolerance (its BLAS sdot
    order is unspecified, optim.py:163).  Backward fusion refuses the policy
    before touching anything."""
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker_clip, args=(2, _free_port(), schedule, out), nprocs=2, join=True,
                       start_method="spawn")
    if schedule == "backward-fusion":
        return
    assert out[0] == out[1], "ranks disagree after the all-gather"
    got = np.frombuffer(out[0], np.float32)
    want = _single_process_clip()
    assert np.allclose(got, want, rtol=1e-5, atol=1e-6), np.abs(got - want).max()


# -- checkpoint / resume under data parallel --------------------------------

def _worker_resume(rank, world, port, schedule, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2104_00237_b200 as of
        from paper_2104_00237_b200.dp import DataParallelFusion

        def fresh():
            g = of.build_model("shared-chain", layers=4, width=6, device="cpu", exact=False,
                               track_input_grad=False)
            pol = of.OptimizerPolicy(KIND, eta=ETA, weight_decay=WD)
            dp = DataParallelFusion(g, pol, bucket_elems=40, update_fn=_oracle_update)
            run = {"backward-fusion": dp.run_backward_fusion, "baseline": dp.run_baseline,
                   "forward-fusion": dp.run_forward_fusion}[schedule]
            return g, dp, run
        xs = _inputs(rank)
        g, dp, run = fresh()
        for x in xs[:2]:
            run(x)
        sd = dp.state_dict()
        g2, dp2, run2 = fresh()
        dp2.load_state_dict(sd)
        for x in xs[2:]:
            run2(x)
        dp2.flush()
        out[rank] = np.concatenate([p.value.detach().numpy().reshape(-1) for p in g2.parameters]).tobytes()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("schedule", ["backward-fusion", "forward-fusion"])
def test_sharded_checkpoint_resume_equals_single_process(schedule):
    """Each rank saves its shard state mid-run; fresh DataParallelFusion objects
    load it and continue: the result equals the uninterrupted single-process
    reference bit for bit."""
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker_resume, args=(2, _free_port(), schedule, out), nprocs=2, join=True,
                       start_method="spawn")
    assert out[0] == out[1]
    assert out[0] == _single_process_reference()


# -- forward-fusion leaders follow the execution order, not registration ----

class _Reordered(torch.nn.Module):
    """Three bias-free layers registered c, a, b but executed a -> b -> c: a
    bucket leader placed by registration order (c) would let a and b read
    their parameters before the deferred update lands."""

    def __init__(self):
        super().__init__()
        gen = torch.Generator().manual_seed(7)
        self.c = torch.nn.Linear(6, 6, bias=False)
        self.a = torch.nn.Linear(6, 6, bias=False)
        self.b = torch.nn.Linear(6, 6, bias=False)
        with torch.no_grad():
            for lin in (self.c, self.a, self.b):
                lin.weight.copy_(torch.rand(6, 6, generator=gen) - 0.5)

    def forward(self, x):
        return self.c(torch.relu(self.b(torch.relu(self.a(x))))).sum()


def _worker_order(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2104_00237_b200 as of
        from paper_2104_00237_b200.dp import DataParallelFusion
        g = of.Graph(_Reordered(), None, track_counts=False)
        pol = of.OptimizerPolicy(KIND, eta=ETA, weight_decay=WD)
        dp = DataParallelFusion(g, pol, bucket_elems=1 << 20, update_fn=_oracle_update)
        assert len(dp.buckets) == 1
        for x in _inputs(rank):
            dp.run_forward_fusion(x)
        assert [g.layers[i].name for i in g.exec_order] == ["a", "b", "c"]
        dp.flush()
        out[rank] = np.concatenate([p.value.detach().numpy().reshape(-1) for p in g.parameters]).tobytes()
    finally:
        dist.destroy_process_group()


def test_forward_fusion_leaders_follow_execution_order():
    from oracle import optim_ref
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker_order, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    assert out[0] == out[1]
    net = _Reordered()
    params = list(net.parameters())
    hp = optim_ref.Hyper(kind=KIND, eta=ETA, weight_decay=WD)
    slots = [dict() for _ in params]
    xs = [_inputs(r) for r in range(2)]
    for it in range(ITERS):
        grads = []
        for r in range(2):
            for p in params:
                p.grad = None
            net(xs[r][it]).backward()
            grads.append([p.grad.numpy().reshape(-1).copy() for p in params])
        for k, p in enumerate(params):
            avg = (grads[0][k] + grads[1][k]) * np.float32(0.5)
            optim_ref.step(KIND, hp, p.detach().numpy().reshape(-1), avg, slots[k], it + 1)
    want = np.concatenate([p.detach().numpy().reshape(-1) for p in params])
    assert np.frombuffer(out[0], np.float32).tobytes() == want.tobytes()
