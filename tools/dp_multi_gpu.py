"""Data parallel across REAL GPUs (one process per device, NCCL): the N>1 path's
numerics check (tests/test_dp_multi_gpu.py runs it when >= 2 GPUs are
visible; it skips on the one-GPU boxes).

    python tools/dp_multi_gpu.py [W]          # prints one JSON line

* transport "nccl": per-bucket NCCL reduce-scatter -> sharded of_policy_step_mt
  -> all-gather (dp.py), every schedule;
* transport "peer": the fused of_dp_step_peer kernel over torch symmetric
  memory (peer loads/stores over NVLink), every schedule;
* "multicast": of_dp_step_multicast (multimem.ld_reduce + multimem.st over an
  NVLS multicast address of torch symmetric memory), when the fabric offers it;
* "clip": baseline and forward fusion with global-norm clipping on both
  transports (NCCL: sq-norm of the reduce-scattered shard; peer:
  of_dp_sqnorm_peer), which must agree across ranks and with each other.

Each rank trains the exact (fixed-order) chain model on its own inputs; every
rank's parameters must equal the reference update (numpy oracle) applied to
the rank-averaged gradient: bit for bit at W = 2 (a sum of two is
order-free), within 1e-6 relative beyond (the collective's summation order),
and within 1e-6 for multicast (the switch's order).
"""

import json
import os
import socket
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from dp_ranks_one_gpu import ETA, ITERS, KIND, LAYERS, WD, WIDTH, _inputs, _reference  # noqa: E402

CLIP = 0.05   # small enough that every iteration clips


def _worker(rank, world, port, transport, schedule, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import paper_2104_00237_b200 as of
        from paper_2104_00237_b200.dp import DataParallelFusion
        if transport == "multicast":
            out[rank] = _multicast(rank, world)
            return
        g = of.build_model("chain", layers=LAYERS, width=WIDTH, seed=0, device="cuda")
        clip = schedule.endswith("+clip")
        pol = of.OptimizerPolicy(KIND, eta=ETA, weight_decay=WD, clip_norm=CLIP if clip else None)
        dpf = DataParallelFusion(g, pol, bucket_elems=2 * WIDTH * WIDTH, transport=transport)
        run = {"backward-fusion": dpf.run_backward_fusion, "baseline": dpf.run_baseline,
               "forward-fusion": dpf.run_forward_fusion}[schedule.replace("+clip", "")]
        for x in _inputs(rank):
            run(torch.from_numpy(x).cuda())
        dpf.flush()
        torch.cuda.synchronize()
        out[rank] = np.concatenate([p.value.detach().cpu().numpy().reshape(-1)
                                    for p in g.parameters]).tobytes()
    finally:
        dist.destroy_process_group()


def _multicast(rank, world):
    """Two steps of of_dp_step_multicast on a flat fp32 bucket; returns the
    parameter buffer, or a skip reason."""
    import torch.distributed._symmetric_memory as symm

    from oracle import optim_ref
    from paper_2104_00237_b200 import kernels
    n = 4 * 1024 * world
    shard = n // world
    grad = symm.empty(n, dtype=torch.float32, device="cuda")
    param = symm.empty(n, dtype=torch.float32, device="cuda")
    hg = symm.rendezvous(grad, dist.group.WORLD.group_name)
    hp_ = symm.rendezvous(param, dist.group.WORLD.group_name)
    if not getattr(hg, "multicast_ptr", 0) or not getattr(hp_, "multicast_ptr", 0):
        return "skip: no multicast address"
    rng = np.random.default_rng(5)
    theta0 = rng.standard_normal(n).astype(np.float32)
    grads = [[np.random.default_rng(100 * r + t).standard_normal(n).astype(np.float32)
              for t in range(2)] for r in range(world)]
    param.copy_(torch.from_numpy(theta0))
    s0 = torch.zeros(shard, device="cuda")
    s1 = torch.zeros(shard, device="cuda")
    scale = torch.full((), 1.0 / world, dtype=torch.float32, device="cuda")
    mb = kernels.McBucket(world, rank, int(hg.multicast_ptr), int(hp_.multicast_ptr), param,
                          s0, s1, rank * shard, shard)
    for t in (1, 2):
        grad.copy_(torch.from_numpy(grads[rank][t - 1]))
        torch.cuda.synchronize()
        hg.barrier()
        kernels.dp_step_multicast(mb, kernels.hparams("adam", 1e-3, 0.9, 0.0, 1e-8, 0.9, 0.999,
                                                      0.9, t), scale, 0, None)
        torch.cuda.synchronize()
        hg.barrier()
    theta = theta0.copy()
    slots = [dict() for _ in range(world)]
    h = optim_ref.Hyper(kind="adam", eta=1e-3)
    for t in (1, 2):
        for r in range(world):
            sl = slice(r * shard, (r + 1) * shard)
            g = grads[0][t - 1][sl].copy()
            for q in range(1, world):
                g = g + grads[q][t - 1][sl]
            g = np.multiply(g, np.float32(1.0 / world))
            th = theta[sl]
            optim_ref.step("adam", h, th, g, slots[r], t)
    got = param.cpu().numpy()
    return {"max_rel": float(np.max(np.abs(got - theta) / np.maximum(np.abs(theta), 1e-6))),
            "grad_zeroed": bool((grad.cpu().numpy() == 0).all())}


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    world = int(sys.argv[1]) if len(sys.argv) > 1 else min(torch.cuda.device_count(), 8)
    res = {"world": world}
    for transport in ("nccl", "peer"):
        for schedule in ("backward-fusion", "baseline", "forward-fusion"):
            out = mp.get_context("spawn").Manager().dict()
            mp.start_processes(_worker, args=(world, _port(), transport, schedule, out),
                               nprocs=world, join=True, start_method="spawn")
            want = np.frombuffer(_reference(world), np.float32)
            got = np.frombuffer(out[0], np.float32)
            res[f"{transport}:{schedule}"] = {
                "ranks_agree": all(out[r] == out[0] for r in range(world)),
                "bitwise_vs_oracle": out[0] == want.tobytes(),
                "max_rel_err": float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-6)))}
    # global-norm clipping (baseline / forward fusion): the two transports'
    # norms differ only in the summation order
    clip = {}
    for transport in ("nccl", "peer"):
        for schedule in ("baseline+clip", "forward-fusion+clip"):
            out = mp.get_context("spawn").Manager().dict()
            mp.start_processes(_worker, args=(world, _port(), transport, schedule, out),
                               nprocs=world, join=True, start_method="spawn")
            clip[(transport, schedule)] = (all(out[r] == out[0] for r in range(world)),
                                           np.frombuffer(out[0], np.float32))
    for schedule in ("baseline+clip", "forward-fusion+clip"):
        a, b = clip[("nccl", schedule)], clip[("peer", schedule)]
        res[f"clip:{schedule}"] = {
            "ranks_agree": a[0] and b[0],
            "nccl_vs_peer_max_rel": float(np.max(np.abs(a[1] - b[1]) / np.maximum(np.abs(a[1]), 1e-6)))}
    out = mp.get_context("spawn").Manager().dict()
    mp.start_processes(_worker, args=(world, _port(), "multicast", None, out), nprocs=world,
                       join=True, start_method="spawn")
    res["multicast"] = dict(out)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
