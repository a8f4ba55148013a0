"""The peer transport with REAL ranks on ONE GPU (diagnostic / GPU test
helper): W processes share cuda:0 and a gloo process group.  torch symmetric
memory refuses two ranks on one device, so the flat buffers are mapped into
the other ranks with CUDA IPC (torch's own tensor-sharing handles, exchanged
with all_gather_object) and the cross-rank barrier is a host barrier after a
device synchronize.  Everything else is the product path: DataParallelFusion
with transport="peer", the of_dp_step_peer kernel reading and writing the
other processes' buffers through their IPC mappings.  Each rank trains the
exact (fixed-order) chain on its own input; every rank's parameters must
equal the reference update applied to the rank-averaged gradient (numpy
oracle), bit for bit; with global-norm clipping ("+clip") within 1e-5 (the
norm's f64 reduction order).

    python tools/dp_ranks_one_gpu.py [W]        # prints one JSON line
"""

import json
import os
import socket
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

KIND, ETA, WD, ITERS, LAYERS, WIDTH = "adam", 1e-2, 1e-3, 3, 4, 8
CLIP = 0.05   # "+clip" schedules: small enough that every iteration clips


def _inputs(rank):
    rng = np.random.default_rng(100 + rank)
    return [rng.uniform(0.1, 1.0, (3, WIDTH)).astype(np.float32) for _ in range(ITERS)]


def _worker(rank, world, port, schedule, out, transport="peer"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2104_00237_b200 as of
        from paper_2104_00237_b200 import dp as dp_mod
        from paper_2104_00237_b200.dp import DataParallelFusion
        from torch.multiprocessing.reductions import reduce_tensor

        class _HostBarrier:
            def __init__(self, ptrs):
                self.buffer_ptrs = ptrs

            def barrier(self, channel=0, timeout_ms=0):
                torch.cuda.synchronize()
                dist.barrier()
                torch.cuda.synchronize()

        keep = []

        def _ipc_symmetric(self, n, dt):
            t = torch.zeros(n, dtype=dt, device=self.device)
            fn, args = reduce_tensor(t)
            handles = [None] * self.world
            dist.all_gather_object(handles, args)
            ptrs = []
            for r, a in enumerate(handles):
                if r == self.rank:
                    ptrs.append(t.data_ptr())
                else:
                    peer = fn(*a)        # cudaIpcOpenMemHandle in this process
                    keep.append(peer)
                    ptrs.append(peer.data_ptr())
            h = _HostBarrier(ptrs)
            if self._sync is None:
                self._sync = h
            return t, h

        dp_mod.DataParallelFusion._symmetric = _ipc_symmetric
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


def _reference(world, clip=None):
    from oracle import chain_ref, optim_ref
    m = chain_ref.build("chain", layers=LAYERS, width=WIDTH, seed=0)
    h = optim_ref.Hyper(kind=KIND, eta=ETA, weight_decay=WD)
    slots = [dict() for _ in m.params]
    xs = [_inputs(r) for r in range(world)]
    def grads_of(x):
        for g in m.grads:
            g[:] = 0
        _, saved = chain_ref._forward(m, x)
        gout = None
        for i in reversed(range(len(m.layer_param))):
            gout = chain_ref._backward_node(m, i, saved, gout)
        return [g.copy() for g in m.grads]

    for it in range(ITERS):
        grads = [grads_of(xs[r][it]) for r in range(world)]
        avg = []
        for k in range(len(m.params)):
            g = grads[0][k].copy()
            for r in range(1, world):
                g = np.add(g, grads[r][k])
            avg.append(np.multiply(g, np.float32(1.0 / world)))
        if clip is not None:   # optim.py:151-172 on the averaged gradient (norm in f64)
            norm = float(np.sqrt(sum(float(np.dot(g.astype(np.float64), g.astype(np.float64)))
                                     for g in avg)))
            if norm > clip:
                avg = [np.multiply(g, np.float32(clip / norm)) for g in avg]
        for k, theta in enumerate(m.params):
            optim_ref.step(KIND, h, theta, avg[k], slots[k], it + 1)
    return np.concatenate(m.params).tobytes()


def main():
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    # "collectives": the reduce-scatter -> sharded kernel -> all-gather path, its
    # collectives carried by the gloo group (NCCL refuses two ranks on one GPU)
    transport = "nccl" if len(sys.argv) > 2 and sys.argv[2] == "collectives" else "peer"
    res = {}
    for schedule in ("backward-fusion", "baseline", "forward-fusion", "baseline+clip",
                     "forward-fusion+clip"):
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        out = mp.get_context("spawn").Manager().dict()
        mp.start_processes(_worker, args=(world, port, schedule, out, transport), nprocs=world,
                           join=True, start_method="spawn")
        same = all(out[r] == out[0] for r in range(world))
        want = _reference(world, CLIP if schedule.endswith("+clip") else None)
        got = np.frombuffer(out[0], np.float32)
        ref = np.frombuffer(want, np.float32)
        res[schedule] = {"ranks_agree": same, "bitwise_vs_oracle": out[0] == want,
                         "max_abs_err": float(np.abs(got - ref).max()),
                         "max_rel_err": float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-6)))}
    print(json.dumps({"world": world, "transport": transport, **res}))


if __name__ == "__main__":
    main()
