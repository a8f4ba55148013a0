#!/usr/bin/env python
"""Benchmark: fused vs unfused training iterations on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (N=1): configs[1] of BASELINE.json -- MobileNetV2 on synthetic
CIFAR-10-shaped data (3x32x32, 10 classes), SGD-momentum (lr 0.1, momentum
0.9, weight decay 5e-4), fp32 weights (TF32 convolutions and matmuls), batch
128 per GPU, channels-last, backward fusion with 1M-element buckets on the
side stream, the whole iteration replayed from a CUDA graph.  One "step" =
one training iteration (forward, backward, every parameter updated), with a
256 MiB L2 flush before it (between its event pair and the previous one's).  The same iteration is also timed with
torch.optim.SGD (foreach, fused), with no update at all (the floor any fusion
can reach), and under our other schedules, eager and graphed; a batch sweep
32..512 and the other BASELINE.json configs (C1, C3, C4, C5) are reported
beside the headline.  N>1 (torchrun): the data-parallel path (dp.py, NCCL
reduce-scatter -> sharded update -> all-gather per bucket, captured in the
graph) against DDP + torch.optim; --force-dp runs that path at N=1.

Prints ONE JSON line (rank 0).  ``value`` = images/s over all ranks with
inputs resident in HBM, device-timed with CUDA events (max over ranks),
median of 3 independently built instances; ``e2e`` = the same through the
public API with pinned-host inputs copied in and the loss read back every
step; ``roofline`` = the update kernel's average launch duration on its
stream (back-to-back replay of one iteration's launches) as algorithmic HBM
bandwidth against MEASURED_PEAKS.json, with the ncu DRAM traffic per launch
(profiles/ncu_traffic.json) and standalone single-pass figures for the
C2-C5 parameter sets; ``cpu_baseline`` / ``cpu_update_baseline`` = the
reference's CPU path (oracle port) on the host cores.

``--impl reference`` times the reference's CPU implementation of the path
(oracle port of optim.py + torch-CPU forward/backward) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "train iter time & images/sec (fused vs unfused) at 1/2/4/8 B200; update HBM GB/s"
UNIT = "images/s"
WORKLOAD = ("C2: MobileNetV2 (torchvision, 10 classes) on synthetic CIFAR-10 shape 3x32x32, "
            "SGD-momentum lr 0.1 m 0.9 wd 5e-4, fp32")


def parse_args(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--model", default="mobilenet_v2_cifar")
    ap.add_argument("--batch", type=int, default=128, help="per-GPU batch")
    ap.add_argument("--schedule", default="backward-fusion",
                    choices=("baseline", "forward-fusion", "backward-fusion"))
    ap.add_argument("--workers", type=int, default=2, help="backward-fusion: 1 inline, >1 side stream")
    ap.add_argument("--ff-bucket-elems", type=int, default=1 << 18,
                    help="forward-fusion buckets (0 = one pre-hook per layer)")
    ap.add_argument("--grad-reset", default="none", choices=("zero", "none"))
    ap.add_argument("--bucket-elems", type=int, default=1 << 20,
                    help="backward-fusion launch groups: 0 = one per layer, else merge layers "
                         "(backward order) into buckets of at least this many elements (1M: "
                         "MobileNetV2's 2.24 M parameters in 3 launches of >= 4 MB, the smallest "
                         "size that leaves the kernel's ~4 us latency floor, still overlapped "
                         "with the backward of the earlier layers)")
    ap.add_argument("--sweep", default="32,64,256,512", help="extra per-GPU batches ('' to skip)")
    ap.add_argument("--graphs", type=int, default=1,
                    help="1: capture each iteration (ours and the torch baseline) as a CUDA graph")
    ap.add_argument("--channels-last", type=int, default=1, help="1: NHWC model and inputs")
    ap.add_argument("--no-extras", action="store_true", help="headline only (for profilers)")
    ap.add_argument("--dp-graphs", type=int, default=1,
                    help="1: capture data-parallel iterations (NCCL collectives included) as CUDA "
                         "graphs too (0: eager data parallel)")
    ap.add_argument("--dp-transport", default="nccl", choices=("nccl", "peer"),
                    help="data parallel: NCCL reduce-scatter/all-gather around the sharded kernel, "
                         "or the fused peer-memory kernel over torch symmetric memory")
    ap.add_argument("--force-dp", action="store_true",
                    help="run the data-parallel code path (NCCL process group, DataParallelFusion, "
                         "DDP baselines) even at one GPU: the N>1 path's smoke test")
    ap.add_argument("--extras", default="c1,c3,c4,c5",
                    help="other BASELINE.json configs timed beside the headline ('' to skip)")
    ap.add_argument("--cpu-iters", type=int, default=2, help="CPU baseline sample iterations")
    ap.add_argument("--instances", type=int, default=5,
                    help="independently built model instances timed for the headline and key rows")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, backend="nccl", force: bool = False):
        import torch
        import torch.distributed as dist
        if self.world > 1 or force:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend, rank=self.rank, world_size=self.world)
            self.pg = dist.group.WORLD
        return self

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------

class Clocks:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(self.NAMES, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# timing helpers
# ---------------------------------------------------------------------------

def timed(step, steps: int, warmup: int, dist: Dist, flush=None) -> float:
    """W warm-up steps, then EXACTLY K steps between barrier+synchronize on both
    sides, device-timed with CUDA events on the current stream; max over ranks.
    With ``flush`` (an L2 flush between timed iterations) each step has its own
    event pair after the flush, and the flush is not part of the step time.
    Returns ms per step."""
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    s = torch.cuda.current_stream()
    n = steps if flush is not None else 1
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    # a start/end range is process-wide (push/pop ranges are per thread and would
    # miss the backward kernels autograd launches from its own thread):
    # ncu --nvtx --nvtx-include timed selects this region
    rng = torch.cuda.nvtx.range_start("timed")
    if flush is None:
        e0[0].record(s)
    for i in range(steps):
        if flush is not None:
            flush()
            e0[i].record(s)
        step()
        if flush is not None:
            e1[i].record(s)
    if flush is None:
        e1[0].record(s)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_end(rng)
    dist.barrier()
    return dist.max(sum(a.elapsed_time(b) for a, b in zip(e0, e1))) / steps


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

# BASELINE.json configs measured here: C2 (the headline) plus C1, C3, C4, C5 as
# single-GPU extras (their multi-GPU data-parallel form runs under torchrun)
WORKLOADS = {
    "c1": {"model": "resnet18_cifar", "batch": 128, "kind": "sgd-momentum",
           "hp": {"eta": 0.1, "alpha": 0.9, "weight_decay": 5e-4},
           "torch": ("SGD", {"lr": 0.1, "momentum": 0.9, "weight_decay": 5e-4}),
           "desc": "ResNet-18 (CIFAR stem) on synthetic 3x32x32, batch 128, SGD-momentum, fp32"},
    "c2": {"model": "mobilenet_v2_cifar", "batch": 128, "kind": "sgd-momentum",
           "hp": {"eta": 0.1, "alpha": 0.9, "weight_decay": 5e-4},
           "torch": ("SGD", {"lr": 0.1, "momentum": 0.9, "weight_decay": 5e-4})},
    "c3": {"model": "vgg16", "batch": 32, "kind": "adam",
           "hp": {"eta": 1e-4, "weight_decay": 1e-4},
           "torch": ("Adam", {"lr": 1e-4, "weight_decay": 1e-4}),
           "desc": "VGG-16 on synthetic 3x224x224, batch 32, Adam (coupled wd 1e-4), fp32"},
    "c4": {"model": "resnet50", "batch": 64, "kind": "adamw", "mixed": True,
           "hp": {"eta": 1e-3, "weight_decay": 0.05},
           "torch": ("AdamW", {"lr": 1e-3, "weight_decay": 0.05}),
           "desc": ("ResNet-50 on synthetic 3x224x224, batch 64, AdamW (wd 0.05); ours: bf16 model "
                    "with fp32 master weights updated in one pass (bf16 grad in, bf16 param out); "
                    "torch: fp32 params under torch.autocast(bf16)")},
    "c5": {"model": "bert_base", "batch": 32, "kind": "adamw",
           "hp": {"eta": 1e-4, "weight_decay": 0.01},
           "torch": ("AdamW", {"lr": 1e-4, "weight_decay": 0.01}),
           "desc": ("BERT-base pre-training (BertForPreTraining, random init), seq 128, batch 32, "
                    "15% MLM labels + NSP, AdamW (wd 0.01), fp32 weights (TF32 matmuls)")},
}


def make_runner(args, batch: int, schedule: str, device, seed=0, workers=None,
                grad_reset=None, opt_impl=None, bucket_elems=None, graphed=None,
                workload="c2", channels_last=None):
    """Returns (step_fn, graph_or_model, policy_or_opt).  ``opt_impl`` selects
    the unfused torch.optim baseline ("foreach" | "fused") or "none" (forward
    + backward only, no update: the lower bound any fusion can reach);
    ``graphed`` captures the whole iteration as a CUDA graph
    (paper_2104_00237_b200.graphs)."""
    import torch

    import paper_2104_00237_b200 as of
    from paper_2104_00237_b200.graphs import CapturedStep
    from paper_2104_00237_b200.models import synthetic_batch

    wl = WORKLOADS[workload]
    mixed = wl.get("mixed", False)
    graphed = args.graphs if graphed is None else graphed
    cl = args.channels_last if channels_last is None else channels_last
    x, y = synthetic_batch(wl["model"], batch, device=device, seed=seed)
    if cl and x.dim() == 4:
        x = x.contiguous(memory_format=torch.channels_last)
    world = getattr(args, "world", 1)
    dp = world > 1 or getattr(args, "dp", False)
    if opt_impl is not None:  # unfused torch.optim baseline (or no update at all)
        g = of.build_classifier(wl["model"], device=device, seed=seed, channels_last=bool(cl))
        if opt_impl == "none-mixed":   # our model math: bf16 module, no autocast, no update
            g.use_master_weights()
            x = x.to(torch.bfloat16) if x.is_floating_point() else x
            opt_impl, mixed = "none", False
        net, loss_fn = g.module, g.loss_fn  # plain module: no hooks until a schedule runs
        name, kw = wl["torch"]
        opt = None
        if opt_impl != "none":
            kw = dict(kw, **({"foreach": True} if opt_impl == "foreach" else {"fused": True}))
            if graphed and name in ("Adam", "AdamW"):
                kw["capturable"] = True
            opt = getattr(torch.optim, name)(net.parameters(), **kw)
        cap_stream = None
        if dp:  # unfused data parallel: DDP all-reduce + torch.optim
            graphed = graphed and bool(args.dp_graphs)
            if graphed:   # DDP stashes autograd nodes on the stream it is built on: the capture's
                cap_stream = torch.cuda.Stream()
                cap_stream.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(cap_stream):
                    net = torch.nn.parallel.DistributedDataParallel(
                        net, device_ids=[device.index], static_graph=True)
                # DDP logs runtime stats from Python in its first 10 iterations
                net._set_ddp_runtime_logging_sample_rate(1 << 30)
            else:
                net = torch.nn.parallel.DistributedDataParallel(net, device_ids=[device.index])
        amp = torch.autocast("cuda", dtype=torch.bfloat16) if mixed else None

        def run(inp):
            if opt is not None:
                opt.zero_grad(set_to_none=True)
            else:
                for p in net.parameters():
                    p.grad = None
            if amp is not None:
                with amp:
                    loss = loss_fn(net(inp[0]), inp[1])
            else:
                loss = loss_fn(net(inp[0]), inp[1])
            loss.backward()
            if opt is not None:
                opt.step()
            return loss
        owner, pol = net, opt
    elif dp:  # data parallel: sharded fused update over NCCL
        cap_stream = None
        from paper_2104_00237_b200.dp import DataParallelFusion
        g = of.build_classifier(wl["model"], device=device, seed=seed, channels_last=bool(cl))
        g.track_counts = False
        if mixed:
            g.use_master_weights()
            x = x.to(torch.bfloat16) if x.is_floating_point() else x
        pol = of.OptimizerPolicy(wl["kind"], **wl["hp"])
        dpf = DataParallelFusion(g, pol, bucket_elems=bucket_elems or args.bucket_elems,
                                 transport=getattr(args, "dp_transport", "nccl"))
        dp_run = {"baseline": dpf.run_baseline, "forward-fusion": dpf.run_forward_fusion,
                  "backward-fusion": dpf.run_backward_fusion}[schedule]
        graphed = graphed and bool(args.dp_graphs)   # NCCL collectives captured in the graph

        def run(inp):
            return dp_run(inp).loss
        owner = g
    else:
        cap_stream = None
        g = of.build_classifier(wl["model"], device=device, seed=seed, channels_last=bool(cl))
        g.track_counts = False  # no per-layer Python pre-hooks unless a schedule needs them
        if mixed:
            g.use_master_weights()
            x = x.to(torch.bfloat16) if x.is_floating_point() else x
        pol = of.OptimizerPolicy(wl["kind"], **wl["hp"], grad_reset=grad_reset or args.grad_reset)
        w = args.workers if workers is None else workers
        ctas, prio = None, "high"
        if w == -1:       # side stream with the update grid capped to a third of the SMs
            w, ctas = 2, max(8, torch.cuda.get_device_properties(device).multi_processor_count // 3)
        elif w == -2:     # side stream at the compute stream's (default) priority
            w, prio = 2, "low"
        if schedule == "baseline":
            def run(inp):
                return of.run_baseline(g, pol, inp, timing=False).loss
        elif schedule == "forward-fusion":
            fbe = args.ff_bucket_elems if bucket_elems is None else bucket_elems
            # forward fusion: an explicit workers=2 selects the side-stream lookahead of one
            # unit, workers=-3 every unit at the first layer
            pre = {2: 1, -3: -1}.get(workers, 0)

            def run(inp):
                return of.run_forward_fusion(g, pol, inp, timing=False, bucket_elems=fbe,
                                             prefetch=pre).loss
        else:
            be = args.bucket_elems if bucket_elems is None else bucket_elems

            def run(inp):
                return of.run_backward_fusion(g, pol, inp, workers=w, timing=False,
                                              bucket_elems=be, update_ctas=ctas,
                                              update_priority=prio).loss
        owner = g
    if graphed:
        ours = isinstance(pol, of.OptimizerPolicy)
        ddp = isinstance(owner, torch.nn.parallel.DistributedDataParallel)
        cap = CapturedStep(run, (x, y), warmup=12 if ddp else 3, policy=pol if ours else None,
                           graph=owner if ours else None, stream=cap_stream if ddp else None)
        return cap, owner, pol

    def step():
        return run((x, y))
    step.run = run
    return step, owner, pol


def measure_update_kernel(args, device, peaks) -> dict:
    """Standalone roofline of the multi-tensor kernel: one pass over a whole
    parameter set (as few launches as the 256-tensor parameter block allows),
    L2 flushed (and its dirty lines written back) before every pass: VGG-16 with Adam (C3, update-bound),
    BERT-base with AdamW (C5), ResNet-50 bf16 + fp32 masters with AdamW (C4:
    bf16 grad in, bf16 parameter out) and MobileNetV2 with SGD-momentum (C2)."""
    import torch

    import paper_2104_00237_b200 as of
    from paper_2104_00237_b200.optim import algorithmic_bytes

    out = {}
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=device)
    for name, model, kind, mixed in (("vgg16_adam", "vgg16", "adam", False),
                                     ("bert_base_adamw", "bert_base", "adamw", False),
                                     ("resnet50_bf16_master_adamw", "resnet50", "adamw", True),
                                     ("mobilenet_v2_sgdm", "mobilenet_v2_cifar", "sgd-momentum", False)):
        g = of.build_classifier(model, device=device)
        if mixed:
            g.use_master_weights()
        pol = of.OptimizerPolicy(kind, eta=1e-4, weight_decay=0.01 if kind == "adamw" else 0.0)
        params = g.parameters
        grads = [torch.randn_like(p.value) * 0.01 for p in params]
        # grad_reset="none" (the headline's): the kernel moves exactly the
        # algorithmic bytes; "zero" would add a 4 B/element gradient write that
        # the byte count does not include.  The step releases the gradients, so
        # each pass hands the same tensors back.
        pol.grad_reset = "none"
        times = []
        for i in range(8):
            pol.begin_iteration()
            for p, gr in zip(params, grads):
                p.value.grad = gr
            flush.zero_()                  # evict the parameter set from L2 ...
            flush.sum()                    # ... and write the flush's dirty lines back now
            torch.cuda._sleep(4_000_000)   # the host builds the tensor list while the GPU waits
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pol.step_params(params)
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                times.append(e0.elapsed_time(e1))
        nbytes = algorithmic_bytes(kind, params)
        t = statistics.median(times) / 1e3
        gbs = nbytes / t / 1e9
        out[name] = {"bytes": nbytes, "us": round(t * 1e6, 2), "achieved_gbs": round(gbs, 1),
                     "frac": round(gbs / peaks["hbm_gbs"], 4), "tensors": len(params),
                     "launches": (len(params) + 255) // 256}
        del g, params
        torch.cuda.empty_cache()
    return out


def ncu_traffic(kernel: str) -> dict | None:
    """DRAM bytes per launch of ``kernel`` from the committed ncu --set full
    capture (profiles/ncu_traffic.json, written by tools/summarize_ncu.py)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    return json.loads(p.read_text()).get(kernel)


def measure_in_situ(args, device, peaks, reps: int = 5) -> dict:
    """Average launch duration of the backward-fusion update kernel on its stream.

    After real training iterations, the exact backward-fusion launch sequence
    of one iteration (same groups, tensors and hyper-parameters) is enqueued on
    the update stream behind a torch.cuda._sleep, with one CUDA event pair
    around the whole sequence: total time / launches is the average launch
    duration, kernel time only (no host issue gaps, and no per-launch event
    records, which would add ~2 us to every few-us launch)."""
    import torch

    from paper_2104_00237_b200.optim import bytes_per_element
    step, g, pol = make_runner(args, args.batch, "backward-fusion", device, workers=2, graphed=False)
    # (launch groups as configured by --bucket-elems)
    for _ in range(3):
        step()
    eng = next(e for k, e in g._engines.items() if k[1])
    native = eng.native
    # element count of every group, from one profiled pass
    step()
    for p in g.parameters:
        if p.value.grad is None:
            p.value.grad = torch.randn_like(p.value) * 0.01
    native.set_profile(True)
    for gi in range(native.num_groups):
        native.launch_group(gi, sync=False)
    native.set_profile(False)
    native.join()
    elems = [n for _, n in native.take_profile()]
    bpe = bytes_per_element(pol.kind, 4)
    ms = []
    for _ in range(reps):
        step()
        # the step released its gradients (grad_reset="none"): give every
        # parameter one again outside the timed sequence, so the replayed
        # launches allocate nothing
        for p in g.parameters:
            if p.value.grad is None:
                p.value.grad = torch.randn_like(p.value) * 0.01
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(eng.stream):
            torch.cuda._sleep(20_000_000)
            e0.record(eng.stream)
            for gi in range(native.num_groups):
                native.launch_group(gi, sync=False)   # queued behind the sleep: kernel time only
            e1.record(eng.stream)
        native.join()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    n = len(elems)
    t = statistics.median(ms) / 1e3
    tot_bytes = sum(elems) * bpe
    gbs = tot_bytes / t / 1e9
    # and live: events around every launch while it runs beside a real backward
    # (eager iterations; the durations include the contention with backward)
    native.set_profile(True)
    for _ in range(reps):
        step()
    native.set_profile(False)
    torch.cuda.synchronize()
    live = native.take_profile()
    live_ms = sum(m for m, _ in live)
    live_bytes = sum(e for _, e in live) * bpe
    live_gbs = live_bytes / (live_ms / 1e3) / 1e9 if live_ms else 0.0
    return {"launches_per_step": n, "avg_bytes": tot_bytes / n, "avg_us": t / n * 1e6,
            "achieved_gbs": gbs, "frac": gbs / peaks["hbm_gbs"],
            "live_beside_backward": {"avg_us": round(live_ms / max(len(live), 1) * 1e3, 3),
                                     "achieved_gbs": round(live_gbs, 1),
                                     "frac": round(live_gbs / peaks["hbm_gbs"], 4),
                                     "launches": len(live)}}


def measure_in_graph(args, device, peaks, flush, reps: int = 20) -> dict:
    """The headline's update launches timed live inside the replayed CUDA
    graph: with the engine's profile mode on during capture, a timing event
    pair around each launch becomes a pair of event-record nodes on the update
    stream, re-recorded by every replay (concurrent with the backward, as in
    the timed steps)."""
    import torch

    import paper_2104_00237_b200 as of
    from paper_2104_00237_b200.graphs import CapturedStep
    from paper_2104_00237_b200.models import synthetic_batch
    from paper_2104_00237_b200.optim import bytes_per_element
    wl = WORKLOADS["c2"]
    g = of.build_classifier(wl["model"], device=device, channels_last=bool(args.channels_last))
    g.track_counts = False
    pol = of.OptimizerPolicy(wl["kind"], **wl["hp"], grad_reset=args.grad_reset)
    x, y = synthetic_batch(wl["model"], args.batch, device=device)
    if args.channels_last:
        x = x.contiguous(memory_format=torch.channels_last)

    def run(inp):
        return of.run_backward_fusion(g, pol, inp, workers=args.workers, timing=False,
                                      bucket_elems=args.bucket_elems).loss
    for _ in range(3):
        run((x, y))
    eng = next(e for k, e in g._engines.items() if k[1])
    native = eng.native
    native.take_profile()
    native.set_profile(True)
    cap = CapturedStep(run, (x, y), policy=pol, graph=g, warmup=1)
    native.set_profile(False)
    n = native.num_groups
    ms, elems = [], []
    for _ in range(reps):
        flush()
        cap()
        torch.cuda.synchronize()
        rec = native.peek_profile(n)
        ms.append(sum(m for m, _ in rec))
        elems = [e for _, e in rec]
    native.take_profile()
    del cap
    t = statistics.median(ms) / 1e3
    tot_bytes = sum(elems) * bytes_per_element(pol.kind, 4)
    gbs = tot_bytes / t / 1e9
    return {"launches_per_step": n, "avg_bytes": tot_bytes / n, "avg_us": t / n * 1e6,
            "achieved_gbs": gbs, "frac": gbs / peaks["hbm_gbs"],
            "replays": reps, "step_us_min_max": [round(min(ms) * 1e3, 3), round(max(ms) * 1e3, 3)]}


def cpu_baseline(args, iters: int) -> dict:
    from oracle import timing
    r = timing.cpu_training_sample(args.model, args.batch, iters, "sgd-momentum",
                                   dict(eta=0.1, alpha=0.9, weight_decay=5e-4))
    return {"value": round(r["images_per_s"], 3), "unit": UNIT, "cores": r["threads"],
            "kind": "port",
            "sample": (f"{iters} iterations at batch {args.batch}: torch-CPU forward/backward on "
                       f"{r['threads']} threads ({r['fwd_bwd_ms']:.0f} ms) + reference update "
                       f"(oracle port of optim.py, numpy, 1 thread, {r['update_ms']:.1f} ms "
                       f"over {r['update_elems']} params)")}


def cpu_update_baseline(std: dict) -> dict:
    """The reference update alone on this host (numpy oracle port, 1 thread)
    next to the kernel's standalone pass over each config's parameter set."""
    from oracle import timing
    rates = {"sgd-momentum": timing.reference_update_rate("sgd-momentum",
                                                         dict(eta=0.1, alpha=0.9, weight_decay=5e-4)),
             "adam": timing.reference_update_rate("adam", dict(eta=1e-4, weight_decay=1e-4))}
    out = {"kind": "port", "cores": 1, "rates": rates, "configs": {}}
    for name, kind in (("vgg16_adam", "adam"), ("bert_base_adamw", "adam"),
                       ("resnet50_bf16_master_adamw", "adam"), ("mobilenet_v2_sgdm", "sgd-momentum")):
        if name not in std:
            continue
        elems = std[name]["bytes"] / 28 if kind == "adam" else std[name]["bytes"] / 20
        cpu_ms = elems / rates[kind]["elems_per_s"] * 1e3
        out["configs"][name] = {"cpu_ms": round(cpu_ms, 1), "gpu_us": std[name]["us"],
                                "ratio": round(cpu_ms * 1e3 / std[name]["us"], 1)}
    return out


def _variants_c2(world: int, dp_graphs: bool = False):
    """(name, schedule, workers, grad_reset, torch optimizer, bucket, CUDA graph, channels-last)"""
    K = 1 << 18
    LB = "fwd+bwd only (no update: lower bound)"
    v = [("torch.optim.SGD(foreach)", "baseline", None, None, "foreach", None, False, False),
         (LB, "baseline", None, None, "none", None, False, False),
         ("graph:" + LB, "baseline", None, None, "none", None, True, False),
         ("cl:graph:" + LB, "baseline", None, None, "none", None, True, True),
         ("torch.optim.SGD(fused)", "baseline", None, None, "fused", None, False, False),
         ("ours:baseline", "baseline", None, None, None, None, False, False),
         ("ours:forward-fusion(per-layer)", "forward-fusion", None, None, None, 0, False, False),
         ("ours:forward-fusion(bucket=256K)", "forward-fusion", None, None, None, K, False, False),
         ("ours:backward-fusion(w=1,per-layer)", "backward-fusion", 1, None, None, 0, False, False),
         ("ours:backward-fusion(w=2,per-layer)", "backward-fusion", 2, None, None, 0, False, False),
         ("ours:backward-fusion(w=1,bucket=256K)", "backward-fusion", 1, None, None, K, False, False),
         ("ours:backward-fusion(w=2,bucket=256K)", "backward-fusion", 2, None, None, K, False, False),
         ("ours:backward-fusion(w=2,bucket=256K,zero)", "backward-fusion", 2, "zero", None, K, False, False),
         ("graph:torch.optim.SGD(foreach)", "baseline", None, None, "foreach", None, True, False),
         ("graph:torch.optim.SGD(fused)", "baseline", None, None, "fused", None, True, False),
         ("graph:ours:baseline", "baseline", None, None, None, None, True, False),
         ("graph:ours:forward-fusion(bucket=256K)", "forward-fusion", None, None, None, K, True, False),
         ("graph:ours:backward-fusion(w=2,per-layer)", "backward-fusion", 2, None, None, 0, True, False),
         ("graph:ours:backward-fusion(w=2,bucket=256K)", "backward-fusion", 2, None, None, K, True, False),
         ("cl:torch.optim.SGD(foreach)", "baseline", None, None, "foreach", None, False, True),
         ("cl:ours:backward-fusion(w=2,bucket=256K)", "backward-fusion", 2, None, None, K, False, True),
         ("cl:graph:torch.optim.SGD(foreach)", "baseline", None, None, "foreach", None, True, True),
         ("cl:graph:ours:backward-fusion(w=2,bucket=256K)", "backward-fusion", 2, None, None, K, True, True),
         ("cl:graph:ours:forward-fusion(bucket=256K)", "forward-fusion", None, None, None, K, True, True),
         ("cl:graph:ours:backward-fusion(w=2,bucket=1M)", "backward-fusion", 2, None, None, 4 * K, True, True),
         ("cl:graph:ours:backward-fusion(w=2,bucket=4M)", "backward-fusion", 2, None, None, 16 * K, True, True),
         ("cl:graph:ours:backward-fusion(w=1,bucket=256K)", "backward-fusion", 1, None, None, K, True, True),
         ("cl:graph:ours:forward-fusion(bucket=1M)", "forward-fusion", None, None, None, 4 * K, True, True),
         ("cl:graph:ours:forward-fusion(bucket=256K,prefetch)", "forward-fusion", 2, None, None, K, True, True),
         ("cl:graph:ours:forward-fusion(bucket=256K,prefetch=all)", "forward-fusion", -3, None, None, K, True, True),
         ("ours:forward-fusion(bucket=256K,prefetch)", "forward-fusion", 2, None, None, K, False, False)]
    if world > 1 and not dp_graphs:
        v = [x for x in v if not x[6]]
    return v


KEY_ROWS = ("torch.optim.SGD(foreach)", "ours:backward-fusion(w=2,bucket=256K)",
            "ours:forward-fusion(bucket=256K)", "graph:torch.optim.SGD(foreach)",
            "graph:ours:backward-fusion(w=2,bucket=256K)", "cl:graph:torch.optim.SGD(foreach)",
            "cl:graph:ours:backward-fusion(w=2,bucket=256K)", "cl:graph:ours:forward-fusion(bucket=256K)",
            "cl:graph:ours:backward-fusion(w=2,bucket=1M)",
            # the floors vary with cuDNN's per-instance algorithm choice as much as the rows
            "fwd+bwd only (no update: lower bound)", "graph:fwd+bwd only (no update: lower bound)",
            "cl:graph:fwd+bwd only (no update: lower bound)")
SWEEP_ROWS = ("torch.optim.SGD(foreach)", "ours:forward-fusion(bucket=256K)",
              "graph:fwd+bwd only (no update: lower bound)",
              "ours:backward-fusion(w=2,bucket=256K)", "graph:torch.optim.SGD(foreach)",
              "graph:ours:backward-fusion(w=2,bucket=256K)", "graph:ours:forward-fusion(bucket=256K)")


def _speedups(row: dict) -> None:
    """Speed-ups against the matching unfused torch baseline (same graph /
    layout mode), and the share of the unfused update phase each schedule
    hides when a forward+backward-only row (the lower bound) is present."""
    def torch_row(prefix):
        for opt in ("SGD", "Adam", "AdamW"):
            r = row.get(f"{prefix}torch.optim.{opt}(foreach)")
            if r:
                return r
        return None
    eager = torch_row("")
    for k, v in row.items():
        mode = k.rsplit("ours:", 1)[0] if "ours:" in k else k.split("torch.optim", 1)[0] \
            if "torch.optim" in k else k.split("fwd+bwd", 1)[0]
        base = torch_row(mode)
        if base:
            v["speedup_vs_unfused_same_mode"] = round(base["ms_per_step"] / v["ms_per_step"], 4)
        if eager:
            v["speedup_vs_eager_torch_foreach"] = round(eager["ms_per_step"] / v["ms_per_step"], 4)
        lb = row.get(mode + "fwd+bwd only (no update: lower bound)")
        if base and lb and k.startswith(mode + "ours:"):
            phase = base["ms_per_step"] - lb["ms_per_step"]
            if phase > 0:
                v["unfused_update_phase_hidden"] = round((base["ms_per_step"] - v["ms_per_step"]) / phase, 3)


def run_ours(args) -> dict:
    import torch

    from paper_2104_00237_b200 import _native
    dist = Dist().init("nccl", force=args.force_dp)
    device = torch.device("cuda", dist.local)
    torch.cuda.set_device(device)
    torch.backends.cudnn.benchmark = True
    # try every cuDNN algorithm: with the default limit (10) the choice varies
    # between model instances and ~1 instance in 4 lands 5-8% off the others
    # (tools/cudnn_variance.py); with 0 every instance of every arm agrees
    torch.backends.cudnn.benchmark_limit = 0
    # fp32 training on B200 the usual way: TF32 tensor cores for matmuls as
    # well as convolutions (cuDNN's default), for every arm alike
    torch.backends.cuda.matmul.allow_tf32 = True
    peaks = load_peaks()
    args.world = dist.world
    args.dp = dist.world > 1 or args.force_dp
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    flush = flush_buf.zero_

    # cuDNN picks per model instance; timings are stable within an instance but
    # differ by up to ~7% between instances (both arms), so the headline is the
    # median over --instances independently built instances, each timed for
    # exactly K steps after W warm-up steps.
    inst = []
    dp_graph_error = None
    with Clocks(dist.local) as clk:
        for _ in range(args.instances):
            try:
                step, g, pol = make_runner(args, args.batch, args.schedule, device)
            except Exception as e:  # noqa: BLE001
                if not (args.dp and args.dp_graphs):
                    raise
                # data-parallel capture failed: measure the eager data-parallel step
                args.dp_graphs = 0
                dp_graph_error = f"{type(e).__name__}: {str(e).splitlines()[0][:160] if str(e) else ''}"
                torch.cuda.synchronize()
                step, g, pol = make_runner(args, args.batch, args.schedule, device)
            n0 = _native.launch_count()
            inst.append(timed(step, args.steps, args.warmup, dist, flush))
            if hasattr(step, "native_launches"):   # CUDA graph: kernel nodes replayed per step
                launches = step.native_launches * args.steps
            else:
                launches = (_native.launch_count() - n0) * args.steps // (args.steps + args.warmup)
            del step, g, pol
            torch.cuda.empty_cache()
    ms = statistics.median(inst)
    clocks = clk.summary()
    value = dist.world * args.batch * 1e3 / ms
    res = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": dist.world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (x~N(0,1) [b,3,32,32], y~U{0..9}; random-init weights)",
           "config": {"workload": WORKLOAD, "model": args.model, "batch_per_gpu": args.batch,
                      "global_batch": args.batch * dist.world, "schedule": args.schedule,
                      "workers": args.workers, "grad_reset": args.grad_reset,
                      "bucket_elems": args.bucket_elems,
                      "cuda_graph": bool(args.graphs) and (not args.dp or bool(args.dp_graphs)),
                      "channels_last": bool(args.channels_last),
                      "parallelism": f"dp{dist.world}",
                      "dp_path": (("sharded fused update: per-bucket NCCL reduce-scatter -> update "
                                   "-> all-gather" if args.dp_transport == "nccl" else
                                   "fused peer-memory kernel per bucket (reduce-scatter + update + "
                                   "all-gather in one kernel over symmetric memory)")
                                  + "; unfused baseline DDP + torch.optim" if args.dp else None),
                      "l2": "256 MiB buffer zeroed before every timed step (outside each step's event pair)",
                      "model_math": ("fp32 parameters/activations; TF32 tensor cores for convolutions "
                                     f"(cudnn.allow_tf32={torch.backends.cudnn.allow_tf32}) and matmuls "
                                     f"(matmul.allow_tf32={torch.backends.cuda.matmul.allow_tf32}); "
                                     "optimizer update exact fp32 (reference arithmetic)")},
           "gpu_launches": int(launches)}
    res["config"]["instances_ms_per_step"] = [round(t, 4) for t in inst]
    if dp_graph_error:
        res["config"]["dp_graph_capture_failed"] = dp_graph_error
    if not args.no_extras:
        sched, failed = {}, {}
        for b in [args.batch] + [int(x) for x in args.sweep.split(",") if x.strip()]:
            row = {}
            for name, sch, w, gr, opt, be, gph, cl in _variants_c2(2 if args.dp else 1, bool(args.dp_graphs)):
                if b != args.batch and name not in SWEEP_ROWS:
                    continue
                ts = []
                try:
                    for _ in range(args.instances if name in KEY_ROWS else 1):
                        st, *_ = make_runner(args, b, sch, device, workers=w, grad_reset=gr,
                                             opt_impl=opt, bucket_elems=be, graphed=gph,
                                             channels_last=cl)
                        ts.append(timed(st, args.steps, args.warmup, dist, flush))
                        del st
                        torch.cuda.empty_cache()
                except Exception as e:  # noqa: BLE001 -- report, keep the other rows
                    failed[f"{b}:{name}"] = f"{type(e).__name__}: {str(e).splitlines()[0][:160] if str(e) else ''}"
                    torch.cuda.synchronize()
                    continue
                t = statistics.median(ts)
                row[name] = {"ms_per_step": round(t, 4), "images_per_s": round(dist.world * b * 1e3 / t, 1)}
                if len(ts) > 1:
                    row[name]["instances_ms"] = [round(x, 4) for x in ts]
            _speedups(row)
            sched[str(b)] = row
        res["schedules"] = sched
        if failed:
            res["failed_rows"] = failed
        row = sched.get(str(args.batch), {})
        headline_graphed = bool(args.graphs) and (not args.dp or bool(args.dp_graphs))
        mode = (("cl:" if args.channels_last else "")
                + ("graph:" if headline_graphed else ""))
        same = row.get(mode + "torch.optim.SGD(foreach)") or row.get("torch.optim.SGD(foreach)")
        eager = row.get("torch.optim.SGD(foreach)")
        lb = row.get(mode + "fwd+bwd only (no update: lower bound)")
        res["vs_unfused_torch"] = {
            "mode": mode or "eager",
            "torch_foreach_ms": same["ms_per_step"] if same else None,
            "speedup": round(same["ms_per_step"] / ms, 4) if same else None,
            "fwd_bwd_only_ms": lb["ms_per_step"] if lb else None,
            "speedup_vs_eager_torch_foreach": round(eager["ms_per_step"] / ms, 4) if eager else None}
        for wl, key in (("c1", "c1_resnet18_sgdm"), ("c3", "c3_vgg16_adam"),
                        ("c4", "c4_resnet50_bf16_adamw"), ("c5", "c5_bert_base_adamw")):
            if wl in args.extras.split(","):
                res[key] = run_extra(args, wl, device, dist, flush)
        res["e2e"] = e2e(args, device, dist, flush)
        # the kernel's own duration is a per-GPU quantity: measured on this
        # GPU's single-process engine whatever the world size
        world, dp, args.world, args.dp = args.world, args.dp, 1, False
        try:
            ins = measure_in_situ(args, device, peaks, 5)
            live = measure_in_graph(args, device, peaks, flush) if args.graphs else None
        finally:
            args.world, args.dp = world, dp
        std = measure_update_kernel(args, device, peaks)
        tr = ncu_traffic("c2_backward_fusion_buckets")
        prim = live or ins
        res["roofline"] = {"bound": "hbm", "kernel": "mt_step_kernel (backward-fusion, side stream)",
                           "achieved": round(prim["achieved_gbs"], 1), "peak": peaks["hbm_gbs"],
                           "unit": "GB/s", "frac": round(prim["frac"], 4),
                           "method": ("CUDA events captured as event-record nodes around each "
                                      "update launch, read after every replay of the headline "
                                      "graph (live, beside the backward)") if live else
                                     "one iteration's launches replayed back to back",
                           "in_graph_live": ({"avg_bytes": round(live["avg_bytes"]),
                                              "avg_us": round(live["avg_us"], 3),
                                              "launches_per_step": live["launches_per_step"]}
                                             if live else None),
                           "traffic": (tr or {}).get("dram_bytes_per_launch"),
                           "traffic_source": (tr or {}).get("source"),
                           "peak_source": peaks["source"],
                           "replayed_back_to_back": {
                               "avg_bytes": round(ins["avg_bytes"]), "avg_us": round(ins["avg_us"], 3),
                               "launches_per_step": ins["launches_per_step"],
                               "frac": round(ins["frac"], 4),
                               "method": "one iteration's launches replayed back to back on their "
                                         "stream after an eager step, one event pair"},
                           "live_eager_beside_backward": ins["live_beside_backward"],
                           "standalone_single_launch": std}
        if dist.rank == 0 and dist.world == 1:
            res["cpu_baseline"] = cpu_baseline(args, args.cpu_iters)
            res["cpu_update_baseline"] = cpu_update_baseline(std)
            from oracle import timing
            res["cpu_harness_baseline"] = dict(timing.reference_harness_breakdown(), kind="port")
    res["clocks"] = clocks
    dist.close()
    return res


OWN_LB = "fwd+bwd only (bf16 module as ours: lower bound for ours)"


def _variants_extra(wl: str):
    """(name, schedule, workers, torch optimizer, bucket, CUDA graph) for the extras."""
    opt = WORKLOADS[wl]["torch"][0]
    LB = "fwd+bwd only (no update: lower bound)"
    v = [(f"torch.optim.{opt}(foreach)", "baseline", None, "foreach", 0, False),
         (f"torch.optim.{opt}(fused)", "baseline", None, "fused", 0, False),
         (LB, "baseline", None, "none", 0, False),
         ("ours:baseline", "baseline", None, None, 0, False),
         ("ours:forward-fusion(per-layer)", "forward-fusion", None, None, 0, False),
         ("ours:backward-fusion(w=2,per-layer)", "backward-fusion", 2, None, 0, False),
         ("ours:backward-fusion(w=2,per-layer,default-prio)", "backward-fusion", -2, None, 0, False),
         # inline on the autograd stream: each update right behind its layer's backward,
         # gradients (and the weights dgrad just read) still in L2 -- the paper's locality
         ("ours:backward-fusion(w=1,per-layer)", "backward-fusion", 1, None, 0, False)]
    if WORKLOADS[wl].get("mixed"):
        v.append((OWN_LB, "baseline", None, "none-mixed", 0, False))
    if wl == "c3":
        v.append(("ours:backward-fusion(w=2,per-layer,capped)", "backward-fusion", -1, None, 0, False))
    else:
        v.append(("ours:forward-fusion(bucket=1M)", "forward-fusion", None, None, 1 << 20, False))
        v.append(("ours:forward-fusion(bucket=1M,prefetch)", "forward-fusion", 2, None, 1 << 20, False))
        v.append(("ours:backward-fusion(w=2,bucket=1M)", "backward-fusion", 2, None, 1 << 20, False))
    # the same iteration captured as one CUDA graph (Adam/AdamW replay through
    # the device-side step index; torch's Adam with capturable=True)
    v += [(f"graph:torch.optim.{opt}(foreach)", "baseline", None, "foreach", 0, True),
          (f"graph:torch.optim.{opt}(fused)", "baseline", None, "fused", 0, True),
          ("graph:" + LB, "baseline", None, "none", 0, True),
          ("graph:ours:baseline", "baseline", None, None, 0, True),
          ("graph:ours:forward-fusion(bucket=1M)", "forward-fusion", None, None, 1 << 20, True),
          ("graph:ours:forward-fusion(bucket=1M,prefetch)", "forward-fusion", 2, None, 1 << 20, True),
          ("graph:ours:backward-fusion(w=2,bucket=1M)", "backward-fusion", 2, None, 1 << 20, True),
          ("graph:ours:backward-fusion(w=1,per-layer)", "backward-fusion", 1, None, 0, True)]
    if WORKLOADS[wl].get("mixed"):
        v.append(("graph:" + OWN_LB, "baseline", None, "none-mixed", 0, True))
    return v


def run_extra(args, wl: str, device, dist, flush) -> dict:
    """One of BASELINE.json's other configs on this GPU, eager and captured as
    CUDA graphs: C1 ResNet-18/CIFAR SGD-momentum, C3 VGG-16 Adam (the
    update-bound case), C4 ResNet-50 bf16 + fp32 masters AdamW, C5 BERT-base
    AdamW."""
    import torch
    b = WORKLOADS[wl]["batch"]
    steps, warm = max(args.steps // 3, 5), 3
    row, failed = {}, {}
    for name, sch, w, opt, be, gph in _variants_extra(wl):
        if gph and args.dp and not args.dp_graphs:
            continue
        try:
            st, *_ = make_runner(args, b, sch, device, workers=w, opt_impl=opt, bucket_elems=be,
                                 graphed=gph, workload=wl, channels_last=wl in ("c4",))
            t = timed(st, steps, warm, dist, flush)
        except Exception as e:  # noqa: BLE001 -- report, keep the other rows
            failed[name] = f"{type(e).__name__}: {str(e).splitlines()[0][:160] if str(e) else ''}"
            torch.cuda.synchronize()
            continue
        row[name] = {"ms_per_step": round(t, 3), "images_per_s": round(dist.world * b * 1e3 / t, 1)}
        del st
        torch.cuda.empty_cache()
    _speedups(row)
    out = {"workload": WORKLOADS[wl]["desc"], "batch_per_gpu": b, "steps": steps, "warmup": warm}
    for mode in ("", "graph:"):
        lb = row.pop(mode + "fwd+bwd only (no update: lower bound)", None)
        own = row.pop(mode + OWN_LB, None)
        key = mode.rstrip(":") or "eager"
        if lb is not None:
            out[f"fwd_bwd_only_ms_{key}"] = lb["ms_per_step"]
        if own is not None:
            # different model math (bf16 module vs fp32 + autocast): ours is judged
            # against its own forward+backward floor, not the torch phase
            out[f"fwd_bwd_only_ms_ours_math_{key}"] = own["ms_per_step"]
            for k, v in row.items():
                if k.startswith(mode + "ours:"):
                    v.pop("unfused_update_phase_hidden", None)
                    v["over_own_fwd_bwd_ms"] = round(v["ms_per_step"] - own["ms_per_step"], 3)
    out["schedules"] = row
    if failed:
        out["failed"] = failed
    return out


def e2e(args, device, dist, flush=None) -> dict:
    """The headline configuration through the public API, end to end: each
    step copies the batch from pinned host memory to the device and reads the
    loss back (CapturedStep copies into its static buffers, then replays).
    Wall clock over the K steps less the device-timed L2 flushes (one before
    every step, like the device-timed value), max over ranks."""
    import torch

    from paper_2104_00237_b200.models import synthetic_batch
    xh, yh = synthetic_batch(args.model, args.batch, device="cpu", seed=1)
    xh, yh = xh.pin_memory(), yh.pin_memory()
    vals = []
    for _ in range(max(1, args.instances)):    # median over instances, like the headline
        vals.append(_e2e_instance(args, device, dist, flush, xh, yh))
        torch.cuda.empty_cache()
    return {"value": round(statistics.median(vals), 2), "unit": UNIT,
            "h2d_bytes_per_step": xh.numel() * xh.element_size() + yh.numel() * yh.element_size(),
            "d2h_bytes_per_step": 4, "instances": [round(v, 1) for v in vals]}


def _e2e_instance(args, device, dist, flush, xh, yh) -> float:
    """Every step: the batch copied in from pinned host memory (graphed: staged
    on a copy stream while the previous replay runs, CapturedStep.stage), the
    iteration, the loss copied out to pinned host memory and read on the host.  Step k's
    loss is read while step k+1 runs (a two-slot pinned ring and an event per
    step), so the host never idles the GPU between steps."""
    import torch
    step, g, pol = make_runner(args, args.batch, args.schedule, device)
    graphed = hasattr(step, "graph")
    run = None if graphed else step.run
    ring = [torch.empty((), dtype=torch.float32).pin_memory() for _ in range(2)]
    events = [torch.cuda.Event(), torch.cuda.Event()]
    losses = []
    # the L2 flush between steps is device-timed and taken out of the wall clock
    fl = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(max(args.steps, args.warmup))]

    def one(k):
        if flush is not None:
            fl[k][0].record()
            flush()
            fl[k][1].record()
        if graphed:
            # this step's batch was staged (host -> device on the step's copy
            # stream) while the previous replay ran; stage the next one now
            if not step.staged:
                step.stage((xh, yh))
            loss = step()
            step.stage((xh, yh))
        else:
            loss = run((xh.to(device, non_blocking=True), yh.to(device, non_blocking=True)))
        ring[k % 2].copy_(loss.detach().float(), non_blocking=True)
        events[k % 2].record()
        if k > 0:                      # the previous step's loss, read on the host now
            events[(k - 1) % 2].synchronize()
            losses.append(float(ring[(k - 1) % 2]))

    def drain(k):
        events[(k - 1) % 2].synchronize()
        losses.append(float(ring[(k - 1) % 2]))
    for k in range(args.warmup):
        one(k)
    drain(args.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    losses.clear()
    t0 = time.perf_counter()
    for k in range(args.steps):
        one(k)
    drain(args.steps)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if flush is not None:
        dt -= sum(a.elapsed_time(b) for a, b in fl[:args.steps]) / 1e3
    dt = dist.max(dt)
    assert len(losses) == args.steps and all(v == v for v in losses), "e2e: a loss was not read"
    return dist.world * args.batch * args.steps / dt


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args) -> dict | None:
    dist = Dist()
    if dist.rank != 0:
        return None
    from oracle import timing
    kw = dict(eta=0.1, alpha=0.9, weight_decay=5e-4)
    timing.cpu_training_sample(args.model, args.batch, 1, "sgd-momentum", kw)  # warm-up
    r = timing.cpu_training_sample(args.model, args.batch, max(args.steps, 1), "sgd-momentum", kw)
    v = round(r["images_per_s"], 3)
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(r["ms_per_iter"], 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": {"workload": WORKLOAD, "model": args.model,
                                             "batch_per_gpu": args.batch, "schedule": "baseline"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["threads"], "kind": "port",
                             "sample": (f"each step: one iteration at batch {args.batch}, "
                                        f"torch-CPU fwd/bwd on {r['threads']} threads + the "
                                        f"reference update (numpy oracle port, 1 thread)")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main(argv=None):
    args = parse_args(argv)
    if args.impl == "reference":
        res = run_reference(args)
    else:
        res = run_ours(args)
    if res is not None and int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
