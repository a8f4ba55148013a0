#!/usr/bin/env python
"""Benchmark: fused vs unfused training iterations on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (N=1): configs[1] of BASELINE.json -- MobileNetV2 on synthetic
CIFAR-10-shaped data (3x32x32, 10 classes), SGD-momentum (lr 0.1, momentum
0.9, weight decay 5e-4), true fp32 (TF32 off for convolutions and matmuls),
batch 128 per GPU, channels-last, backward fusion with 1M-element buckets on
the side stream, the whole iteration replayed from a CUDA graph.  One "step"
= one training iteration (forward, backward, every parameter updated), with a
256 MiB L2 flush before it (outside its event pair).  Its same-mode
comparators -- our own unfused update (ours:baseline), forward fusion,
torch.optim.SGD (foreach, fused) and forward+backward with no update (the
floor any fusion can reach) -- are built --instances times each, interleaved
instance by instance, and every row is the median over its instances.
N>1 (torchrun): the data-parallel path (dp.py, NCCL reduce-scatter ->
sharded update -> all-gather per bucket, captured in the graph) against
DDP + torch.optim; --force-dp runs that path at N=1.

Prints ONE compact JSON line (rank 0, < 2 KB).  ``value`` = images/s over all
ranks with inputs resident in HBM, device-timed with CUDA events (max over
ranks); ``unfused`` = the comparators' medians and the speed-ups against
them; ``e2e`` = the same step through the public API with pinned-host inputs
copied in and the loss read back every step; ``roofline`` = the update
kernel's average launch duration, timed live inside the replayed headline
graph, as algorithmic HBM bandwidth against MEASURED_PEAKS.json, with the ncu
DRAM traffic per launch (profiles/ncu_traffic.json); ``cpu_baseline`` = the
reference's CPU path (oracle port) on the host cores.  Every row, instance
and diagnostic (batch sweep --sweep, the other configs --extras c1,c3,c4,c5,
standalone single-launch rooflines) goes to --extras-out.

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

if int(os.environ.get("WORLD_SIZE", "1")) > 1 or "--force-dp" in sys.argv:
    # NCCL reads its debug settings when the library loads (with torch), so
    # they are set here, before any import of torch: rank 0's communicator
    # lines (ranks, transport, NVLS) go to stdout ahead of the result line --
    # the process group is destroyed before that line is printed -- and the
    # other ranks stay quiet, so the result stays the last stdout line
    # (the GPU image presets NCCL_DEBUG=VERSION, so a lower level is raised).
    # NCCL writes them to a file that main() echoes before the result: NCCL
    # logs once more while the process exits, after anything printed here.
    if os.environ.get("RANK", "0") == "0" and \
            os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
        import tempfile
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
        os.environ["NCCL_DEBUG_FILE"] = os.path.join(tempfile.gettempdir(),
                                                     f"optfuse_bench_nccl_{os.getpid()}.log")
        NCCL_LOG = os.environ["NCCL_DEBUG_FILE"]
NCCL_LOG = globals().get("NCCL_LOG")

METRIC = "train iter time & images/sec (fused vs unfused) at 1/2/4/8 B200; update HBM GB/s"
UNIT = "images/s"

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
    ap.add_argument("--graphs", type=int, default=1,
                    help="1: capture each iteration (ours and the torch baseline) as a CUDA graph")
    ap.add_argument("--channels-last", type=int, default=1, help="1: NHWC model and inputs")
    ap.add_argument("--tf32", type=int, default=0,
                    help="1: TF32 tensor cores for convolutions and matmuls (every arm; the line "
                         "then says dtype tf32).  Default 0: true fp32")
    ap.add_argument("--dp-graphs", type=int, default=1,
                    help="1: capture data-parallel iterations (NCCL collectives included) as CUDA "
                         "graphs too (0: eager data parallel)")
    ap.add_argument("--dp-transport", default="nccl", choices=("nccl", "peer"),
                    help="data parallel: NCCL reduce-scatter/all-gather around the sharded kernel, "
                         "or the fused peer-memory kernel over torch symmetric memory")
    ap.add_argument("--force-dp", action="store_true",
                    help="run the data-parallel code path (NCCL process group, DataParallelFusion, "
                         "DDP baselines) even at one GPU: the N>1 path's smoke test")
    ap.add_argument("--instances", type=int, default=5,
                    help="independently built instances of every arm, interleaved; rows are medians")
    ap.add_argument("--sweep", default="", help="extra per-GPU batches, e.g. 32,64,256,512")
    ap.add_argument("--extras", default="",
                    help="other BASELINE.json configs to time, e.g. c1,c3,c4,c5 (written to --extras-out)")
    ap.add_argument("--standalone", type=int, default=1,
                    help="1: standalone single-launch roofline of the C2-C5 parameter sets (extras)")
    ap.add_argument("--extras-out", default="gpurun_out/bench_extras.json",
                    help="where every row, instance and diagnostic goes ('' = nowhere); the "
                         "printed line stays compact")
    ap.add_argument("--in-situ", type=int, default=1,
                    help="1: also time the C3 (VGG-16 Adam) backward-fusion launches live (roofline.in_situ_c3_large)")
    ap.add_argument("--headline-only", action="store_true",
                    help="time the headline arm only, nothing else (for profilers)")
    ap.add_argument("--cpu-iters", type=int, default=10, help="CPU baseline: timed iterations")
    ap.add_argument("--cpu-warmup", type=int, default=2, help="CPU baseline: warm-up iterations")
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
    "c5m": {"model": "bert_base", "batch": 32, "kind": "adamw", "mixed": True,
            "hp": {"eta": 1e-4, "weight_decay": 0.01},
            "torch": ("AdamW", {"lr": 1e-4, "weight_decay": 0.01}),
            "desc": ("BERT-base pre-training, seq 128, batch 32, AdamW (wd 0.01), bf16 module with "
                     "fp32 master weights (ours; torch: fp32 params under autocast bf16); adds the "
                     "consumer-fused rows (Linear weights updated inside their wgrad GEMM)")},
    "c5": {"model": "bert_base", "batch": 32, "kind": "adamw",
           "hp": {"eta": 1e-4, "weight_decay": 0.01},
           "torch": ("AdamW", {"lr": 1e-4, "weight_decay": 0.01}),
           "desc": ("BERT-base pre-training (BertForPreTraining, random init), seq 128, batch 32, "
                    "15% MLM labels + NSP, AdamW (wd 0.01), fp32 weights (TF32 matmuls)")},
}


def make_runner(args, batch: int, schedule: str, device, seed=0, workers=None,
                grad_reset=None, opt_impl=None, bucket_elems=None, graphed=None,
                workload="c2", channels_last=None, consumer=False):
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
            cf = None
            if consumer:   # Linear weights updated inside their wgrad GEMM (tcgen05)
                from paper_2104_00237_b200.consumer import ConsumerFusion
                cf = ConsumerFusion(g, pol)

            def run(inp):
                return of.run_backward_fusion(g, pol, inp, workers=w, timing=False,
                                              bucket_elems=be, update_ctas=ctas,
                                              update_priority=prio, consumer=cf).loss
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


def measure_live_launches(args, wl: str, device, peaks, iters: int = 3) -> dict:
    """In-situ roofline of one config's backward-fusion launches (per layer,
    side stream, eager): a CUDA event pair around every update launch while it
    runs beside the backward (engine profile mode), algorithmic bytes of each
    launch / its duration.  Reported over all launches and over the large
    ones (>= 64 MB: the update-bound layers, e.g. VGG-16's fc6 at 2.9 GB)."""
    import torch

    from paper_2104_00237_b200.optim import bytes_per_element_of
    world, dp, args.world, args.dp = getattr(args, "world", 1), getattr(args, "dp", False), 1, False
    try:
        step, g, pol = make_runner(args, WORKLOADS[wl]["batch"], "backward-fusion", device, workers=2,
                                   bucket_elems=0, graphed=False, workload=wl,
                                   channels_last=wl in ("c4",))
    finally:
        args.world, args.dp = world, dp
    for _ in range(3):
        step()
    eng = next(e for k, e in g._engines.items() if k[1])
    eng.native.take_profile()
    eng.native.set_profile(True)
    for _ in range(iters):
        step()
    eng.native.set_profile(False)
    torch.cuda.synchronize()
    rec = eng.native.take_profile()
    bpe = bytes_per_element_of(pol.kind, g.parameters[0])

    def summ(rows):
        if not rows:
            return None
        b = sum(n for _, n in rows) * bpe
        t = sum(ms for ms, _ in rows) / 1e3
        return {"launches": len(rows) // iters, "bytes_per_step": b // iters,
                "achieved_gbs": round(b / t / 1e9, 1), "frac": round(b / t / 1e9 / peaks["hbm_gbs"], 4)}
    big = max(rec, key=lambda r: r[1])
    out = {"all": summ(rec), "large": summ([r for r in rec if r[1] * bpe >= 64 << 20]),
           "largest_launch": {"bytes": big[1] * bpe, "us": round(big[0] * 1e3, 2),
                              "frac": round(big[1] * bpe / (big[0] / 1e3) / 1e9 / peaks["hbm_gbs"], 4)},
           "method": "event pair around each launch, side stream beside the eager backward"}
    del step, g, pol
    torch.cuda.empty_cache()
    return out


def cpu_baseline(args) -> dict:
    """The reference arm's measurement (same function, same workload) on a
    bounded sample: W warm-up + K timed iterations on all host cores."""
    from oracle import timing
    r = timing.cpu_training_sample(args.model, args.batch, args.cpu_iters, "sgd-momentum",
                                   dict(eta=0.1, alpha=0.9, weight_decay=5e-4),
                                   warmup=args.cpu_warmup)
    return {"value": round(r["images_per_s"], 3), "unit": UNIT, "cores": r["threads"],
            "kind": "port",
            "sample": (f"{args.cpu_warmup}+{args.cpu_iters} iterations at batch {args.batch}, "
                       f"pinned to {r['threads']} cores: torch-CPU fwd/bwd "
                       f"{r['fwd_bwd_ms']:.0f} ms + reference update (numpy oracle port of "
                       f"optim.py, 1 thread) {r['update_ms']:.1f} ms")}


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
        ours = row.get(mode + "ours:baseline")
        if ours and k.startswith(mode + "ours:") and k != mode + "ours:baseline":
            v["speedup_vs_ours_unfused"] = round(ours["ms_per_step"] / v["ms_per_step"], 4)
        lb = row.get(mode + "fwd+bwd only (no update: lower bound)")
        if base and lb and k.startswith(mode + "ours:"):
            phase = base["ms_per_step"] - lb["ms_per_step"]
            if phase > 0:
                v["unfused_update_phase_hidden"] = round((base["ms_per_step"] - v["ms_per_step"]) / phase, 3)


def _headline_name(args) -> str:
    if args.schedule == "baseline":
        return "ours:baseline"
    if args.schedule == "forward-fusion":
        return f"ours:forward-fusion(bucket={_kname(args.ff_bucket_elems)})"
    return f"ours:backward-fusion(w={args.workers},bucket={_kname(args.bucket_elems)})"


def _kname(n: int) -> str:
    if n <= 0:
        return "per-layer"
    return f"{n >> 20}M" if n % (1 << 20) == 0 else f"{n >> 10}K"


def headline_arms(args) -> list:
    """The headline and its same-mode comparators (same graph / layout mode,
    same model math), timed interleaved instance by instance:
    (row name, make_runner keyword arguments)."""
    arms = [(_headline_name(args), {})]
    if args.schedule != "baseline":
        arms.append(("ours:baseline", {"schedule": "baseline"}))
    if args.schedule != "forward-fusion":
        arms.append((f"ours:forward-fusion(bucket={_kname(1 << 18)})",
                     {"schedule": "forward-fusion", "bucket_elems": 1 << 18}))
    if args.schedule != "backward-fusion":
        arms.append((f"ours:backward-fusion(w=2,bucket={_kname(args.bucket_elems)})",
                     {"schedule": "backward-fusion", "workers": 2,
                      "bucket_elems": args.bucket_elems}))
    arms += [("torch.optim.SGD(foreach)", {"schedule": "baseline", "opt_impl": "foreach"}),
             ("torch.optim.SGD(fused)", {"schedule": "baseline", "opt_impl": "fused"}),
             (FLOOR, {"schedule": "baseline", "opt_impl": "none"})]
    if getattr(args, "dp", False) or getattr(args, "force_dp", False):
        # data parallel: the torch arms run under DDP, so the no-update arm is DDP's
        # forward + backward + gradient all-reduce -- a floor for the DDP arms only
        arms = [(FLOOR_DDP if n == FLOOR else "DDP+" + n if n.startswith("torch") else n, kw)
                for n, kw in arms]
    return arms


FLOOR = "fwd+bwd only (no update: lower bound)"
FLOOR_DDP = "DDP fwd+bwd+all-reduce only (no update; floor of the DDP arms)"


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
    # true fp32 (the reference's arithmetic): no TF32 tensor cores in any arm
    # unless --tf32 1 asks for the (labelled) TF32 variant
    torch.backends.cudnn.allow_tf32 = bool(args.tf32)
    torch.backends.cuda.matmul.allow_tf32 = bool(args.tf32)
    peaks = load_peaks()
    args.world = dist.world
    args.dp = dist.world > 1 or args.force_dp
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    flush = flush_buf.zero_

    # Every arm is built --instances times; the instances of all arms are
    # interleaved (instance i of every arm, then instance i+1), each timed for
    # exactly K steps after W warm-up steps; each row is the median over its
    # instances.  cuDNN picks per model instance, and the GPU drifts between
    # slow and fast windows, so interleaving keeps the
    # fused/unfused comparison inside the same windows.
    arms = headline_arms(args)
    if args.headline_only:
        arms = arms[:1]
    elif args.graphs and not args.dp:
        # the same fused / unfused pair eager (no CUDA graph): the host issues
        # every kernel there, and fusion hides its updates in the host's gaps
        arms += [("eager:" + n, dict(kw, graphed=False)) for n, kw in arms
                 if n in (arms[0][0], "ours:baseline", "torch.optim.SGD(foreach)")]
    times = {name: [] for name, _ in arms}
    head = arms[0][0]
    launches = 0
    dp_graph_error = None
    with Clocks(dist.local) as clk:
        for _ in range(args.instances):
            for name, kw in arms:
                kw = dict(kw)
                sched = kw.pop("schedule", args.schedule)
                try:
                    step, g, pol = make_runner(args, args.batch, sched, device, **kw)
                except Exception as e:  # noqa: BLE001
                    if not (args.dp and args.dp_graphs):
                        raise
                    # data-parallel capture failed: measure the eager data-parallel step
                    args.dp_graphs = 0
                    dp_graph_error = f"{type(e).__name__}: {str(e).splitlines()[0][:160] if str(e) else ''}"
                    torch.cuda.synchronize()
                    step, g, pol = make_runner(args, args.batch, sched, device, **kw)
                n0 = _native.launch_count()
                times[name].append(timed(step, args.steps, args.warmup, dist, flush))
                if name == head:
                    if hasattr(step, "native_launches"):   # CUDA graph: kernel nodes per replay
                        launches = step.native_launches * args.steps
                    else:
                        launches = (_native.launch_count() - n0) * args.steps // (args.steps + args.warmup)
                del step, g, pol
                torch.cuda.empty_cache()
    clocks = clk.summary()
    med = {k: statistics.median(v) for k, v in times.items()}
    ms = med[head]
    value = dist.world * args.batch * 1e3 / ms
    graphed = bool(args.graphs) and (not args.dp or bool(args.dp_graphs))
    mode = ("graph" if graphed else "eager") + (", NHWC" if args.channels_last else "")
    math = "fp32 (TF32 off)" if not args.tf32 else "fp32 weights, TF32 tensor cores"
    if args.dp:
        mode += f", data parallel over {args.dp_transport}"
    workload = (f"C2 MobileNetV2 (10 classes) on synthetic 3x32x32, batch {args.batch}/GPU, "
                f"SGD-momentum, {math}; {head}, {mode}")

    def ratio(name):
        return round(med[name] / ms, 4) if name in med else None

    def med_ms(name):
        return round(med[name], 4) if name in med else None

    unfused_torch = "DDP + " if args.dp else ""
    tp = "DDP+" if args.dp else ""
    res = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": dist.world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f32" if not args.tf32 else "tf32",
           "data": "synthetic x~N(0,1), y~U{0..9}; random-init weights",
           "config": {"workload": workload, "global_batch": args.batch * dist.world,
                      "parallelism": f"dp{dist.world}", "instances": args.instances,
                      "l2": "256 MiB flush before every timed step, outside its events"},
           "unfused": {"ours_baseline_ms": med_ms("ours:baseline"),
                       "torch_foreach_ms": med_ms(tp + "torch.optim.SGD(foreach)"),
                       "torch_fused_ms": med_ms(tp + "torch.optim.SGD(fused)"),
                       ("ddp_fwd_bwd_ms" if tp else "fwd_bwd_floor_ms"): med_ms(FLOOR_DDP if tp else FLOOR),
                       "speedup_vs_ours_unfused": ratio("ours:baseline"),
                       "speedup_vs_torch_foreach": ratio(tp + "torch.optim.SGD(foreach)"),
                       "speedup_vs_torch_fused": ratio(tp + "torch.optim.SGD(fused)"),
                       "torch_arm": unfused_torch + "torch.optim, same mode"},
           "gpu_launches": int(launches)}
    if "eager:" + head in med:
        eh = med["eager:" + head]
        res["unfused"]["eager"] = {
            "fused_ms": round(eh, 4), "ours_baseline_ms": med_ms("eager:ours:baseline"),
            "torch_foreach_ms": med_ms("eager:torch.optim.SGD(foreach)"),
            "speedup_vs_ours_unfused": round(med["eager:ours:baseline"] / eh, 4),
            "speedup_vs_torch_foreach": round(med["eager:torch.optim.SGD(foreach)"] / eh, 4)}
    extras = {"rows": {k: {"ms_per_step": round(med[k], 4),
                           "images_per_s": round(dist.world * args.batch * 1e3 / med[k], 1),
                           "instances_ms": [round(t, 4) for t in v]} for k, v in times.items()},
              "mode": mode, "model_math": math,
              "torch_backends": {"cudnn.allow_tf32": torch.backends.cudnn.allow_tf32,
                                 "matmul.allow_tf32": torch.backends.cuda.matmul.allow_tf32,
                                 "cudnn.benchmark_limit": 0}}
    if dp_graph_error:
        extras["dp_graph_capture_failed"] = dp_graph_error
    if args.headline_only:
        res["clocks"] = clocks
        dist.close()
        return res
    res["e2e"] = e2e(args, device, dist, flush)
    extras["e2e_instances"] = res["e2e"].pop("instances")
    # the kernel's own duration is a per-GPU quantity: measured on this GPU's
    # single-process engine whatever the world size
    world, dp, args.world, args.dp = args.world, args.dp, 1, False
    try:
        live = measure_in_graph(args, device, peaks, flush) if args.graphs else None
        ins = measure_in_situ(args, device, peaks, 5)
    finally:
        args.world, args.dp = world, dp
    tr = ncu_traffic("c2_backward_fusion_buckets")
    prim = live or ins
    res["roofline"] = {"bound": "hbm", "kernel": "mt_step_kernel",
                       "achieved": round(prim["achieved_gbs"], 1), "peak": peaks["hbm_gbs"],
                       "unit": "GB/s", "frac": round(prim["frac"], 4),
                       "traffic": (tr or {}).get("dram_bytes_per_launch"),
                       "bytes_per_launch": round(prim["avg_bytes"]),
                       "us_per_launch": round(prim["avg_us"], 3),
                       "launches_per_step": prim["launches_per_step"]}
    if args.in_situ:
        # the update-bound config's large layers (VGG-16 Adam), live beside its backward
        c3 = measure_live_launches(args, "c3", device, peaks)
        res["roofline"]["in_situ_c3_large"] = {k: c3["large"][k] for k in ("achieved_gbs", "frac")}
        extras["in_situ_c3"] = c3
    extras["roofline"] = {
        "method": ("CUDA events captured as event-record nodes around each update launch of the "
                   "headline graph, read after every replay (live, beside the backward)")
        if live else "one iteration's launches replayed back to back",
        "peak_source": peaks["source"], "traffic_source": (tr or {}).get("source"),
        "in_graph_live": live, "replayed_back_to_back": ins}
    if args.sweep:
        extras["batch_sweep"] = run_sweep(args, device, dist, flush)
    for wl in [w for w in args.extras.split(",") if w.strip()]:
        extras[wl] = run_extra(args, wl, device, dist, flush)
    if args.standalone:
        std = measure_update_kernel(args, device, peaks)
        extras["standalone_single_launch"] = std
    if dist.rank == 0 and dist.world == 1:
        res["cpu_baseline"] = cpu_baseline(args)
        if args.standalone:
            extras["cpu_update_baseline"] = cpu_update_baseline(std)
    res["clocks"] = clocks
    dist.close()
    if dist.rank == 0 and args.extras_out:
        out = Path(args.extras_out)
        out.parent.mkdir(parents=True, exist_ok=True)
        extras["headline_line"] = res
        out.write_text(json.dumps(extras, indent=1))
        res["extras"] = str(out)
    return res


def run_sweep(args, device, dist, flush) -> dict:
    """Batch sweep (C2: per-GPU batch 32..512) of the headline, ours unfused
    and torch foreach, interleaved per instance."""
    import torch
    out = {}
    arms = [a for a in headline_arms(args)
            if a[0] in (_headline_name(args), "ours:baseline", "torch.optim.SGD(foreach)", FLOOR)]
    for b in [int(x) for x in args.sweep.split(",") if x.strip()]:
        times = {n: [] for n, _ in arms}
        for _ in range(args.instances):
            for name, kw in arms:
                kw = dict(kw)
                sched = kw.pop("schedule", args.schedule)
                st, *_ = make_runner(args, b, sched, device, **kw)
                times[name].append(timed(st, args.steps, args.warmup, dist, flush))
                del st
                torch.cuda.empty_cache()
        row = {}
        for n, v in times.items():
            t = statistics.median(v)
            row[n] = {"ms_per_step": round(t, 4), "images_per_s": round(dist.world * b * 1e3 / t, 1),
                      "instances_ms": [round(x, 4) for x in v]}
        h = row[_headline_name(args)]["ms_per_step"]
        for n in ("ours:baseline", "torch.optim.SGD(foreach)"):
            if n in row:
                row[_headline_name(args)][f"speedup_vs_{n}"] = round(row[n]["ms_per_step"] / h, 4)
        out[str(b)] = row
    return out



OWN_LB = "fwd+bwd only (bf16 module as ours: lower bound for ours)"


def _variants_extra(wl: str):
    """(name, schedule, workers, torch optimizer, bucket, CUDA graph) for the extras."""
    opt = WORKLOADS[wl]["torch"][0]
    LB = FLOOR
    v = []
    for gph, pre in ((False, ""), (True, "graph:")):
        # (graph mode: Adam/AdamW replay through the device-side step index;
        # torch's Adam with capturable=True)
        v += [(f"{pre}torch.optim.{opt}(foreach)", "baseline", None, "foreach", 0, gph),
              (f"{pre}torch.optim.{opt}(fused)", "baseline", None, "fused", 0, gph),
              (pre + LB, "baseline", None, "none", 0, gph),
              (pre + "ours:baseline", "baseline", None, None, 0, gph),
              (pre + "ours:forward-fusion(per-layer)", "forward-fusion", None, None, 0, gph),
              (pre + "ours:forward-fusion(bucket=1M)", "forward-fusion", None, None, 1 << 20, gph),
              (pre + "ours:backward-fusion(w=2,per-layer)", "backward-fusion", 2, None, 0, gph),
              (pre + "ours:backward-fusion(w=2,bucket=1M)", "backward-fusion", 2, None, 1 << 20, gph),
              # inline on the autograd stream: each update right behind its layer's backward,
              # gradients (and the weights dgrad just read) still in L2 -- the paper's locality
              (pre + "ours:backward-fusion(w=1,per-layer)", "backward-fusion", 1, None, 0, gph)]
        if WORKLOADS[wl].get("mixed"):
            v.append((pre + OWN_LB, "baseline", None, "none-mixed", 0, gph))
        if wl == "c5m":
            v.append((pre + "ours:backward-fusion(w=2,per-layer)+consumer", "backward-fusion+consumer",
                      2, None, 0, gph))
            v.append((pre + "ours:backward-fusion(w=1,per-layer)+consumer", "backward-fusion+consumer",
                      1, None, 0, gph))
    return v


def run_extra(args, wl: str, device, dist, flush) -> dict:
    """One of BASELINE.json's other configs on this GPU, eager and captured as
    CUDA graphs: C1 ResNet-18/CIFAR SGD-momentum, C3 VGG-16 Adam (the
    update-bound case), C4 ResNet-50 bf16 + fp32 masters AdamW, C5 BERT-base
    AdamW.  Every row is built --instances times, instances interleaved across
    rows (instance i of every row, then i+1); each row is the median."""
    import torch
    b = WORKLOADS[wl]["batch"]
    steps, warm = max(args.steps // 2, 10), 3
    variants = [v for v in _variants_extra(wl) if not (v[5] and args.dp and not args.dp_graphs)]
    times, failed = {v[0]: [] for v in variants}, {}
    for _ in range(args.instances):
        for name, sch, w, opt, be, gph in variants:
            if name in failed:
                continue
            try:
                cons = sch.endswith("+consumer")
                st, *_ = make_runner(args, b, sch.replace("+consumer", ""), device, workers=w,
                                     opt_impl=opt, bucket_elems=be, graphed=gph, workload=wl,
                                     channels_last=wl in ("c4",), consumer=cons)
                times[name].append(timed(st, steps, warm, dist, flush))
            except Exception as e:  # noqa: BLE001 -- report, keep the other rows
                failed[name] = f"{type(e).__name__}: {str(e).splitlines()[0][:160] if str(e) else ''}"
                torch.cuda.synchronize()
                continue
            del st
            torch.cuda.empty_cache()
    row = {}
    for name, ts in times.items():
        if ts:
            t = statistics.median(ts)
            row[name] = {"ms_per_step": round(t, 3), "images_per_s": round(dist.world * b * 1e3 / t, 1),
                         "instances_ms": [round(x, 3) for x in ts]}
    _speedups(row)
    out = {"workload": WORKLOADS[wl]["desc"], "batch_per_gpu": b, "steps": steps, "warmup": warm,
           "instances": args.instances}
    for mode in ("", "graph:"):
        lb = row.pop(mode + FLOOR, None)
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
    r = timing.cpu_training_sample(args.model, args.batch, max(args.steps, 1), "sgd-momentum", kw,
                                   warmup=max(args.warmup, 1))
    v = round(r["images_per_s"], 3)
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(r["ms_per_iter"], 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic x~N(0,1), y~U{0..9}; random-init weights",
            "config": {"workload": (f"C2 MobileNetV2 (10 classes) on synthetic 3x32x32, batch "
                                    f"{args.batch}, SGD-momentum, fp32; reference CPU path "
                                    f"(unfused: forward, backward, per-parameter update)"),
                       "global_batch": args.batch, "parallelism": "cpu"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["threads"], "kind": "port",
                             "sample": (f"each step: one iteration at batch {args.batch}, pinned "
                                        f"to {r['threads']} cores: torch-CPU fwd/bwd + the "
                                        f"reference update (numpy oracle port, 1 thread)")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main(argv=None):
    args = parse_args(argv)
    if args.impl == "reference":
        res = run_reference(args)
    else:
        res = run_ours(args)
    if NCCL_LOG and os.path.exists(NCCL_LOG):   # rank 0's communicator lines, before the result
        with open(NCCL_LOG) as fh:
            sys.stdout.write(fh.read())
    if res is not None and int(os.environ.get("RANK", "0")) == 0:
        line = json.dumps(res, separators=(",", ":"))
        if len(line) > 2048:
            print(f"bench: result line is {len(line)} bytes (> 2 KB)", file=sys.stderr)
        print(line, flush=True)


if __name__ == "__main__":
    main()
