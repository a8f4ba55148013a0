"""PDL probe (GPU box): one config's baseline (or other schedule) as a captured
step; device time per replay (CUDA events, L2 flushed, median of 20) and one
replay's CUPTI timeline (kernel busy time, span, our update kernel and the gap
in front of it).  Run once per library (OPTFUSE_B200_LIB) to compare builds.

    python tools/pdl_probe.py c4 baseline
"""

import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
    sched = sys.argv[2] if len(sys.argv) > 2 else "baseline"
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.benchmark_limit = 0
    dev = torch.device("cuda", 0)
    args = bench.parse_args([])
    args.world, args.dp = 1, False
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    if sched == "floor":   # forward + backward only (our bf16 model math for C4)
        kw = dict(opt_impl="none-mixed" if bench.WORKLOADS[wl].get("mixed") else "none")
        sched = "baseline"
    else:
        kw = {} if sched == "baseline" else dict(workers=2, bucket_elems=1 << 20)
    step, g, pol = bench.make_runner(args, bench.WORKLOADS[wl]["batch"], sched, dev, graphed=True,
                                     workload=wl, channels_last=wl in ("c4",), **kw)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        buf.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    from torch.profiler import ProfilerActivity, profile
    buf.zero_()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                 if e.device_type.name == "CUDA" and not e.name.startswith(("Memcpy", "Memset"))),
                key=lambda k: k[0])
    busy = sum(e - s for s, e, _ in ks)
    upd = [k for k in ks if "mt_step_kernel" in k[2]]
    out = {"config": wl, "schedule": sched, "ms_median": round(statistics.median(ts), 4),
           "ms_min": round(min(ts), 4), "kernels": len(ks),
           "span_us": round(ks[-1][1] - ks[0][0], 1), "kernel_busy_us": round(busy, 1)}
    if upd:
        i = ks.index(upd[0])
        out["update_us"] = round(upd[0][1] - upd[0][0], 2)
        out["gap_before_update_us"] = round(upd[0][0] - max(e for s, e, _ in ks[:i]), 2) if i else None
    print(json.dumps(out))


if __name__ == "__main__":
    main()
