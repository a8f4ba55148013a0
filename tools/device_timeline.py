"""Device-timeline proof of overlap (CUPTI via torch.profiler): for one
backward-fusion iteration, where each update launch (mt_step_kernel, side
stream) ran relative to the backward's kernels on the compute stream.

    python tools/device_timeline.py [c2|c3|c5] > profiles/r02_device_timeline_<cfg>.json

The schedule trace (trace.py, the reference's format) records HOST issue
order; this records DEVICE start/end timestamps: per update launch, its
stream, duration, and the fraction of its duration during which a kernel of
another stream (the backward) was executing.  Also the backward-only span
after the last update ends (the part of the step the update did not extend).
"""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_00237_b200 as of  # noqa: E402
from paper_2104_00237_b200.models import synthetic_batch  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    wl = bench.WORKLOADS[cfg]
    cl = cfg == "c2"
    g = of.build_classifier(wl["model"], device="cuda", channels_last=cl)
    g.track_counts = False
    x, y = synthetic_batch(wl["model"], wl["batch"], device="cuda")
    if cl:
        x = x.contiguous(memory_format=torch.channels_last)
    pol = of.OptimizerPolicy(wl["kind"], **wl["hp"], grad_reset="none")
    be = (1 << 20) if cfg == "c2" else 0

    def step():
        of.run_backward_fusion(g, pol, (x, y), workers=2, timing=False, bucket_elems=be)
    for _ in range(4):
        step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    kern = []
    for e in prof.events():
        if e.device_type.name != "CUDA" or e.name.startswith("Memcpy") or e.name.startswith("Memset"):
            continue
        tr = e.time_range
        stream = getattr(e, "stream", None)
        kern.append({"name": e.name, "start": tr.start, "end": tr.end,
                     "stream": stream if stream is not None else e.thread})
    kern.sort(key=lambda k: k["start"])
    upd = [k for k in kern if "mt_step_kernel" in k["name"]]
    other = [k for k in kern if "mt_step_kernel" not in k["name"]]
    rows = []
    for u in upd:
        dur = u["end"] - u["start"]
        # union of other-stream kernel intervals intersected with [start, end)
        # (kernels of one stream never overlap, so any overlap is another stream's)
        iv = sorted((max(o["start"], u["start"]), min(o["end"], u["end"])) for o in other
                    if o["end"] > u["start"] and o["start"] < u["end"])
        covered, cur = 0.0, None
        for a, b in iv:
            if cur is None or a > cur[1]:
                if cur:
                    covered += cur[1] - cur[0]
                cur = [a, b]
            else:
                cur[1] = max(cur[1], b)
        if cur:
            covered += cur[1] - cur[0]
        rows.append({"start_us": round(u["start"] - kern[0]["start"], 2), "dur_us": round(dur, 2),
                     "stream": u["stream"],
                     "overlapped_by_backward": round(covered / dur, 3) if dur > 0 else None})
    t0, t1 = kern[0]["start"], max(k["end"] for k in kern)
    last_upd = max(u["end"] for u in upd) if upd else t0
    last_bwd = max(o["end"] for o in other)
    out = {"config": cfg, "schedule": "backward-fusion w=2 (side stream)" + (", 1M buckets" if be else ", per layer"),
           "kernels": len(kern), "update_launches": len(upd),
           "iteration_kernel_span_us": round(t1 - t0, 1),
           "update_kernel_us_total": round(sum(r["dur_us"] for r in rows), 2),
           "update_time_overlapped_by_backward": round(
               sum(r["dur_us"] * (r["overlapped_by_backward"] or 0) for r in rows)
               / max(sum(r["dur_us"] for r in rows), 1e-9), 3),
           "last_update_end_minus_last_other_kernel_end_us": round(last_upd - last_bwd, 2),
           "updates": rows}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
