"""Backward fusion on a GPU-bound step (diagnostic): one config (c3 | c4 | c5),
graphed, true fp32 (TF32 off, as bench.py); side-stream update grid capped at
various CTA counts, both stream priorities, per-layer and 1M buckets, against
the baseline schedule.  Arms are interleaved, --instances rounds, medians."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_00237_b200 as of  # noqa: E402
from paper_2104_00237_b200.graphs import CapturedStep  # noqa: E402
from paper_2104_00237_b200.models import synthetic_batch  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.benchmark_limit = 0
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    dev = torch.device("cuda", 0)
    args = bench.parse_args([])
    args.world, args.dp = 1, False
    dist = bench.Dist()
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    W = bench.WORKLOADS[wl]
    arms = [("baseline", "baseline", {})]
    for bucket, tag in ((1 << 20, "1M"), (0, "layer")):
        for cap in (0, 8, 16, 32, 74):
            for prio in ("high", "low"):
                if prio == "low" and cap not in (0, 16):
                    continue
                kw = dict(workers=2, bucket_elems=bucket, update_ctas=cap, update_priority=prio)
                arms.append((f"bf_{tag}_cap{cap}_{prio}", "backward-fusion", kw))
    arms.append(("bf_layer_inline", "backward-fusion", dict(workers=1, bucket_elems=0)))
    if len(sys.argv) > 3 and sys.argv[3] == "inline":   # inline buckets vs the side stream only
        arms = [("baseline", "baseline", {}),
                ("bf_1M_cap0_high", "backward-fusion", dict(workers=2, bucket_elems=1 << 20)),
                ("bf_layer_inline", "backward-fusion", dict(workers=1, bucket_elems=0)),
                ("bf_1M_inline", "backward-fusion", dict(workers=1, bucket_elems=1 << 20)),
                ("bf_4M_inline", "backward-fusion", dict(workers=1, bucket_elems=1 << 22))]
    instances = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    res = {name: [] for name, _, _ in arms}
    for _ in range(instances):
        for name, sched, kw in arms:
            g = of.build_classifier(W["model"], device=dev, channels_last=wl in ("c4",))
            g.track_counts = False
            x, y = synthetic_batch(W["model"], W["batch"], device=dev)
            if W.get("mixed"):
                g.use_master_weights()
                x = x.to(torch.bfloat16)
            pol = of.OptimizerPolicy(W["kind"], **W["hp"], grad_reset="none")
            if sched == "baseline":
                run = lambda inp: of.run_baseline(g, pol, inp, timing=False).loss  # noqa: E731
            else:
                run = lambda inp, kw=kw: of.run_backward_fusion(g, pol, inp, timing=False, **kw).loss  # noqa: E731
            cap = CapturedStep(run, (x, y), policy=pol, graph=g)
            res[name].append(round(bench.timed(cap, 10, 3, dist, buf.zero_), 3))
            del cap, g
            torch.cuda.empty_cache()
    import statistics
    out = {name: {"median_ms": statistics.median(v), "instances_ms": v} for name, v in res.items()}
    base = out["baseline"]["median_ms"]
    for v in out.values():
        v["vs_baseline"] = round(base / v["median_ms"], 4)
    print(json.dumps({wl: out}))


if __name__ == "__main__":
    main()
