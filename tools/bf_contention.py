"""Backward fusion on a GPU-bound step (diagnostic): BERT-base b32 AdamW,
graphed; side-stream update grid capped at various CTA counts and both
stream priorities, against the baseline schedule and the floor."""

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
    torch.backends.cuda.matmul.allow_tf32 = True
    dev = torch.device("cuda", 0)
    args = bench.parse_args([])
    args.world, args.dp = 1, False
    dist = bench.Dist()
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    W = bench.WORKLOADS[wl]
    out = {}
    for name, sched, kw in (("baseline", "baseline", {}),
                            ("bf_1M", "backward-fusion", dict(workers=2, bucket_elems=1 << 20)),
                            ("bf_1M_cap37", "backward-fusion", dict(workers=2, bucket_elems=1 << 20, update_ctas=37)),
                            ("bf_1M_cap74", "backward-fusion", dict(workers=2, bucket_elems=1 << 20, update_ctas=74)),
                            ("bf_1M_cap148", "backward-fusion", dict(workers=2, bucket_elems=1 << 20, update_ctas=148)),
                            ("bf_1M_cap296", "backward-fusion", dict(workers=2, bucket_elems=1 << 20, update_ctas=296)),
                            ("bf_1M_low", "backward-fusion", dict(workers=2, bucket_elems=1 << 20, update_priority="low")),
                            ("bf_1M_cap74_low", "backward-fusion", dict(workers=2, bucket_elems=1 << 20, update_ctas=74, update_priority="low")),
                            ("bf_4M_cap148", "backward-fusion", dict(workers=2, bucket_elems=1 << 22, update_ctas=148))):
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
        out[name] = round(bench.timed(cap, 10, 3, dist, buf.zero_), 3)
        del cap, g
        torch.cuda.empty_cache()
    print(json.dumps({wl: out}))


if __name__ == "__main__":
    main()
