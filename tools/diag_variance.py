"""Diagnose run-to-run variance of graphed MobileNetV2 steps (not a bench)."""
import sys, time
sys.path.insert(0, ".")
import torch
import bench

args = bench.parse_args([])
args.world = 1
dist = bench.Dist()
dev = torch.device("cuda", 0)
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for bm in (True, False):
    torch.backends.cudnn.benchmark = bm
    for rep in range(3):
        for name, kw in (("torch", dict(opt_impl="foreach")), ("bf256K", dict(bucket_elems=1 << 18)),
                         ("bf4M", dict(bucket_elems=1 << 22))):
            sch = "baseline" if "opt_impl" in kw else "backward-fusion"
            st, *_ = bench.make_runner(args, 128, sch, dev, graphed=True, channels_last=True, **kw)
            ts = [bench.timed(st, 50, 5, dist, flush_buf.zero_) for _ in range(3)]
            print(f"benchmark={bm} rep={rep} {name:8s} " + " ".join(f"{t:.3f}" for t in ts), flush=True)
            del st
            torch.cuda.empty_cache()
