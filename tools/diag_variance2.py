"""Is the first graphed BF instance in a process systematically faster? (diagnostic)"""
import sys
sys.path.insert(0, ".")
import torch
import bench

order = sys.argv[1].split(",")
args = bench.parse_args([])
args.world = 1
dist = bench.Dist()
dev = torch.device("cuda", 0)
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
keep = []
for name in order:
    kw = dict(opt_impl="foreach") if name == "torch" else dict(bucket_elems=1 << 18)
    if name.endswith("w1"):
        kw["workers"] = 1
    sch = "baseline" if name == "torch" else "backward-fusion"
    st, g, pol = bench.make_runner(args, 128, sch, dev, graphed=True, channels_last=True, **kw)
    ts = [bench.timed(st, 50, 5, dist, flush_buf.zero_) for _ in range(2)]
    print(f"{' '.join(order)} :: {name:8s} " + " ".join(f"{t:.3f}" for t in ts), flush=True)
    if "keep" in sys.argv:
        keep.append((st, g, pol))
