"""Per-kernel device time of the headline step in its graphed form (CUPTI via
torch.profiler; ncu cannot replay cuDNN's semi-persistent batch-norm kernel as
a graph node).  Prints a markdown table."""

import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402


def main():
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.benchmark_limit = 0
    torch.backends.cuda.matmul.allow_tf32 = False   # true fp32, as bench.py
    torch.backends.cudnn.allow_tf32 = False
    dev = torch.device("cuda", 0)
    args = bench.parse_args([])
    args.world, args.dp = 1, False
    st, *_ = bench.make_runner(args, args.batch, args.schedule, dev)
    for _ in range(10):
        st()
    torch.cuda.synchronize()
    reps = 5
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            st()
        torch.cuda.synchronize()
    agg = defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type.name != "CUDA" or e.device_time_total <= 0:
            continue
        a = agg[e.name[:80]]
        a[0] += 1
        a[1] += e.device_time_total
    total = sum(v[1] for v in agg.values())
    print(f"# Headline step, graphed (MobileNetV2 b128 CL, BF 1M buckets): kernels per step\n")
    print(f"CUPTI device time over {reps} replays (torch.profiler), per step: "
          f"{total / reps:.1f} us of kernel time.\n")
    print("| kernel | per step | us per step | share |\n|---|---|---|---|")
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"| `{name}` | {n / reps:.0f} | {us / reps:.1f} | {us / total:.4f} |")
    ours = {k: v for k, v in agg.items() if "mt_step" in k or "of_" in k or "mt_copy" in k}
    o = sum(v[1] for v in ours.values())
    print(f"\nliboptfuse_b200 kernels: {sum(v[0] for v in ours.values()) / reps:.0f} per step, "
          f"{o / reps:.1f} us per step, share {o / total:.4f} of kernel time "
          "(on the side stream, concurrent with backward).")


if __name__ == "__main__":
    main()
