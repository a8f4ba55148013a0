"""Fast vs slow model instances (diagnostic): build graphed channels-last
MobileNetV2 forward+backward steps until one lands in the fast mode, then
replay the fastest and the slowest once each inside NVTX ranges "fast" /
"slow" (for ncu --nvtx-include)."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import bench  # noqa: E402
import paper_2104_00237_b200 as of  # noqa: E402
from paper_2104_00237_b200.graphs import CapturedStep  # noqa: E402
from paper_2104_00237_b200.models import synthetic_batch  # noqa: E402


def main():
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.benchmark_limit = 0
    torch.backends.cuda.matmul.allow_tf32 = True
    dev = torch.device("cuda", 0)
    dist = bench.Dist()
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    x, y = synthetic_batch("mobilenet_v2_cifar", 128, device=dev)
    x = x.contiguous(memory_format=torch.channels_last)
    caps = []
    for i in range(30):
        g = of.build_classifier("mobilenet_v2_cifar", device=dev, channels_last=True)
        net = g.module

        def run(inp, net=net):
            for p in net.parameters():
                p.grad = None
            loss = F.cross_entropy(net(inp[0]), inp[1])
            loss.backward()
            return loss
        cap = CapturedStep(run, (x, y), warmup=3)
        t = bench.timed(cap, 20, 5, dist, buf.zero_)
        caps.append((t, cap, g))
        if len(caps) >= 4 and min(c[0] for c in caps) < 0.95 * max(c[0] for c in caps):
            break
    caps.sort(key=lambda c: c[0])
    fast, slow = caps[0], caps[-1]
    from torch.profiler import ProfilerActivity, profile
    per = {}
    for name, (t, cap, g) in (("fast", fast), ("slow", slow)):
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(3):
                cap()
            torch.cuda.synchronize()
        per[name] = {e.key[:70]: e.device_time_total / 3 for e in prof.key_averages()
                     if e.device_time_total > 0}
    keys = sorted(set(per["fast"]) | set(per["slow"]),
                  key=lambda k: -abs(per["slow"].get(k, 0) - per["fast"].get(k, 0)))
    diff = [(k, round(per["fast"].get(k, 0), 1), round(per["slow"].get(k, 0), 1)) for k in keys[:15]]
    print(json.dumps({"times": [round(c[0], 4) for c in caps], "fast": round(fast[0], 4),
                      "slow": round(slow[0], 4),
                      "total_us": {n: round(sum(v.values()), 1) for n, v in per.items()},
                      "top_diffs_us(fast,slow)": diff}))


if __name__ == "__main__":
    main()
