"""Where forward fusion's extra time goes in the graphed MobileNetV2 step
(diagnostic): torch.profiler over 3 replays of floor / BF / FF graphs,
per-kernel device time, and the step time of each."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402


def main():
    torch.backends.cudnn.benchmark = True
    torch.backends.cudnn.benchmark_limit = 0
    torch.backends.cuda.matmul.allow_tf32 = True
    dev = torch.device("cuda", 0)
    args = bench.parse_args([])
    args.world, args.dp = 1, False
    dist = bench.Dist()
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {}
    for name, sch, opt, w, be in (("floor", "baseline", "none", None, 0),
                                  ("bf_1M", "backward-fusion", None, 2, 1 << 20),
                                  ("ff_256K", "forward-fusion", None, None, 1 << 18),
                                  ("ff_1M", "forward-fusion", None, None, 1 << 20)):
        st, *_ = bench.make_runner(args, 128, sch, dev, workers=w, opt_impl=opt, bucket_elems=be,
                                   graphed=True, channels_last=True)
        t = bench.timed(st, 30, 10, dist, buf.zero_)
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(3):
                st()
            torch.cuda.synchronize()
        per = {e.key[:60]: round(e.device_time_total / 3, 1) for e in prof.key_averages()
               if e.device_time_total > 0}
        out[name] = {"ms": round(t, 4), "kernel_us": round(sum(per.values()), 1), "kernels": per}
        del st
        torch.cuda.empty_cache()
    base = out["floor"]["kernels"]
    summary = {}
    for name in ("bf_1M", "ff_256K", "ff_1M"):
        k = out[name]["kernels"]
        extra = sorted(((key, round(k.get(key, 0) - base.get(key, 0), 1)) for key in set(k) | set(base)),
                       key=lambda kv: -abs(kv[1]))[:8]
        summary[name] = {"ms": out[name]["ms"], "kernel_us": out[name]["kernel_us"], "extra_vs_floor": extra}
    summary["floor"] = {"ms": out["floor"]["ms"], "kernel_us": out["floor"]["kernel_us"]}
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
