"""cuDNN algorithm choice vs model instance (diagnostic, GPU box): the graphed
channels-last MobileNetV2 step timed over several independently built
instances, forward+backward only and with backward fusion, for a given
torch.backends.cudnn.benchmark_limit (0 = try every algorithm)."""

import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    limit = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    # limit < 0: no benchmarking at all (cuDNN's heuristics pick)
    torch.backends.cudnn.benchmark = limit >= 0
    torch.backends.cudnn.benchmark_limit = max(limit, 0)
    torch.backends.cuda.matmul.allow_tf32 = True
    args = bench.parse_args(["--steps", "30", "--warmup", "10"])
    args.world, args.dp = 1, False
    dev = torch.device("cuda", 0)
    dist = bench.Dist()
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {}
    for name, opt in (("floor", "none"), ("bf_1M", None), ("torch_foreach", "foreach")):
        ts = []
        for _ in range(n):
            st, *_ = bench.make_runner(args, 128, "backward-fusion" if opt is None else "baseline", dev,
                                       workers=2, opt_impl=opt, bucket_elems=1 << 20, graphed=True,
                                       channels_last=True)
            ts.append(round(bench.timed(st, 30, 10, dist, buf.zero_), 4))
            del st
            torch.cuda.empty_cache()
        out[name] = {"median": statistics.median(ts), "instances": ts}
    print(json.dumps({"benchmark_limit": limit, **out}))


if __name__ == "__main__":
    main()
