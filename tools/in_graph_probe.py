"""Per-replay spread of the in-graph live update timing (bench.measure_in_graph)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

args = bench.parse_args([])
args.world, args.dp = 1, False
torch.backends.cudnn.benchmark = True
torch.backends.cudnn.benchmark_limit = 0
dev = torch.device("cuda:0")
peaks = bench.load_peaks()
buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
out = {}
for bucket in (1 << 22, 1 << 20, 1 << 18):
    args.bucket_elems = bucket
    out[str(bucket)] = bench.measure_in_graph(args, dev, peaks, buf.zero_, reps=40)
print(json.dumps(out))
