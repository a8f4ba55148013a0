"""A/B of update-kernel builds (GPU box): for every build/ab/*.so, in its own
process (OPTFUSE_B200_LIB), the standalone single-launch roofline of the C2-C5
parameter sets, the headline's bucket launches timed live inside the replayed
graph, and the same launches queued back to back (bench.py's functions)."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, str(ROOT))
    import torch
    import bench
    args = bench.parse_args([])
    dev = torch.device("cuda")
    peaks = bench.load_peaks()
    out = {"standalone": {k: [v["us"], v["frac"]] for k, v in bench.measure_update_kernel(args, dev, peaks).items()}}
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    r = bench.measure_in_graph(args, dev, peaks, lambda: flush_buf.zero_())
    out["in_graph"] = [round(r["avg_us"], 3), round(r["frac"], 4)]
    r = bench.measure_in_situ(args, dev, peaks)
    out["queued"] = [round(r["avg_us"], 3), round(r["frac"], 4)]
    out["live_eager"] = [r["live_beside_backward"]["avg_us"], r["live_beside_backward"]["frac"]]
    print(json.dumps(out))
    sys.exit(0)

res = {}
for rep in range(int(os.environ.get("AB_REPS", "2"))):
    for so in sorted((ROOT / "build" / "ab").glob("*.so")):
        env = dict(os.environ, OPTFUSE_B200_LIB=str(so))
        out = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-600:]
        print(so.name, line, flush=True)
        try:
            res.setdefault(so.stem, []).append(json.loads(line))
        except ValueError:
            res.setdefault(so.stem, []).append({"error": line})
print(json.dumps(res))
