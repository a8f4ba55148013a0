"""Standalone update-kernel roofline for each build/variants/*.so (GPU box):
one subprocess per variant with OPTFUSE_B200_LIB pointing at it."""

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
    r = bench.measure_update_kernel(None, torch.device("cuda"), bench.load_peaks())
    print(json.dumps({k: [v["us"], v["frac"]] for k, v in r.items()}))
    sys.exit(0)

for so in sorted((ROOT / "build" / "variants").glob("*.so")):
    env = dict(os.environ, OPTFUSE_B200_LIB=str(so))
    out = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True, text=True)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
    print(so.name, line, flush=True)
