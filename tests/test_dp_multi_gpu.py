"""Data parallel across >= 2 real GPUs over NCCL / NVLink (tools/dp_multi_gpu.py):
both transports and every schedule against the numpy oracle of the
rank-averaged update, plus the NVLS multicast kernel's numerics.  The driver's
GPU boxes have one GPU, so this skips there; it is the N>1 path's check on an
8-GPU node."""

import json
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_data_parallel_across_gpus():
    world = min(torch.cuda.device_count(), 4)
    proc = subprocess.run([sys.executable, str(ROOT / "tools" / "dp_multi_gpu.py"), str(world)],
                          capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr[-3000:]
    res = json.loads(proc.stdout.strip().splitlines()[-1])
    for transport in ("nccl", "peer"):
        for sched in ("backward-fusion", "baseline", "forward-fusion"):
            r = res[f"{transport}:{sched}"]
            assert r["ranks_agree"], (transport, sched)
            if world == 2:
                assert r["bitwise_vs_oracle"], (transport, sched, r)
            else:
                assert r["max_rel_err"] <= 1e-6, (transport, sched, r)
    for schedule in ("baseline+clip", "forward-fusion+clip"):
        r = res[f"clip:{schedule}"]
        assert r["ranks_agree"] and r["nccl_vs_peer_max_rel"] <= 1e-5, (schedule, r)
    for rank, r in res["multicast"].items():
        if isinstance(r, str):          # fabric without NVLS multicast
            assert r.startswith("skip"), r
            continue
        assert r["grad_zeroed"] and r["max_rel"] <= 1e-6, (rank, r)
