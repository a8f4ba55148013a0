"""Data parallel with real ranks: W processes share the one GPU
(tools/dp_ranks_one_gpu.py).  Peer transport: their flat buffers are mapped into
each other with CUDA IPC and of_dp_step_peer reads and writes the other
processes' memory.  Collectives transport: the reduce-scatter / all-gather
run over gloo on the CUDA tensors around the sharded kernel.  Every schedule must leave every rank with the reference
update of the rank-averaged gradient, bit for bit (exact chain model)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("world,mode", [(2, "peer"), (3, "peer"), (2, "collectives")])
def test_data_parallel_real_ranks_one_gpu(world, mode):
    """mode "peer": the fused peer kernel over CUDA-IPC mappings; "collectives":
    reduce-scatter -> sharded kernel -> all-gather with the collectives carried
    by gloo on the CUDA tensors (NCCL refuses two ranks on one device)."""
    proc = subprocess.run([sys.executable, str(ROOT / "tools" / "dp_ranks_one_gpu.py"), str(world),
                           mode],
                          capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr[-2000:]
    res = json.loads(proc.stdout.strip().splitlines()[-1])
    assert res["world"] == world
    for sched in ("backward-fusion", "baseline", "forward-fusion"):
        assert res[sched]["ranks_agree"], sched
        assert res[sched]["bitwise_vs_oracle"], (sched, res[sched]["max_abs_err"])
    for sched in ("baseline+clip", "forward-fusion+clip"):   # peer: of_dp_sqnorm_peer
        assert res[sched]["ranks_agree"], sched
        assert res[sched]["max_rel_err"] <= 1e-5, (sched, res[sched])
