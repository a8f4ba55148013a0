"""Shared test configuration.

Markers: ``gpu`` -- needs a CUDA B200 (run with ``-m gpu`` on the GPU box);
everything else runs on a CPU-only host (``-m "not gpu"``).
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def policy_golden():
    return dict(np.load(GOLDEN / "policy_steps.npz"))


@pytest.fixture(scope="session")
def traj_golden():
    return dict(np.load(GOLDEN / "trajectories.npz"))


@pytest.fixture(scope="session")
def spec_kats():
    import json
    with open(GOLDEN / "spec_kats.json") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def traces_golden():
    import json
    with open(GOLDEN / "traces.json") as fh:
        return json.load(fh)
