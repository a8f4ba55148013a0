"""The device half of the Appendix B.2 guard, tested adversarially.

Reference: a parameter may be updated in place only once its gradient is
complete AND no backward node still has to read its old value
(schedule.py:54-59 ``check_inplace_safety``, graph.py:117-122 -- the input
gradient is computed from the OLD theta).

On the GPU the host half holds by autograd ordering (a node's input-gradient
kernels are enqueued before its AccumulateGrad hook fires); the device half is
the event the backward-fusion engine records on the compute stream at hook
time and the update side stream waits on (optfuse_engine.cpp launch_group).
Here a layer's backward enqueues its weight gradient, then a long device
sleep, then the input gradient that reads W: the hook fires (host) while the
device is still asleep.  With the event edge the side-stream update waits for
the input gradient and the trajectory equals the unfused baseline bit for bit;
with the edge removed (test-only switch) the update lands inside the sleep,
the input gradient reads the NEW weight and the trajectory diverges -- so the
passing test is evidence of the guard, not of lucky timing.
"""

import numpy as np
import pytest
import torch

import paper_2104_00237_b200 as of

pytestmark = pytest.mark.gpu
DEV = "cuda"
SLEEP_CYCLES = 60_000_000      # ~30 ms at B200 clocks: far longer than the host's hook latency


class _SleepyMatmul(torch.autograd.Function):
    """x @ w whose backward computes dW, sleeps on the device, then dX = g @ W^T
    (the read of the old weight that the guard protects)."""

    @staticmethod
    def forward(ctx, x, w):
        ctx.save_for_backward(x, w)
        return x @ w

    @staticmethod
    def backward(ctx, gout):
        x, w = ctx.saved_tensors
        gw = x.t() @ gout
        torch.cuda._sleep(SLEEP_CYCLES)
        gx = gout @ w.t()
        return gx, gw


class _Net(torch.nn.Module):
    def __init__(self, width=64):
        super().__init__()
        gen = torch.Generator().manual_seed(3)
        self.l1 = torch.nn.Linear(width, width, bias=False)
        self.l2 = torch.nn.Linear(width, width, bias=False)
        with torch.no_grad():
            self.l1.weight.copy_((torch.rand(width, width, generator=gen) - 0.5) * 0.3)
            self.l2.weight.copy_((torch.rand(width, width, generator=gen) - 0.5) * 0.3)

    def forward(self, x):
        h = torch.relu(_SleepyMatmul.apply(x, self.l1.weight))
        return (_SleepyMatmul.apply(h, self.l2.weight) ** 2).sum()


def _run(schedule: str, skip_wait: bool = False, iters: int = 3):
    torch.manual_seed(0)
    g = of.Graph(_Net().to(DEV), None, track_counts=False)
    pol = of.OptimizerPolicy("sgd-momentum", eta=0.05, alpha=0.9, grad_reset="none")
    xs = [torch.rand(32, 64, generator=torch.Generator().manual_seed(i)).to(DEV) for i in range(iters)]
    for x in xs:
        if schedule == "baseline":
            of.run_baseline(g, pol, x, timing=False)
        else:
            of.run_backward_fusion(g, pol, x, workers=2, timing=False)
            eng = next(e for k, e in g._engines.items() if k[1])
            eng.native._debug_skip_ready_wait(skip_wait)
    torch.cuda.synchronize()
    return np.concatenate([p.value.detach().cpu().numpy().reshape(-1) for p in g.parameters])


def test_side_stream_update_waits_for_the_old_weight_readers():
    want = _run("baseline")
    got = _run("backward-fusion")
    assert got.tobytes() == want.tobytes()


def test_removing_the_event_edge_breaks_the_trajectory():
    """The control: same run with the ready-event wait dropped must differ
    (the switch takes effect from the second iteration: the engine is created
    by the first)."""
    want = _run("baseline")
    bad = _run("backward-fusion", skip_wait=True)
    assert bad.tobytes() != want.tobytes()
    assert np.isfinite(bad).all()
