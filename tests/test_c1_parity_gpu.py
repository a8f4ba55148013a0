"""North-star parity on a benchmarked configuration (C1): ResNet-18 on
synthetic CIFAR-10-shaped data, SGD-momentum (lr 0.1, momentum 0.9, coupled
weight decay 5e-4), true fp32 (TF32 off, deterministic cuDNN), BatchNorm in
train mode, 100 iterations.

GPU side: the product path -- baseline, backward fusion (side stream,
per-layer) and forward fusion (+ flush) on cuda.  CPU side: the reference's
path -- torch-CPU forward/backward (the reference's own autodiff only runs its
synthetic chains) + the reference update (oracle.optim_ref.step, the
bit-exact restatement of optim.py:74-148) on every parameter.

What can and cannot be equal:
* the three GPU schedules produce the same trajectory bit for bit (same
  kernels, only the issue point of each update moves);
* one step from identical parameters (teacher forcing: the CPU path restarted
  from the GPU's parameters) agrees per tensor to 1e-5 norm-wise relative --
  the only difference is cuDNN's vs oneDNN's convolution/BN reduction order;
* a free-running 100-step trajectory cannot stay at 1e-5: training is a
  chaotic map, and the ~1e-7 per-step reduction-order differences grow
  geometrically.  The test records the growth (per-tensor error at steps 1,
  10, 50, 100) and asserts the loss curves are indistinguishable (relative
  difference well below the step-to-step loss change).
With OPTFUSE_PARITY_OUT=<file> the curves are written as JSON
(profiles/r02_c1_parity.json comes from this).
"""

import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import paper_2104_00237_b200 as of
from paper_2104_00237_b200.models import synthetic_batch

pytestmark = pytest.mark.gpu

DEV = "cuda"
ITERS = 100
BATCH = 32
HP = dict(eta=0.1, alpha=0.9, weight_decay=5e-4)
CHECKPOINTS = (1, 10, 50, 100)


def _setup_numerics():
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False


def _batches():
    return [synthetic_batch("resnet18_cifar", BATCH, device="cpu", seed=s) for s in range(8)]


def _gpu_run(schedule, batches):
    g = of.build_classifier("resnet18_cifar", device=DEV, seed=0)   # BN in train mode
    pol = of.OptimizerPolicy("sgd-momentum", **HP)
    losses, snaps = [], {}
    dev_batches = [(x.to(DEV), y.to(DEV)) for x, y in batches]
    for it in range(1, ITERS + 1):
        inp = dev_batches[(it - 1) % len(dev_batches)]
        if schedule == "baseline":
            rep = of.run_baseline(g, pol, inp, timing=False)
        elif schedule == "backward-fusion":
            rep = of.run_backward_fusion(g, pol, inp, workers=2, timing=False)
        else:
            rep = of.run_forward_fusion(g, pol, inp, timing=False)
        losses.append(float(rep.loss))
        if it in CHECKPOINTS:
            if schedule == "forward-fusion":
                # an observation point: apply the deferred updates (as eval would)
                of.flush_pending_updates(g, pol)
            snaps[it] = [p.value.detach().cpu().numpy().copy() for p in g.parameters]
    return losses, snaps, g


def _cpu_net():
    import torchvision
    torch.manual_seed(0)
    m = torchvision.models.resnet18(num_classes=10)
    m.conv1 = torch.nn.Conv2d(3, 64, kernel_size=3, stride=1, padding=1, bias=False)
    m.maxpool = torch.nn.Identity()
    return m


def _cpu_step(net, params, slots, hp, x, y, t):
    from oracle import optim_ref
    loss = F.cross_entropy(net(x), y)
    loss.backward()
    for p, sl in zip(reversed(params), reversed(slots)):
        optim_ref.step("sgd-momentum", hp, p.detach().numpy().reshape(-1),
                       p.grad.numpy().reshape(-1), sl, t)
    return float(loss)


def _rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


@pytest.fixture(scope="module")
def runs():
    from oracle import optim_ref
    _setup_numerics()
    torch.set_num_threads(max(1, min(16, os.cpu_count() or 1)))
    batches = _batches()
    gpu = {s: _gpu_run(s, batches) for s in ("baseline", "backward-fusion", "forward-fusion")}
    net = _cpu_net()
    params = [p for p in net.parameters() if p.requires_grad]
    hp = optim_ref.Hyper(kind="sgd-momentum", **HP)
    slots = [dict() for _ in params]
    losses, snaps = [], {}
    for it in range(1, ITERS + 1):
        x, y = batches[(it - 1) % len(batches)]
        losses.append(_cpu_step(net, params, slots, hp, x, y, it))
        if it in CHECKPOINTS:
            snaps[it] = [p.detach().numpy().copy() for p in params]
    return gpu, (losses, snaps), batches


def test_gpu_schedules_bitwise_identical(runs):
    gpu, _, _ = runs
    base_losses, base_snaps, _ = gpu["baseline"]
    for s in ("backward-fusion", "forward-fusion"):
        losses, snaps, _ = gpu[s]
        assert losses == base_losses, s
        for it in CHECKPOINTS:
            for a, b in zip(snaps[it], base_snaps[it]):
                assert a.tobytes() == b.tobytes(), (s, it)


def test_one_step_from_identical_parameters_within_1e5(runs):
    """Teacher forcing: at several points of the GPU trajectory, restart the
    CPU reference path from the GPU's parameters, momentum and BN statistics
    and take one step; every tensor agrees with the GPU's next step to 1e-5
    (norm-wise relative)."""
    from oracle import optim_ref
    _setup_numerics()
    batches = runs[2]
    record = {}
    for start in (0, 20, 60):
        g = of.build_classifier("resnet18_cifar", device=DEV, seed=0)
        pol = of.OptimizerPolicy("sgd-momentum", **HP)
        for it in range(1, start + 1):
            x, y = batches[(it - 1) % len(batches)]
            of.run_baseline(g, pol, (x.to(DEV), y.to(DEV)), timing=False)
        net = _cpu_net()
        net.load_state_dict({k: v.detach().cpu() for k, v in g.module.state_dict().items()})
        params = [p for p in net.parameters() if p.requires_grad]
        names = [n for n, p in net.named_parameters() if p.requires_grad]
        assert names == [p.name for p in g.parameters]
        slots = [{"momentum": gp.history["momentum"].detach().cpu().numpy().reshape(-1).copy()}
                 if "momentum" in gp.history else {} for gp in g.parameters]
        before = [gp.value.detach().cpu().numpy().copy() for gp in g.parameters]
        x, y = batches[start % len(batches)]
        of.run_baseline(g, pol, (x.to(DEV), y.to(DEV)), timing=False)
        _cpu_step(net, params, slots, optim_ref.Hyper(kind="sgd-momentum", **HP), x, y, start + 1)
        worst_p = worst_d = 0.0
        for gp, cp, b in zip(g.parameters, params, before):
            got, want = gp.value.detach().cpu().numpy(), cp.detach().numpy()
            r = _rel(want, got)
            worst_p = max(worst_p, r)
            assert r <= 1e-5, (start, gp.name, r)
            worst_d = max(worst_d, _rel(want - b, got - b))   # the update itself
        record[start] = {"param_rel_max": worst_p, "update_rel_max": worst_d}
        assert worst_d <= 1e-2, (start, worst_d)
    out = os.environ.get("OPTFUSE_PARITY_OUT")
    if out:
        with open(out + ".one_step.json", "w") as f:
            json.dump(record, f, indent=1)


def test_free_running_losses_indistinguishable(runs):
    gpu, (cpu_losses, cpu_snaps), _ = runs
    losses, snaps, g = gpu["baseline"]
    rel = [abs(a - b) / abs(b) for a, b in zip(losses, cpu_losses)]
    growth = {}
    for it in CHECKPOINTS:
        errs = [_rel(a, b) for a, b in zip(snaps[it], cpu_snaps[it])]
        growth[it] = {"max": max(errs), "median": float(np.median(errs))}
    # the per-iteration loss change of training itself (the signal)
    steps = [abs(a - b) / abs(b) for a, b in zip(cpu_losses[1:], cpu_losses[:-1])]
    out = os.environ.get("OPTFUSE_PARITY_OUT")
    if out:
        with open(out, "w") as f:
            json.dump({"config": "C1 ResNet-18/CIFAR b32, SGD-m lr 0.1 m 0.9 wd 5e-4, fp32 (TF32 off), "
                                 "BN train, deterministic cuDNN, 8 synthetic batches cycled",
                       "gpu_losses": losses, "cpu_losses": cpu_losses,
                       "loss_rel_diff_max": max(rel), "loss_rel_diff_median": float(np.median(rel)),
                       "loss_step_change_median": float(np.median(steps)),
                       "param_rel_err_by_step": growth,
                       "tensors": [p.name for p in g.parameters]}, f, indent=1)
    assert growth[1]["max"] <= 1e-5, growth[1]
    # indistinguishable: far below the training signal over the whole run
    assert max(rel[:10]) <= 1e-4, rel[:10]
    assert float(np.median(rel)) <= 0.05 * float(np.median(steps)), (np.median(rel), np.median(steps))
    assert abs(np.mean(losses[-10:]) - np.mean(cpu_losses[-10:])) <= 0.05 * np.mean(cpu_losses[-10:])
