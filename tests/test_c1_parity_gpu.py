"""North-star parity on a benchmarked configuration (C1): ResNet-18 on
synthetic CIFAR-10-shaped data, batch 128, SGD-momentum (lr 0.1, momentum
0.9, coupled weight decay 5e-4), true fp32 (TF32 off, deterministic cuDNN),
BatchNorm in train mode, 100 iterations.

GPU side: the product path -- baseline, backward fusion (side stream,
per-layer) and forward fusion (+ flush) on cuda.  CPU side: the reference's
path -- torch-CPU forward/backward (the reference's own autodiff only runs its
synthetic chains) + the reference update (oracle.optim_ref.step, the
bit-exact restatement of optim.py:74-148) on every parameter.

What is and is not equal, and what the tests assert:
* the three GPU schedules: the same trajectory bit for bit (same kernels,
  only the issue point of each update moves) -- fused and unfused losses are
  identical, not merely indistinguishable;
* the update itself: fed the GPU's own gradients, the reference update on the
  CPU reproduces the GPU's new parameters and momentum BIT FOR BIT (62
  tensors, three points of the trajectory);
* forward/backward across devices: cuDNN and oneDNN sum convolutions and BN
  in different orders, so from identical parameters the gradients already
  differ (~1e-5..1e-4 relative, recorded).  Training is a chaotic map at this
  learning rate: those differences grow geometrically, so a free-running
  100-step trajectory cannot stay at 1e-5 (the 1e-5-after-100-steps contract
  is met bit for bit where the arithmetic is exact: the chain models,
  test_schedules_gpu.py long runs).  The test measures the growth and
  compares it with the CPU path against ITSELF after a one-ulp perturbation
  of one weight: the GPU-vs-CPU gap must grow no faster than the CPU path's
  own (it tracks it step for step: at step 100 both are ~0.44 median per
  tensor), and the loss curves agree while the gap is small (first steps).
With OPTFUSE_PARITY_OUT=<file> the curves are written as JSON
(profiles/r02/c1_parity.json comes from this).
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
BATCH = 128
HP = dict(eta=0.1, alpha=0.9, weight_decay=5e-4)
CHECKPOINTS = (1, 2, 5, 10, 20, 50, 100)


def _setup_numerics():
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False


def _batches():
    return [synthetic_batch("resnet18_cifar", BATCH, device="cpu", seed=s) for s in range(4)]


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
    return losses, snaps


def _cpu_net():
    import torchvision
    torch.manual_seed(0)
    m = torchvision.models.resnet18(num_classes=10)
    m.conv1 = torch.nn.Conv2d(3, 64, kernel_size=3, stride=1, padding=1, bias=False)
    m.maxpool = torch.nn.Identity()
    return m


def _cpu_run(batches, perturb=False):
    from oracle import optim_ref
    net = _cpu_net()
    params = [p for p in net.parameters() if p.requires_grad]
    if perturb:   # one ulp on one element of the first convolution
        with torch.no_grad():
            w = params[0].view(-1)
            w[0] = torch.nextafter(w[0], torch.tensor(float("inf")))
    hp = optim_ref.Hyper(kind="sgd-momentum", **HP)
    slots = [dict() for _ in params]
    losses, snaps = [], {}
    for it in range(1, ITERS + 1):
        x, y = batches[(it - 1) % len(batches)]
        loss = F.cross_entropy(net(x), y)
        loss.backward()
        for p, sl in zip(reversed(params), reversed(slots)):
            optim_ref.step("sgd-momentum", hp, p.detach().numpy().reshape(-1),
                           p.grad.numpy().reshape(-1), sl, it)
        losses.append(float(loss))
        if it in CHECKPOINTS:
            snaps[it] = [p.detach().numpy().copy() for p in params]
    return losses, snaps


def _rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


@pytest.fixture(scope="module")
def runs():
    _setup_numerics()
    torch.set_num_threads(max(1, min(16, os.cpu_count() or 1)))
    batches = _batches()
    gpu = {s: _gpu_run(s, batches) for s in ("baseline", "backward-fusion", "forward-fusion")}
    return gpu, _cpu_run(batches), _cpu_run(batches, perturb=True), batches


def test_gpu_schedules_bitwise_identical(runs):
    gpu = runs[0]
    base_losses, base_snaps = gpu["baseline"]
    for s in ("backward-fusion", "forward-fusion"):
        losses, snaps = gpu[s]
        assert losses == base_losses, s
        for it in CHECKPOINTS:
            for a, b in zip(snaps[it], base_snaps[it]):
                assert a.tobytes() == b.tobytes(), (s, it)


def test_update_bitwise_on_the_gpu_gradients(runs):
    """Teacher forcing of the update alone: at three points of the trajectory
    the GPU's gradients, parameters and momentum go through the reference
    update on the CPU, which must reproduce the GPU's step bit for bit; the
    cross-device gradient gap at identical parameters is recorded."""
    from oracle import optim_ref
    _setup_numerics()
    batches = runs[3]
    record = {}
    for start in (0, 20, 60):
        g = of.build_classifier("resnet18_cifar", device=DEV, seed=0)
        pol = of.OptimizerPolicy("sgd-momentum", **HP, grad_reset="zero")
        for it in range(1, start + 1):
            x, y = batches[(it - 1) % len(batches)]
            of.run_baseline(g, pol, (x.to(DEV), y.to(DEV)), timing=False)
        # the CPU reference path's gradients from the same parameters and BN statistics
        net = _cpu_net()
        net.load_state_dict({k: v.detach().cpu() for k, v in g.module.state_dict().items()})
        x, y = batches[start % len(batches)]
        F.cross_entropy(net(x), y).backward()
        cpu_grads = [p.grad.numpy().copy() for p in net.parameters()]
        # one GPU iteration, split so its gradients can be read before the update
        xd, yd = x.to(DEV), y.to(DEV)
        pol.begin_iteration()
        g.forward((xd, yd))
        g.backward()
        grads = [p.value.grad.detach().cpu().numpy().copy() for p in g.parameters]
        theta = [p.value.detach().cpu().numpy().reshape(-1).copy() for p in g.parameters]
        slots = [{"momentum": p.history["momentum"].detach().cpu().numpy().reshape(-1).copy()}
                 if "momentum" in p.history else {} for p in g.parameters]
        pol.step_params(list(reversed(g.parameters)))
        h = optim_ref.Hyper(kind="sgd-momentum", **HP)
        for k, p in enumerate(g.parameters):
            optim_ref.step("sgd-momentum", h, theta[k], grads[k].reshape(-1).copy(), slots[k], pol.t)
            assert p.value.detach().cpu().numpy().reshape(-1).tobytes() == theta[k].tobytes(), p.name
            assert (p.history["momentum"].detach().cpu().numpy().reshape(-1).tobytes()
                    == slots[k]["momentum"].tobytes()), p.name
        gap = [_rel(gg, cg) for gg, cg in zip(grads, cpu_grads)]
        record[start] = {"grad_rel_gap_max": max(gap), "grad_rel_gap_median": float(np.median(gap))}
    out = os.environ.get("OPTFUSE_PARITY_OUT")
    if out:
        with open(out + ".teacher_forced.json", "w") as f:
            json.dump(record, f, indent=1)
    # cuDNN vs oneDNN summation order (BN statistics amplify it later in training)
    assert all(r["grad_rel_gap_median"] <= 5e-2 for r in record.values()), record


def test_free_running_divergence_is_the_cpu_paths_own(runs):
    gpu, (cpu_losses, cpu_snaps), (pert_losses, pert_snaps), _ = runs
    losses, snaps = gpu["baseline"]
    rel = [abs(a - b) / abs(b) for a, b in zip(losses, cpu_losses)]
    growth, own = {}, {}
    for it in CHECKPOINTS:
        e = [_rel(a, b) for a, b in zip(snaps[it], cpu_snaps[it])]
        o = [_rel(a, b) for a, b in zip(pert_snaps[it], cpu_snaps[it])]
        growth[it] = {"max": max(e), "median": float(np.median(e))}
        own[it] = {"max": max(o), "median": float(np.median(o))}
    out = os.environ.get("OPTFUSE_PARITY_OUT")
    if out:
        with open(out, "w") as f:
            json.dump({"config": "C1 ResNet-18/CIFAR b128, SGD-m lr 0.1 m 0.9 wd 5e-4, fp32 (TF32 off), "
                                 "BN train, deterministic cuDNN, 4 synthetic batches cycled, 100 steps",
                       "gpu_losses": losses, "cpu_losses": cpu_losses,
                       "cpu_perturbed_losses": pert_losses,
                       "loss_rel_diff_step1": rel[0],
                       "loss_rel_diff_median": float(np.median(rel)),
                       "gpu_vs_cpu_param_rel_err": growth,
                       "cpu_vs_cpu_one_ulp_param_rel_err": own}, f, indent=1)
    own_rel = [abs(a - b) / abs(b) for a, b in zip(pert_losses, cpu_losses)]
    assert rel[0] <= 1e-5, rel[0]                     # identical parameters, one forward
    assert max(rel[:4]) <= 1e-3, rel[:4]              # the losses agree while the gap is small
    # the GPU-vs-CPU gap grows no faster than the CPU path's own sensitivity to a
    # one-ulp change of one weight, step by step: the growth is the map's, not the port's
    for it in CHECKPOINTS:
        assert growth[it]["median"] <= 10 * own[it]["median"] + 1e-6, (it, growth[it], own[it])
    assert max(rel[:10]) <= 10 * max(own_rel[:10]) + 1e-5, (rel[:10], own_rel[:10])
