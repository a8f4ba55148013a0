"""Kernel parity on the GPU: the sm_100a update kernels against the pinned
oracle (bit-exact for the reference kinds) and torch AdamW (tolerance)."""

import ctypes

import numpy as np
import pytest
import torch

import paper_2104_00237_b200 as of
from paper_2104_00237_b200 import _native as nat
from paper_2104_00237_b200 import kernels
from oracle import optim_ref

pytestmark = pytest.mark.gpu
DEV = "cuda"
KINDS = optim_ref.KINDS
ETA = {"sgd": 0.01, "sgd-momentum": 0.01, "adagrad": 0.01, "rmsprop": 1e-3,
       "adadelta": 1.0, "adam": 1e-3}
TDT = {"f32": torch.float32, "f64": torch.float64}


def _param(arr, pid=0):
    return of.Parameter(pid, torch.nn.Parameter(torch.from_numpy(arr.copy()).to(DEV)))


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("wd", [0.0, 1e-2])
def test_golden_policy_trajectories(policy_golden, kind, prec, wd):
    key = f"{kind}|{prec}|wd{wd}"
    p = _param(policy_golden[key + "|theta0"])
    grads = policy_golden[key + "|grads"]
    traj = policy_golden[key + "|traj"]
    pol = of.OptimizerPolicy(kind=kind, eta=ETA[kind], weight_decay=wd)
    for s in range(grads.shape[0]):
        pol.begin_iteration()
        p.value.grad = torch.from_numpy(grads[s].copy()).to(DEV)
        pol.step(p)
        got = p.value.detach().cpu().numpy()
        assert got.tobytes() == traj[s].tobytes(), f"step {s + 1}: max diff {np.abs(got - traj[s]).max()}"
        assert not p.value.grad.any(), "grad must be zero after the step (optim.py:111)"
    for name in pol.history_slots():
        assert p.history[name].cpu().numpy().tobytes() == policy_golden[key + "|slot|" + name].tobytes()


def _resnet18_shapes():
    g = of.build_classifier("resnet18_cifar", device="cpu")
    return [tuple(p.value.shape) for p in g.parameters]


@pytest.mark.parametrize("kind,hp", [("sgd-momentum", dict(eta=0.1, alpha=0.9, weight_decay=5e-4)),
                                     ("adam", dict(eta=1e-3, weight_decay=1e-4)),
                                     ("adadelta", dict(eta=1.0, weight_decay=1e-4))])
def test_multi_tensor_resnet18_shapes_bitwise(kind, hp):
    """100 injected-gradient steps over the 62 ResNet-18/CIFAR tensors (11.17 M
    elements, one multi-tensor launch per step) equal the oracle bit for bit."""
    shapes = _resnet18_shapes()
    rng = np.random.default_rng(0)
    thetas = [(rng.standard_normal(int(np.prod(s))) * 0.05).astype(np.float32) for s in shapes]
    params = [_param(t, i) for i, t in enumerate(thetas)]
    pol = of.OptimizerPolicy(kind=kind, **hp)
    ref_slots = [dict() for _ in shapes]
    h = optim_ref.Hyper(kind=kind, **hp)
    steps = 100 if kind == "sgd-momentum" else 12
    for s in range(steps):
        pol.begin_iteration()
        grads = [(rng.standard_normal(t.size) * 0.01).astype(np.float32) for t in thetas]
        for p, g in zip(params, grads):
            p.value.grad = torch.from_numpy(g).to(DEV)
        pol.step_params(reversed(params))
        for t, g, sl in zip(thetas, grads, ref_slots):
            optim_ref.step(kind, h, t, g, sl, s + 1)
    for p, t, sl in zip(params, thetas, ref_slots):
        assert p.value.detach().cpu().numpy().reshape(-1).tobytes() == t.tobytes()
        for name in pol.history_slots():
            assert p.history[name].cpu().numpy().reshape(-1).tobytes() == sl[name].tobytes()


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
@pytest.mark.parametrize("kind", ["sgd-momentum", "adam"])
def test_unaligned_and_ragged_views(offset, kind):
    """Parameters that are views at unaligned offsets of one buffer, with sizes
    that are not multiples of the vector width or tile (scalar path + tails)."""
    sizes = [1, 3, 4, 5, 4095, 4096, 4097, 70001]
    total = sum(sizes) + offset
    rng = np.random.default_rng(offset)
    flat_p = torch.from_numpy(rng.standard_normal(total).astype(np.float32)).to(DEV)
    flat_g = torch.zeros(total, device=DEV)
    params, thetas, o = [], [], offset
    for i, n in enumerate(sizes):
        v = torch.nn.Parameter(flat_p[o:o + n])
        params.append(of.Parameter(i, v))
        thetas.append(flat_p[o:o + n].cpu().numpy().copy())
        o += n
    pol = of.OptimizerPolicy(kind=kind, eta=1e-2)
    h = optim_ref.Hyper(kind=kind, eta=1e-2)
    slots = [dict() for _ in sizes]
    o = offset
    views = []
    for n in sizes:
        views.append(flat_g[o:o + n])
        o += n
    for s in range(5):
        pol.begin_iteration()
        for p, v in zip(params, views):
            v.copy_(torch.randn(v.numel(), device=DEV))
            p.value.grad = v
        host_g = [v.cpu().numpy().copy() for v in views]
        pol.step_params(params)
        for t, g, sl in zip(thetas, host_g, slots):
            optim_ref.step(kind, h, t, g, sl, s + 1)
    for p, t in zip(params, thetas):
        assert p.value.detach().cpu().numpy().tobytes() == t.tobytes()
    assert not flat_g.any()


def test_many_tensors_chunked_launches():
    """> 256 tensors (two launches per step: 256 + 44) and tiny tensors."""
    rng = np.random.default_rng(3)
    arrs = [rng.standard_normal(int(n)).astype(np.float32) for n in rng.integers(1, 300, 300)]
    params = [_param(a, i) for i, a in enumerate(arrs)]
    pol = of.OptimizerPolicy("adam", eta=1e-3)
    h = optim_ref.Hyper(kind="adam", eta=1e-3)
    slots = [dict() for _ in arrs]
    for s in range(3):
        pol.begin_iteration()
        gs = [rng.standard_normal(a.size).astype(np.float32) for a in arrs]
        for p, g in zip(params, gs):
            p.value.grad = torch.from_numpy(g).to(DEV)
        n0 = nat.launch_count()
        pol.step_params(params)
        assert nat.launch_count() - n0 == 2  # 256 + 44
        for a, g, sl in zip(arrs, gs, slots):
            optim_ref.step("adam", h, a, g, sl, s + 1)
    for p, a in zip(params, arrs):
        assert p.value.detach().cpu().numpy().tobytes() == a.tobytes()


def test_grad_reset_none_releases_gradients():
    rng = np.random.default_rng(5)
    a = rng.standard_normal(1000).astype(np.float32)
    p = _param(a)
    pol = of.OptimizerPolicy("sgd-momentum", eta=0.1, grad_reset="none")
    h = optim_ref.Hyper(kind="sgd-momentum", eta=0.1)
    sl = {}
    for s in range(3):
        pol.begin_iteration()
        g = rng.standard_normal(1000).astype(np.float32)
        p.value.grad = torch.from_numpy(g.copy()).to(DEV)
        pol.step(p)
        assert p.value.grad is None
        optim_ref.step("sgd-momentum", h, a, g, sl, s + 1)
    assert p.value.detach().cpu().numpy().tobytes() == a.tobytes()


def test_missing_grad_steps_with_zero_gradient():
    """The reference steps every parameter, even one without contributions."""
    a = np.linspace(-1, 1, 77).astype(np.float32)
    p = _param(a)
    pol = of.OptimizerPolicy("sgd-momentum", eta=0.1, weight_decay=0.01)
    pol.begin_iteration()
    pol.step(p)
    optim_ref.step("sgd-momentum", optim_ref.Hyper("sgd-momentum", eta=0.1, weight_decay=0.01),
                   a, np.zeros_like(a), {}, 1)
    assert p.value.detach().cpu().numpy().tobytes() == a.tobytes()


def _raw_list(ps, gs, s0=None, s1=None, sh=None):
    tl = kernels.TensorList(len(ps))
    for i in range(len(ps)):
        tl.set(i, ps[i], gs[i], s0[i] if s0 else None, s1[i] if s1 else None,
               sh[i] if sh else None)
    tl.set_dtypes(ps[0].dtype, gs[0].dtype)
    return tl


def test_bf16_grads_fp32_master_and_bf16_shadow():
    """Mixed precision: bf16 gradients into fp32 master weights, bf16 shadow
    written in the same pass; equals the fp32 kernel fed the upcast grads."""
    torch.manual_seed(0)
    n = [5000, 3, 131073]
    master = [torch.randn(k, device=DEV) for k in n]
    m = [torch.zeros(k, device=DEV) for k in n]
    v = [torch.zeros(k, device=DEV) for k in n]
    shadow = [torch.empty(k, device=DEV, dtype=torch.bfloat16) for k in n]
    ref_p = [x.cpu().numpy().copy() for x in master]
    ref_s = [dict() for _ in n]
    h = optim_ref.Hyper(kind="adam", eta=1e-3, weight_decay=1e-4)
    for t in range(1, 4):
        g16 = [torch.randn(k, device=DEV).to(torch.bfloat16) for k in n]
        host_g = [g.float().cpu().numpy() for g in g16]
        tl = _raw_list(master, g16, m, v, shadow)
        hp = kernels.hparams("adam", 1e-3, 0.9, 1e-4, 1e-8, 0.9, 0.999, 0.9, t)
        kernels.policy_step(tl, hp, None, nat.OF_FLAG_SHADOW_BF16 | nat.OF_FLAG_ZERO_GRAD, None)
        for i, g in enumerate(g16):
            assert not g.any()
        for i in range(len(n)):
            optim_ref.step("adam", h, ref_p[i], host_g[i], ref_s[i], t)
    for i in range(len(n)):
        assert master[i].cpu().numpy().tobytes() == ref_p[i].tobytes()
        assert torch.equal(shadow[i], master[i].to(torch.bfloat16))


def test_adamw_matches_torch_adamw():
    """AdamW is pinned to torch.optim.AdamW(foreach=False) on CPU (no reference)."""
    rng = np.random.default_rng(7)
    th = rng.standard_normal(10007).astype(np.float32)
    p = _param(th)
    pol = of.OptimizerPolicy("adamw", eta=1e-3, weight_decay=0.05)
    ref = torch.nn.Parameter(torch.from_numpy(th.copy()))
    opt = torch.optim.AdamW([ref], lr=1e-3, weight_decay=0.05, foreach=False)
    for s in range(20):
        g = rng.standard_normal(10007).astype(np.float32)
        pol.begin_iteration()
        p.value.grad = torch.from_numpy(g.copy()).to(DEV)
        pol.step(p)
        ref.grad = torch.from_numpy(g.copy())
        opt.step()
    got = p.value.detach().cpu().numpy()
    want = ref.detach().numpy()
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel < 1e-6, rel
    assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-3)) < 1e-5
    st = opt.state[ref]
    np.testing.assert_allclose(p.history["exp_avg"].cpu().numpy(), st["exp_avg"].numpy(),
                               rtol=1e-5, atol=1e-9)
    np.testing.assert_allclose(p.history["exp_avg_sq"].cpu().numpy(), st["exp_avg_sq"].numpy(),
                               rtol=1e-5, atol=1e-12)


def test_sqnorm_and_clip_factor():
    rng = np.random.default_rng(11)
    gs = [rng.standard_normal(int(k)).astype(np.float32) for k in (1, 7, 4096, 123457, 3)]
    g = of.build_model("chain", layers=1, width=1, device=DEV)  # container for parameters
    params = [_param(np.zeros_like(x), i) for i, x in enumerate(gs)]
    for p, x in zip(params, gs):
        p.value.grad = torch.from_numpy(x).to(DEV)
    g.parameters = params
    want_sq = sum(float(np.dot(x.astype(np.float64), x.astype(np.float64))) for x in gs)
    norm = want_sq ** 0.5
    f = of.clip_by_global_norm(g, 1.0)
    assert abs(float(f) - 1.0 / norm) <= 1e-12 * (1.0 / norm)
    assert params[0]._grad_scale is not None
    assert float(of.clip_by_global_norm(g, 1e9)) == 1.0
    # deterministic: same bits twice
    a = float(of.clip_by_global_norm(g, 0.5))
    b = float(of.clip_by_global_norm(g, 0.5))
    assert a == b


def test_spec_kats_on_gpu(spec_kats):
    p = _param(np.array([1.0], np.float32))
    p.value.grad = torch.tensor([2.0], device=DEV)
    pol = of.OptimizerPolicy("sgd", eta=0.1)
    pol.begin_iteration()
    pol.step(p)
    assert p.value.detach().cpu().tolist() == spec_kats["sgd"]["theta"]
    assert p.value.grad.cpu().tolist() == [0.0]
    p = _param(np.array([1.0], np.float32))
    pol = of.OptimizerPolicy("sgd-momentum", eta=0.1, alpha=0.9)
    got = []
    for _ in range(2):
        pol.begin_iteration()
        p.value.grad = p.value.detach().clone()
        pol.step(p)
        got.append(float(p.value))
    assert got == spec_kats["sgd_momentum"]["theta"]
    p = _param(np.array([1.0], np.float32))
    pol = of.OptimizerPolicy("sgd", eta=1.0, weight_decay=0.1)
    pol.begin_iteration()
    pol.step(p)
    assert p.value.detach().cpu().tolist() == spec_kats["weight_decay"]["theta"]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("max_ctas", [1, 7, 49, 148])
def test_capped_grid_same_bits(max_ctas, dtype):
    """A capped grid (background update on the side stream) walks the same
    tiles with fewer CTAs: identical results."""
    rng = np.random.default_rng(max_ctas)
    sizes = [3, 4097, 300001, 77]
    ps = [torch.from_numpy(rng.standard_normal(n).astype(dtype)).to(DEV) for n in sizes]
    gs = [torch.from_numpy(rng.standard_normal(n).astype(dtype)).to(DEV) for n in sizes]
    ms = [torch.zeros(n, device=DEV, dtype=ps[0].dtype) for n in sizes]
    vs = [torch.zeros(n, device=DEV, dtype=ps[0].dtype) for n in sizes]
    ref = [(p.cpu().numpy().copy(), g.cpu().numpy().copy()) for p, g in zip(ps, gs)]
    tl = _raw_list(ps, gs, ms, vs)
    hp = kernels.hparams("adam", 1e-3, 0.9, 1e-4, 1e-8, 0.9, 0.999, 0.9, 1, max_ctas=max_ctas)
    kernels.policy_step(tl, hp, None, 0, None)
    h = optim_ref.Hyper(kind="adam", eta=1e-3, weight_decay=1e-4)
    for p, (th, g) in zip(ps, ref):
        optim_ref.step("adam", h, th, g, {}, 1)
        assert p.cpu().numpy().tobytes() == th.tobytes()


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("kind", ["sgd-momentum", "adam"])
@pytest.mark.parametrize("mixed", [False, True])
def test_peer_step_simulated_ranks_on_one_gpu(world, kind, mixed):
    """of_dp_step_peer with W "ranks" whose buffers all live on this GPU (plain
    device pointers stand in for the NVLink peer mappings): the multi-peer
    logic -- rank-order gradient sum, 1/W scale, the update of each owned
    shard, parameter writes into every peer, gradient zeroing in every peer --
    against the oracle on the averaged gradient, bit for bit (fp32, and bf16
    parameters with fp32 master shards)."""
    rng = np.random.default_rng(5)
    n = 4 * world * 37
    S = n // world
    eta, wd = ETA[kind], 1e-3
    theta0 = rng.standard_normal(n).astype(np.float32)
    grads = [rng.standard_normal(n).astype(np.float32) for _ in range(world)]
    if mixed:   # bf16 model: parameters and gradients are bf16, masters fp32
        grads = [torch.from_numpy(g).to(torch.bfloat16).float().numpy() for g in grads]
        params = [torch.from_numpy(theta0).to(DEV).to(torch.bfloat16) for _ in range(world)]
        gbufs = [torch.from_numpy(g).to(DEV).to(torch.bfloat16) for g in grads]
        masters = [torch.from_numpy(theta0[r * S:(r + 1) * S].copy()).to(DEV) for r in range(world)]
    else:
        params = [torch.from_numpy(theta0.copy()).to(DEV) for _ in range(world)]
        gbufs = [torch.from_numpy(g.copy()).to(DEV) for g in grads]
        masters = [None] * world
    names = optim_ref.SLOTS[kind]
    states = [[torch.zeros(S, device=DEV) for _ in names] + [None, None] for _ in range(world)]
    scale = torch.full((), 1.0 / world, dtype=torch.float32, device=DEV)
    pdt = torch.bfloat16 if mixed else torch.float32
    for t in (1, 2):
        hp = kernels.hparams(kind, eta, 0.9, wd, 1e-8, 0.9, 0.999, 0.9, t)
        if t == 2:   # fresh gradients for the second step
            for w in range(world):
                gbufs[w].copy_(torch.from_numpy(grads[w]).to(gbufs[w].dtype))
        for r in range(world):
            pb = kernels.PeerBucket(world, r, pdt, pdt, [g.data_ptr() for g in gbufs],
                                    [p.data_ptr() for p in params], masters[r], states[r][0],
                                    states[r][1], r * S, S)
            kernels.dp_step_peer(pb, hp, scale, 0, None)
    torch.cuda.synchronize()
    theta = theta0.copy()
    slots = {}
    h = optim_ref.Hyper(kind=kind, eta=eta, weight_decay=wd)
    for t in (1, 2):
        g = grads[0].copy()
        for w in range(1, world):
            g = np.add(g, grads[w])
        g = np.multiply(g, np.float32(1.0 / world))
        optim_ref.step(kind, h, theta, g, slots, t)
    for r in range(world):
        assert not gbufs[r].float().any(), f"rank {r}: gradient not zeroed"
        if mixed:
            want = torch.from_numpy(theta).to(torch.bfloat16)
            assert torch.equal(params[r].cpu(), want), f"rank {r}: bf16 parameters"
            got_m = masters[r].cpu().numpy()
            assert got_m.tobytes() == theta[r * S:(r + 1) * S].tobytes()
        else:
            assert params[r].cpu().numpy().tobytes() == theta.tobytes(), f"rank {r}: parameters"
        for k, name in enumerate(names):
            got = states[r][k].cpu().numpy()
            assert got.tobytes() == slots[name][r * S:(r + 1) * S].tobytes(), (r, name)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("mixed", [False, True])
def test_peer_sqnorm_simulated_ranks_on_one_gpu(world, mixed):
    """of_dp_sqnorm_peer with W "ranks" on this GPU: each rank's partial is
    Σ over its shard of (Σ_w g_w)², the peers summed in rank order in the
    gradient's compute type exactly as of_dp_step_peer sums them; the ranks'
    partials add up to the numpy f64 value (reduction order: 1e-12), and
    accumulate=1 adds to the output."""
    rng = np.random.default_rng(world)
    n = 4 * world * 1031
    S = n // world
    grads = [rng.standard_normal(n).astype(np.float32) for _ in range(world)]
    if mixed:
        grads = [torch.from_numpy(g).to(torch.bfloat16).float().numpy() for g in grads]
        gbufs = [torch.from_numpy(g).to(DEV).to(torch.bfloat16) for g in grads]
    else:
        gbufs = [torch.from_numpy(g.copy()).to(DEV) for g in grads]
    gsum = grads[0].copy()
    for w in range(1, world):
        gsum = np.add(gsum, grads[w])           # f32, rank order
    ws = torch.empty(kernels.sqnorm_workspace_len(), dtype=torch.float64, device=DEV)
    pdt = torch.bfloat16 if mixed else torch.float32
    total = 0.0
    for r in range(world):
        out = torch.full((), 7.0, dtype=torch.float64, device=DEV)
        pb = kernels.PeerBucket(world, r, pdt, pdt, [g.data_ptr() for g in gbufs],
                                [g.data_ptr() for g in gbufs], None, None, None, r * S, S)
        kernels.dp_sqnorm_peer(pb, ws, out, False, None)
        want = float(np.sum(gsum[r * S:(r + 1) * S].astype(np.float64) ** 2))
        assert abs(out.item() - want) <= 1e-12 * want, (r, out.item(), want)
        kernels.dp_sqnorm_peer(pb, ws, out, True, None)     # accumulate
        assert abs(out.item() - 2 * want) <= 2e-12 * want
        total += want
    assert total > 0
    for w in range(world):   # the reduction only reads the gradients
        assert torch.equal(gbufs[w].float().cpu(), torch.from_numpy(grads[w]))


def test_copy_mt_many_tensors_any_alignment():
    """of_copy_mt: >256 tensors (two launches), odd byte counts and unaligned views."""
    torch.manual_seed(0)
    base = torch.randn(100000, device=DEV)
    srcs, dsts = [], []
    off = 1
    for i in range(300):
        n = int(torch.randint(1, 200, (1,)))
        srcs.append(base[off:off + n])            # 4-byte aligned only for most
        dsts.append(torch.empty(n, device=DEV))
        off += n + 1
    srcs.append(torch.randn(12345, device=DEV, dtype=torch.float64))
    dsts.append(torch.empty(12345, device=DEV, dtype=torch.float64))
    srcs.append(torch.randn(7, device=DEV).to(torch.bfloat16))
    dsts.append(torch.empty(7, device=DEV, dtype=torch.bfloat16))
    kernels.copy_mt(kernels.CopyList(dsts, srcs))
    torch.cuda.synchronize()
    for d, s in zip(dsts, srcs):
        assert torch.equal(d, s)


def test_tensor_beyond_2_31_elements():
    """One 2^31 + 6157-element tensor (26 GB with its gradient and momentum):
    64-bit element offsets; checked bitwise against the oracle on windows at
    the head, across the 2^31 boundary and at the ragged tail."""
    n = (1 << 31) + 6157
    if torch.cuda.get_device_properties(0).total_memory < 64 << 30:
        pytest.skip("needs a large-memory GPU")
    gen = torch.Generator(device=DEV).manual_seed(11)
    val = torch.randn(n, device=DEV, generator=gen)
    grad = torch.randn(n, device=DEV, generator=gen)
    wins = [(0, 4096), ((1 << 31) - 4096, (1 << 31) + 4096), (n - 5000, n)]
    before = [(val[a:b].cpu().numpy().copy(), grad[a:b].cpu().numpy().copy()) for a, b in wins]
    p = of.Parameter(0, torch.nn.Parameter(val))
    del val
    p.value.grad = grad
    del grad
    pol = of.OptimizerPolicy("sgd-momentum", eta=0.1, grad_reset="none")
    h = optim_ref.Hyper(kind="sgd-momentum", eta=0.1)
    pol.begin_iteration()
    pol.step(p)
    torch.cuda.synchronize()
    for (a, b), (th, g) in zip(wins, before):
        optim_ref.step("sgd-momentum", h, th, g, {}, 1)
        assert p.value[a:b].detach().cpu().numpy().tobytes() == th.tobytes(), (a, b)
    del p
    torch.cuda.empty_cache()


def test_empty_tensors_in_a_list():
    """Zero-element parameters beside ordinary ones: skipped by the packer,
    the others updated bitwise."""
    rng = np.random.default_rng(8)
    sizes = [0, 513, 0, 4096, 0, 7]
    arrs = [rng.standard_normal(s).astype(np.float32) for s in sizes]
    params = [_param(a, i) for i, a in enumerate(arrs)]
    pol = of.OptimizerPolicy("adam", eta=1e-3)
    h = optim_ref.Hyper(kind="adam", eta=1e-3)
    slots = [dict() for _ in arrs]
    for s in range(3):
        pol.begin_iteration()
        gs = [rng.standard_normal(a.size).astype(np.float32) for a in arrs]
        for p, g in zip(params, gs):
            p.value.grad = torch.from_numpy(g).to(DEV)
        pol.step_params(params)
        for a, g, sl in zip(arrs, gs, slots):
            optim_ref.step("adam", h, a, g, sl, s + 1)
    for p, a in zip(params, arrs):
        assert p.value.detach().cpu().numpy().tobytes() == a.tobytes()


class _Multicast1:
    """A one-device NVLS multicast object bound to a fresh physical allocation
    (CUDA driver API): ``uva`` is the unicast mapping, ``mva`` the multicast
    one.  None of torch's symmetric memory: it builds no multicast object for
    a single rank."""

    def __init__(self, nbytes: int):
        from cuda.bindings import driver as d
        self.d = d

        def ok(r):
            err, *rest = r if isinstance(r, tuple) else (r,)
            if err != d.CUresult.CUDA_SUCCESS:
                raise RuntimeError(str(err))
            return rest[0] if len(rest) == 1 else rest
        self.ok = ok
        torch.zeros(1, device=DEV)                     # primary context current
        dev = ok(d.cuDeviceGet(torch.cuda.current_device()))
        if not ok(d.cuDeviceGetAttribute(
                d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)):
            pytest.skip("no multicast support")
        fd = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        mp = d.CUmulticastObjectProp()
        mp.numDevices = 1
        mp.handleTypes = fd
        mp.size = nbytes
        gran = ok(d.cuMulticastGetGranularity(
            mp, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        size = (nbytes + gran - 1) // gran * gran
        mp.size = size
        self.size = size
        err, mc = d.cuMulticastCreate(mp)
        if err != d.CUresult.CUDA_SUCCESS:
            # the single-GPU boxes report multicast support but refuse to
            # create a one-device multicast object (CUDA_ERROR_INVALID_VALUE)
            pytest.skip(f"cuMulticastCreate: {err}")
        self.mc = mc
        ok(d.cuMulticastAddDevice(self.mc, dev))
        ap = d.CUmemAllocationProp()
        ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.requestedHandleTypes = fd
        ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = int(torch.cuda.current_device())
        self.mem = ok(d.cuMemCreate(size, ap, 0))
        ok(d.cuMulticastBindMem(self.mc, 0, self.mem, 0, size, 0))
        acc = d.CUmemAccessDesc()
        acc.location = ap.location
        acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uva = ok(d.cuMemAddressReserve(size, gran, 0, 0))
        ok(d.cuMemMap(self.uva, size, 0, self.mem, 0))
        ok(d.cuMemSetAccess(self.uva, size, [acc], 1))
        self.mva = ok(d.cuMemAddressReserve(size, gran, 0, 0))
        ok(d.cuMemMap(self.mva, size, 0, self.mc, 0))
        ok(d.cuMemSetAccess(self.mva, size, [acc], 1))

    def write(self, arr: np.ndarray) -> None:
        torch.cuda.synchronize()
        self.ok(self.d.cuMemcpyHtoD(self.uva, arr.ctypes.data, arr.nbytes))

    def read(self, n: int) -> np.ndarray:
        torch.cuda.synchronize()
        out = np.empty(n, dtype=np.float32)
        self.ok(self.d.cuMemcpyDtoH(out.ctypes.data, self.uva, out.nbytes))
        return out

    def close(self) -> None:
        d = self.d
        for va in (self.mva, self.uva):
            d.cuMemUnmap(va, self.size)
            d.cuMemAddressFree(va, self.size)
        d.cuMulticastUnbind(self.mc, torch.cuda.current_device(), 0, self.size)
        d.cuMemRelease(self.mem)
        d.cuMemRelease(self.mc)


@pytest.mark.parametrize("kind", ["sgd-momentum", "adam"])
def test_multicast_step_world1_against_oracle(kind):
    """of_dp_step_multicast through a real NVLS multicast object of one GPU:
    the in-switch reduced gradient load, the update and the multicast
    parameter and zero-gradient stores, bit for bit against the oracle (two
    steps, the shard in the middle of the buffer)."""
    n, begin, S = 4 * 1000, 4 * 100, 4 * 700
    gm, pm = _Multicast1(4 * n), _Multicast1(4 * n)
    try:
        rng = np.random.default_rng(12)
        theta0 = rng.standard_normal(n).astype(np.float32)
        grads = [rng.standard_normal(n).astype(np.float32) for _ in range(2)]
        pm.write(theta0)
        names = optim_ref.SLOTS[kind]
        states = [torch.zeros(S, device=DEV) for _ in names] + [None, None]
        eta, wd = ETA[kind], 1e-3
        mb = kernels.McBucket(1, 0, int(gm.mva), int(pm.mva), None, states[0], states[1], begin, S)
        mb.struct.local_param = int(pm.uva)
        for t in (1, 2):
            gm.write(grads[t - 1])
            kernels.dp_step_multicast(mb, kernels.hparams(kind, eta, 0.9, wd, 1e-8, 0.9, 0.999,
                                                          0.9, t), None, 0, None)
            g = gm.read(n)
            assert not g[begin:begin + S].any(), "shard gradient not zeroed"
            assert g[:begin].tobytes() == grads[t - 1][:begin].tobytes()
        theta = theta0[begin:begin + S].copy()
        slots = {}
        h = optim_ref.Hyper(kind=kind, eta=eta, weight_decay=wd)
        for t in (1, 2):
            optim_ref.step(kind, h, theta, grads[t - 1][begin:begin + S].copy(), slots, t)
        got = pm.read(n)
        assert got[begin:begin + S].tobytes() == theta.tobytes()
        assert got[:begin].tobytes() == theta0[:begin].tobytes()
        for k, name in enumerate(names):
            assert states[k].cpu().numpy().tobytes() == slots[name].tobytes(), name
    finally:
        gm.close()
        pm.close()


def test_multicast_step_argument_errors():
    """of_dp_step_multicast rejects bad buckets before any launch."""
    st = torch.zeros(8, device=DEV)
    buf = torch.zeros(64, device=DEV)
    hp = kernels.hparams("sgd-momentum", 0.1, 0.9, 0.0, 1e-8, 0.9, 0.999, 0.9, 1)
    cases = [
        kernels.McBucket(1, 0, buf.data_ptr(), buf.data_ptr(), buf, st, None, 2, 8),      # begin % 4
        kernels.McBucket(1, 1, buf.data_ptr(), buf.data_ptr(), buf, st, None, 0, 8),      # rank
        kernels.McBucket(1, 0, 0, buf.data_ptr(), buf, st, None, 0, 8),                   # NULL mc
        kernels.McBucket(1, 0, buf.data_ptr() + 4, buf.data_ptr(), buf, st, None, 0, 8),  # align
        kernels.McBucket(1, 0, buf.data_ptr(), buf.data_ptr(), buf, None, None, 0, 8),    # state0
        kernels.McBucket(1, 0, buf.data_ptr(), buf.data_ptr(), buf, st, None, 0, 8,
                         dtype=torch.bfloat16),                                            # dtype
        kernels.McBucket(1, 0, buf.data_ptr(), buf.data_ptr(), buf, st, None, 0, 8,
                         dtype=torch.float64),                                             # dtype
    ]
    n0 = nat.launch_count()
    for mb in cases:
        with pytest.raises(Exception):
            kernels.dp_step_multicast(mb, hp, None, 0, None)
    assert nat.launch_count() == n0
