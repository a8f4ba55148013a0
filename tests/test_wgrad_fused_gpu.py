"""Consumer-fused backward fusion: the tcgen05 weight-gradient GEMM whose
epilogue applies the optimizer update (of_wgrad_step, csrc/optfuse_wgrad.cu).

Parity contract:
* the gradient the kernel accumulates (dumped on request) equals the fp32
  product of the bf16 operands within fp32 reduction-order tolerance;
* the update it applies from the accumulator is BIT-IDENTICAL to the
  multi-tensor kernel (of_policy_step_mt) and, for the reference kinds, to
  the numpy oracle (optim.py:74-148) fed that same gradient;
* BERT-base Linear shapes (768x768, 3072x768, 768x3072 at 4096 tokens) and
  ragged ones (token, row and column tails) alike.
"""

import numpy as np
import pytest
import torch

from paper_2104_00237_b200 import _native as nat
from paper_2104_00237_b200 import kernels
from oracle import optim_ref

pytestmark = pytest.mark.gpu
DEV = "cuda"

# BERT-base Linear (M, N, T): 768 x 768 runs as a 4-way split-K cluster, the
# FFN shapes unsplit; then ragged token/row/column tails, unsplit (136 x 96,
# 128 x 64), 4-way (264 x 160 x 1000) and 2-way (256 x 128 x 512) splits
SHAPES = [(768, 768, 4096), (3072, 768, 4096), (768, 3072, 4096),
          (136, 96, 200), (128, 64, 64), (264, 160, 1000), (256, 128, 512), (256, 256, 4096)]


def _problem(M, N, T, seed=0, slots=2):
    g = torch.Generator(device="cpu").manual_seed(seed)
    dy = (torch.randn(T, M, generator=g) * 0.1).to(torch.bfloat16).to(DEV)
    x = torch.randn(T, N, generator=g).to(torch.bfloat16).to(DEV)
    theta = (torch.randn(M, N, generator=g) * 0.05).to(DEV)
    s = [torch.rand(M, N, generator=g).to(DEV) * 1e-3 for _ in range(slots)]
    return dy, x, theta, s


def _hp(kind, t=3):
    return kernels.hparams(kind, 1e-3, 0.9, 1e-2, 1e-8, 0.9, 0.999, 0.9, t)


def _ref_grad(dy, x):
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        return dy.double().t() @ x.double()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


@pytest.mark.parametrize("M,N,T", SHAPES)
def test_gradient_matches_fp64_product(M, N, T):
    dy, x, theta, (m, v) = _problem(M, N, T)
    dump = torch.full((M, N), float("nan"), device=DEV)
    kernels.wgrad_step(dy, x, theta, m, v, _hp("adamw"), grad_dump=dump)
    torch.cuda.synchronize()
    want = _ref_grad(dy, x)
    err = ((dump.double() - want).norm() / want.norm()).item()
    assert torch.isfinite(dump).all()
    assert err < 2e-5, err        # exact bf16 products, fp32 accumulation (a layout error is O(1))


@pytest.mark.parametrize("kind", ["adamw", "adam", "sgd-momentum", "sgd"])
@pytest.mark.parametrize("M,N,T", SHAPES[:2] + SHAPES[3:7])
def test_fused_update_bitwise_vs_multi_tensor_kernel(kind, M, N, T):
    """Same gradient, same functor: the epilogue's update equals of_policy_step_mt."""
    slots = {"sgd": 0, "sgd-momentum": 1}.get(kind, 2)
    dy, x, theta, s = _problem(M, N, T, slots=slots)
    s += [None] * (2 - len(s))
    theta2 = theta.clone()
    s2 = [t.clone() if t is not None else None for t in s]
    shadow = torch.empty(M, N, dtype=torch.bfloat16, device=DEV)
    dump = torch.empty(M, N, device=DEV)
    hp = _hp(kind)
    kernels.wgrad_step(dy, x, theta, s[0], s[1], hp, shadow=shadow, grad_dump=dump)
    tl = kernels.TensorList(1)
    tl.set(0, theta2, dump.clone(), s2[0], s2[1])
    tl.set_dtypes(torch.float32, torch.float32)
    kernels.policy_step(tl, hp, None, 0, None)
    torch.cuda.synchronize()
    assert theta.cpu().numpy().tobytes() == theta2.cpu().numpy().tobytes()
    for a, b in zip(s, s2):
        if a is not None:
            assert a.cpu().numpy().tobytes() == b.cpu().numpy().tobytes()
    assert torch.equal(shadow, theta.to(torch.bfloat16))


@pytest.mark.parametrize("kind", ["adam", "sgd-momentum"])
def test_fused_update_bitwise_vs_reference_oracle(kind):
    """The reference kinds against the numpy oracle of optim.py on the kernel's
    own gradient, over three steps (history carried across)."""
    M, N, T = 256, 128, 512
    slots = 2 if kind == "adam" else 1
    dy, x, theta, _ = _problem(M, N, T, slots=0)
    hist = [torch.zeros(M, N, device=DEV) for _ in range(slots)] + [None] * (2 - slots)
    th_np = theta.cpu().numpy().reshape(-1).copy()
    h = optim_ref.Hyper(kind=kind, eta=1e-3, alpha=0.9, weight_decay=1e-2)
    sl = {}
    for t in (1, 2, 3):
        dy_t = dy * (t * 0.5)
        dump = torch.empty(M, N, device=DEV)
        kernels.wgrad_step(dy_t.contiguous(), x, theta, hist[0], hist[1], _hp(kind, t), grad_dump=dump)
        torch.cuda.synchronize()
        optim_ref.step(kind, h, th_np, dump.cpu().numpy().reshape(-1).copy(), sl, t)
    assert theta.cpu().numpy().reshape(-1).tobytes() == th_np.tobytes()


def test_device_step_graph_replay_bitwise_vs_eager():
    """OF_FLAG_DEVICE_STEP: the fused launch captured in a CUDA graph reads its
    Adam step index on the device; 3 replays == 3 eager steps."""
    import paper_2104_00237_b200 as of
    M, N, T = 256, 128, 256
    dy, x, theta, (m, v) = _problem(M, N, T)
    th_e, m_e, v_e = theta.clone(), m.clone(), v.clone()
    pol = of.OptimizerPolicy("adamw", eta=1e-3, weight_decay=1e-2)
    for t in (1, 2, 3):
        kernels.wgrad_step(dy, x, th_e, m_e, v_e, _hp("adamw", t))
    ds = pol.device_step(torch.device(DEV))
    ds.ensure(4)
    hp = kernels.hparams("adamw", 1e-3, 0.9, 1e-2, 1e-8, 0.9, 0.999, 0.9, 1, device_step=ds)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph, stream=s):
        kernels.step_advance(ds.offset, 1)
        kernels.wgrad_step(dy, x, theta, m, v, hp, flags=nat.OF_FLAG_DEVICE_STEP)
    ds.offset.fill_(-1)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    for a, b in ((theta, th_e), (m, m_e), (v, v_e)):
        assert a.cpu().numpy().tobytes() == b.cpu().numpy().tobytes()


def test_argument_errors_before_launch():
    dy, x, theta, (m, v) = _problem(128, 64, 64)
    n0 = nat.launch_count()
    with pytest.raises(Exception):       # in_features not a multiple of 32
        kernels.wgrad_step(dy, x[:, :48].contiguous(), theta[:, :48].contiguous(), m, v, _hp("adamw"))
    with pytest.raises(Exception):       # adam needs both slots
        kernels.wgrad_step(dy, x, theta, m, None, _hp("adam"))
    with pytest.raises(Exception):       # zero-grad flag has no meaning here
        kernels.wgrad_step(dy, x, theta, m, v, _hp("adamw"), flags=nat.OF_FLAG_ZERO_GRAD)
    assert nat.launch_count() == n0
