"""Consumer-fused backward fusion in a real model (consumer.ConsumerFusion):
BERT (tiny config) as a bf16 module with fp32 masters, AdamW, every eligible
Linear weight updated inside its weight-gradient GEMM (of_wgrad_step), the
rest by the ordinary backward-fusion launches.

* first iteration from identical weights: every parameter the consumer kernel
  does not own is updated BIT-IDENTICALLY to plain backward fusion (same
  gradients -- the input-gradient GEMMs read the old weights in both), and
  the consumer-owned weights match the fp32 reference update of the fp64
  product dY^T X to fp32 accumulation tolerance;
* the tied MLM decoder weight (= word embeddings, two producers) is never
  consumer-fused;
* the whole iteration captured as a CUDA graph replays bit-identically to
  eager (device-side Adam step index in the fused epilogue too).
"""

import numpy as np
import pytest
import torch

import paper_2104_00237_b200 as of
from paper_2104_00237_b200.consumer import ConsumerFusion

pytestmark = pytest.mark.gpu
DEV = "cuda"
TINY_BERT = dict(num_hidden_layers=2, hidden_size=64, num_attention_heads=4, intermediate_size=128,
                 vocab_size=512, max_position_embeddings=64, attn_implementation="sdpa")


def _bert(seed=0):
    g = of.build_classifier("bert_base", device=DEV, seed=seed, config=TINY_BERT)
    g.track_counts = False
    g.use_master_weights()
    return g


def _inp():
    return of.models.synthetic_batch("bert_base", 8, device=DEV, seed=0, seq=32, vocab=512)


def _masters(g):
    return [p.master.detach().clone() for p in g.parameters]


def test_eligible_layers_and_tied_weight_excluded():
    g = _bert()
    pol = of.OptimizerPolicy("adamw", eta=1e-3, weight_decay=0.01)
    cf = ConsumerFusion(g, pol)
    names = {g.parameters[i].name for i in cf.ids}
    assert names and all(n.endswith(".weight") for n in names)
    assert not any("decoder" in n or "word_embeddings" in n for n in names)
    # 2 layers x (q, k, v, attention out, intermediate, output) + pooler + MLM transform
    assert len(cf.ids) == 2 * 6 + 2


def test_first_iteration_matches_plain_backward_fusion():
    from torch.nn.attention import SDPBackend, sdpa_kernel
    torch.backends.cuda.matmul.allow_tf32 = False
    inp = _inp()
    res = {}
    for mode in ("plain", "consumer"):
        g = _bert()
        pol = of.OptimizerPolicy("adamw", eta=1e-3, weight_decay=0.01, grad_reset="none")
        cf = ConsumerFusion(g, pol) if mode == "consumer" else None
        before = _masters(g)
        with sdpa_kernel(SDPBackend.MATH):
            of.run_backward_fusion(g, pol, inp, workers=2, timing=False, consumer=cf)
        torch.cuda.synchronize()
        res[mode] = (g, before, cf)
    gp, before, _ = res["plain"]
    gc, _, cf = res["consumer"]
    assert cf.launches == len(cf.ids)
    for k, (a, b) in enumerate(zip(gc.parameters, gp.parameters)):
        if k in cf.id_set:
            d_c = (a.master - before[k]).double()
            d_p = (b.master - before[k]).double()
            # AdamW's first step is ~eta * sign(g): the fp32 vs bf16-rounded
            # gradient flips only elements with |g| at bf16 resolution
            rel = ((d_c - d_p).norm() / d_p.norm()).item()
            assert rel < 5e-2, (a.name, rel)
            assert torch.equal(a.value, a.master.to(torch.bfloat16))
        else:
            assert a.master.cpu().numpy().tobytes() == b.master.cpu().numpy().tobytes(), a.name


def test_consumer_weights_follow_the_fp64_product():
    """One step, Adam (reference kind) on the consumer weights: the update the
    epilogue applied equals the oracle update of the exact fp64 gradient
    dY^T X to within the fp32 accumulation of that gradient."""
    from torch.nn.attention import SDPBackend, sdpa_kernel
    g = _bert()
    pol = of.OptimizerPolicy("adam", eta=1e-3, weight_decay=0.0, grad_reset="none")
    cf = ConsumerFusion(g, pol)
    seen = {}
    orig = cf.step_weight

    def spy(pid, gy2, x2):
        a, b = gy2.double(), x2.double()
        seen[pid] = ((a.t() @ b).float().cpu().numpy(),
                     (a.abs().t() @ b.abs()).cpu().numpy(), a.shape[0])
        orig(pid, gy2, x2)
    cf.step_weight = spy
    before = _masters(g)
    with sdpa_kernel(SDPBackend.MATH):
        of.run_backward_fusion(g, pol, _inp(), workers=2, timing=False, consumer=cf)
    torch.cuda.synchronize()
    from oracle import optim_ref
    h = optim_ref.Hyper(kind="adam", eta=1e-3)
    for pid in cf.ids:
        gref, gabs, tokens = seen[pid]
        gref, gabs = gref.reshape(-1), gabs.reshape(-1)
        th = before[pid].cpu().numpy().reshape(-1).copy()
        optim_ref.step("adam", h, th, gref.copy(), {}, 1)
        got = g.parameters[pid].master.cpu().numpy().reshape(-1)
        # The kernel's gradient is the fp32 tensor-core accumulation of exact
        # bf16 products, in an order of its own: |g_kernel - g| <= K u sum|a||b|
        # (u = 2^-24, the worst-case summation bound).  Adam's first step is
        # -eta g / (|g| + eps), whose slope in g is eta eps / (|g| + eps)^2, so
        # each element may differ from the oracle's step by that slope times
        # the gradient bound, plus a few ulp of theta for the roundings.
        gerr = tokens * 2.0 ** -24 * gabs + np.spacing(np.abs(gref))
        slope = h.eta * h.epsilon / (np.abs(gref).astype(np.float64) + h.epsilon) ** 2
        # (the roundings are those of theta_old + delta: ulps of the larger
        # operand, not of a result that cancels towards zero)
        mag = np.maximum(np.abs(before[pid].cpu().numpy().reshape(-1)), np.float32(h.eta))
        tol = 4 * np.spacing(mag).astype(np.float64) + slope * gerr
        err = np.abs(got.astype(np.float64) - th.astype(np.float64))
        bad = err > tol
        assert not bad.any(), (g.parameters[pid].name, int(bad.sum()), float(err[bad].max()),
                               float(tol[bad].min()))
        # and most elements (|g| well above eps) step by eta * sign(g) to ~2 ulp
        big = np.abs(gref) > 1e4 * h.epsilon
        assert np.allclose(got[big], th[big], rtol=0, atol=5e-9), g.parameters[pid].name


def test_captured_consumer_step_bitwise_vs_eager():
    from torch.nn.attention import SDPBackend, sdpa_kernel

    from paper_2104_00237_b200.graphs import CapturedStep
    inp = _inp()
    out = {}
    for mode in ("eager", "graph"):
        g = _bert()
        pol = of.OptimizerPolicy("adamw", eta=1e-3, weight_decay=0.01, grad_reset="none")
        cf = ConsumerFusion(g, pol)
        step = lambda i: of.run_backward_fusion(g, pol, i, workers=2, timing=False,  # noqa: E731
                                               bucket_elems=1 << 16, consumer=cf).loss
        with sdpa_kernel(SDPBackend.MATH):
            if mode == "eager":
                for _ in range(6):
                    step(inp)
            else:
                static = (inp[0].clone(), tuple(t.clone() for t in inp[1]))
                cap = CapturedStep(step, static, policy=pol, warmup=3, graph=g)
                for _ in range(3):
                    cap()
        torch.cuda.synchronize()
        out[mode] = np.concatenate([p.master.cpu().numpy().reshape(-1) for p in g.parameters])
    assert out["eager"].tobytes() == out["graph"].tobytes()
