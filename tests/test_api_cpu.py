"""Host-side contract of the GPU API that needs no device: validation, error
types and raise-before-mutate (optim.py:53-61, :82-87; schedule.py:174-177),
graph discovery, and the product/oracle separation."""

import re
from pathlib import Path

import pytest
import torch

import paper_2104_00237_b200 as of
from paper_2104_00237_b200 import errors

PKG = Path(of.__file__).resolve().parent


def test_error_types_match_reference_bases():
    assert issubclass(of.ConfigError, ValueError)
    assert issubclass(of.ShapeError, ValueError)
    assert issubclass(of.StateError, RuntimeError)
    assert issubclass(of.SchedulingContractError, RuntimeError)
    assert issubclass(of.GlobalInfoRequired, RuntimeError)
    assert issubclass(of.NumericError, ArithmeticError)


@pytest.mark.parametrize("kw", [dict(kind="lbfgs"), dict(eta=0.0), dict(eta=-1.0),
                                dict(alpha=1.0), dict(alpha=-0.1), dict(weight_decay=-1e-4),
                                dict(grad_reset="keep")])
def test_policy_validation(kw):
    with pytest.raises(of.ConfigError):
        of.OptimizerPolicy(**kw)


def test_policy_defaults_and_global_info():
    p = of.OptimizerPolicy()
    assert (p.kind, p.eta, p.alpha, p.weight_decay, p.epsilon, p.beta1, p.beta2, p.rho) == (
        "sgd", 0.01, 0.9, 0.0, 1e-8, 0.9, 0.999, 0.9)
    assert not p.requires_global_info
    assert of.OptimizerPolicy(clip_norm=1.0).requires_global_info
    assert of.OptimizerPolicy(kind="newton").requires_global_info
    assert of.OptimizerPolicy(kind="adam").history_slots() == ("exp_avg", "exp_avg_sq")
    assert of.OptimizerPolicy(kind="adamw").history_slots() == ("exp_avg", "exp_avg_sq")


def test_backward_fusion_rejects_global_info_without_mutation():
    g = of.build_model("chain", layers=3, width=4, device="cpu")
    before = [p.value.detach().clone() for p in g.parameters]
    pol = of.OptimizerPolicy("adam", clip_norm=1.0)
    with pytest.raises(of.GlobalInfoRequired):
        of.run_backward_fusion(g, pol, torch.ones(2, 4))
    assert pol.t == 0
    assert all(torch.equal(a, p.value) for a, p in zip(before, g.parameters))
    with pytest.raises(of.GlobalInfoRequired):
        of.run_backward_fusion(g, of.OptimizerPolicy("newton"), torch.ones(2, 4))


def test_newton_cannot_drive_a_schedule():
    g = of.build_model("chain", layers=2, width=2, device="cpu")
    with pytest.raises(of.ConfigError):
        of.run_baseline(g, of.OptimizerPolicy("newton"), torch.ones(1, 2))
    with pytest.raises(of.ConfigError):
        of.OptimizerPolicy("newton").step(g.parameters[0])


def test_step_contract_errors_before_mutation():
    g = of.build_model("chain", layers=2, width=2, device="cpu")
    p = g.parameters[0]
    p.count = 1
    with pytest.raises(of.SchedulingContractError):
        of.OptimizerPolicy("sgd").step(p)
    assert p.history == {} and p.value.grad is None
    p.count = 0
    with pytest.raises(of.ConfigError, match="CUDA"):
        of.OptimizerPolicy("sgd-momentum").step(p)
    assert p.history == {} and p.value.grad is None


def test_workers_validation():
    g = of.build_model("chain", layers=2, width=2, device="cpu")
    with pytest.raises(of.ConfigError):
        of.run_backward_fusion(g, of.OptimizerPolicy("sgd"), torch.ones(1, 2), workers=0)


def test_build_model_errors():
    with pytest.raises(of.ConfigError):
        of.build_model("resnet", device="cpu")
    with pytest.raises(of.ConfigError):
        of.build_model("chain", layers=0, device="cpu")
    with pytest.raises(of.ConfigError):
        of.build_model("shared-chain", layers=4, width=2, share_groups=[[0]], device="cpu")
    with pytest.raises(of.ConfigError):
        of.build_model("shared-chain", layers=4, width=2, share_groups=[[0, 9]], device="cpu")
    with pytest.raises(of.ConfigError):
        of.build_model("shared-chain", layers=4, width=2, share_groups=[[0, 1], [1, 2]],
                       device="cpu")
    with pytest.raises(of.ConfigError):
        of.build_model("chain", layers=2, width=2, share_groups=[[0, 1]], device="cpu")
    with pytest.raises(of.ShapeError):
        of.build_model("chain", layers=2, width=2, precision="f16", device="cpu")


def test_graph_discovery_shared_and_counts():
    g = of.build_model("shared-chain", layers=4, width=3, device="cpu")
    assert len(g.parameters) == 3 and len(g.layers) == 4
    assert [p.id for L in g.layers for p in L.params] == [0, 1, 0, 2]
    assert [L.index for L in g.parameters[0].layers] == [0, 2]
    g.forward(torch.ones(2, 3))
    assert [p.count for p in g.parameters] == [2, 1, 1]
    assert not of.check_inplace_safety(g.parameters[0], g)
    g.backward()
    assert [p.count for p in g.parameters] == [0, 0, 0]
    assert of.check_inplace_safety(g.parameters[0], g)
    with pytest.raises(of.StateError):
        g.backward()


def test_synthetic_init_matches_reference_seeding(traj_golden):
    import numpy as np
    for model, kw in (("chain", dict(layers=3, width=4)), ("shared-chain", dict(layers=4, width=4)),
                      ("mul-probe", dict(width=3))):
        for prec in ("f32", "f64"):
            g = of.build_model(model, **kw, precision=prec, device="cpu")
            flat = np.concatenate([p.value.detach().numpy().reshape(-1) for p in g.parameters])
            assert flat.tobytes() == traj_golden[f"cell|adam|{model}|{prec}|init"].tobytes()
            xs = of.iteration_inputs(g, 2, 0, 10, device="cpu")
            assert np.stack([x.numpy() for x in xs]).tobytes() == \
                traj_golden[f"cell|adam|{model}|{prec}|inputs"].tobytes()


def test_exact_chain_cpu_matches_oracle_gradients():
    """The fixed-order autograd port reproduces the reference gradients bitwise
    (checked on CPU torch; the GPU run uses the same op sequence)."""
    import numpy as np
    from oracle import chain_ref
    g = of.build_model("chain", layers=3, width=4, device="cpu")
    m = chain_ref.build("chain", layers=3, width=4)
    x = of.iteration_inputs(g, 2, 0, 1, device="cpu")[0]
    g.forward(x)
    g.backward()
    chain_ref.run_baseline(m, chain_ref.Policy("sgd", eta=1e-30), x.numpy())
    # the oracle stepped with a negligible eta and reset grads; recompute grads
    m2 = chain_ref.build("chain", layers=3, width=4)
    loss, saved = chain_ref._forward(m2, x.numpy())
    gout = None
    for i in reversed(range(3)):
        gout = chain_ref._backward_node(m2, i, saved, gout)
    for p, ref in zip(g.parameters, m2.grads):
        assert p.value.grad.numpy().reshape(-1).tobytes() == ref.tobytes()
    assert g.input_grad.numpy().tobytes() == gout.tobytes()


def test_classifier_discovery():
    g = of.build_classifier("mobilenet_v2_cifar", device="cpu")
    assert len(g.parameters) == 158
    assert sum(p.value.numel() for p in g.parameters) == 2_236_682
    g = of.build_classifier("resnet18_cifar", device="cpu")
    assert len(g.parameters) == 62
    assert sum(p.value.numel() for p in g.parameters) == 11_173_962


def test_bert_base_discovery_and_loss():
    """C5's network: BERT-base pre-training, 206 tensors / 110.1 M parameters
    (SURVEY.md §8(a)2), the MLM decoder tied to the word embeddings."""
    g = of.build_classifier("bert_base", device="cpu")
    assert len(g.parameters) == 206
    assert sum(p.value.numel() for p in g.parameters) == 110_106_428
    emb = g.module.net.bert.embeddings.word_embeddings.weight
    p = g.parameter_of(emb)
    assert len(p.layers) == 2   # embedding lookup + MLM decoder
    small = of.build_classifier("bert_base", device="cpu",
                                config=dict(num_hidden_layers=1, hidden_size=32,
                                            num_attention_heads=2, intermediate_size=64,
                                            vocab_size=100))
    ids, (labels, nsp) = of.models.synthetic_batch("bert_base", 3, device="cpu", seq=16, vocab=100)
    assert ids.shape == labels.shape == (3, 16) and nsp.shape == (3,)
    assert ((labels == -100) | (labels == ids)).all()
    loss = small.forward((ids, (labels, nsp)))
    assert loss.dim() == 0 and torch.isfinite(loss)


def test_tied_parameters_are_one_parameter():
    emb = torch.nn.Embedding(10, 4)
    head = torch.nn.Linear(4, 10, bias=False)
    head.weight = emb.weight
    g = of.Graph(torch.nn.Sequential(emb, head), None)
    assert len(g.parameters) == 1 and len(g.layers) == 2
    assert [L.index for L in g.parameters[0].layers] == [0, 1]


def test_product_never_imports_oracle():
    pat = re.compile(r"^\s*(from|import)\s+oracle\b", re.M)
    for f in PKG.rglob("*.py"):
        assert not pat.search(f.read_text()), f"{f} imports the test oracle"


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2104_00237_b200 import _native
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setenv("OPTFUSE_B200_LIB", str(tmp_path / "nope.so"))
    with pytest.raises(errors.NativeLibraryError, match="no CPU fallback"):
        _native.lib()


def test_checkpoint_rejects_foreign_or_mismatched_state():
    from paper_2104_00237_b200 import checkpoint
    g = of.build_model("chain", layers=2, width=3, device="cpu")
    pol = of.OptimizerPolicy("adam")
    with pytest.raises(errors.ConfigError):
        checkpoint.load_state_dict(g, pol, {"format": "something-else"})
    sd = {"format": "optfuse-b200/1", "policy": {"kind": "sgd"}, "model": {}, "history": {},
          "master": {}}
    with pytest.raises(errors.ConfigError, match="checkpoint is for"):
        checkpoint.load_state_dict(g, pol, sd)


def test_same_layout_ignores_strides_of_size_one_dims():
    from paper_2104_00237_b200.kernels import same_layout
    w = torch.empty(16, 32, 1, 1)
    g = torch.empty_strided((16, 32, 1, 1), (32, 1, 32, 32))   # channels-last strides
    assert w.stride() != g.stride() and same_layout(w, g)
    a = torch.empty(4, 3, 3, 3).contiguous(memory_format=torch.channels_last)
    b = torch.empty(4, 3, 3, 3)
    assert not same_layout(a, b)
    assert not same_layout(torch.empty(4), torch.empty(4, dtype=torch.float64))
    assert not same_layout(torch.empty(8)[::2], torch.empty(4))


def test_device_step_table_holds_the_hosts_bias_corrections():
    """OF_FLAG_DEVICE_STEP reads (1 - beta1**t, 1 - beta2**t) from this table:
    the very Python doubles optim.py:145-146 computes, filled ahead of use."""
    from paper_2104_00237_b200.optim import DeviceStep
    pol = of.OptimizerPolicy("adam", beta1=0.9, beta2=0.999)
    pol.t = 5
    ds = DeviceStep(pol, torch.device("cpu"))
    assert ds.filled >= 6 and ds.table.dtype == torch.float64
    for t in (1, 2, 5, ds.filled - 1):
        assert float(ds.table[t, 0]) == 1 - 0.9 ** t and float(ds.table[t, 1]) == 1 - 0.999 ** t
    ds.ensure(ds.filled + 10)
    t = ds.filled - 1
    assert float(ds.table[t, 1]) == 1 - 0.999 ** t
    with pytest.raises(errors.StateError):
        ds.ensure(DeviceStep.ROWS)
