"""numpy restatement of the reference's synthetic graphs and schedules (test oracle).

Restates, for the parity tests only:

* parameter/input initialisation -- tensor.py:78-83 (PCG64 uniform), graph.py:291-292
  (per-parameter SeedSequence([seed, pid])), bench.py:102-103 and :226-228
  (per-iteration inputs);
* the three models of build_model -- graph.py:295-342 (chain, shared-chain, mul-probe);
* forward / backward arithmetic -- graph.py:171-231 (x @ W with the fixed rank-1
  accumulation order of tensor.py:91-104, relu mask, sum loss) and graph.py:85-131
  (grad accumulation, input gradient from the parameter's current value);
* the schedules -- schedule.py:71-95 (baseline), :98-160 (forward-fusion + flush),
  :163-207 (serial backward-fusion with the in-place safety guard :54-59).

The per-parameter update is oracle.optim_ref.step.  Pinned against the reference
by tests/test_oracle_golden.py.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import optim_ref

DTYPES = {"f32": np.float32, "f64": np.float64}


def param_seed(seed: int, pid: int) -> int:
    """graph.py:291-292."""
    return int(np.random.SeedSequence([seed, pid]).generate_state(1)[0])


def uniform(shape, lo: float, hi: float, seed: int, precision: str) -> np.ndarray:
    """tensor.py:78-83, returned already shaped."""
    rng = np.random.Generator(np.random.PCG64(seed))
    vals = rng.uniform(lo, hi, size=int(np.prod(shape)))
    return vals.astype(DTYPES[precision]).reshape(shape)


def fixed_matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """tensor.py:91-104: one rank-1 update per contraction index, ascending."""
    out = np.zeros((a.shape[0], b.shape[1]), dtype=a.dtype)
    for k in range(a.shape[1]):
        out += np.multiply.outer(a[:, k], b[k, :])
    return out


@dataclass
class Model:
    kind: str                       # chain | shared-chain | mul-probe
    width: int
    precision: str
    params: list                    # flat arrays (owned values)
    layer_param: list               # layer index -> parameter index
    grads: list = field(default_factory=list)

    def __post_init__(self):
        self.grads = [np.zeros_like(p) for p in self.params]
        self.pending = [False] * len(self.params)
        self.updated = [False] * len(self.params)
        self.pending_t = None

    def shape_of(self, pid: int):
        return (self.width,) if self.kind == "mul-probe" else (self.width, self.width)

    def input_shape(self, batch: int):
        return (self.width,) if self.kind == "mul-probe" else (batch, self.width)


def build(kind: str, layers: int = 1, width: int = 1, share_groups=None, seed: int = 0,
          precision: str = "f32", init_range=None) -> Model:
    """graph.py:295-342."""
    if kind == "mul-probe":
        lo, hi = init_range if init_range else (0.5, 1.5)
        p = uniform((width,), lo, hi, param_seed(seed, 0), precision).reshape(-1)
        return Model(kind, width, precision, [p], [0])
    owner = list(range(layers))
    if kind == "shared-chain":
        groups = share_groups if share_groups is not None else [[0, min(2, layers - 1)]]
        for group in groups:
            head = min(group)
            for idx in group:
                owner[idx] = head
    lo, hi = init_range if init_range else (-1.0 / width ** 0.5, 1.0 / width ** 0.5)
    by_owner: dict = {}
    params, layer_param = [], []
    for i in range(layers):
        if owner[i] not in by_owner:
            pid = len(params)
            by_owner[owner[i]] = pid
            params.append(uniform((width, width), lo, hi, param_seed(seed, pid), precision).reshape(-1))
        layer_param.append(by_owner[owner[i]])
    return Model(kind, width, precision, params, layer_param)


def iteration_inputs(model: Model, batch: int, seed: int, iters: int) -> list:
    """bench.py:226-228 with make_input (bench.py:102-103)."""
    base = int(np.random.SeedSequence([seed, 9173]).generate_state(1)[0])
    return [uniform(model.input_shape(batch), 0.1, 1.0, base + i, model.precision)
            for i in range(iters)]


class Policy:
    """OptimizerPolicy state: hyper-parameters, step counter t, history slots."""

    def __init__(self, kind: str, clip_norm=None, **hp):
        self.hp = optim_ref.Hyper(kind=kind, **hp)
        self.clip_norm = clip_norm
        self.t = 0
        self.slots: dict = {}

    @property
    def requires_global_info(self) -> bool:
        return self.clip_norm is not None

    def step(self, model: Model, pid: int, step_t=None) -> None:
        t = self.t if step_t is None else step_t
        optim_ref.step(self.hp.kind, self.hp, model.params[pid], model.grads[pid],
                       self.slots.setdefault(pid, {}), t)
        model.pending[pid] = False


class GlobalInfoRequired(RuntimeError):
    pass


def _forward(model: Model, x: np.ndarray, pre_node=None):
    """graph.py:171-231; returns (loss, per-node saved tensors)."""
    saved = []
    loss = 0.0
    n = len(model.layer_param)
    for i, pid in enumerate(model.layer_param):
        if pre_node is not None:
            pre_node(i)
        if model.kind == "mul-probe":
            theta = model.params[pid]
            saved.append((x.copy(), None))
            out = theta * x
            loss = float(out.sum())
            continue
        w = model.params[pid].reshape(model.width, model.width)
        pre = fixed_matmul(x, w)
        mask = (pre > 0).astype(pre.dtype)
        saved.append((x, mask))
        x = pre * mask
        if i == n - 1:
            loss = float(x.sum())
    return loss, saved


def _backward_node(model: Model, i: int, saved, gout):
    """graph.py:85-131 for node i: accumulate, then the input gradient from
    the parameter's CURRENT value (before any fused update of it)."""
    pid = model.layer_param[i]
    x, mask = saved[i]
    if model.kind == "mul-probe":
        contrib = x if gout is None else gout * x
        model.grads[pid] += contrib
        return model.params[pid].copy()
    gm = mask if gout is None else gout * mask
    contrib = fixed_matmul(x.T, gm).reshape(-1)
    model.grads[pid] += contrib
    w = model.params[pid].reshape(model.width, model.width)
    return fixed_matmul(gm, w.T)


def run_baseline(model: Model, policy: Policy, x: np.ndarray):
    """schedule.py:71-95; returns (loss, input_grad)."""
    policy.t += 1
    loss, saved = _forward(model, x)
    gout = None
    for i in reversed(range(len(model.layer_param))):
        gout = _backward_node(model, i, saved, gout)
    if policy.clip_norm is not None:
        optim_ref.clip_by_global_norm(model.grads, policy.clip_norm)
    for pid in reversed(range(len(model.params))):
        policy.step(model, pid)
    return loss, gout


def run_forward_fusion(model: Model, policy: Policy, x: np.ndarray):
    """schedule.py:98-138: pending updates applied just before each node."""
    policy.t += 1

    def apply_pending(i):
        pid = model.layer_param[i]
        if model.pending[pid] and not model.updated[pid]:
            policy.step(model, pid, step_t=model.pending_t)
            model.updated[pid] = True

    loss, saved = _forward(model, x, apply_pending)
    gout = None
    for i in reversed(range(len(model.layer_param))):
        gout = _backward_node(model, i, saved, gout)
    if policy.clip_norm is not None:
        optim_ref.clip_by_global_norm(model.grads, policy.clip_norm)
    model.pending = [True] * len(model.params)
    model.updated = [False] * len(model.params)
    model.pending_t = policy.t
    return loss, gout


def flush_pending_updates(model: Model, policy: Policy) -> int:
    """schedule.py:141-160 (layer order, frozen step index, idempotent)."""
    flushed = 0
    for pid in model.layer_param:
        if not model.pending[pid]:
            continue
        policy.step(model, pid, step_t=model.pending_t)
        flushed += 1
    return flushed


def run_backward_fusion(model: Model, policy: Policy, x: np.ndarray):
    """schedule.py:163-207 (serial): step each parameter right after the
    backward node that completes its gradient and releases its last reader."""
    if policy.requires_global_info:
        raise GlobalInfoRequired("backward-fusion cannot host a global-norm clip")
    policy.t += 1
    loss, saved = _forward(model, x)
    n = len(model.layer_param)
    remaining = [model.layer_param.count(pid) for pid in range(len(model.params))]
    gout = None
    for i in reversed(range(n)):
        gout = _backward_node(model, i, saved, gout)
        pid = model.layer_param[i]
        remaining[pid] -= 1       # count -= 1 and reader discarded (graph.py:110,129)
        if remaining[pid] == 0:   # check_inplace_safety (schedule.py:54-59)
            policy.step(model, pid)
    return loss, gout
