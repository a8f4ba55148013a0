"""Update policies on the GPU: the reference's OptimizerPolicy, executed by the
sm_100a multi-tensor kernels.

Mirrors /root/reference/pkg/src/optfuse/optim.py:
  * ``OptimizerPolicy`` -- same fields, defaults, validation (optim.py:34-72);
  * ``OptimizerPolicy.step(param, step_t=None, trace=None)`` -- same contract
    (optim.py:74-115): newton and count != 0 raise before anything is touched,
    history is allocated lazily as zeros, the gradient is reset (zeroed in the
    kernel, or released when ``grad_reset="none"``), the parameter is updated
    in place;
  * ``clip_by_global_norm(graph, max_norm)`` (optim.py:151-172) -- the squared
    norm is reduced on the device; the factor is *not* applied in a second
    pass over the gradients but carried as a device scalar into the next step
    of every parameter (bitwise the same as scaling the gradient first).

B200 additions: ``step_params`` updates a whole list of parameters in one
kernel launch (the per-layer / per-bucket unit of the fused schedules), the
``adamw`` kind (torch.optim.AdamW semantics, not in the reference), and the
``stream`` argument that the backward-fusion engine uses to issue updates on
its side stream.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from . import kernels
from . import trace as tr
from .errors import ConfigError, NumericError, SchedulingContractError, StateError

KINDS = ("sgd", "sgd-momentum", "newton", "adagrad", "rmsprop", "adadelta", "adam", "adamw")

_HISTORY_SLOTS = {
    "sgd": (),
    "sgd-momentum": ("momentum",),
    "adagrad": ("sum_sq",),
    "rmsprop": ("square_avg",),
    "adadelta": ("square_avg", "acc_delta"),
    "adam": ("exp_avg", "exp_avg_sq"),
    "adamw": ("exp_avg", "exp_avg_sq"),
}

GRAD_RESETS = ("zero", "none")


@dataclass
class OptimizerPolicy:
    """One update rule and its constants (optim.py:34-72).

    ``t`` counts begun iterations and feeds the Adam bias corrections; the
    schedulers advance it exactly once per iteration.  ``grad_reset`` chooses
    how a step resets the gradient: ``"zero"`` (reference semantics,
    optim.py:111 -- the kernel writes zeros, gradients stay allocated) or
    ``"none"`` (the gradient tensor is released after the step, so the next
    backward's AccumulateGrad steals its input instead of adding into it).
    """

    kind: str = "sgd"
    eta: float = 0.01
    alpha: float = 0.9
    weight_decay: float = 0.0
    epsilon: float = 1e-8
    beta1: float = 0.9
    beta2: float = 0.999
    rho: float = 0.9
    clip_norm: float | None = None
    t: int = 0
    grad_reset: str = "zero"
    _lists: dict = field(default_factory=dict, repr=False, compare=False)
    _hp_cache: tuple = field(default=(None, None), repr=False, compare=False)
    _dstep_buf: object = field(default=None, repr=False, compare=False)
    _dstep: object = field(default=None, repr=False, compare=False)   # active while capturing

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ConfigError(f"unknown optimizer {self.kind!r}, expected one of {KINDS}")
        if self.eta <= 0:
            raise ConfigError(f"step size must be > 0, got {self.eta}")
        if not 0 <= self.alpha < 1:
            raise ConfigError(f"momentum decay must be in [0, 1), got {self.alpha}")
        if self.weight_decay < 0:
            raise ConfigError(f"weight decay must be >= 0, got {self.weight_decay}")
        if self.grad_reset not in GRAD_RESETS:
            raise ConfigError(f"grad_reset must be one of {GRAD_RESETS}, got {self.grad_reset!r}")

    @property
    def requires_global_info(self) -> bool:
        """True iff no parameter may be updated before all gradients exist."""
        return self.clip_norm is not None or self.kind == "newton"

    def history_slots(self) -> tuple:
        return _HISTORY_SLOTS.get(self.kind, ())

    def begin_iteration(self) -> None:
        self.t += 1

    # -- single-parameter API (the reference's plugin boundary) -------------

    def step(self, param, step_t: int | None = None, trace: tr.ScheduleTrace | None = None,
             stream=None) -> None:
        """Apply this policy's update to one parameter, in place."""
        self.step_params((param,), step_t=step_t, trace=trace, stream=stream)

    # -- multi-tensor API (one kernel launch) --------------------------------

    def check_steppable(self, params) -> None:
        """The contract checks of optim.py:82-87; raises before any mutation."""
        if self.kind == "newton":
            raise ConfigError("newton needs the full Hessian and has no per-parameter step")
        for p in params:
            if p.count != 0:
                raise SchedulingContractError(
                    f"parameter {p.id} still has {p.count} pending gradient contributions")
            if not p._layout_ok:
                _check_layout(p, p.value.grad)

    def step_params(self, params, step_t: int | None = None,
                    trace: tr.ScheduleTrace | None = None, stream=None,
                    hold: list | None = None) -> None:
        """Update every parameter of ``params`` with one multi-tensor launch.

        Arithmetic per parameter is exactly ``step`` (parameters are
        independent, optim.py:3-5).  ``stream``: CUDA stream to launch on
        (default: current).  ``hold``: when given and ``grad_reset == "none"``,
        released gradient tensors are appended to it so the caller can keep
        them alive until ``stream`` has been joined.
        """
        params = tuple(params)
        if not params:
            return
        self.check_steppable(params)
        t = self.t if step_t is None else step_t
        if self.kind in ("adam", "adamw") and t < 1:
            raise StateError(f"{self.kind} step needs step index t >= 1 (call begin_iteration)")
        slots = _HISTORY_SLOTS[self.kind]
        # group by gradient scale (global-norm clip factor) -- normally one group
        scale = params[0]._grad_scale
        if any(p._grad_scale is not scale for p in params):
            by_scale: dict = {}
            for p in params:
                by_scale.setdefault(id(p._grad_scale), []).append(p)
            for group in by_scale.values():
                self.step_params(group, step_t=step_t, trace=trace, stream=stream, hold=hold)
            return

        key = tuple(id(p) for p in params)
        tl = self._lists.get(key)
        if tl is None:
            tl = kernels.TensorList(len(params))
            self._lists[key] = tl
        zero = self.grad_reset == "zero"
        self.prepare(params)
        s_a = slots[0] if slots else None
        s_b = slots[1] if len(slots) > 1 else None
        mixed = params[0].master is not None
        for i, p in enumerate(params):
            v = p.value
            h = p.history
            if mixed:   # fp32 master updated, bf16 parameter written as the shadow
                tl.set(i, p.master, v.grad, h[s_a] if s_a else None, h[s_b] if s_b else None, v)
            else:
                tl.set(i, v, v.grad, h[s_a] if s_a else None, h[s_b] if s_b else None, None)
        p0 = params[0]
        tl.set_dtypes(p0.master.dtype if mixed else p0.value.dtype, p0.value.grad.dtype)
        flags = ((nat.OF_FLAG_ZERO_GRAD if zero else 0) | (nat.OF_FLAG_SHADOW_BF16 if mixed else 0)
                 | self.device_step_flag)
        kernels.policy_step(tl, self._hparams(t), scale, flags, stream)
        if trace is not None:
            for p in params:
                trace.record_mem(tr.PARAM, p.id, tr.READ)
                trace.record_mem(tr.GRAD, p.id, tr.READ)
                if slots:
                    trace.record_mem(tr.HISTORY, p.id, tr.READ)
                    trace.record_mem(tr.HISTORY, p.id, tr.WRITE)
                trace.record_mem(tr.GRAD, p.id, tr.WRITE)
                trace.record_mem(tr.PARAM, p.id, tr.WRITE)
        for p in params:
            p.pending = False
            p._grad_scale = None
            if not zero:
                if hold is not None and p.value.grad is not None:
                    hold.append(p.value.grad)
                p.value.grad = None

    def prepare(self, params, hold: list | None = None) -> None:
        """Allocate, on the current stream, what a step of ``params`` needs:
        zero history slots on first use (optim.py:90-94) and a zero gradient
        for a parameter that received no contribution this iteration (the
        reference steps every parameter, with g = 0, schedule.py:87)."""
        for p in params:
            v = p.value
            if v.grad is None:
                v.grad = torch.zeros_like(v)
        self.prepare_history(params)

    def prepare_history(self, params) -> None:
        """Zero history slots on first use (optim.py:90-94)."""
        slots = _HISTORY_SLOTS[self.kind]
        for p in params:
            h = p.history
            if len(h) < len(slots):
                ref = p.master if p.master is not None else p.value
                for name in slots:
                    if name not in h:
                        h[name] = torch.zeros_like(ref, memory_format=torch.preserve_format)

    # -- CUDA-graph replay of step-dependent kinds ----------------------------

    @property
    def device_step_flag(self) -> int:
        """OF_FLAG_DEVICE_STEP while a CUDA graph is being captured."""
        return nat.OF_FLAG_DEVICE_STEP if self._dstep is not None else 0

    def device_step(self, device) -> "DeviceStep":
        """The device-resident step index of this policy (created on first use)."""
        ds = self._dstep_buf
        if ds is None or ds.betas != (self.beta1, self.beta2):
            ds = DeviceStep(self, device)
            self._dstep_buf = ds
        return ds

    def _hparams(self, t: int) -> nat.OfHparams:
        key = (t, self.kind, self.eta, self.alpha, self.weight_decay, self.epsilon,
               self.beta1, self.beta2, self.rho, id(self._dstep))
        cached_key, hp = self._hp_cache
        if cached_key != key:
            hp = kernels.hparams(self.kind, self.eta, self.alpha, self.weight_decay, self.epsilon,
                                 self.beta1, self.beta2, self.rho, t, device_step=self._dstep)
            self._hp_cache = (key, hp)
        return hp


def bytes_per_element(kind: str, param_itemsize: int = 4, grad_itemsize: int | None = None,
                      shadow: bool = False) -> int:
    """Algorithmic HBM bytes of one element update: read
    theta, grad and every history slot; write theta and every slot (+ a bf16
    shadow).  Gradient zeroing is not counted."""
    slots = len(_HISTORY_SLOTS[kind])
    g = param_itemsize if grad_itemsize is None else grad_itemsize
    return param_itemsize * (2 + 2 * slots) + g + (2 if shadow else 0)


class DeviceStep:
    """Device-resident step index for CUDA-graph replay (OF_FLAG_DEVICE_STEP).

    A captured launch reads its step index as ``t_base + offset`` when it runs,
    where ``t_base`` is the host step index at capture and ``offset`` (one
    device int64) is advanced by the graph's first node on every replay; the
    Adam bias corrections come from ``table[t] = (1 - beta1**t, 1 - beta2**t)``,
    filled on the host with the very Python expressions of optim.py:145-146, so
    a replayed step is bit-identical to the eager one.  The table is allocated
    once (its address is baked into the graph) and filled ahead of use."""

    ROWS = 1 << 20      # 16 MiB: a million replayed iterations
    CHUNK = 4096

    def __init__(self, policy, device):
        self.betas = (policy.beta1, policy.beta2)
        self.offset = torch.zeros(1, dtype=torch.int64, device=device)
        self.table = torch.zeros((self.ROWS, 2), dtype=torch.float64, device=device)
        self.filled = 0
        self.ensure(policy.t + 1)

    def ensure(self, t: int) -> None:
        """Rows up to index ``t`` are valid (stream-ordered host copy)."""
        if t < self.filled:
            return
        if t >= self.ROWS:
            raise StateError(f"step index {t} beyond the device step table ({self.ROWS} rows)")
        hi = min(self.ROWS, max(t + 1, self.filled + self.CHUNK))
        b1, b2 = self.betas
        rows = [(1 - b1 ** k, 1 - b2 ** k) for k in range(self.filled, hi)]
        self.table[self.filled:hi].copy_(torch.tensor(rows, dtype=torch.float64))
        self.filled = hi


def algorithmic_bytes(kind: str, params) -> int:
    total = 0
    for p in params:
        if hasattr(p, "value"):
            total += p.value.numel() * bytes_per_element_of(kind, p)
        else:
            total += p.numel() * bytes_per_element(kind, p.element_size())
    return total


def _check_layout(p, g) -> None:
    """Parameter, gradient, history (and master) must share one dense layout:
    the kernels walk the buffers in storage order."""
    v = p.value
    if not v.is_cuda:
        raise ConfigError(f"parameter {p.id} is on {v.device}; the update kernels run on CUDA only")
    m = p.master
    if m is not None:
        if v.dtype != torch.bfloat16 or m.dtype != torch.float32:
            raise ConfigError(f"parameter {p.id}: master weights need a bf16 parameter and an "
                              f"fp32 master, got {v.dtype} / {m.dtype}")
        if m.shape != v.shape or not _same_order(m, v) or m.device != v.device:
            raise ConfigError(f"parameter {p.id}: master layout differs from the parameter's")
    elif v.dtype not in (torch.float32, torch.float64):
        raise ConfigError(f"parameter {p.id} has dtype {v.dtype}; expected float32 or float64 "
                          "(or bf16 with master weights)")
    if not kernels.is_dense(v):
        raise ConfigError(f"parameter {p.id} is not dense; the update kernels need dense storage")
    if g is None:
        return  # checked again once a gradient exists
    if g.shape != v.shape or not _same_order(g, v) or g.device != v.device:
        raise ConfigError(f"parameter {p.id}: gradient layout {tuple(g.stride())} on {g.device} "
                          f"differs from parameter layout {tuple(v.stride())} on {v.device}")
    if g.dtype != v.dtype:
        raise ConfigError(f"parameter {p.id}: gradient dtype {g.dtype} with parameter {v.dtype}")
    p._layout_ok = True


def _same_order(a, b) -> bool:
    """Same element order in memory: strides agree on every dimension of size
    > 1 (a size-1 dimension's stride is arbitrary -- e.g. a 1x1 convolution
    weight is both contiguous and channels-last) and both are dense."""
    return (all(sa == sb for n, sa, sb in zip(a.shape, a.stride(), b.stride()) if n > 1)
            and kernels.is_dense(a) and kernels.is_dense(b))


def bytes_per_element_of(kind: str, p) -> int:
    """Algorithmic bytes per element for this parameter's storage (mixed: bf16
    grad in, fp32 master + history, bf16 shadow out)."""
    if p.master is not None:
        return bytes_per_element(kind, 4, 2, shadow=True)
    return bytes_per_element(kind, p.value.element_size())


def _clip_buffers(graph, dev):
    """Per-graph clip scalars (sq-norm, f64 factor, f32 coef, workspace),
    allocated once and rewritten in place by every clip: a captured CUDA graph
    bakes their addresses into its launches (forward fusion's deferred updates
    read the factor of the previous replay), so they must never move."""
    bufs = getattr(graph, "_clip_bufs", None)
    if bufs is None or bufs[0].device != dev:
        bufs = (torch.zeros((), dtype=torch.float64, device=dev),
                torch.ones((), dtype=torch.float64, device=dev),
                torch.ones((), dtype=torch.float32, device=dev),
                torch.empty(kernels.sqnorm_workspace_len(), dtype=torch.float64, device=dev))
        graph._clip_bufs = bufs
    return bufs


def clip_factor(graph, max_norm: float, trace: tr.ScheduleTrace | None = None, stream=None):
    """Device half of the global-norm clip: returns (factor, coef), a 0-dim
    float64 factor (optim.py:165-168) and its float32 rounding, both
    persistent per-graph buffers rewritten by the next clip."""
    params = graph.parameters
    dev = params[0].value.device
    sq, factor, coef, ws = _clip_buffers(graph, dev)
    by_dtype: dict = {}
    for p in params:
        if trace is not None:
            trace.record_mem(tr.GRAD, p.id, tr.READ)
        g = p.value.grad
        if g is not None:
            by_dtype.setdefault(g.dtype, []).append(g)
    if not by_dtype:
        sq.zero_()
    first = True
    for dt, gl in by_dtype.items():
        tl = kernels.TensorList(len(gl))
        for i, g in enumerate(gl):
            tl.set(i, None, g)
        tl.set_dtypes(dt if dt != torch.bfloat16 else torch.float32, dt)
        kernels.sqnorm(tl, ws, sq, accumulate=not first, stream=stream)
        first = False
    kernels.clip_coef(sq, max_norm, coef, factor, stream)
    if trace is not None:
        for p in params:
            trace.record_mem(tr.GRAD, p.id, tr.WRITE)
    return factor, coef


def grad_scale_for(p, factor, coef):
    """The scale tensor a parameter's update multiplies its gradient by
    (optim.py:170 ``p.grad.data *= factor``): numpy scales an f64 gradient by
    the double factor, an f32 one by the factor rounded to f32."""
    ref = p.master if p.master is not None else p.value
    return factor if ref.dtype == torch.float64 else coef


def clip_by_global_norm(graph, max_norm: float, trace: tr.ScheduleTrace | None = None,
                        stream=None) -> torch.Tensor:
    """Global-norm clip (optim.py:151-172) as a device reduction.

    Returns the clip factor as a 0-dim float64 CUDA tensor (1.0 when nothing
    is clipped; a copy, so it keeps this clip's value); ``float(result)``
    gives the reference's return value (and synchronises).  The factor is
    attached to every parameter and folded into its next update -- the
    reference's in-place ``grad *= factor`` without a second pass over the
    gradients (in f64 for f64 parameters, f32 otherwise).
    """
    factor, coef = clip_factor(graph, max_norm, trace, stream)
    for p in graph.parameters:
        p._grad_scale = grad_scale_for(p, factor, coef)
    return factor.clone()


def newton_step(theta, grad_fn, hessian_fn, eta: float = 1.0):
    """Full-Hessian toy validator (optim.py:175-194).  Not on the fused path:
    it couples every coordinate, so no schedule can host it (schedule.py:62-64);
    kept for API completeness and evaluated on the host in float64."""
    th = np.asarray(theta.detach().cpu().numpy() if isinstance(theta, torch.Tensor) else theta)
    d = th.size
    if d > 16:
        raise ConfigError(f"newton step is limited to dimension <= 16, got {d}")
    g = np.asarray(grad_fn(th.copy()), dtype=np.float64).reshape(d)
    h = np.asarray(hessian_fn(th.copy()), dtype=np.float64).reshape(d, d)
    try:
        direction = np.linalg.solve(h, g)
    except np.linalg.LinAlgError as e:
        raise NumericError(f"Hessian is singular: {e}") from e
    if not np.all(np.isfinite(direction)):
        raise NumericError("Hessian solve produced non-finite values")
    new = th.astype(np.float64).reshape(d) - eta * direction
    out = new.astype(th.dtype).reshape(th.shape)
    return torch.from_numpy(out) if isinstance(theta, torch.Tensor) else out
