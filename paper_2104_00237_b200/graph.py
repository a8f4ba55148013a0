"""Graph: a PyTorch module as the reference's schedulers see a training graph.

The reference builds its own eager tape (/root/reference/pkg/src/optfuse/graph.py).
On B200, PyTorch autograd is the tape; what the schedulers need from it is
exactly the reference's per-parameter scheduling state and its two hook sites:

* ``Parameter`` (graph.py:27-45): the trainable tensor plus ``history``
  (optimizer slots, device tensors), ``count`` (forward usages still owing a
  gradient contribution), ``updated`` (forward-fusion latch) and ``pending``
  (deferred update).
* the forward hook site (graph.py:171-218): a forward pre-hook on every layer
  -- a module owning parameters directly -- that increments ``count`` and
  runs the schedule's ``pre_node_hook`` *before* the layer executes;
* the gradient-ready site (graph.py:85-131): a C++ PostAccumulateGradHook on
  every parameter, installed by the native engine (engine.py).  AccumulateGrad
  fires it once, after every use of the parameter has contributed
  (shared/tied parameters included) and after the consuming node computed its
  input gradient from the old value, which is Appendix B.2's in-place safety
  condition (schedule.py:54-59) on the host.

A layer is a module with direct parameters; a parameter shared by several
layers (tied embeddings, ``shared-chain``) is one ``Parameter`` bound to each.
"""

from __future__ import annotations

import torch

from . import trace as tr
from .errors import ConfigError, StateError


class Parameter:
    """A trainable tensor plus its scheduling state (graph.py:27-45).

    While a native fusion engine owns the forward-fusion flags of the graph,
    ``pending`` and ``updated`` read and write them there.
    """

    __slots__ = ("id", "name", "value", "history", "count", "_updated", "_pending",
                 "_grad_scale", "_layout_ok", "layers", "_flags", "master")

    def __init__(self, pid: int, value: torch.Tensor, name: str = ""):
        self.id = pid
        self.name = name
        self.value = value
        self.history: dict = {}
        self.count = 0
        self._updated = False
        self._pending = False
        self._grad_scale = None
        self._layout_ok = False
        self.layers: list = []
        self._flags = None
        self.master = None   # fp32 master copy when the model runs in bf16

    @property
    def pending(self) -> bool:
        f = self._flags
        return self._pending if f is None else f.is_pending(self.id)

    @pending.setter
    def pending(self, v: bool) -> None:
        f = self._flags
        if f is None:
            self._pending = bool(v)
        else:
            f.set_pending(self.id, bool(v))

    @property
    def updated(self) -> bool:
        f = self._flags
        return self._updated if f is None else f.is_updated(self.id)

    @updated.setter
    def updated(self, v: bool) -> None:
        f = self._flags
        if f is None:
            self._updated = bool(v)
        else:
            f.set_updated(self.id, bool(v))

    @property
    def grad(self):
        return self.value.grad

    def __repr__(self) -> str:
        return f"Parameter(id={self.id}, name={self.name!r}, shape={tuple(self.value.shape)})"


class Layer:
    """A module that owns parameters directly: one node of the reference's tape."""

    __slots__ = ("index", "name", "module", "params")

    def __init__(self, index: int, name: str, module: torch.nn.Module, params: list):
        self.index = index
        self.name = name
        self.module = module
        self.params = params

    def __repr__(self) -> str:
        return f"Layer({self.index}, {self.name!r}, params={[p.id for p in self.params]})"


class Graph:
    """A training graph: parameter registry, layers and per-iteration state.

    ``module(x)`` must return the network output; the loss is
    ``loss_fn(output, target)`` for ``inp = (x, target)``, or the output itself
    when ``loss_fn`` is None (the synthetic models return their scalar loss).
    """

    def __init__(self, module: torch.nn.Module, loss_fn=None, *, model: str = "module",
                 precision: str = "f32", width: int = 0, track_counts: bool = True,
                 track_input_grad: bool = False):
        self.module = module
        self.loss_fn = loss_fn
        self.model = model
        self.precision = precision
        self.width = width
        self.track_counts = track_counts
        self.track_input_grad = track_input_grad
        self.parameters: list = []
        self.layers: list = []
        by_tensor: dict = {}
        for mname, mod in module.named_modules():
            own = [(n, t) for n, t in mod.named_parameters(recurse=False) if t.requires_grad]
            if not own:
                continue
            layer = Layer(len(self.layers), mname, mod, [])
            for n, t in own:
                p = by_tensor.get(id(t))
                if p is None:
                    p = Parameter(len(self.parameters), t, f"{mname}.{n}" if mname else n)
                    by_tensor[id(t)] = p
                    self.parameters.append(p)
                if p not in layer.params:
                    layer.params.append(p)
                    p.layers.append(layer)
            self.layers.append(layer)
        self._by_tensor = by_tensor
        # per-iteration state
        self.pending_step_t = None
        self.pending_scale = None     # clip factor riding with the deferred updates
        self._forward_done = False
        self._loss = None
        self._input = None
        self._trace = None
        self._pre_node_hook = None
        self._prev_fwd_task = None
        self._ff_hook = None          # forward-fusion apply(layer), set by the schedule
        self._engines: dict = {}      # native fusion engines, by configuration
        self._flag_owner = None       # engine holding the pending/updated flags
        self._hook_owner = None       # engine whose C++ hooks sit on the parameters
        self.master_weights = False
        self._pre_handles = None
        self._leader_handles = None   # bucketed forward fusion: hooks on bucket leaders only
        self.exec_order = None        # layer indices in first-execution order (recorded)
        # bumped whenever deferred updates are applied from the host outside an
        # iteration (flush, checkpoint, state_dict): a CUDA graph captured
        # before that would apply them again on its next replay
        self.flush_gen = 0

    # -- mixed precision -------------------------------------------------------

    def use_master_weights(self, dtype=torch.bfloat16) -> None:
        """Run the module in ``dtype`` (bf16) and keep fp32 master weights.

        Every parameter gets an fp32 ``master`` copy taken from its current
        value; the module (parameters and buffers) is cast to ``dtype``.  The
        update kernels then read the bf16 gradient, update the fp32 master and
        history, and write the bf16 parameter back in the same pass
        (OF_FLAG_SHADOW_BF16: 2+4+8 B read, 4+8+2 B written per element).
        Must be called before any optimizer state exists."""
        if dtype != torch.bfloat16:
            raise ConfigError("master weights are supported for bfloat16 models")
        if self._engines or any(p.history for p in self.parameters):
            raise StateError("use_master_weights must precede the first update")
        for p in self.parameters:
            if p.value.dtype != torch.float32:
                raise ConfigError(f"parameter {p.id} is {p.value.dtype}; masters start from float32")
            p.master = p.value.detach().clone()
        self.module.to(dtype)
        for p in self.parameters:
            p.value.grad = None
            p._layout_ok = False
        self.master_weights = True

    # -- structure ---------------------------------------------------------

    @property
    def device(self) -> torch.device:
        return self.parameters[0].value.device

    def parameter_of(self, tensor: torch.Tensor) -> Parameter:
        return self._by_tensor[id(tensor)]

    def node_params(self) -> dict:
        return {layer.index: [p.id for p in layer.params] for layer in self.layers}

    @property
    def input_grad(self):
        """dL/d(input) of the last backward (needs ``track_input_grad``)."""
        return None if self._input is None else self._input.grad

    # -- hook sites ----------------------------------------------------------

    def _make_pre_hook(self, layer: Layer):
        def pre_hook(module, args):
            # hooks first, then the usage count (graph.py:195 before :200)
            extra = None
            if self._ff_hook is not None:
                extra = self._ff_hook(layer)
            if self._pre_node_hook is not None:
                more = self._pre_node_hook(layer)
                if more:
                    extra = (extra or []) + list(more)
            if self.track_counts:
                for p in layer.params:
                    p.count += 1
            if self._trace is not None:
                deps = [] if self._prev_fwd_task is None else [self._prev_fwd_task]
                if extra:
                    deps.extend(extra)
                self._prev_fwd_task = self._trace.add_task(tr.FORWARD, layer.index, deps)
            return None
        return pre_hook

    def _sync_pre_hooks(self, needed: bool) -> None:
        """Forward pre-hooks cost host time on every layer call, so they are
        installed only while something uses them (counts, forward fusion, a
        pre_node_hook or a trace)."""
        if needed and self._pre_handles is None:
            self._pre_handles = [L.module.register_forward_pre_hook(self._make_pre_hook(L))
                                 for L in self.layers]
        elif not needed and self._pre_handles is not None:
            for h in self._pre_handles:
                h.remove()
            self._pre_handles = None

    def set_leader_hooks(self, leaders) -> None:
        """Install forward pre-hooks on the given (layer, callback) pairs only,
        replacing any previous leader hooks (``leaders=None`` removes them)."""
        if self._leader_handles is not None:
            for h in self._leader_handles:
                h.remove()
            self._leader_handles = None
        if leaders:
            def make(fn):
                if getattr(fn, "is_hook", False):   # already hook(module, args) -> None
                    return fn
                def hook(module, args):
                    fn()
                    return None  # a non-None return would replace the layer's input
                return hook
            self._leader_handles = [L.module.register_forward_pre_hook(make(fn))
                                    for L, fn in leaders]

    def set_flag_owner(self, eng) -> None:
        """Move the forward-fusion flags into ``eng`` (a native engine) or back
        to the Parameter objects (``eng=None``)."""
        old = self._flag_owner
        if old is eng:
            return
        state = [(p.pending, p.updated) for p in self.parameters]
        for p, (pend, upd) in zip(self.parameters, state):
            p._flags = None
            p._pending, p._updated = pend, upd
            if eng is not None:
                eng.set_pending(p.id, pend)
                eng.set_updated(p.id, upd)
                p._flags = eng
        self._flag_owner = eng

    # -- execution -----------------------------------------------------------

    def forward(self, inp, trace: tr.ScheduleTrace | None = None, pre_node_hook=None):
        """Run the module; returns the scalar loss as a 0-dim device tensor.

        Resets every usage count (graph.py:186-187); each executing layer
        increments its parameters' counts after ``pre_node_hook(layer)`` ran.
        """
        if self.track_counts:
            for p in self.parameters:
                p.count = 0
        self._trace = trace
        self._pre_node_hook = pre_node_hook
        self._prev_fwd_task = None
        self._sync_pre_hooks(self.track_counts or self._ff_hook is not None
                             or pre_node_hook is not None or trace is not None)
        if isinstance(inp, (tuple, list)):
            x, target = inp[0], inp[1]
        else:
            x, target = inp, None
        if self.track_input_grad:
            x = x.detach().requires_grad_(True)
            self._input = x
        try:
            out = self.module(x)
            loss = out if self.loss_fn is None else self.loss_fn(out, target)
        finally:
            self._pre_node_hook = None
        self._loss = loss
        self._forward_done = True
        return loss

    def backward(self, trace: tr.ScheduleTrace | None = None) -> None:
        """Reverse pass over this iteration's loss (graph.py:274-281)."""
        if not self._forward_done:
            raise StateError("backward requires a completed forward pass this iteration")
        self._forward_done = False
        loss, self._loss = self._loss, None
        self._trace = trace
        try:
            loss.backward()
        finally:
            self._trace = None
        if self.track_counts:
            for p in self.parameters:
                p.count = 0  # every contribution has been accumulated

    def zero_grads(self) -> None:
        """graph.py:283-288."""
        for p in self.parameters:
            if p.value.grad is not None:
                p.value.grad.zero_()
            p.count = 0

    def allocate_grads(self) -> None:
        """Give every parameter a persistent zero gradient (reference layout:
        a Parameter always owns a gradient buffer, graph.py:34)."""
        for p in self.parameters:
            if p.value.grad is None:
                p.value.grad = torch.zeros_like(p.value)
