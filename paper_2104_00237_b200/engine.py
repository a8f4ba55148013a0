"""Python face of the native hook scheduler (csrc/optfuse_engine.cpp).

One ``FusionEngine`` per (graph, optimizer kind, stream mode, bucketing)
holds, in C++: the parameter tensors and their history slots, the launch
groups, the per-parameter ``pending``/``updated`` flags of forward fusion,
the update side stream's events, and a PostAccumulateGradHook on every
parameter.  Python only arms it once per iteration.
"""

from __future__ import annotations

import torch

from . import _native as nat
from . import kernels
from .errors import NativeLibraryError

_mod = None


def native_engine_module():
    """Import the compiled engine extension; no fallback."""
    global _mod
    if _mod is None:
        nat.lib()  # the kernel library it links against must load first
        try:
            from . import _optfuse_engine as m
        except ImportError as e:
            raise NativeLibraryError(
                f"native engine extension not built ({e}); run "
                "`python -c 'import __graft_entry__ as g; g.build()'`") from e
        _mod = m
    return _mod


def launch_groups(graph, bucket_elems: int = 0, exclude=frozenset()) -> list:
    """Backward-fusion launch groups as lists of parameter ids.

    Each parameter belongs to the first layer (registration order) binding it,
    so a shared parameter is updated once, when its last use has contributed.
    With ``bucket_elems > 0`` consecutive layer groups are merged, in backward
    order (last layer first), until a bucket holds at least that many
    elements -- fewer, larger launches for networks of many small layers.
    """
    groups, seen = [], set(exclude)   # excluded: updated by their consumer kernel
    for layer in graph.layers:
        ids = [p.id for p in layer.params if p.id not in seen]
        seen.update(ids)
        if ids:
            groups.append(ids)
    if bucket_elems <= 0:
        return groups
    numel = {p.id: p.value.numel() for p in graph.parameters}
    buckets, cur, size = [], [], 0
    for ids in reversed(groups):
        cur = cur + ids
        size += sum(numel[i] for i in ids)
        if size >= bucket_elems:
            buckets.append(cur)
            cur, size = [], 0
    if cur:
        buckets.append(cur)
    return buckets


class FusionEngine:
    def __init__(self, graph, policy, side_stream: bool, bucket_elems: int = 0,
                 priority: str = "high", exclude=frozenset()):
        m = native_engine_module()
        self.graph = graph
        self.kind = policy.kind
        self.side = side_stream
        self.bucket_elems = bucket_elems
        self.groups = launch_groups(graph, bucket_elems, exclude)
        # CUDA stream priorities: lower number = higher priority (-1 is the
        # highest torch exposes, 0 the default)
        self.stream = (torch.cuda.Stream(priority=-1 if priority == "high" else 0)
                       if side_stream else None)
        params = graph.parameters
        # history slots exist before the engine captures their pointers
        policy.prepare_history(params)
        self.native = m.Engine([p.value for p in params], self.groups,
                               [[p.id for p in L.params] for L in graph.layers],
                               self.stream.cuda_stream if self.stream is not None else 0)
        slots = policy.history_slots()
        self.mixed = graph.master_weights
        for p in params:
            a = p.history[slots[0]] if slots else None
            b = p.history[slots[1]] if len(slots) > 1 else None
            self.native.set_slots(p.id, a, b, p.master)
        self._hp_key = None
        self.ff_bucket_elems = 0
        self.ff_prefetch = False
        self.ff_leaders = None

    def configure(self, policy, step_t: int, grad_scale=None, max_ctas: int = 0) -> None:
        """Hyper-parameters (and the frozen step index) of the next launches.
        ``max_ctas`` caps each update's grid (0: fill the GPU)."""
        ds = policy._dstep
        key = (step_t, policy.kind, policy.eta, policy.alpha, policy.weight_decay, policy.epsilon,
               policy.beta1, policy.beta2, policy.rho, policy.grad_reset, id(grad_scale), max_ctas,
               id(ds))
        if key == self._hp_key:
            return
        hp = kernels.hparams(policy.kind, policy.eta, policy.alpha, policy.weight_decay,
                             policy.epsilon, policy.beta1, policy.beta2, policy.rho, step_t)
        zero = policy.grad_reset == "zero"
        flags = ((nat.OF_FLAG_ZERO_GRAD if zero else 0) | (nat.OF_FLAG_SHADOW_BF16 if self.mixed else 0)
                 | policy.device_step_flag)
        self.native.set_hparams(hp.kind, hp.eta, hp.alpha, hp.weight_decay, hp.epsilon, hp.beta1,
                                hp.beta2, hp.rho, hp.bias_correction1, hp.bias_correction2,
                                flags, not zero, grad_scale, max_ctas,
                                ds.offset if ds is not None else None,
                                ds.table if ds is not None else None, step_t)
        self._hp_key = key

    @property
    def launches(self) -> int:
        return self.native.launches
