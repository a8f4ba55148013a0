"""Consumer-fused backward fusion: the update of a Linear layer's weight runs in
the epilogue of the GEMM that produces its gradient.

The reference's backward fusion (schedule.py:163-207) updates a parameter as
soon as its gradient is complete.  On B200 the gradient of a weight tile is
complete when the tensor cores finish its accumulation in TMEM, so the
B200-native form of the schedule applies the update right there
(of_wgrad_step, csrc/optfuse_wgrad.cu): the weight gradient is never written
to HBM and no separate update launch exists.  The Appendix B.2 guard
(schedule.py:54-59) is stream order: the layer's input-gradient GEMM -- the
only reader of the old weight -- is issued first on the same stream.

Scope: bf16 modules with fp32 master weights (``graph.use_master_weights()``,
the C4 / BERT-mixed configuration); every ``nn.Linear`` whose weight belongs
to that layer alone (a tied weight, e.g. BERT's MLM decoder = word
embeddings, keeps the ordinary path: its gradient has a second producer) and
whose shape fits the kernel (in_features % 32 == 0, out_features % 8 == 0).
Biases, LayerNorms and embeddings keep the ordinary backward-fusion launches.
The same arithmetic as the multi-tensor kernel applied to the fp32
accumulator (the unfused mixed path first rounds the gradient to bf16).

    cf = ConsumerFusion(graph, policy)
    run_backward_fusion(graph, policy, inp, workers=2, consumer=cf)

Outside ``run_backward_fusion(..., consumer=cf)`` (other schedules, eval,
``torch.autograd.grad``) the patched layers produce an ordinary weight
gradient.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F

from . import _native as nat
from . import kernels
from .errors import ConfigError


class _FusedLinear(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, cf, pid):
        ctx.cf, ctx.pid, ctx.has_bias = cf, pid, bias is not None
        ctx.save_for_backward(x, weight)
        return F.linear(x, weight, bias)

    @staticmethod
    def backward(ctx, gy):
        x, w = ctx.saved_tensors
        gy2 = gy.reshape(-1, gy.shape[-1])
        x2 = x.reshape(-1, x.shape[-1])
        # the input gradient reads the OLD weight: issued before the update
        gx = (gy2 @ w).view(*gy.shape[:-1], w.shape[1]) if ctx.needs_input_grad[0] else None
        gb = gy2.sum(0) if ctx.has_bias else None
        cf = ctx.cf
        if cf.active:
            cf.step_weight(ctx.pid, gy2.contiguous(), x2.contiguous())
            gw = None
        else:
            gw = gy2.t() @ x2
        return gx, gw, gb, None, None


class ConsumerFusion:
    """Patches the eligible Linear layers of ``graph`` (see module docstring)."""

    def __init__(self, graph, policy):
        if not graph.master_weights:
            raise ConfigError("consumer fusion runs on bf16 modules with fp32 master weights "
                              "(graph.use_master_weights())")
        if policy.requires_global_info:
            raise ConfigError("consumer fusion is backward fusion: no global-information policy")
        self.graph = graph
        self.policy = policy
        self.active = False
        self.launches = 0
        self.ids: list = []
        policy.prepare_history(graph.parameters)
        slots = policy.history_slots()
        self._slots = slots
        for layer in graph.layers:
            mod = layer.module
            if type(mod) is not torch.nn.Linear:
                continue
            p = graph.parameter_of(mod.weight)
            if len(p.layers) != 1 or mod.in_features % 32 or mod.out_features % 8:
                continue
            if mod.weight.dtype != torch.bfloat16 or p.master is None:
                continue
            self.ids.append(p.id)
            mod.forward = self._make_forward(mod, p.id)
        if not self.ids:
            raise ConfigError("no Linear layer of this graph is eligible for consumer fusion")
        self.id_set = frozenset(self.ids)

    def _make_forward(self, mod, pid):
        def forward(x):
            return _FusedLinear.apply(x, mod.weight, mod.bias, self, pid)
        return forward

    def step_weight(self, pid: int, gy2: torch.Tensor, x2: torch.Tensor) -> None:
        """dW = gy2^T x2 fused with the policy step of parameter ``pid``."""
        pol = self.policy
        p = self.graph.parameters[pid]
        h = p.history
        s = self._slots
        flags = pol.device_step_flag
        kernels.wgrad_step(gy2, x2, p.master, h[s[0]] if s else None,
                           h[s[1]] if len(s) > 1 else None, pol._hparams(pol.t),
                           shadow=p.value, flags=flags)
        self.launches += 1

    @property
    def numel(self) -> int:
        return sum(self.graph.parameters[i].value.numel() for i in self.ids)


def supported() -> bool:
    """The fused wgrad kernel is in the loaded library (ABI 3)."""
    return hasattr(nat.lib(), "of_wgrad_step")
