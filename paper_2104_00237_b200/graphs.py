"""CUDA-graph capture of a whole fused training iteration.

Eager PyTorch issues ~600 kernels per MobileNetV2 iteration from the host, so
at small batch the step is host-bound.  ``CapturedStep`` records one
iteration of any schedule -- forward (with forward-fusion update launches
before each layer), backward (with backward-fusion launches on the update
side stream, joined back by events) and the baseline's update phase -- into a
CUDA graph and replays it.  The graph preserves the schedule: each update
node depends on exactly the events the engine recorded at its issue point
(gradient-ready for backward fusion, the preceding layer for forward fusion),
so replay runs the same DAG with no host in the loop.

Constraints (checked): the policy's hyper-parameters must not change between
replays -- kinds whose update depends on the step index (adam, adamw bias
corrections) are rejected -- and inputs are copied into static buffers.
"""

from __future__ import annotations

import torch

from .errors import ConfigError

_STEP_INDEPENDENT = ("sgd", "sgd-momentum", "adagrad", "rmsprop", "adadelta")


class CapturedStep:
    """``step_fn(inputs) -> loss`` captured once, replayed by ``__call__``.

    ``static_inputs`` is a tensor or tuple of tensors on the device; each call
    copies the given inputs into them (``non_blocking``) before replay.
    """

    def __init__(self, step_fn, static_inputs, policy=None, warmup: int = 3):
        if policy is not None and policy.kind not in _STEP_INDEPENDENT:
            raise ConfigError(f"{policy.kind!r} depends on the step index; it cannot be "
                              "replayed from a captured graph with fixed hyper-parameters")
        self.static = static_inputs if isinstance(static_inputs, tuple) else (static_inputs,)
        self.step_fn = step_fn
        cur = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            for _ in range(warmup):
                step_fn(self._arg())
        cur.wait_stream(side)
        torch.cuda.synchronize()
        from . import _native
        n0 = _native.launch_count()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.loss = step_fn(self._arg())
        # liboptfuse_b200 kernel nodes in the graph (each replay launches them all)
        self.native_launches = _native.launch_count() - n0

    def _arg(self):
        return self.static if len(self.static) > 1 else self.static[0]

    def __call__(self, inputs=None):
        if inputs is not None:
            src = inputs if isinstance(inputs, tuple) else (inputs,)
            for dst, s in zip(self.static, src):
                dst.copy_(s, non_blocking=True)
        self.graph.replay()
        return self.loss
