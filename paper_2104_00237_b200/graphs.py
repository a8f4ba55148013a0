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

Step-dependent policies (adam, adamw: the bias corrections change every
iteration) are captured with OF_FLAG_DEVICE_STEP: the graph's first node
advances a device step offset, and every captured update reads its step index
as (host index at capture + offset) from a table of the host's own bias
corrections, so replay j is bit-identical to eager iteration t_capture + j.
The host policy's ``t`` (and a forward-fusion graph's ``pending_step_t``) is
advanced per replay so that flushes and checkpoints after replays see the
right step; stepping the policy eagerly between replays is rejected, and so
is a replay after the host applied the deferred updates (a flush, observe,
or state_dict between replays): the captured forward would apply them again.

Constraints: inputs are copied into static buffers; a forward-fusion step
must be captured with ``graph=``: the gradients one replay produces are what
the next replay's forward reads, and the capture routes them (see __init__).
"""

from __future__ import annotations

import torch

from .errors import StateError

_STEP_INDEPENDENT = ("sgd", "sgd-momentum", "adagrad", "rmsprop", "adadelta")


_CAPTURE_STREAMS: dict = {}


def _capture_stream(device):
    """One warm-up/capture stream per device, shared by every CapturedStep
    (captures run one at a time): each new stream that runs a matmul gets its
    own cuBLAS workspace, kept for the life of the process."""
    s = _CAPTURE_STREAMS.get(device)
    if s is None:
        s = _CAPTURE_STREAMS[device] = torch.cuda.Stream(device)
    return s


class CapturedStep:
    """``step_fn(inputs) -> loss`` captured once, replayed by ``__call__``.

    ``static_inputs`` is a tensor or (nested) tuple of tensors on the device;
    each call copies the given inputs into them (``non_blocking``) before
    replay.  ``policy``: the OptimizerPolicy the step drives (needed for
    step-dependent kinds); ``graph``: the Graph (keeps its forward-fusion
    ``pending_step_t`` in step with the replays).
    """

    def __init__(self, step_fn, static_inputs, policy=None, warmup: int = 3, graph=None,
                 stream=None):
        self.static = static_inputs if isinstance(static_inputs, tuple) else (static_inputs,)
        self.step_fn = step_fn
        self.policy = policy
        self.owner = graph
        cur = torch.cuda.current_stream()
        # warm-up and capture stream (a caller whose module stashed autograd
        # nodes on a stream, e.g. DDP, passes that stream)
        side = stream if stream is not None else _capture_stream(cur.device)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            for _ in range(warmup):
                step_fn(self._arg())
        cur.wait_stream(side)
        torch.cuda.synchronize()
        # Forward fusion reads, in iteration i+1, the gradients iteration i
        # produced.  The captured forward-fusion launches read the gradients
        # that exist now (the last warm-up iteration's); every replay's
        # backward writes its gradients into the graph's own pool.  So the
        # captured iteration ends with one multi-tensor copy of its gradients
        # into the buffers the next replay's forward reads (held here).  With
        # grad_reset="zero" the gradients are persistent and need nothing.
        self.grad_reset_forced = False
        self._ff_prev = None
        owner = getattr(graph, "_flag_owner", None)
        ff = owner is not None and owner.num_pending() > 0
        if ff and policy is not None and policy.grad_reset == "none":
            prev = [p.value.grad for p in graph.parameters]
            if all(g is not None for g in prev):
                self._ff_prev = prev
            else:             # some parameter has no gradient: keep them resident instead
                policy.grad_reset = "zero"
                self.grad_reset_forced = True
        from . import _native, kernels
        self.dstep = None
        if policy is not None and policy.kind not in _STEP_INDEPENDENT:
            self.dstep = policy.device_step(torch.device("cuda", torch.cuda.current_device()))
            self.dstep.ensure(policy.t + 1)
            torch.cuda.synchronize()
        n0 = _native.launch_count()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=side):
            if self.dstep is not None:
                kernels.step_advance(self.dstep.offset, 1)   # first node of every replay
                policy._dstep = self.dstep
                try:
                    self.loss = step_fn(self._arg())
                finally:
                    policy._dstep = None
            else:
                self.loss = step_fn(self._arg())
            if self._ff_prev is not None:
                cur = [p.value.grad for p in graph.parameters]
                if any(g is None for g in cur):
                    raise StateError("forward fusion left a parameter without a gradient")
                # one multi-tensor copy kernel (torch's foreach copy costs ~10x
                # more on MobileNetV2's 158 small tensors)
                ok = [kernels.same_layout(d, c) for d, c in zip(self._ff_prev, cur)]
                for d, c, k in zip(self._ff_prev, cur, ok):
                    if not k:
                        d.copy_(c)
                same = [(d, c) for d, c, k in zip(self._ff_prev, cur, ok) if k]
                if same:
                    kernels.copy_mt(kernels.CopyList([d for d, _ in same], [c for _, c in same],
                                                     checked=True))
        # liboptfuse_b200 kernel nodes in the graph (each replay launches them all)
        self.native_launches = _native.launch_count() - n0
        if self.dstep is not None:
            self.dstep.offset.fill_(-1)     # replay j runs with offset j
        self.replays = 0
        self._t = policy.t if policy is not None else None
        self._flush_gen = getattr(graph, "flush_gen", None)
        self._stage = None        # device staging copy of the next call's inputs
        self._staged = False

    def _arg(self):
        return self.static if len(self.static) > 1 else self.static[0]

    def __call__(self, inputs=None):
        pol = self.policy
        if self.owner is not None and getattr(self.owner, "flush_gen", None) != self._flush_gen:
            # the host applied the deferred (forward-fusion) updates this graph's
            # next replay would apply again from the same gradients
            raise StateError("deferred updates were applied on the host (flush / observe / "
                             "state_dict) after this step was captured; replaying would apply "
                             "them twice -- capture again to continue")
        if pol is not None:
            if pol.t != self._t:
                raise StateError("the policy was stepped outside this captured graph; "
                                 "capture again to continue with replays")
            if self.replays > 0:      # the capture's own iteration never ran: replay 0 is t_capture
                pol.t += 1
                self._t = pol.t
                if self.owner is not None and self.owner.pending_step_t is not None:
                    self.owner.pending_step_t = pol.t
            if self.dstep is not None:
                self.dstep.ensure(pol.t + 1)
        if inputs is not None:
            if self._staged:
                raise StateError("inputs were staged for this call; call it without inputs")
            src = inputs if isinstance(inputs, tuple) else (inputs,)
            _copy_into(self.static, src)
        elif self._staged:
            cur = torch.cuda.current_stream()
            cur.wait_event(self._stage_ready)
            _copy_into(self.static, self._stage)      # on-device, ~1 µs per MB
            self._stage_free.record(cur)
            self._staged = False
        self.graph.replay()
        self.replays += 1
        return self.loss


    @property
    def staged(self) -> bool:
        """Inputs are staged for the next call."""
        return self._staged

    def stage(self, inputs) -> None:
        """Starts copying the NEXT call's inputs (ideally pinned host tensors)
        into a device staging buffer on a copy stream, overlapping whatever
        runs now (typically the previous replay).  The next ``__call__()``
        without inputs consumes them: one on-device copy into the static
        inputs, ordered behind the staging copy.  The host tensors must stay
        unchanged until that call has been issued."""
        if self._staged:
            raise StateError("inputs already staged; call the step before staging more")
        src = inputs if isinstance(inputs, tuple) else (inputs,)
        if self._stage is None:
            self._copy_stream = torch.cuda.Stream()
            self._stage = _empty_like_nested(self.static, self._copy_stream)
            self._stage_ready = torch.cuda.Event()
            self._stage_free = torch.cuda.Event()
            self._stage_free.record()
        cs = self._copy_stream
        cs.wait_event(self._stage_free)           # the last staged inputs were consumed
        with torch.cuda.stream(cs):
            _copy_into(self._stage, src)
        self._stage_ready.record(cs)
        self._staged = True


def _empty_like_nested(t, stream):
    """Allocated on the current stream, also used on ``stream`` (so that its
    memory is not reused before that stream's copies into it are done)."""
    if isinstance(t, (tuple, list)):
        return type(t)(_empty_like_nested(x, stream) for x in t)
    e = torch.empty_like(t)
    e.record_stream(stream)
    return e


def _copy_into(dst, src) -> None:
    for d, s in zip(dst, src):
        if isinstance(d, (tuple, list)):
            _copy_into(d, s)
        else:
            d.copy_(s, non_blocking=True)
