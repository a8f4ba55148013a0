"""The three training schedules on the GPU.

Mirrors /root/reference/pkg/src/optfuse/schedule.py: the same functions,
arguments, return type and error behaviour, all three producing the same
parameter trajectory (bit-identical on one device: same kernels, same
per-parameter arithmetic, only the issue point of each update moves).

* ``run_baseline`` (schedule.py:71-95): forward, backward, optional global
  clip, then every update -- here one multi-tensor launch.
* ``run_forward_fusion`` (schedule.py:98-138) + ``flush_pending_updates``
  (:141-160): a layer's deferred update is issued on the compute stream by
  that layer's forward pre-hook, immediately before the kernels that read the
  weight, so the update's write of theta and the forward's read of theta are
  adjacent in the stream (and in L2).
* ``run_backward_fusion`` (:163-207): each layer's update is issued from the
  post-accumulate-grad hook as soon as its gradients are complete.  With
  ``workers=1`` it is issued inline on the autograd stream (the serial
  reference order); with ``workers>1`` it goes to a high-priority side stream
  behind an event recorded at hook time -- that event is the device-side half
  of the Appendix B.2 guard (every kernel reading the old theta was enqueued
  before it) -- and overlaps the backward of the preceding layers.  The
  compute stream joins the side stream once at the end of backward, before
  the next forward can read any updated weight.  This is the GPU form of the
  reference's ``_ParallelRunner`` (schedule.py:210-311): updates outrank
  backward work through stream priority instead of a heap.
"""

from __future__ import annotations

import torch

from . import trace as tr
from .errors import ConfigError, GlobalInfoRequired
from .graph import Graph, Parameter
from .optim import OptimizerPolicy, clip_by_global_norm

BASELINE = "baseline"
FORWARD_FUSION = "forward-fusion"
BACKWARD_FUSION = "backward-fusion"
SCHEDULES = (BASELINE, FORWARD_FUSION, BACKWARD_FUSION)
STAGES = ("forward", "backward", "optimizer")


class StepReport:
    """What one iteration did (schedule.py:35-51).

    ``loss`` is the 0-dim device tensor (no host sync); ``float(report.loss)``
    is the reference's float.  ``stage_ms`` is measured with CUDA events on the
    compute stream and resolved lazily (first access synchronises).  Fused
    updates are billed to the stage that issues them, so fused schedules
    report an optimizer stage of zero.
    """

    def __init__(self, schedule: str, loss, trace, events=None, fused: bool = False,
                 pending_updates: int = 0):
        self.schedule = schedule
        self.loss = loss
        self.trace = trace
        self.pending_updates = pending_updates
        self._events = events
        self._fused = fused
        self._stage_ms = None

    @property
    def stage_ms(self) -> dict:
        if self._stage_ms is None:
            ev = self._events
            if not ev:
                self._stage_ms = {s: 0.0 for s in STAGES}
            else:
                ev[-1].synchronize()
                out = {"forward": ev[0].elapsed_time(ev[1]), "backward": ev[1].elapsed_time(ev[2])}
                out["optimizer"] = 0.0 if self._fused else ev[2].elapsed_time(ev[3])
                self._stage_ms = out
        return self._stage_ms

    @property
    def total_ms(self) -> float:
        return sum(self.stage_ms.values())


def check_inplace_safety(param: Parameter, graph: Graph) -> bool:
    """True iff ``param`` may be updated in place now (schedule.py:54-59).

    Condition (1), gradient complete, is ``count == 0``.  Condition (2), no
    backward node still to read the old value, holds on the host whenever the
    gradient is complete: autograd runs a node's input-gradient computation
    before its AccumulateGrad; on the device it is enforced by the event the
    backward-fusion engine records at hook time.
    """
    return param.count == 0


def _reject_newton(policy: OptimizerPolicy) -> None:
    if policy.kind == "newton":
        raise ConfigError("newton has no per-parameter step and cannot drive a schedule")


class _Marks:
    __slots__ = ("events", "stream")

    def __init__(self, on: bool):
        self.events = [] if on else None
        self.stream = torch.cuda.current_stream() if on else None

    def mark(self) -> None:
        if self.events is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(self.stream)
            self.events.append(ev)


class _TraceHooks:
    """Records backward-node tasks (and nothing else) when a trace is on."""

    def __init__(self, graph: Graph, trace: tr.ScheduleTrace):
        self.graph = graph
        self.trace = trace
        self.done: set = set()
        self.prev = trace.tasks[-1].task_id if trace.tasks else None
        self.last_of: dict = {}

    def backward_nodes_for(self, p: Parameter) -> list:
        """Record the backward node of every layer binding ``p`` not yet
        recorded (reverse layer order); returns the task ids."""
        ids = []
        for layer in sorted(p.layers, key=lambda L: -L.index):
            if layer.index in self.done:
                continue
            self.done.add(layer.index)
            deps = () if self.prev is None else (self.prev,)
            self.prev = self.trace.add_task(tr.BACKWARD, layer.index, deps)
            ids.append(self.prev)
        if ids:
            self.last_of[p.id] = ids[-1]
        return ids

    def __call__(self, p: Parameter) -> None:
        self.backward_nodes_for(p)


def run_baseline(graph: Graph, policy: OptimizerPolicy, inp, *, timing: bool = True,
                 trace: bool = False) -> StepReport:
    """Three contiguous phases; the update phase is one multi-tensor launch."""
    _reject_newton(policy)
    policy.begin_iteration()
    tc = tr.ScheduleTrace(BASELINE) if trace else None
    marks = _Marks(timing)
    marks.mark()
    loss = graph.forward(inp, tc)
    marks.mark()
    if tc is not None:
        graph.install_grad_ready_hooks()
        graph._grad_ready = _TraceHooks(graph, tc)
    try:
        graph.backward(tc)
    finally:
        graph._grad_ready = None
    marks.mark()
    prev = tc.tasks[-1].task_id if tc is not None and tc.tasks else None
    if policy.clip_norm is not None:
        clip_by_global_norm(graph, policy.clip_norm, tc)
        if tc is not None:
            prev = tc.add_task(tr.CLIP_BARRIER, -1, (prev,))
    order = list(reversed(graph.parameters))
    policy.step_params(order, trace=tc)
    if tc is not None:
        for p in order:
            prev = tc.add_task(tr.OPT_STEP, p.id, (prev,))
    marks.mark()
    return StepReport(BASELINE, loss, tc, marks.events)


def run_forward_fusion(graph: Graph, policy: OptimizerPolicy, inp, *, timing: bool = True,
                       trace: bool = False) -> StepReport:
    """Lazy schedule: deferred updates applied just before each layer's forward.

    The ``updated`` latch applies a shared parameter once; new gradients are
    deferred at the end of backward, tagged with this iteration's step index
    (schedule.py:130-133).  Global-information transforms are legal: the clip
    factor is computed once all gradients exist and rides along with the
    deferred updates.
    """
    _reject_newton(policy)
    policy.begin_iteration()
    tc = tr.ScheduleTrace(FORWARD_FUSION) if trace else None
    step_t = graph.pending_step_t

    def apply_pending(layer):
        todo = [p for p in layer.params if p.pending and not p.updated]
        if not todo:
            return None
        policy.step_params(todo, step_t=step_t, trace=tc)
        for p in todo:
            p.updated = True
        if tc is None:
            return None
        return [tc.add_task(tr.OPT_STEP, p.id, ()) for p in todo]

    marks = _Marks(timing)
    marks.mark()
    graph._ff_hook = apply_pending
    try:
        loss = graph.forward(inp, tc)
    finally:
        graph._ff_hook = None
    # a pending parameter whose layer did not run this forward is applied now,
    # before this iteration's gradients accumulate on top of its old ones
    leftover = [p for p in graph.parameters if p.pending]
    if leftover:
        policy.step_params(leftover, step_t=step_t, trace=tc)
    marks.mark()
    if tc is not None:
        graph.install_grad_ready_hooks()
        graph._grad_ready = _TraceHooks(graph, tc)
    try:
        graph.backward(tc)
    finally:
        graph._grad_ready = None
    if policy.clip_norm is not None:
        clip_by_global_norm(graph, policy.clip_norm, tc)
        if tc is not None:
            tc.add_task(tr.CLIP_BARRIER, -1, (tc.tasks[-1].task_id,))
    for p in graph.parameters:
        p.pending = True
        p.updated = False
    graph.pending_step_t = policy.t
    marks.mark()
    marks.mark()
    return StepReport(FORWARD_FUSION, loss, tc, marks.events, fused=True,
                      pending_updates=len(graph.parameters))


def flush_pending_updates(graph: Graph, policy: OptimizerPolicy,
                          trace: tr.ScheduleTrace | None = None) -> int:
    """Apply every deferred update as the next forward pass would (layer order,
    frozen step index); idempotent (schedule.py:141-160).  Must precede any
    observation of parameter values (eval, state_dict, checkpoint)."""
    todo = []
    seen: set = set()
    for layer in graph.layers:
        for p in layer.params:
            if p.pending and p.id not in seen:
                seen.add(p.id)
                todo.append(p)
    if not todo:
        return 0
    policy.step_params(todo, step_t=graph.pending_step_t, trace=trace)
    if trace is not None:
        prev = None
        for p in todo:
            prev = trace.add_task(tr.FLUSH, p.id, () if prev is None else (prev,))
    return len(todo)


class BackwardFusionEngine:
    """Per-graph state of backward fusion: launch groups, readiness counters,
    the update side stream and its events (the GPU ``_ParallelRunner``).

    Launch groups are layers: each parameter belongs to the first layer that
    binds it, so a shared parameter is updated once, after its last use (its
    AccumulateGrad fires once, after all contributions).
    """

    def __init__(self, graph: Graph, side_stream: bool):
        self.graph = graph
        groups, seen = [], set()
        for layer in graph.layers:
            ps = [p for p in layer.params if p.id not in seen]
            seen.update(p.id for p in ps)
            if ps:
                groups.append(ps)
        self.groups = groups
        self.group_of = {}
        for gi, ps in enumerate(groups):
            for p in ps:
                self.group_of[p.id] = gi
        self.size = [len(g) for g in groups]
        self.ready = [0] * len(groups)
        self.launched = [False] * len(groups)
        self.stream = torch.cuda.Stream(priority=-1) if side_stream else None
        self.events = [torch.cuda.Event() for _ in groups] if side_stream else None
        self.join = torch.cuda.Event() if side_stream else None
        self.hold: list = []
        self.policy = None
        self.trace_hooks = None
        # optional instrumentation: (start event, end event, params) per
        # side-stream launch, for the bench's in-situ kernel timing
        self.profile = None

    def begin(self, policy: OptimizerPolicy, tc) -> None:
        self.policy = policy
        self.ready = [0] * len(self.groups)
        self.launched = [False] * len(self.groups)
        self.trace_hooks = _TraceHooks(self.graph, tc) if tc is not None else None

    def on_grad_ready(self, p: Parameter) -> None:
        p.count = 0
        if self.trace_hooks is not None:
            self.trace_hooks.backward_nodes_for(p)
        gi = self.group_of[p.id]
        self.ready[gi] += 1
        if self.ready[gi] == self.size[gi]:
            self._launch(gi)

    def _launch(self, gi: int) -> None:
        params = self.groups[gi]
        policy = self.policy
        tc = self.trace_hooks.trace if self.trace_hooks is not None else None
        if self.stream is None:
            policy.step_params(params, trace=tc)
        else:
            policy.prepare(params, hold=self.hold)
            ev = self.events[gi]
            ev.record(torch.cuda.current_stream())
            self.stream.wait_event(ev)
            if self.profile is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(self.stream)
                policy.step_params(params, trace=tc, stream=self.stream, hold=self.hold)
                e1.record(self.stream)
                self.profile.append((e0, e1, params))
            else:
                policy.step_params(params, trace=tc, stream=self.stream, hold=self.hold)
        self.launched[gi] = True
        if tc is not None:
            for p in params:
                dep = self.trace_hooks.last_of.get(p.id)
                tc.add_task(tr.OPT_STEP, p.id, () if dep is None else (dep,))

    def finish(self) -> None:
        # groups that did not complete during backward (parameters that got no
        # gradient this iteration): the reference still steps them with g = 0
        for gi, done in enumerate(self.launched):
            if not done:
                for p in self.groups[gi]:
                    p.count = 0
                self._launch(gi)
        if self.stream is not None:
            self.join.record(self.stream)
            torch.cuda.current_stream().wait_event(self.join)
        self.hold.clear()
        self.policy = None
        self.trace_hooks = None


def run_backward_fusion(graph: Graph, policy: OptimizerPolicy, inp, workers: int = 1, *,
                        timing: bool = True, trace: bool = False) -> StepReport:
    """Eager schedule: update each layer as soon as its gradients are complete.

    Raises GlobalInfoRequired, mutating nothing, for policies or transforms
    that must see all gradients first (schedule.py:174-177).
    """
    if policy.requires_global_info:
        raise GlobalInfoRequired(
            f"backward-fusion cannot host {policy.kind!r}"
            + (" with global-norm clipping" if policy.clip_norm is not None else ""))
    _reject_newton(policy)
    if workers < 1:
        raise ConfigError(f"workers must be >= 1, got {workers}")
    side = workers > 1
    eng = graph._bf_engine
    if eng is None or (eng.stream is not None) != side:
        eng = BackwardFusionEngine(graph, side)
        graph._bf_engine = eng
    policy.begin_iteration()
    tc = tr.ScheduleTrace(BACKWARD_FUSION) if trace else None
    marks = _Marks(timing)
    marks.mark()
    loss = graph.forward(inp, tc)
    marks.mark()
    graph.install_grad_ready_hooks()
    eng.begin(policy, tc)
    graph._grad_ready = eng.on_grad_ready
    try:
        graph.backward(tc)
        eng.finish()
    finally:
        graph._grad_ready = None
    marks.mark()
    marks.mark()
    return StepReport(BACKWARD_FUSION, loss, tc, marks.events, fused=True)
