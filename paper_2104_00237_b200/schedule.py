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

import functools

import torch

from . import checkpoint
from . import trace as tr
from .errors import ConfigError, GlobalInfoRequired
from .graph import Graph, Parameter
from .optim import OptimizerPolicy, clip_by_global_norm, clip_factor, grad_scale_for

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
        # the iteration's backward has run: the caller gets a plain device value
        self.loss = loss.detach() if isinstance(loss, torch.Tensor) else loss
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


class _TraceRecorder:
    """Host-side schedule trace from the engine's gradient-ready callback:
    records the backward node(s) a ready parameter completes and, for backward
    fusion, the step task of each launch group once all its members are ready
    (the same counting the native engine does)."""

    def __init__(self, graph: Graph, trace: tr.ScheduleTrace, groups=None):
        self.graph = graph
        self.trace = trace
        self.done: set = set()
        self.prev = trace.tasks[-1].task_id if trace.tasks else None
        self.last_of: dict = {}
        self.groups = groups
        if groups is not None:
            self.group_of = {pid: gi for gi, g in enumerate(groups) for pid in g}
            self.ready = [0] * len(groups)
            self.stepped = [False] * len(groups)

    def backward_nodes_for(self, p: Parameter) -> None:
        for layer in sorted(p.layers, key=lambda L: -L.index):
            if layer.index in self.done:
                continue
            self.done.add(layer.index)
            deps = () if self.prev is None else (self.prev,)
            self.prev = self.trace.add_task(tr.BACKWARD, layer.index, deps)
            self.last_of[p.id] = self.prev

    def steps_for_group(self, gi: int) -> None:
        self.stepped[gi] = True
        for pid in self.groups[gi]:
            dep = self.last_of.get(pid)
            self.trace.add_task(tr.OPT_STEP, pid, () if dep is None else (dep,))

    def __call__(self, pid: int) -> None:
        p = self.graph.parameters[pid]
        p.count = 0
        self.backward_nodes_for(p)
        if self.groups is not None:
            gi = self.group_of[pid]
            self.ready[gi] += 1
            if self.ready[gi] == len(self.groups[gi]):
                self.steps_for_group(gi)

    def finish(self) -> None:
        if self.groups is not None:
            for gi, done in enumerate(self.stepped):
                if not done:
                    self.steps_for_group(gi)


_ALL_IN_ONE = 1 << 62   # bucket size that merges every layer into one launch group


def _engine(graph: Graph, policy: OptimizerPolicy, side: bool, bucket_elems: int = 0,
            priority: str = "high", exclude=frozenset()):
    from .engine import FusionEngine
    key = ((policy.kind, side, bucket_elems) + (() if priority == "high" else (priority,))
           + ((("consumer", exclude),) if exclude else ()))
    eng = graph._engines.get(key)
    if eng is None:
        eng = FusionEngine(graph, policy, side, bucket_elems, priority, exclude)
        graph._engines[key] = eng
    return eng


def _own_hooks(graph: Graph, eng) -> None:
    """One post-accumulate-grad hook slot per tensor: make ``eng`` its owner."""
    if graph._hook_owner is not eng:
        eng.native.install_hooks()
        graph._hook_owner = eng


def _traced_backward(graph: Graph, policy: OptimizerPolicy, tc) -> None:
    """Backward of an unfused schedule with the engine hooks reporting
    gradient readiness (no launches) to the trace recorder."""
    eng = _engine(graph, policy, False)
    rec = _TraceRecorder(graph, tc)
    _own_hooks(graph, eng)
    eng.native.set_callback(rec)
    eng.native.bf_begin(False)
    try:
        graph.backward(tc)
    finally:
        eng.native.disarm()
        eng.native.set_callback(None)


def _leave_forward_fusion(graph: Graph, policy: OptimizerPolicy) -> None:
    """Switching away from forward fusion: drop its leader hooks and apply any
    update it still defers, so no schedule ever reads a stale parameter."""
    graph.set_leader_hooks(None)
    owner = graph._flag_owner
    if owner is not None and owner.num_pending():
        flush_pending_updates(graph, policy)


def run_baseline(graph: Graph, policy: OptimizerPolicy, inp, *, timing: bool = True,
                 trace: bool = False) -> StepReport:
    """Three contiguous phases; the update phase is one multi-tensor launch."""
    _reject_newton(policy)
    checkpoint.attach(graph, policy)
    _leave_forward_fusion(graph, policy)
    policy.begin_iteration()
    tc = tr.ScheduleTrace(BASELINE) if trace else None
    marks = _Marks(timing)
    marks.mark()
    loss = graph.forward(inp, tc)
    marks.mark()
    if tc is not None:
        _traced_backward(graph, policy, tc)
    else:
        graph.backward()
    marks.mark()
    prev = tc.tasks[-1].task_id if tc is not None and tc.tasks else None
    if policy.clip_norm is not None:
        clip_by_global_norm(graph, policy.clip_norm, tc)
        if tc is not None:
            prev = tc.add_task(tr.CLIP_BARRIER, -1, (prev,))
    order = list(reversed(graph.parameters))
    if tc is None and policy.clip_norm is None and graph.device.type == "cuda":
        # the same single multi-tensor launch, its tensor list kept by the
        # native engine (one group: every parameter, backward order): no
        # per-parameter Python on the host, which an eager step pays for
        policy.check_steppable(order)
        eng = _engine(graph, policy, False, _ALL_IN_ONE)
        eng.configure(policy, policy.t, None, 0)
        eng.native.launch_group(0, sync=False)
        eng.native.join()
        for p in order:
            p.pending = False
            p._grad_scale = None
    else:
        policy.step_params(order, trace=tc)
    if tc is not None:
        for p in order:
            prev = tc.add_task(tr.OPT_STEP, p.id, (prev,))
    marks.mark()
    return StepReport(BASELINE, loss, tc, marks.events)


def ff_units(graph: Graph, bucket_elems: int) -> tuple:
    """Forward-fusion buckets over the recorded execution order: each
    parameter goes to the bucket of the first layer that uses it; a bucket
    closes once it holds ``bucket_elems`` elements.  Returns (units as lists
    of parameter ids, leader layer of each unit)."""
    units, leaders, seen = [], [], set()
    cur, size, lead = [], 0, None
    for li in graph.exec_order:
        layer = graph.layers[li]
        ids = [p.id for p in layer.params if p.id not in seen]
        if not ids:
            continue
        seen.update(ids)
        if lead is None:
            lead = layer
        cur += ids
        size += sum(graph.parameters[i].value.numel() for i in ids)
        if size >= bucket_elems:
            units.append(cur)
            leaders.append(lead)
            cur, size, lead = [], 0, None
    if cur:
        units.append(cur)
        leaders.append(lead)
    return units, leaders


def run_forward_fusion(graph: Graph, policy: OptimizerPolicy, inp, *, timing: bool = True,
                       trace: bool = False, bucket_elems: int = 0,
                       prefetch: int = 0) -> StepReport:
    """Lazy schedule: deferred updates applied just before each layer's forward.

    The layer's forward pre-hook calls the native engine, which launches the
    update of that layer's pending, not yet ``updated`` parameters on the
    compute stream (the latch applies a shared parameter once); new gradients
    are deferred at the end of backward, tagged with this iteration's step
    index (schedule.py:130-133).  Global-information transforms are legal: the
    clip factor is computed once all gradients exist and rides along with the
    deferred updates as a device scalar.

    ``bucket_elems > 0`` groups consecutive layers (in the execution order
    recorded by the first iteration) into buckets whose pending updates are
    issued together right before the bucket's first layer, so only bucket
    leaders carry a pre-hook.

    ``prefetch=d`` (B200 addition; True = 1) issues the updates of units
    u+1 .. u+d on a side stream when unit u's pre-hook runs, so they overlap
    the forward of the units before them; each unit's pre-hook waits for its
    own update.  ``prefetch=-1``: every unit at the first pre-hook.  Same
    trajectory, bit for bit.
    """
    _reject_newton(policy)
    checkpoint.attach(graph, policy)
    if bucket_elems < 0:
        raise ConfigError(f"bucket_elems must be >= 0, got {bucket_elems}")
    tc = tr.ScheduleTrace(FORWARD_FUSION) if trace else None
    depth = 0 if tc is not None else (1 << 30 if prefetch is not True and prefetch < 0
                                      else int(prefetch))
    prefetch = depth > 0
    eng = _engine(graph, policy, prefetch)
    graph.set_flag_owner(eng.native)
    policy.begin_iteration()
    if graph.pending_step_t is not None:
        eng.configure(policy, graph.pending_step_t, graph.pending_scale)
    native = eng.native
    if prefetch:
        def ff_layer(u, _f=native.ff_unit_lookahead, _d=depth):
            return _f(u, _d)
    else:
        ff_layer = native.ff_layer
    if bucket_elems == 0 and tc is None:
        # after the first iteration, one unit per executed layer in execution
        # order (a shared parameter belongs to the layer that uses it first):
        # the per-layer schedule, with hooks that call the engine directly
        bucket_elems = 1
    bucketed = bucket_elems > 0 and tc is None and graph.exec_order is not None
    if bucketed:
        if eng.ff_bucket_elems != bucket_elems or eng.ff_prefetch != depth:
            units, leaders = ff_units(graph, bucket_elems)
            native.set_ff_units(units)
            eng.ff_bucket_elems = bucket_elems
            eng.ff_prefetch = depth
            hooks = []
            for i, L in enumerate(leaders):
                h = functools.partial(native.ff_hook, i, depth)   # no Python frame per layer
                h.is_hook = True
                hooks.append((L, h))
            eng.ff_leaders = hooks
        graph.set_leader_hooks(eng.ff_leaders)
        apply_pending = None
    else:
        if eng.ff_bucket_elems:
            native.reset_ff_units()
            eng.ff_bucket_elems = 0
        graph.set_leader_hooks(None)
        order = [] if graph.exec_order is None else None
        seen = set()

        if tc is None:
            def apply_pending(layer):
                if order is not None and layer.index not in seen:
                    seen.add(layer.index)
                    order.append(layer.index)
                ff_layer(layer.index)
                return None
        else:
            def apply_pending(layer):
                todo = [p.id for p in layer.params if p.pending and not p.updated]
                ff_layer(layer.index)
                return [tc.add_task(tr.OPT_STEP, pid, ()) for pid in todo]

    marks = _Marks(timing)
    marks.mark()
    graph._ff_hook = apply_pending
    try:
        loss = graph.forward(inp, tc)
    finally:
        graph._ff_hook = None
    if not bucketed and tc is None and order is not None:
        graph.exec_order = order
    if prefetch:
        native.ff_join()   # prefetched units whose layer did not run
    # a pending parameter whose layer did not run this forward is applied now,
    # before this iteration's gradients accumulate on top of its old ones
    if native.num_pending():
        native.flush()
    marks.mark()
    if tc is not None:
        _traced_backward(graph, policy, tc)
    else:
        graph.backward()
    scale = None
    if policy.clip_norm is not None:
        factor, coef = clip_factor(graph, policy.clip_norm, tc)
        # one scale for the whole engine: the f64 factor for an f64 graph
        scale = grad_scale_for(graph.parameters[0], factor, coef)
        if tc is not None:
            tc.add_task(tr.CLIP_BARRIER, -1, (tc.tasks[-1].task_id,))
    native.set_all_pending()
    graph.pending_step_t = policy.t
    graph.pending_scale = scale
    marks.mark()
    marks.mark()
    return StepReport(FORWARD_FUSION, loss, tc, marks.events, fused=True,
                      pending_updates=len(graph.parameters))


def flush_pending_updates(graph: Graph, policy: OptimizerPolicy,
                          trace: tr.ScheduleTrace | None = None) -> int:
    """Apply every deferred update as the next forward pass would (layer order,
    frozen step index); idempotent (schedule.py:141-160).  Must precede any
    observation of parameter values (eval, state_dict, checkpoint)."""
    owner = graph._flag_owner
    todo = []
    seen: set = set()
    for layer in graph.layers:
        for p in layer.params:
            if p.pending and p.id not in seen:
                seen.add(p.id)
                todo.append(p)
    if not todo:
        return 0
    if owner is not None:
        # the engine that holds the flags (forward fusion with or without
        # the side-stream lookahead uses different engines)
        eng = next((e for e in graph._engines.values() if e.native is owner), None)
        if eng is None:
            eng = _engine(graph, policy, False)
        eng.configure(policy, graph.pending_step_t, graph.pending_scale)
        n = eng.native.flush()
    else:
        policy.step_params(todo, step_t=graph.pending_step_t)
        n = len(todo)
    if n:
        graph.flush_gen += 1
    if trace is not None:
        prev = None
        for p in todo:
            prev = trace.add_task(tr.FLUSH, p.id, () if prev is None else (prev,))
    return n


def default_update_ctas() -> int:
    """Default grid cap of a side-stream backward-fusion update: none.

    Measured on B200: capping the update to a third of the SMs
    does not buy overlap -- cuDNN/CUTLASS convolution CTAs leave no room for a
    co-resident update CTA, so a capped update only runs longer -- so the
    update fills the GPU and relies on stream priority.  ``update_ctas`` keeps
    the cap available for models whose backward kernels under-fill the SMs."""
    return 0


def run_backward_fusion(graph: Graph, policy: OptimizerPolicy, inp, workers: int = 1, *,
                        timing: bool = True, trace: bool = False,
                        bucket_elems: int = 0, update_ctas: int | None = None,
                        update_priority: str = "high", consumer=None) -> StepReport:
    """Eager schedule: update each layer as soon as its gradients are complete.

    ``workers=1`` issues each update inline on the autograd stream;
    ``workers>1`` on the engine's high-priority side stream behind an event
    (the device half of the Appendix B.2 guard), overlapping the backward of
    the preceding layers; ``update_ctas`` optionally caps each update's grid
    so it streams alongside the backward (default 0: uncapped).
    ``bucket_elems`` merges consecutive layers (backward order) into launch
    groups of at least that many elements.  ``update_priority`` ("high" |
    "low") is the side stream's priority: high mirrors the reference runner's
    step-first heap; low lets a GPU-bound backward keep the SMs and the
    updates fill the gaps.
    ``consumer`` (a consumer.ConsumerFusion of this graph and policy): its
    Linear weights are updated inside their weight-gradient GEMM (no gradient
    in memory, no separate launch); every other parameter as above.
    Raises GlobalInfoRequired, mutating nothing, for policies or transforms
    that must see all gradients first (schedule.py:174-177).
    """
    if policy.requires_global_info:
        raise GlobalInfoRequired(
            f"backward-fusion cannot host {policy.kind!r}"
            + (" with global-norm clipping" if policy.clip_norm is not None else ""))
    _reject_newton(policy)
    checkpoint.attach(graph, policy)
    if workers < 1:
        raise ConfigError(f"workers must be >= 1, got {workers}")
    if bucket_elems < 0:
        raise ConfigError(f"bucket_elems must be >= 0, got {bucket_elems}")
    if update_priority not in ("high", "low"):
        raise ConfigError(f"update_priority must be 'high' or 'low', got {update_priority!r}")
    if consumer is not None and (consumer.graph is not graph or consumer.policy is not policy):
        raise ConfigError("consumer fusion was built for another graph or policy")
    if consumer is not None and trace:
        raise ConfigError("schedule traces do not cover consumer-fused layers")
    _leave_forward_fusion(graph, policy)
    eng = _engine(graph, policy, workers > 1, bucket_elems,
                  update_priority if workers > 1 else "high",
                  consumer.id_set if consumer is not None else frozenset())
    policy.begin_iteration()
    if workers > 1 and update_ctas is None:
        update_ctas = default_update_ctas()
    eng.configure(policy, policy.t, None, update_ctas if workers > 1 else 0)
    tc = tr.ScheduleTrace(BACKWARD_FUSION) if trace else None
    marks = _Marks(timing)
    marks.mark()
    loss = graph.forward(inp, tc)
    marks.mark()
    native = eng.native
    _own_hooks(graph, eng)
    rec = None
    if tc is not None:
        rec = _TraceRecorder(graph, tc, eng.groups)
        native.set_callback(rec)
    native.bf_begin(True)
    if consumer is not None:
        consumer.active = True
    try:
        graph.backward(tc)
    finally:
        native.disarm()
        if consumer is not None:
            consumer.active = False
        if rec is not None:
            native.set_callback(None)
    native.bf_finish()
    if rec is not None:
        rec.finish()
    marks.mark()
    marks.mark()
    return StepReport(BACKWARD_FUSION, loss, tc, marks.events, fused=True)
