"""Data-parallel fused optimizer: per-bucket gradient reduce-scatter, sharded
update, parameter all-gather.

The reference is single-process; the paper only claims DDP compatibility
(PAPER.md:1815-1818).  On B200 the update is element-wise and per-parameter,
so it shards naturally: rank r owns a contiguous 1/W slice of every bucket
(and only that slice of the optimizer history -- state memory / W).

Layout (per bucket = consecutive layers in backward order, ``launch_groups``):
  flat_param [padded]  -- the module's parameters become views into it, each
                          starting on a 128-byte boundary (gaps stay zero:
                          a zero gradient on a zero parameter updates to zero)
  flat_grad  [padded]  -- gradients copied in per bucket (one multi-tensor copy;
                          AccumulateGrad keeps stealing its input)
  grad_shard [S], history shards [S] per slot, S = padded / W (padded to W*4
  elements so every shard starts 16-byte aligned for the vector path)

Backward fusion: when the last gradient of a bucket is accumulated, the
bucket's pipeline is issued on the communication stream behind an event:
copy gradients in -> ``reduce_scatter_tensor(SUM)`` -> the multi-tensor update
kernel on the shard (1/W folded in as the device gradient scale) ->
``all_gather_into_tensor`` back into flat_param.  It overlaps the backward of
the remaining layers; the compute stream joins once at the end of backward.
Forward fusion: the reduce-scatter happens in backward, the update +
all-gather of each bucket are issued by its first layer's forward pre-hook,
with the next bucket prefetched on the communication stream.

``transport="peer"`` replaces the three steps by ONE kernel over NVLink peer
memory (``of_dp_step_peer``): flat_param and flat_grad live in torch symmetric
memory, so every rank can address every peer's buffers; the shard owner sums
its shard of the gradients over the peers, updates it, writes the result into
every peer's flat_param and zeroes the gradient shard it read, between two
cross-rank barriers.  No staging buffer, no reduce-scatter output, and the
all-gather traffic is issued by the same threads that computed the values.
Global-norm clipping on this transport: after a barrier, one kernel per bucket
(``of_dp_sqnorm_peer``) sums the squares of the peer-summed gradient shard in
f64 (the same rank-order sum the fused step uses), then the scalar is
all-reduced and the factor folded into the steps' gradient scale, as on the
NCCL transport.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _native as nat
from . import kernels
from .engine import launch_groups
from .errors import ConfigError, GlobalInfoRequired, StateError

DEFAULT_BUCKET_ELEMS = 1 << 22  # 16 MiB of fp32 per bucket
TRANSPORTS = ("nccl", "peer")


class _Bucket:
    __slots__ = ("index", "params", "offsets", "flat_param", "flat_grad", "grad_shard", "slots",
                 "shard", "master", "tl", "peer", "hparam", "hgrad", "sq_tl", "grad_views", "gathered",
                 "ready",
                 "event", "done", "leader", "pending")

    def __init__(self, index):
        self.index = index


class DataParallelFusion:
    """Sharded fused optimizer of one Graph across a process group."""

    def __init__(self, graph, policy, *, group=None, bucket_elems: int = DEFAULT_BUCKET_ELEMS,
                 update_fn=None, transport: str = "nccl"):
        if not dist.is_initialized():
            raise StateError("torch.distributed is not initialised")
        if policy.kind == "newton":
            raise ConfigError("newton has no per-parameter step")
        if transport not in TRANSPORTS:
            raise ConfigError(f"transport must be one of {TRANSPORTS}, got {transport!r}")
        if transport == "peer" and (update_fn is not None or graph.device.type != "cuda"):
            raise ConfigError("the peer transport runs the fused CUDA kernel over symmetric memory")
        self.transport = transport
        self.graph = graph
        self.policy = policy
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.update_fn = update_fn
        self.device = graph.device
        self.cuda = self.device.type == "cuda"
        if self.cuda and update_fn is None:
            kernels.sqnorm_workspace_len()  # the kernel library must load (no fallback)
        elif update_fn is None:
            raise ConfigError("the sharded update runs on CUDA; pass update_fn only for host tests")
        self.comm = torch.cuda.Stream() if self.cuda else None
        self._sync = None
        self.barrier_timeout_ms = 0   # peer transport: 0 = wait indefinitely
        slots = policy.history_slots()
        # mixed precision (C4): the module runs in bf16 with fp32 masters
        # (Graph.use_master_weights).  Gradients are reduce-scattered in bf16;
        # rank r keeps the fp32 master and history of its shard only; the
        # kernel writes the updated bf16 parameters straight into the shard of
        # flat_param (OF_FLAG_SHADOW_BF16) and only bf16 is all-gathered.
        self.mixed = bool(getattr(graph, "master_weights", False))
        self.flags = nat.OF_FLAG_SHADOW_BF16 if self.mixed else 0
        src = dist.get_global_rank(group, 0) if group else 0
        unit = self.world * 4
        self.buckets = []
        for bi, ids in enumerate(launch_groups(graph, bucket_elems)):
            b = _Bucket(bi)
            b.params = [graph.parameters[i] for i in ids]
            dt = b.params[0].value.dtype
            if any(p.value.dtype != dt for p in b.params):
                raise ConfigError("a data-parallel bucket needs one dtype")
            if self.mixed and any(p.master is None for p in b.params):
                raise ConfigError("master weights: every parameter needs an fp32 master")
            mdt = torch.float32 if self.mixed else dt
            # every parameter starts on a 128-byte boundary of the flat buffers:
            # cuDNN/cuBLAS pick their kernels (and so their rounding) by operand
            # alignment, and a view at an odd bf16 offset would change both
            align = max(1, 128 // torch.empty((), dtype=dt).element_size())
            b.offsets = []
            n = 0
            for p in b.params:
                b.offsets.append(n)
                n += -(-p.value.numel() // align) * align
            padded = -(-n // unit) * unit
            S = padded // self.world
            if transport == "peer":   # symmetric buffers, mapped into every peer
                b.flat_param, b.hparam = self._symmetric(padded, dt)
                b.flat_grad, b.hgrad = self._symmetric(padded, dt)
            else:
                b.flat_param = torch.zeros(padded, dtype=dt, device=self.device)
                b.flat_grad = torch.zeros(padded, dtype=dt, device=self.device)
            flat_master = torch.zeros(padded, dtype=mdt, device=self.device) if self.mixed else None
            with torch.no_grad():
                for p, off in zip(b.params, b.offsets):
                    v = p.value
                    if not _dense(v):
                        raise ConfigError(f"parameter {p.id} must be dense (contiguous or "
                                          "channels-last) for data parallel")
                    # views with the parameter's own strides: a channels-last
                    # weight keeps its memory layout inside the flat buffer
                    pv = torch.as_strided(b.flat_param, v.size(), v.stride(), off)
                    pv.copy_(v)
                    if self.mixed:
                        torch.as_strided(flat_master, v.size(), v.stride(), off).copy_(p.master)
                    v.data = pv
                    v.grad = None
            # where each parameter's gradient lands in flat_grad (same strides)
            b.grad_views = [torch.as_strided(b.flat_grad, p.value.size(), p.value.stride(), off)
                            for p, off in zip(b.params, b.offsets)]
            if self.mixed:
                dist.broadcast(flat_master, src=src, group=group)
                with torch.no_grad():
                    b.flat_param.copy_(flat_master)
            else:
                dist.broadcast(b.flat_param, src=src, group=group)
            b.shard = slice(self.rank * S, (self.rank + 1) * S)
            # (the peer transport reads the shard straight from every peer's
            # flat_grad: no reduce-scatter destination)
            b.grad_shard = torch.zeros(S if transport == "nccl" else 0, dtype=dt, device=self.device)
            b.slots = {name: torch.zeros(S, dtype=mdt, device=self.device) for name in slots}
            # the owned fp32 master shard (state memory / W); the full-size
            # per-parameter masters are released: a non-DP schedule on this
            # graph now fails loudly instead of updating stale masters
            b.master = flat_master[b.shard].clone() if self.mixed else None
            del flat_master
            if self.cuda:
                tl = kernels.TensorList(1)
                pv = b.flat_param[b.shard]
                if self.mixed:
                    tl.set(0, b.master, b.grad_shard, b.slots[slots[0]] if slots else None,
                           b.slots[slots[1]] if len(slots) > 1 else None, pv)
                else:
                    tl.set(0, pv, b.grad_shard, b.slots[slots[0]] if slots else None,
                           b.slots[slots[1]] if len(slots) > 1 else None)
                tl.set_dtypes(mdt, dt)
                b.tl = tl
                if transport == "peer":
                    sl = [b.slots[k] for k in slots] + [None, None]
                    b.peer = kernels.PeerBucket(
                        self.world, self.rank, dt, dt, b.hgrad.buffer_ptrs, b.hparam.buffer_ptrs,
                        b.master, sl[0], sl[1], b.shard.start, S)
                b.event = torch.cuda.Event()
                b.done = torch.cuda.Event()
            b.ready = 0
            b.pending = False
            b.gathered = False
            self.buckets.append(b)
        if self.mixed:
            for p in graph.parameters:
                p.master = None
        # single-device engines hold the parameters' old storage: drop them
        graph._engines.clear()
        self.bucket_of = {p.id: b for b in self.buckets for p in b.params}
        self.scale = None
        if self.cuda:
            self.scale = torch.full((), 1.0 / self.world, dtype=torch.float32, device=self.device)
        # global-norm clipping (baseline / forward fusion; backward fusion
        # rejects it): factor of the averaged gradient, folded with 1/W into
        # the sharded updates' device gradient scale
        self._clip_gscale = None
        self._host_factor = None
        if policy.clip_norm is not None and self.cuda:
            dev = self.device
            self._sq = torch.zeros((), dtype=torch.float64, device=dev)
            self._factor = torch.zeros((), dtype=torch.float64, device=dev)
            self._coef = torch.zeros((), dtype=torch.float32, device=dev)
            self._clip_gscale = torch.zeros((), dtype=torch.float32, device=dev)
            self._ws = torch.empty(kernels.sqnorm_workspace_len(), dtype=torch.float64, device=dev)
            for b in self.buckets:
                if transport == "peer":   # of_dp_sqnorm_peer reads the shard from every peer
                    continue
                tl = kernels.TensorList(1)
                tl.set(0, None, b.grad_shard)
                tl.set_dtypes(torch.float32 if self.mixed else b.grad_shard.dtype, b.grad_shard.dtype)
                b.sq_tl = tl
        self._hooks = None
        self._mode = None
        self._leader_handles = None
        self.join_event = torch.cuda.Event() if self.cuda else None

    @property
    def _pending_t(self):
        """Step index frozen when forward fusion deferred the updates
        (schedule.py:133); kept on the Graph, where a CUDA-graph replay
        (CapturedStep) advances it."""
        return self.graph.pending_step_t

    @_pending_t.setter
    def _pending_t(self, t) -> None:
        self.graph.pending_step_t = t

    def _symmetric(self, n: int, dt):
        """A zeroed flat buffer in torch symmetric memory and its handle (the
        peers' mappings of it: ``buffer_ptrs``; cross-rank ``barrier``)."""
        import torch.distributed._symmetric_memory as symm_mem
        t = symm_mem.empty(n, dtype=dt, device=self.device)
        t.zero_()
        grp = self.group if self.group is not None else dist.group.WORLD
        h = symm_mem.rendezvous(t, grp)
        if self._sync is None:
            self._sync = h
        return t, h

    # -- global-norm clipping ---------------------------------

    def _clip(self) -> None:
        """After every bucket's reduce-scatter: Σ g² over this rank's summed
        gradient shards (f64, fixed order), one all-reduce of that scalar, the
        norm of the averaged gradient sqrt(total) / W and the clip factor of
        optim.py:165-168; the update kernels then multiply their summed
        gradient by f32(factor) * (1/W)."""
        W = self.world
        if not self.cuda:   # host stand-in (gloo tests): same quantities in torch
            total = torch.zeros((), dtype=torch.float64)
            for b in self.buckets:
                g = b.grad_shard.double()
                total += (g * g).sum()
            dist.all_reduce(total, group=self.group)
            norm = float(total.sqrt()) / W
            mx = self.policy.clip_norm
            self._host_factor = 1.0 if norm <= mx else mx / norm
            return
        if self.transport == "peer":
            # on the communication stream, like the peer steps (barrier order):
            # barrier (every rank's gradients complete), then Σ over this rank's
            # shard of the peer-summed gradient squared -- the same rank-order
            # sum the fused step will use -- then the same all-reduce and factor
            cur = torch.cuda.current_stream()
            on_comm = cur == self.comm
            if not on_comm:
                self.comm.wait_stream(cur)
            with torch.cuda.stream(self.comm):
                self._sync.barrier(channel=0, timeout_ms=self.barrier_timeout_ms)
                for i, b in enumerate(self.buckets):
                    kernels.dp_sqnorm_peer(b.peer, self._ws, self._sq, i > 0, None)
                self._finish_clip()
            if not on_comm:
                cur.wait_stream(self.comm)
            return
        for i, b in enumerate(self.buckets):
            kernels.sqnorm(b.sq_tl, self._ws, self._sq, i > 0, None)
        self._finish_clip()

    def _finish_clip(self) -> None:
        W = self.world
        dist.all_reduce(self._sq, group=self.group)
        self._sq.div_(float(W * W))
        kernels.clip_coef(self._sq, self.policy.clip_norm, self._coef, self._factor, None)
        torch.mul(self._coef, 1.0 / W, out=self._clip_gscale)

    def _gscale(self):
        return self._clip_gscale if self._clip_gscale is not None else self.scale

    # -- the per-bucket pipeline ----------------------------------------------

    def _gather_grads(self, b) -> None:
        if b.gathered:
            b.gathered = False
            return
        self._gather_grads_host(b)

    def _gather_grads_host(self, b) -> None:
        """Copy the bucket's gradients into flat_grad with one multi-tensor copy
        and release them.  AccumulateGrad steals each incoming gradient
        (``p.grad`` is None), where persistent views into flat_grad would cost
        one add kernel per parameter per step (+0.3 ms on MobileNetV2 in a
        CUDA graph).  Alignment gaps and padding are never written: zero."""
        dst, src = [], []
        for p, view in zip(b.params, b.grad_views):
            g = p.value.grad
            if g is None:          # no contribution this iteration: the reference steps with 0
                view.zero_()
                continue
            dst.append(view)
            src.append(g)
        if src:
            if self.cuda:   # one multi-tensor copy kernel (a gradient in another layout: copy_)
                ok = [kernels.same_layout(d, s) for d, s in zip(dst, src)]
                for d, s, k in zip(dst, src, ok):
                    if not k:
                        d.copy_(s)
                pd = [d for d, k in zip(dst, ok) if k]
                if pd:
                    ps = [s for s, k in zip(src, ok) if k]
                    kernels.copy_mt(kernels.CopyList(pd, ps, checked=True))
            else:
                torch._foreach_copy_(dst, src)
        for p, g in zip(b.params, [p.value.grad for p in b.params]):
            if g is not None and self.cuda:
                g.record_stream(torch.cuda.current_stream())   # freed after this stream's copy
            p.value.grad = None

    def _reduce_scatter(self, b) -> None:
        self._gather_grads(b)
        if self.transport == "peer":
            return   # the fused kernel reads every peer's gradients in place
        dist.reduce_scatter_tensor(b.grad_shard, b.flat_grad, op=dist.ReduceOp.SUM, group=self.group)

    def _update_and_gather(self, b, t: int) -> None:
        if self.transport == "peer":
            # barrier: every rank's gradients of this bucket are complete; one
            # kernel sums the shard over the peers, updates it and writes it
            # to every peer; barrier: those writes (and the gradient zeroing)
            # landed before any rank reads parameters or accumulates again
            # All of them go on the communication stream, whatever stream the
            # caller is on: the barriers of one rank then run in host issue
            # order, which is the same on every rank.
            cur = torch.cuda.current_stream()
            on_comm = cur == self.comm
            if not on_comm:
                self.comm.wait_stream(cur)
            with torch.cuda.stream(self.comm):
                self._sync.barrier(channel=0, timeout_ms=self.barrier_timeout_ms)
                kernels.dp_step_peer(b.peer, self.policy._hparams(t), self._gscale(),
                                     self.policy.device_step_flag, None)
                self._sync.barrier(channel=0, timeout_ms=self.barrier_timeout_ms)
            if not on_comm:
                cur.wait_stream(self.comm)
            return
        if self.update_fn is not None:
            if self.mixed:    # host stand-in: fp32 grad shard, master updated, bf16 written back
                g = b.grad_shard.float().mul_(1.0 / self.world)
                if self._host_factor is not None:
                    g.mul_(self._host_factor)
                self.update_fn(b.master, g, b.slots, t)
                with torch.no_grad():
                    b.flat_param[b.shard].copy_(b.master)
            else:
                b.grad_shard.mul_(1.0 / self.world)
                if self._host_factor is not None:
                    b.grad_shard.mul_(self._host_factor)
                self.update_fn(b.flat_param[b.shard], b.grad_shard, b.slots, t)
        else:
            kernels.policy_step(b.tl, self.policy._hparams(t), self._gscale(),
                                self.flags | self.policy.device_step_flag, None)
        dist.all_gather_into_tensor(b.flat_param, b.flat_param[b.shard], group=self.group)

    def _on_stream(self, stream):
        return torch.cuda.stream(stream) if stream is not None else _NullCtx()

    # -- hooks -------------------------------------------------------------------

    def _install(self) -> None:
        if self._hooks is not None:
            return
        if self.cuda:
            # the native engine's C++ gradient-ready hooks count readiness per
            # bucket and call back into Python once per bucket (not once per
            # parameter); no launches of its own
            from .engine import native_engine_module
            g = self.graph
            eng = native_engine_module().Engine(
                [p.value for p in g.parameters], [[p.id for p in b.params] for b in self.buckets],
                [[p.id for p in L.params] for L in g.layers], self.comm.cuda_stream)
            # the engine gathers each completed bucket's gradients into flat_grad
            # on the communication stream (one of_copy_mt), then calls back
            for gi, b in enumerate(self.buckets):
                eng.set_group_views(gi, b.grad_views)
            eng.set_group_callback(self._on_bucket_ready)
            eng.install_hooks()
            g._hook_owner = eng
            self._eng = eng
            self._hooks = [eng]
            return
        hooks = []
        for p in self.graph.parameters:
            hooks.append(p.value.register_post_accumulate_grad_hook(
                lambda t, p=p: self._on_grad_ready(p)))
        self._hooks = hooks

    def _on_bucket_ready(self, gi: int) -> None:
        b = self.buckets[gi]
        if self._mode is None:
            return
        b.ready = len(b.params)
        b.gathered = True       # the engine already copied the gradients into flat_grad
        self._bucket_ready(b)

    def _backward(self) -> None:
        eng = getattr(self, "_eng", None)
        if eng is not None:
            eng.bf_begin(False)
        try:
            self.graph.backward()
        finally:
            if eng is not None:
                eng.disarm()

    def _on_grad_ready(self, p) -> None:
        b = self.bucket_of.get(p.id)
        if b is None or self._mode is None:
            return
        b.ready += 1
        if b.ready == len(b.params):
            self._bucket_ready(b)

    def _bucket_ready(self, b) -> None:
        cur = torch.cuda.current_stream() if self.cuda else None
        if self.cuda:
            b.event.record(cur)
            self.comm.wait_event(b.event)
        with self._on_stream(self.comm):
            self._reduce_scatter(b)
            if self._mode == "backward-fusion":
                self._update_and_gather(b, self.policy.t)
            else:
                b.pending = True
            if self.cuda:
                b.done.record(self.comm)

    def _finish_backward(self) -> None:
        for b in self.buckets:
            if b.ready < len(b.params):  # parameters without gradients this iteration
                self._bucket_ready(b)
        if self.policy.clip_norm is not None:   # forward fusion: the deferred updates need it
            with self._on_stream(self.comm):
                self._clip()
        if self.cuda:
            self.join_event.record(self.comm)
            torch.cuda.current_stream().wait_event(self.join_event)
        for b in self.buckets:
            b.ready = 0

    # -- schedules -----------------------------------------------------------------

    def run_backward_fusion(self, inp, *, timing: bool = False):
        """Forward, then backward with each bucket's RS -> update -> AG issued
        as soon as the bucket's gradients are complete."""
        from .schedule import StepReport
        pol = self.policy
        if pol.requires_global_info:
            raise GlobalInfoRequired("backward-fusion cannot host a global-information policy")
        self._install()
        self._apply_deferred()
        pol.begin_iteration()
        loss = self.graph.forward(inp)
        self._mode = "backward-fusion"
        self._backward()
        self._finish_backward()
        self._mode = None
        return StepReport("backward-fusion", loss, None, fused=True)

    def run_baseline(self, inp, *, timing: bool = False):
        """Unfused data parallel: full forward, full backward, then per bucket
        RS -> update -> AG on the compute stream."""
        from .schedule import StepReport
        self._apply_deferred()
        self.policy.begin_iteration()
        loss = self.graph.forward(inp)
        self.graph.backward()
        if self.policy.clip_norm is not None:   # global information: every shard first
            for b in reversed(self.buckets):
                self._reduce_scatter(b)
            self._clip()
            for b in reversed(self.buckets):
                self._update_and_gather(b, self.policy.t)
        else:
            for b in reversed(self.buckets):
                self._reduce_scatter(b)
                self._update_and_gather(b, self.policy.t)
        return StepReport("baseline", loss, None)

    def run_forward_fusion(self, inp, *, timing: bool = False):
        """RS during backward; update + AG deferred to each bucket's first layer
        in the next forward (next bucket prefetched on the comm stream)."""
        from .schedule import StepReport
        self._install()
        record = self._leader_handles is None and self.graph.exec_order is None
        if record:
            # leaders must be the first EXECUTED layer of each bucket (module
            # registration order can differ): record the order in this forward,
            # which has no deferred bucket to apply yet, and place them after it
            self._apply_deferred()
        else:
            self._install_leaders()
        self.policy.begin_iteration()
        if record:
            loss = self._forward_recording(inp)
            self._install_leaders()
        else:
            loss = self.graph.forward(inp)
        self._apply_deferred()          # buckets whose leader did not run
        self._mode = "forward-fusion"
        self._backward()
        self._finish_backward()
        self._mode = None
        self._pending_t = self.policy.t
        return StepReport("forward-fusion", loss, None, fused=True,
                          pending_updates=sum(len(b.params) for b in self.buckets if b.pending))

    def _forward_recording(self, inp):
        """Forward pass that records the layers' first-execution order into
        ``graph.exec_order`` (temporary pre-hooks on every layer)."""
        order, seen = [], set()

        def note(i):
            if i not in seen:
                seen.add(i)
                order.append(i)
        hs = [L.module.register_forward_pre_hook(lambda m, a, i=L.index: note(i))
              for L in self.graph.layers]
        try:
            loss = self.graph.forward(inp)
        finally:
            for h in hs:
                h.remove()
        self.graph.exec_order = order
        return loss

    def _install_leaders(self) -> None:
        if self._leader_handles is not None:
            return
        order = self.graph.exec_order or [L.index for L in self.graph.layers]
        pos = {li: k for k, li in enumerate(order)}
        fwd = []
        for b in self.buckets:
            first = min((pos.get(L.index, len(pos)) for p in b.params for L in p.layers))
            fwd.append((first, b))
        fwd.sort(key=lambda x: x[0])
        self._fwd_buckets = [b for _, b in fwd]
        handles = []
        for k, (first, b) in enumerate(fwd):
            if first >= len(order):
                continue
            layer = self.graph.layers[order[first]]
            handles.append(layer.module.register_forward_pre_hook(
                lambda m, a, k=k: self._leader(k)))
        self._leader_handles = handles

    def _leader(self, k: int):
        bs = self._fwd_buckets
        b = bs[k]
        t = self._pending_t
        # a bucket made pending by the previous backward needs no wait: that
        # backward ended with the compute stream joining the communication
        # stream (and an event recorded then may predate a CUDA-graph capture)
        if b.pending:
            self._issue_deferred(b, t, None)
        elif self.cuda:   # prefetched on the communication stream in this forward
            torch.cuda.current_stream().wait_event(b.done)
        if k + 1 < len(bs) and bs[k + 1].pending:   # prefetch the next bucket
            nb = bs[k + 1]
            self.comm.wait_stream(torch.cuda.current_stream()) if self.cuda else None
            self._issue_deferred(nb, t, self.comm)
        return None

    def _issue_deferred(self, b, t, stream) -> None:
        with self._on_stream(stream):
            self._update_and_gather(b, t)
            b.pending = False
            if self.cuda:
                b.done.record(torch.cuda.current_stream())

    def _apply_deferred(self) -> None:
        t = self._pending_t
        for b in self.buckets:
            if b.pending:   # (ordered after its reduce-scatter by the backward's join)
                self._update_and_gather(b, t)
                b.pending = False

    def flush(self) -> int:
        """Apply every deferred bucket update now (host-side observation point)."""
        n = sum(len(b.params) for b in self.buckets if b.pending)
        self._apply_deferred()
        if n:
            self.graph.flush_gen += 1
        return n

    # -- checkpoint / resume ---------------------------------------------------

    def state_dict(self) -> dict:
        """This rank's training state: pending updates applied first, then the
        module tensors (identical on every rank after the all-gather), the
        policy and, per bucket, the history (and fp32 master) of the shard this
        rank owns.  Each rank saves its own; resume with the same world size
        and buckets."""
        from .checkpoint import _POLICY_FIELDS
        self.flush()
        with torch.no_grad():
            return {"format": "optfuse-b200-dp/1", "world": self.world, "rank": self.rank,
                    "buckets": [{"shard": (b.shard.start, b.shard.stop),
                                 "slots": {k: v.detach().clone() for k, v in b.slots.items()},
                                 "master": b.master.detach().clone() if b.master is not None else None}
                                for b in self.buckets],
                    "model": {k: v.detach().clone() for k, v in self.graph.module.state_dict().items()},
                    "policy": {f: getattr(self.policy, f) for f in _POLICY_FIELDS},
                    "pending_t": self._pending_t}

    def load_state_dict(self, sd: dict) -> None:
        from .checkpoint import _POLICY_FIELDS
        if sd.get("format") != "optfuse-b200-dp/1":
            raise ConfigError("not an optfuse-b200 data-parallel checkpoint")
        if sd["world"] != self.world or sd["rank"] != self.rank:
            raise ConfigError(f"checkpoint of rank {sd['rank']}/{sd['world']}, this is "
                              f"{self.rank}/{self.world}")
        if len(sd["buckets"]) != len(self.buckets) or any(
                tuple(bs["shard"]) != (b.shard.start, b.shard.stop)
                for bs, b in zip(sd["buckets"], self.buckets)):
            raise ConfigError("checkpoint buckets differ from this model's")
        if sd["policy"]["kind"] != self.policy.kind:
            raise ConfigError(f"checkpoint is for {sd['policy']['kind']!r}, policy is {self.policy.kind!r}")
        if any(b.pending for b in self.buckets):
            raise StateError("flush pending updates before loading a checkpoint")
        for f in _POLICY_FIELDS:
            setattr(self.policy, f, sd["policy"][f])
        with torch.no_grad():
            # module tensors land in the flat buffers the parameters view
            self.graph.module.load_state_dict(sd["model"])
            for bs, b in zip(sd["buckets"], self.buckets):
                for k, v in bs["slots"].items():
                    b.slots[k].copy_(v)
                if b.master is not None:
                    b.master.copy_(bs["master"])
        self._pending_t = sd.get("pending_t")


def _dense(t) -> bool:
    """Non-overlapping and dense: the elements fill [0, numel) of its storage
    span in some stride order (contiguous, channels-last, ...)."""
    return kernels.is_dense(t)


class _NullCtx:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False
