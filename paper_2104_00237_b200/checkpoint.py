"""Observation points and checkpoint / resume for fused training.

The reference has no serialization but fixes the semantics that
matter: under forward fusion the raw parameter values are stale until
``flush_pending_updates`` (schedule.py:141-160), and any observation -- eval,
``state_dict``, a checkpoint -- must flush first.  This module
makes that automatic:

* ``attach(graph, policy)`` (called by every schedule) remembers the policy
  and installs a ``state_dict`` pre-hook on the root module, so
  ``graph.module.state_dict()`` applies pending updates before reading;
* ``observe(graph)`` flushes and returns the number of updates applied (use
  it before eval or any host read of the weights);
* ``state_dict(graph, policy)`` / ``load_state_dict(graph, policy, sd)`` save
  and restore the full training state: module tensors, the policy constants
  and step counter, every history slot and (mixed precision) the fp32 master
  weights.  Resuming continues the trajectory bit for bit.

Backward fusion needs nothing extra: every schedule joins its update stream
into the compute stream before returning, so a read issued afterwards on the
compute stream sees the updated values.
"""

from __future__ import annotations

import torch

from .errors import ConfigError, StateError

_POLICY_FIELDS = ("kind", "eta", "alpha", "weight_decay", "epsilon", "beta1", "beta2", "rho",
                  "clip_norm", "t", "grad_reset")


def attach(graph, policy) -> None:
    """Remember ``policy`` as the one driving ``graph``; first call installs the
    flush-before-read hook on the root module."""
    graph._policy = policy
    if getattr(graph, "_sd_hook", None) is None:
        def pre_hook(module, prefix, keep_vars):
            observe(graph)
        graph._sd_hook = graph.module.register_state_dict_pre_hook(pre_hook)


def _num_pending(graph) -> int:
    owner = graph._flag_owner
    if owner is not None:
        return int(owner.num_pending())
    return sum(1 for p in graph.parameters if p.pending)


def observe(graph, policy=None) -> int:
    """Apply every deferred forward-fusion update (no-op otherwise)."""
    from .schedule import flush_pending_updates
    if _num_pending(graph) == 0:
        return 0
    policy = policy or getattr(graph, "_policy", None)
    if policy is None:
        raise StateError("pending updates but no policy attached to this graph")
    return flush_pending_updates(graph, policy)


def state_dict(graph, policy) -> dict:
    """Flush, then snapshot everything a resumed run needs (tensors cloned on
    their device; ``torch.save`` moves them as usual)."""
    observe(graph, policy)
    with torch.no_grad():
        hist = {p.name: {k: v.detach().clone() for k, v in p.history.items()}
                for p in graph.parameters if p.history}
        master = {p.name: p.master.detach().clone() for p in graph.parameters
                  if p.master is not None}
        return {"format": "optfuse-b200/1",
                "model": {k: v.detach().clone() for k, v in graph.module.state_dict().items()},
                "policy": {f: getattr(policy, f) for f in _POLICY_FIELDS},
                "history": hist, "master": master}


def load_state_dict(graph, policy, sd: dict) -> None:
    """Restore a snapshot taken by ``state_dict`` into a graph built the same
    way (same network, same ``use_master_weights`` choice) and a policy of the
    same kind.  Tensors are copied in place, so engines, tensor lists and
    CUDA graphs built on this graph stay valid."""
    if sd.get("format") != "optfuse-b200/1":
        raise ConfigError("not an optfuse-b200 checkpoint")
    if sd["policy"]["kind"] != policy.kind:
        raise ConfigError(f"checkpoint is for {sd['policy']['kind']!r}, policy is {policy.kind!r}")
    if _num_pending(graph):
        raise StateError("flush pending updates before loading a checkpoint")
    for f in _POLICY_FIELDS:
        setattr(policy, f, sd["policy"][f])
    graph.module.load_state_dict(sd["model"])
    by_name = {p.name: p for p in graph.parameters}
    if set(sd["master"]) != {p.name for p in graph.parameters if p.master is not None}:
        raise ConfigError("checkpoint and graph disagree on master weights")
    with torch.no_grad():
        for name, m in sd["master"].items():
            by_name[name].master.copy_(m)
        for name, slots in sd["history"].items():
            p = by_name[name]
            ref = p.master if p.master is not None else p.value
            for k, v in slots.items():
                if k not in p.history:
                    p.history[k] = torch.empty_like(ref, memory_format=torch.preserve_format)
                p.history[k].copy_(v)
    graph.pending_step_t = None
    graph.pending_scale = None
