"""Generate the golden fixtures by running the REFERENCE implementation.

    PYTHONDONTWRITEBYTECODE=1 OPTFUSE_REF=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Imports the unmodified reference package (`optfuse`, read-only under
/root/reference) and records, as small .npz/.json fixtures in this directory:

* policy_steps.npz -- OptimizerPolicy.step (optim.py:74-148) trajectories for the
  six local kinds x {f32, f64} x {no decay, coupled decay}, with injected grads;
* spec_kats.json   -- the SPEC.md known-answer examples (SPEC.md:213-215, 233-235,
  287/307) evaluated by the reference;
* trajectories.npz -- verify-grid cells (bench.py:241-273: 10 iterations, batch 2,
  eta 0.01) for every kind x {chain(3,4), shared-chain(4,4), mul-probe(3)} x
  {f32, f64}, seed 0, under baseline / forward-fusion(+flush) / backward-fusion,
  plus 100-iteration chain(8,32) f32 runs (sgd-momentum with decay, adam eta=1e-4)
  and clip runs (baseline+clip vs forward-fusion+clip, f32; baseline+clip, f64);
* traces.json      -- schedule traces (trace.py:102-112 export format) and
  critical-path depths (locality.py:92-100) for chain(n) baseline / BF.

The GPU box never runs this script (no /root/reference there); it only reads
the committed fixtures.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("OPTFUSE_REF", "/root/reference/pkg/src")
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import optfuse  # noqa: E402
from optfuse import bench as rbench  # noqa: E402
from optfuse.graph import Parameter  # noqa: E402
from optfuse.tensor import Tensor  # noqa: E402

OUT = Path(__file__).resolve().parent
KINDS = ("sgd", "sgd-momentum", "adagrad", "rmsprop", "adadelta", "adam")
ETA = {"sgd": 0.01, "sgd-momentum": 0.01, "adagrad": 0.01, "rmsprop": 1e-3,
       "adadelta": 1.0, "adam": 1e-3}


def policy_steps() -> None:
    rng = np.random.default_rng(20210401)
    n, steps = 263, 8
    arrays = {}
    for prec, dt in (("f32", np.float32), ("f64", np.float64)):
        for wd in (0.0, 1e-2):
            for kind in KINDS:
                key = f"{kind}|{prec}|wd{wd}"
                theta0 = rng.uniform(-1, 1, n).astype(dt)
                grads = (rng.standard_normal((steps, n)) * 0.1).astype(dt)
                grads[:, :7] = 0  # exact-zero gradients exercise eps paths
                p = Parameter(0, Tensor((n,), theta0.copy()))
                pol = optfuse.OptimizerPolicy(kind=kind, eta=ETA[kind], weight_decay=wd)
                traj = []
                for s in range(steps):
                    pol.begin_iteration()
                    p.grad.data[:] = grads[s]
                    pol.step(p)
                    assert not p.grad.data.any()
                    traj.append(p.value.data.copy())
                arrays[key + "|theta0"] = theta0
                arrays[key + "|grads"] = grads
                arrays[key + "|traj"] = np.stack(traj)
                for name in pol.history_slots():
                    arrays[key + "|slot|" + name] = p.history[name].data.copy()
    np.savez_compressed(OUT / "policy_steps.npz", **arrays)


def spec_kats() -> dict:
    out = {}
    # SPEC.md:213 sgd eta=0.1 theta=1 grad=2 -> 0.8, grad reset
    p = Parameter(0, optfuse.from_list([1.0]))
    p.grad = optfuse.from_list([2.0])
    pol = optfuse.OptimizerPolicy("sgd", eta=0.1)
    pol.begin_iteration()
    pol.step(p)
    out["sgd"] = {"theta": p.value.data.tolist(), "grad": p.grad.data.tolist()}
    # SPEC.md:214 momentum on theta^2/2 (grad = theta), eta 0.1 alpha 0.9
    p = Parameter(0, optfuse.from_list([1.0]))
    pol = optfuse.OptimizerPolicy("sgd-momentum", eta=0.1, alpha=0.9)
    thetas, bufs = [], []
    for _ in range(2):
        pol.begin_iteration()
        p.grad.data[:] = p.value.data
        pol.step(p)
        thetas.append(float(p.value.data[0]))
        bufs.append(float(p.history["momentum"].data[0]))
    out["sgd_momentum"] = {"theta": thetas, "momentum": bufs}
    # SPEC.md:215 decay-only sgd
    p = Parameter(0, optfuse.from_list([1.0]))
    pol = optfuse.OptimizerPolicy("sgd", eta=1.0, weight_decay=0.1)
    pol.begin_iteration()
    pol.step(p)
    out["weight_decay"] = {"theta": p.value.data.tolist()}
    # SPEC.md:233-235 clip
    clip = {}
    for max_norm in (10.0, 1.0):
        g = optfuse.build_model("mul-probe", width=1)
        q = optfuse.build_model("mul-probe", width=1)
        g.parameters = [g.parameters[0], q.parameters[0]]
        g.parameters[0].grad = optfuse.from_list([3.0])
        g.parameters[1].grad = optfuse.from_list([4.0])
        factor = optfuse.clip_by_global_norm(g, max_norm)
        clip[str(max_norm)] = {"factor": factor,
                               "grads": [float(x.grad.data[0]) for x in g.parameters]}
    g = optfuse.build_model("mul-probe", width=2)
    clip["zero"] = {"factor": optfuse.clip_by_global_norm(g, 1.0)}
    out["clip"] = clip
    # SPEC.md:287/307, acceptance #2: the Appendix B.2 race oracle
    race = {}
    for sched in ("baseline", "backward-fusion"):
        g = optfuse.build_model("mul-probe", width=1, init_range=(2.0, 2.0))
        pol = optfuse.OptimizerPolicy("sgd", eta=0.1)
        inp = optfuse.from_list([3.0])
        run = optfuse.run_baseline if sched == "baseline" else optfuse.run_backward_fusion
        rep = run(g, pol, inp)
        race[sched] = {"loss": rep.loss, "theta": float(g.parameters[0].value.data[0]),
                       "input_grad": float(g.input_grad.data[0])}
    out["race"] = race
    with open(OUT / "spec_kats.json", "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    return out


MODELS = (("chain", {"layers": 3, "width": 4}),
          ("shared-chain", {"layers": 4, "width": 4}),
          ("mul-probe", {"width": 3}))


def _run(model, kw, prec, seed, kind, sched, inputs, eta=0.01, wd=0.0, clip=None, flush=True):
    g = optfuse.build_model(model, **kw, seed=seed, precision=prec)
    pol = optfuse.OptimizerPolicy(kind=kind, eta=eta, weight_decay=wd, clip_norm=clip)
    losses, input_grads = [], []
    for inp in inputs:
        if sched == "baseline":
            rep = optfuse.run_baseline(g, pol, inp)
        elif sched == "forward-fusion":
            rep = optfuse.run_forward_fusion(g, pol, inp)
        else:
            rep = optfuse.run_backward_fusion(g, pol, inp)
        losses.append(rep.loss)
        input_grads.append(g.input_grad.data.copy())
    stale = [p.value.data.copy() for p in g.parameters]
    if sched == "forward-fusion" and flush:
        assert optfuse.flush_pending_updates(g, pol) == len(g.parameters)
        assert optfuse.flush_pending_updates(g, pol) == 0
    params = [p.value.data.copy() for p in g.parameters]
    return np.array(losses), params, stale, np.stack(input_grads)


def trajectories() -> None:
    arrays = {}
    for kind in KINDS:
        for model, kw in MODELS:
            for prec in ("f32", "f64"):
                seed = 0
                g0 = optfuse.build_model(model, **kw, seed=seed, precision=prec)
                inputs = rbench._iteration_inputs(g0, 2, seed, 10)
                key = f"cell|{kind}|{model}|{prec}"
                arrays[key + "|inputs"] = np.stack([i.data for i in inputs])
                arrays[key + "|init"] = np.concatenate([p.value.data for p in g0.parameters])
                for sched in ("baseline", "forward-fusion", "backward-fusion"):
                    losses, params, stale, ig = _run(model, kw, prec, seed, kind, sched, inputs)
                    arrays[f"{key}|{sched}|losses"] = losses
                    arrays[f"{key}|{sched}|params"] = np.concatenate(params)
                    arrays[f"{key}|{sched}|input_grads"] = ig
                    if sched == "forward-fusion":
                        arrays[f"{key}|{sched}|stale"] = np.concatenate(stale)
    # 100 fp32 iterations (the north-star parity length)
    for kind, eta, wd in (("sgd-momentum", 0.01, 5e-4), ("adam", 1e-4, 0.0)):
        g0 = optfuse.build_model("chain", layers=8, width=32, seed=0, precision="f32")
        inputs = rbench._iteration_inputs(g0, 32, 0, 100)
        key = f"long|{kind}"
        for sched in ("baseline", "forward-fusion", "backward-fusion"):
            losses, params, _, _ = _run("chain", {"layers": 8, "width": 32}, "f32", 0, kind,
                                        sched, inputs, eta=eta, wd=wd)
            arrays[f"{key}|{sched}|losses"] = losses
            arrays[f"{key}|{sched}|params"] = np.concatenate(params)
        arrays[f"{key}|hp"] = np.array([eta, wd])
    # global-norm clip: baseline+clip == forward-fusion+clip (acceptance #8)
    for kind in ("sgd-momentum", "adam"):
        g0 = optfuse.build_model("chain", layers=3, width=4, seed=0, precision="f32")
        inputs = rbench._iteration_inputs(g0, 2, 0, 10)
        for sched in ("baseline", "forward-fusion"):
            losses, params, _, _ = _run("chain", {"layers": 3, "width": 4}, "f32", 0, kind,
                                        sched, inputs, clip=0.05)
            arrays[f"clip|{kind}|{sched}|losses"] = losses
            arrays[f"clip|{kind}|{sched}|params"] = np.concatenate(params)
    # the same in f64: numpy scales f64 gradients by the double factor itself
    for kind in ("sgd-momentum", "adam"):
        g0 = optfuse.build_model("chain", layers=3, width=4, seed=0, precision="f64")
        inputs = rbench._iteration_inputs(g0, 2, 0, 10)
        losses, params, _, _ = _run("chain", {"layers": 3, "width": 4}, "f64", 0, kind,
                                    "baseline", inputs, clip=0.05)
        arrays[f"clip64|{kind}|baseline|losses"] = losses
        arrays[f"clip64|{kind}|baseline|params"] = np.concatenate(params)
    np.savez_compressed(OUT / "trajectories.npz", **arrays)


def traces() -> None:
    out = {"depth": {}, "lines": {}}
    for n in range(1, 33):
        row = {}
        for sched in ("baseline", "backward-fusion"):
            g = optfuse.build_model("chain", layers=n, width=2, seed=0)
            pol = optfuse.OptimizerPolicy("sgd", eta=0.01)
            inp = optfuse.uniform((1, 2), 0.1, 1.0, 0)
            run = optfuse.run_baseline if sched == "baseline" else optfuse.run_backward_fusion
            rep = run(g, pol, inp)
            row[sched] = optfuse.critical_path_depth(rep.trace)
        out["depth"][str(n)] = row
    for sched in ("baseline", "forward-fusion", "backward-fusion"):
        g = optfuse.build_model("chain", layers=3, width=4, seed=0)
        pol = optfuse.OptimizerPolicy("sgd-momentum", eta=0.01)
        inp = optfuse.uniform((2, 4), 0.1, 1.0, 0)
        run = {"baseline": optfuse.run_baseline, "forward-fusion": optfuse.run_forward_fusion,
               "backward-fusion": optfuse.run_backward_fusion}[sched]
        run(g, pol, inp)
        rep = run(g, pol, inp)  # steady state (FF has pending updates)
        out["lines"][sched] = [ln for ln in rep.trace.export_lines() if ln.startswith("task")]
    with open(OUT / "traces.json", "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def main() -> None:
    policy_steps()
    spec_kats()
    trajectories()
    traces()
    for f in sorted(OUT.glob("*.npz")) + sorted(OUT.glob("*.json")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
