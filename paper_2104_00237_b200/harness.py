"""GPU report harness.

Produces the reference harness's reports (/root/reference/pkg/src/optfuse/bench.py)
from runs on the device, so the B200 numbers sit beside the paper's figures in
the same shape:

  mode        report
  ----------  ---------------------------------------------------------------
  time        stage means (CUDA events), total mean/median, speed-up vs baseline
  breakdown   Fig. 3: schedule / stage / ms for the three schedules
  sweep       Fig. 4: TSV ``idx  forward-fusion  backward-fusion`` per batch
              size (speed-up or saved ms; ``skip:<Error>`` when a schedule
              cannot host the policy)
  optimizers  App. C.3: update-stage ratio and both speed-ups per optimizer
  verify      cross-schedule equivalence grid on the device (bit-exact)
  trace       one steady-state iteration's host issue trace

Models: the reference's synthetic graphs with exact arithmetic, plus the
benchmark CNNs of BASELINE.json.
"""

from __future__ import annotations

import statistics
from dataclasses import dataclass, replace

import torch

from . import models
from .errors import ConfigError
from .optim import OptimizerPolicy
from .schedule import (BACKWARD_FUSION, BASELINE, FORWARD_FUSION, SCHEDULES,
                       flush_pending_updates, run_backward_fusion, run_baseline,
                       run_forward_fusion)

MODES = ("time", "trace", "verify", "breakdown", "sweep", "optimizers")
STAGES = ("forward", "backward", "optimizer")
LOCAL_OPTIMIZERS = ("sgd", "sgd-momentum", "adagrad", "rmsprop", "adadelta", "adam")
CSV_HEADER = "\t".join(("idx", FORWARD_FUSION, BACKWARD_FUSION))
SKIP_MARKER = "skip"
MODEL_CHOICES = models.SYNTHETIC + tuple(models.CLASSIFIERS) + tuple(models.NETWORKS)
VERIFY_MODELS = (("chain", dict(layers=3, width=4)), ("shared-chain", dict(layers=4, width=4)),
                 ("mul-probe", dict(width=3)))
_RUNNERS = {BASELINE: run_baseline, FORWARD_FUSION: run_forward_fusion,
            BACKWARD_FUSION: run_backward_fusion}


@dataclass
class BenchConfig:
    """Harness settings: the reference's fields plus the B200 knobs."""

    model: str = "chain"
    layers: int = 8
    width: int = 32
    optimizer: str = "adam"
    eta: float = 0.001
    weight_decay: float = 0.0
    clip_norm: float | None = None
    schedule: str = BACKWARD_FUSION
    precision: str = "f32"
    batch: int = 32
    batch_sweep: tuple | None = None
    iters: int = 100
    warmup: int = 10
    workers: int = 1
    seed: int = 0
    out: str | None = None
    mode: str = "time"
    metric: str = "speedup"
    bucket_elems: int = 0
    grad_reset: str = "zero"
    device: str = "cuda"
    dtype: str = "fp32"
    tf32: int = 0

    def __post_init__(self):
        checks = (
            (self.mode in MODES, f"unknown mode {self.mode!r}, expected one of {MODES}"),
            (self.schedule in SCHEDULES, f"unknown schedule {self.schedule!r}"),
            (self.model in MODEL_CHOICES, f"unknown model {self.model!r}"),
            (self.iters >= 1, f"measured iterations must be >= 1, got {self.iters}"),
            (self.warmup >= 0, f"warmup must be >= 0, got {self.warmup}"),
            (self.batch >= 1, f"batch must be >= 1, got {self.batch}"),
            (self.metric in ("speedup", "saved"), f"metric must be speedup|saved, got {self.metric!r}"),
            (self.dtype in ("fp32", "bf16"), f"dtype must be fp32|bf16, got {self.dtype!r}"),
            (self.dtype == "fp32" or self.model not in models.SYNTHETIC,
             "--dtype bf16 (bf16 module + fp32 master weights) is for the benchmark networks"),
            (self.batch_sweep is None or 1 <= self.batch_sweep[0] <= self.batch_sweep[1],
             f"batch sweep needs 1 <= lo <= hi, got {self.batch_sweep}"),
        )
        for ok, msg in checks:
            if not ok:
                raise ConfigError(msg)

    def batch_sizes(self) -> list:
        if self.batch_sweep is None:
            return [self.batch]
        return list(range(self.batch_sweep[0], self.batch_sweep[1] + 1))


class _Session:
    """One model + policy + input, driven by one schedule."""

    def __init__(self, cfg: BenchConfig, batch: int):
        self.cfg = cfg
        if cfg.model in models.SYNTHETIC:
            self.graph = models.build_model(cfg.model, layers=cfg.layers, width=cfg.width,
                                            seed=cfg.seed, precision=cfg.precision,
                                            device=cfg.device, track_input_grad=False)
            self.inp = models.make_input(self.graph, batch, cfg.seed)
        else:
            if cfg.precision != "f32":
                raise ConfigError("the benchmark networks run in f32 (or --dtype bf16)")
            self.graph = models.build_classifier(cfg.model, device=cfg.device, seed=cfg.seed)
            self.graph.track_counts = False
            self.inp = models.synthetic_batch(cfg.model, batch, device=cfg.device, seed=cfg.seed)
            if cfg.dtype == "bf16":   # bf16 module, fp32 masters updated in the same pass
                self.graph.use_master_weights()
                x, y = self.inp
                self.inp = (x.to(torch.bfloat16) if x.is_floating_point() else x, y)
        self.policy = OptimizerPolicy(kind=cfg.optimizer, eta=cfg.eta,
                                      weight_decay=cfg.weight_decay, clip_norm=cfg.clip_norm,
                                      grad_reset=cfg.grad_reset)

    def step(self, schedule: str, **kw):
        extra = {}
        if schedule != BASELINE:
            extra["bucket_elems"] = self.cfg.bucket_elems
        if schedule == BACKWARD_FUSION:
            extra["workers"] = self.cfg.workers
        return _RUNNERS[schedule](self.graph, self.policy, self.inp, **extra, **kw)


def measure(cfg: BenchConfig, schedule: str, batch: int) -> dict:
    """Warm-up, then measured iterations; mean per-stage ms plus the mean and
    median of the totals.  Stage times are CUDA events on the compute stream."""
    sess = _Session(cfg, batch)
    for _ in range(cfg.warmup):
        sess.step(schedule)
    reps = [sess.step(schedule) for _ in range(cfg.iters)]
    torch.cuda.synchronize()
    stats = {stage: statistics.fmean(r.stage_ms[stage] for r in reps) for stage in STAGES}
    totals = [r.total_ms for r in reps]
    stats.update(total=statistics.fmean(totals), median=statistics.median(totals))
    return stats


# -- TSV (Fig. 4 data) ----------------------------------------------------------

def format_csv(rows) -> list:
    def cell(v):
        return v if isinstance(v, str) else repr(float(v))
    return [CSV_HEADER] + ["\t".join((str(i), cell(a), cell(b))) for i, a, b in rows]


def emit_csv(rows, path: str) -> None:
    with open(path, "w") as fh:
        fh.writelines(line + "\n" for line in format_csv(rows))


def parse_csv(path: str) -> list:
    def value(text):
        try:
            return float(text)
        except ValueError:
            return text
    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines or lines[0] != CSV_HEADER:
        raise ConfigError(f"unexpected header {lines[0] if lines else ''!r}")
    return [(int(a), value(b), value(c)) for a, b, c in (ln.split("\t") for ln in lines[1:])]


# -- reports ----------------------------------------------------------------------

def sweep(cfg: BenchConfig) -> list:
    out = []
    for b in cfg.batch_sizes():
        base = measure(cfg, BASELINE, b)["total"]
        cells = []
        for schedule in (FORWARD_FUSION, BACKWARD_FUSION):
            try:
                t = measure(cfg, schedule, b)["total"]
            except Exception as e:  # a schedule that cannot host the policy
                cells.append(f"{SKIP_MARKER}:{type(e).__name__}")
            else:
                cells.append(base - t if cfg.metric == "saved" else base / t)
        out.append((b, *cells))
    return out


def breakdown(cfg: BenchConfig) -> list:
    return [(s, stage, ms) for s in SCHEDULES
            for stage, ms in ((k, v) for k, v in measure(cfg, s, cfg.batch).items()
                              if k in STAGES)]


def compare_optimizers(cfg: BenchConfig) -> list:
    decay = cfg.weight_decay if cfg.weight_decay > 0 else 1e-4
    table = [("sgd-no-decay", "sgd", 0.0)] + [(k, k, decay) for k in LOCAL_OPTIMIZERS]
    out = []
    for name, kind, wd in table:
        sub = replace(cfg, optimizer=kind, weight_decay=wd, clip_norm=None)
        t = {s: measure(sub, s, cfg.batch) for s in SCHEDULES}
        base = t[BASELINE]["total"]
        out.append((name, t[BASELINE]["optimizer"] / base, base / t[FORWARD_FUSION]["total"],
                    base / t[BACKWARD_FUSION]["total"]))
    return out


def verify_cell(optimizer: str, model: str, build_kwargs: dict, precision: str, seed: int,
                iters: int = 10, batch: int = 2, device: str = "cuda") -> list:
    """Baseline, forward fusion (+flush) and backward fusion inline and on the
    side stream must end with bit-identical parameters on the device."""
    finals = {}
    for label, run, kw in (("baseline", run_baseline, {}),
                           ("forward", run_forward_fusion, {}),
                           ("backward-inline", run_backward_fusion, {"workers": 1}),
                           ("backward-side-stream", run_backward_fusion, {"workers": 2})):
        g = models.build_model(model, **build_kwargs, seed=seed, precision=precision,
                               device=device, track_input_grad=False)
        pol = OptimizerPolicy(kind=optimizer, eta=0.01)
        for x in models.iteration_inputs(g, batch, seed, iters):
            run(g, pol, x, timing=False, **kw)
        flush_pending_updates(g, pol)
        finals[label] = b"".join(p.value.detach().cpu().numpy().tobytes() for p in g.parameters)
    tag = f"{optimizer}/{model}/{precision}/seed{seed}"
    return [f"{tag}: {k} parameters not bitwise equal to baseline"
            for k, v in finals.items() if v != finals["baseline"]]


def verify_grid(iters: int = 10, seeds=(0, 1, 2), batch: int = 2,
                precisions=("f32", "f64"), device: str = "cuda") -> tuple:
    grid = [(o, m, kw, p, s) for o in LOCAL_OPTIMIZERS for m, kw in VERIFY_MODELS
            for p in precisions for s in seeds]
    failures = []
    for cell in grid:
        failures += verify_cell(*cell, iters=iters, batch=batch, device=device)
    return len(grid), failures


def _write(path, lines) -> None:
    if path:
        with open(path, "w") as fh:
            fh.writelines(line + "\n" for line in lines)


def _mode_verify(cfg):
    cells, failures = verify_grid(device=cfg.device)
    lines = [f"verified {cells} cells"] + (failures or ["all trajectories equivalent"])
    return {"lines": lines, "failures": failures, "cells": cells, "exit_code": int(bool(failures))}


def _mode_trace(cfg):
    sess = _Session(cfg, cfg.batch)
    for _ in range(max(cfg.warmup, 1)):
        sess.step(cfg.schedule)
    report = sess.step(cfg.schedule, trace=True)
    lines = report.trace.export_lines()
    _write(cfg.out, lines)
    return {"lines": lines, "trace": report.trace, "exit_code": 0}


def _mode_breakdown(cfg):
    rows = breakdown(cfg)
    lines = ["schedule\tstage\tms"] + [f"{s}\t{stage}\t{ms:.4f}" for s, stage, ms in rows]
    _write(cfg.out, lines)
    return {"lines": lines, "rows": rows, "exit_code": 0}


def _mode_sweep(cfg):
    rows = sweep(cfg)
    if cfg.out:
        emit_csv(rows, cfg.out)
    return {"lines": format_csv(rows), "rows": rows, "exit_code": 0}


def _mode_optimizers(cfg):
    rows = compare_optimizers(cfg)
    lines = ["optimizer\tratio\tforward-fusion\tbackward-fusion"]
    lines += ["\t".join((n, f"{r:.6f}", f"{a:.6f}", f"{b:.6f}")) for n, r, a, b in rows]
    _write(cfg.out, lines)
    return {"lines": lines, "rows": rows, "exit_code": 0}


def _mode_time(cfg):
    stats = measure(cfg, cfg.schedule, cfg.batch)
    lines = [f"{k}_ms={stats[k]:.4f}" for k in STAGES + ("total", "median")]
    if cfg.schedule != BASELINE:
        base = measure(cfg, BASELINE, cfg.batch)["total"]
        lines += [f"baseline_total_ms={base:.4f}", f"speedup={base / stats['total']:.4f}"]
    _write(cfg.out, lines)
    return {"lines": lines, "stats": stats, "exit_code": 0}


def run_bench(cfg: BenchConfig) -> dict:
    """Run one mode; returns its display lines, rows and the exit code."""
    handler = {"verify": _mode_verify, "trace": _mode_trace, "breakdown": _mode_breakdown,
               "sweep": _mode_sweep, "optimizers": _mode_optimizers, "time": _mode_time}[cfg.mode]
    import torch
    if not str(cfg.device).startswith("cuda"):
        out = handler(cfg)
    else:
        # fp32 means fp32: no TF32 tensor-core rounding in the networks'
        # convolutions and matmuls unless asked for (bench.py does the same)
        prev = (torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32)
        torch.backends.cudnn.allow_tf32 = torch.backends.cuda.matmul.allow_tf32 = bool(cfg.tf32)
        try:
            out = handler(cfg)
        finally:
            torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32 = prev
    out["mode"] = cfg.mode
    return out
