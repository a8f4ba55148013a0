"""``python -m paper_2104_00237_b200.cli`` -- the GPU harness from the shell.

Accepts the reference CLI's flags (/root/reference/pkg/src/optfuse/cli.py:22-49)
so existing sweep scripts run unchanged, plus the B200 knobs
(``--bucket-elems``, ``--grad-reset``, ``--device``, ``--dtype``) and the
benchmark networks (the BASELINE.json CNNs and ``bert_base``) as ``--model``
choices.  Multi-GPU runs go through ``bench.py`` under torchrun.  Exit status: 2 for a configuration error, 1 when the
verify grid finds a mismatch, 0 otherwise.
"""

from __future__ import annotations

import argparse
import sys

from .errors import ConfigError
from .harness import MODEL_CHOICES, MODES, BenchConfig, run_bench
from .optim import KINDS
from .schedule import SCHEDULES


def _lo_hi(text: str) -> tuple:
    parts = text.split(":")
    if len(parts) != 2 or not all(p.strip().lstrip("-").isdigit() for p in parts):
        raise argparse.ArgumentTypeError(f"expected lo:hi, got {text!r}")
    return int(parts[0]), int(parts[1])


# (flag, BenchConfig field, argparse keywords) -- one row per option
_OPTIONS = (
    ("--model", "model", dict(default="chain", choices=MODEL_CHOICES)),
    ("--layers", "layers", dict(type=int, default=8)),
    ("--width", "width", dict(type=int, default=32)),
    ("--optimizer", "optimizer", dict(default="adam", choices=[k for k in KINDS if k != "newton"])),
    ("--eta", "eta", dict(type=float, default=0.001)),
    ("--weight-decay", "weight_decay", dict(type=float, default=0.0)),
    ("--clip-norm", "clip_norm", dict(type=float, default=None)),
    ("--schedule", "schedule", dict(default="backward-fusion", choices=SCHEDULES)),
    ("--batch", "batch", dict(type=int, default=32)),
    ("--batch-sweep", "batch_sweep", dict(type=_lo_hi, default=None, metavar="LO:HI")),
    ("--iters", "iters", dict(type=int, default=100)),
    ("--warmup", "warmup", dict(type=int, default=10)),
    ("--workers", "workers", dict(type=int, default=1,
                                  help="backward fusion: 1 inline, >1 on the update side stream")),
    ("--precision", "precision", dict(default="f32", choices=("f32", "f64"))),
    ("--seed", "seed", dict(type=int, default=0)),
    ("--mode", "mode", dict(default="time", choices=MODES)),
    ("--metric", "metric", dict(default="speedup", choices=("speedup", "saved"))),
    ("--out", "out", dict(default=None)),
    ("--bucket-elems", "bucket_elems", dict(type=int, default=0,
                                            help="launch groups of >= this many elements")),
    ("--grad-reset", "grad_reset", dict(default="zero", choices=("zero", "none"))),
    ("--device", "device", dict(default="cuda")),
    ("--dtype", "dtype", dict(default="fp32", choices=("fp32", "bf16"),
                              help="bf16: bf16 module with fp32 master weights (networks only)")),
    ("--tf32", "tf32", dict(type=int, default=0,
                            help="1: TF32 tensor cores for the networks' convolutions and matmuls")),
)


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="optfuse-b200", description="Fused-optimizer schedules on B200: time, sweep, verify.")
    for flag, field, kw in _OPTIONS:
        parser.add_argument(flag, dest=field, **kw)
    return parser


def main(argv=None) -> int:
    ns = build_parser().parse_args(argv)
    try:
        result = run_bench(BenchConfig(**{field: getattr(ns, field) for _, field, _ in _OPTIONS}))
    except ConfigError as err:
        sys.stderr.write(f"error: {err}\n")
        return 2
    sys.stdout.write("".join(line + "\n" for line in result["lines"]))
    return result["exit_code"]


if __name__ == "__main__":
    sys.exit(main())
