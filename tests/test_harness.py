"""GPU report harness and CLI (reference bench.py / cli.py formats)."""

import subprocess
import sys

import pytest

from paper_2104_00237_b200 import cli, harness
from paper_2104_00237_b200.errors import ConfigError

REFERENCE_FLAGS = ["--model", "chain", "--layers", "3", "--width", "4", "--optimizer", "adam",
                   "--eta", "0.01", "--weight-decay", "0.0", "--schedule", "baseline",
                   "--batch", "2", "--batch-sweep", "1:3", "--iters", "2", "--warmup", "1",
                   "--workers", "2", "--precision", "f64", "--seed", "1", "--mode", "time",
                   "--metric", "saved"]


def test_cli_accepts_every_reference_flag():
    ns = cli.build_parser().parse_args(REFERENCE_FLAGS + ["--clip-norm", "1.0", "--out", "x"])
    assert ns.batch_sweep == (1, 3) and ns.precision == "f64" and ns.clip_norm == 1.0


@pytest.mark.parametrize("kw", [dict(mode="plot"), dict(schedule="lazy"), dict(iters=0),
                                dict(warmup=-1), dict(batch=0), dict(metric="ratio"),
                                dict(batch_sweep=(3, 1)), dict(model="resnet152"),
                                dict(dtype="fp16"), dict(model="chain", dtype="bf16")])
def test_config_validation(kw):
    with pytest.raises(ConfigError):
        harness.BenchConfig(**kw)


def test_cli_exit_code_2_on_config_error(capsys):
    assert cli.main(["--iters", "0"]) == 2
    assert "error:" in capsys.readouterr().err


def test_sweep_tsv_round_trip(tmp_path):
    rows = [(1, 1.25, "skip:GlobalInfoRequired"), (2, 0.1 + 0.2, 1.0)]
    path = tmp_path / "s.tsv"
    harness.emit_csv(rows, str(path))
    text = path.read_text().splitlines()
    assert text[0] == "idx\tforward-fusion\tbackward-fusion" and len(text) == 3
    assert harness.parse_csv(str(path)) == rows
    bad = tmp_path / "b.tsv"
    bad.write_text("a\tb\tc\n")
    with pytest.raises(ConfigError):
        harness.parse_csv(str(bad))


def test_batch_sizes():
    assert harness.BenchConfig(batch_sweep=(2, 5)).batch_sizes() == [2, 3, 4, 5]
    assert harness.BenchConfig(batch=7).batch_sizes() == [7]


@pytest.mark.gpu
def test_verify_grid_on_device_all_cells_equivalent():
    cells, failures = harness.verify_grid()
    assert cells == 108
    assert failures == []


@pytest.mark.gpu
def test_breakdown_and_sweep_reports():
    cfg = harness.BenchConfig(model="chain", layers=4, width=16, iters=3, warmup=1, batch=4,
                              optimizer="sgd-momentum", eta=0.01, batch_sweep=(1, 2))
    rows = harness.breakdown(cfg)
    assert [(s, st) for s, st, _ in rows] == [(s, st) for s in harness.SCHEDULES
                                              for st in harness.STAGES]
    assert all(ms == 0.0 for s, st, ms in rows if st == "optimizer" and s != "baseline")
    clip = harness.BenchConfig(model="chain", layers=2, width=8, iters=2, warmup=1,
                               clip_norm=0.1, batch_sweep=(1, 2))
    out = harness.sweep(clip)
    assert [r[0] for r in out] == [1, 2] and all(r[2] == "skip:GlobalInfoRequired" for r in out)
    assert all(isinstance(r[1], float) for r in out)


@pytest.mark.gpu
def test_cli_time_mode_on_a_cnn():
    proc = subprocess.run([sys.executable, "-m", "paper_2104_00237_b200.cli", "--model",
                           "mobilenet_v2_cifar", "--optimizer", "sgd-momentum", "--batch", "16",
                           "--iters", "3", "--warmup", "2", "--workers", "2",
                           "--bucket-elems", "262144", "--mode", "time"],
                          capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr
    keys = [ln.split("=")[0] for ln in proc.stdout.split()]
    assert keys == ["forward_ms", "backward_ms", "optimizer_ms", "total_ms", "median_ms",
                    "baseline_total_ms", "speedup"]


@pytest.mark.gpu
def test_cli_bf16_master_weights_on_a_cnn():
    proc = subprocess.run([sys.executable, "-m", "paper_2104_00237_b200.cli", "--model",
                           "resnet18_cifar", "--optimizer", "adamw", "--batch", "16", "--dtype", "bf16",
                           "--iters", "3", "--warmup", "2", "--workers", "2", "--mode", "breakdown"],
                          capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr
    assert "backward-fusion" in proc.stdout
