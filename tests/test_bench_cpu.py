"""bench.py contract pieces that run without a GPU: the reference arm's JSON
line, the speed-up/floor bookkeeping and the variant tables."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_reference_arm_json_line(capsys):
    bench.main(["--impl", "reference", "--steps", "1", "--warmup", "1"])
    line = capsys.readouterr().out.strip().splitlines()[-1]
    d = json.loads(line)
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == "images/s"
    assert d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "images/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_speedups_and_hidden_update_phase():
    row = {"cl:graph:torch.optim.SGD(foreach)": {"ms_per_step": 2.8},
           "cl:graph:fwd+bwd only (no update: lower bound)": {"ms_per_step": 2.6},
           "cl:graph:ours:backward-fusion(w=2,bucket=1M)": {"ms_per_step": 2.65},
           "torch.optim.SGD(foreach)": {"ms_per_step": 8.0}}
    bench._speedups(row)
    ours = row["cl:graph:ours:backward-fusion(w=2,bucket=1M)"]
    assert abs(ours["speedup_vs_unfused_same_mode"] - 2.8 / 2.65) < 1e-3
    assert abs(ours["unfused_update_phase_hidden"] - 0.75) < 1e-3
    assert abs(ours["speedup_vs_eager_torch_foreach"] - 8.0 / 2.65) < 1e-3


def test_variant_tables_are_well_formed():
    for world, dpg in ((1, False), (2, False), (2, True)):
        names = [v[0] for v in bench._variants_c2(world, dpg)]
        assert len(names) == len(set(names))
        if world > 1 and not dpg:
            assert not any(v[6] for v in bench._variants_c2(world, dpg))
    for wl in ("c1", "c3", "c4", "c5"):
        names = [v[0] for v in bench._variants_extra(wl)]
        assert len(names) == len(set(names))
        assert f"torch.optim.{bench.WORKLOADS[wl]['torch'][0]}(foreach)" in names
    assert bench.OWN_LB in [v[0] for v in bench._variants_extra("c4")]


def test_defaults():
    a = bench.parse_args([])
    assert a.gpus == 1 and a.warmup >= 3 and a.bucket_elems == 1 << 20 and a.dp_graphs == 1
