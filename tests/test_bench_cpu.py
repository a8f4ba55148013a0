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
    import argparse
    for sched in ("baseline", "forward-fusion", "backward-fusion"):
        args = bench.parse_args(["--schedule", sched])
        arms = bench.headline_arms(args)
        names = [a[0] for a in arms]
        assert len(names) == len(set(names))
        assert names[0] == bench._headline_name(args)
        # the same-mode comparators the line reports
        for need in ("ours:baseline", "torch.optim.SGD(foreach)", "torch.optim.SGD(fused)",
                     bench.FLOOR):
            assert need in names
    for wl in ("c1", "c3", "c4", "c5"):
        names = [v[0] for v in bench._variants_extra(wl)]
        assert len(names) == len(set(names))
        assert f"torch.optim.{bench.WORKLOADS[wl]['torch'][0]}(foreach)" in names
        assert "ours:baseline" in names and "graph:ours:baseline" in names
    assert bench.OWN_LB in [v[0] for v in bench._variants_extra("c4")]


def test_compact_line_fits_2kb():
    """A fully populated result line (the shape run_ours prints) stays under 2 KB."""
    import json
    long = "x" * 60
    res = {"metric": bench.METRIC, "value": 12345.67, "unit": "images/s", "n_gpus": 8, "steps": 30,
           "warmup": 10, "ms_per_step": 2.5311, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic x~N(0,1), y~U{0..9}; random-init weights",
           "config": {"workload": "C2 MobileNetV2 (10 classes) on synthetic 3x32x32, batch 128/GPU, "
                                  "SGD-momentum, fp32 (TF32 off); ours:backward-fusion(w=2,bucket=1M), "
                                  "graph, NHWC, data parallel over nccl",
                      "global_batch": 1024, "parallelism": "dp8", "instances": 5,
                      "l2": "256 MiB flush before every timed step, outside its events"},
           "unfused": {"ours_baseline_ms": 2.5311, "torch_foreach_ms": 2.5311, "torch_fused_ms": 2.5311,
                       "fwd_bwd_floor_ms": 2.5311, "speedup_vs_ours_unfused": 1.0123,
                       "speedup_vs_torch_foreach": 1.0123, "speedup_vs_torch_fused": 1.0123,
                       "torch_arm": "DDP + torch.optim, same mode"},
           "gpu_launches": 90,
           "e2e": {"value": 12345.67, "unit": "images/s", "h2d_bytes_per_step": 1573888,
                   "d2h_bytes_per_step": 4},
           "roofline": {"bound": "hbm", "kernel": "mt_step_kernel", "achieved": 1561.9, "peak": 6546.9,
                        "unit": "GB/s", "frac": 0.2392, "traffic": 8960853, "bytes_per_launch": 14911213,
                        "us_per_launch": 9.547, "launches_per_step": 3},
           "cpu_baseline": {"value": 777.489, "unit": "images/s", "cores": 16, "kind": "port",
                            "sample": "2+10 iterations at batch 128, pinned to 16 cores: torch-CPU "
                                      "fwd/bwd 150 ms + reference update (numpy oracle port of "
                                      "optim.py, 1 thread) 10.1 ms"},
           "clocks": {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": [], "samples": 77},
           "extras": "gpurun_out/bench_extras.json"}
    assert len(long) == 60
    assert len(json.dumps(res, separators=(",", ":"))) < 2048


def test_defaults():
    a = bench.parse_args([])
    assert a.gpus == 1 and a.warmup >= 3 and a.bucket_elems == 1 << 20 and a.dp_graphs == 1
    assert a.tf32 == 0 and a.instances >= 5 and a.extras == "" and a.sweep == ""
