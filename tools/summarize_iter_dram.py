"""Summarise tools/iter_dram.sh's ncu CSVs: per config and schedule, the DRAM
bytes (read + write) and kernel time of one training iteration, split into
the update kernels (mt_step_kernel) and everything else, next to the update's
algorithmic bytes.

    python tools/summarize_iter_dram.py gpurun_out > profiles/r02_iter_dram.md
"""

import csv
import io
import re
import sys
from collections import defaultdict
from pathlib import Path

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def load(path: Path):
    text = path.read_text(errors="replace")
    start = text.find('"ID"')
    if start < 0:
        return None
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    kern = defaultdict(lambda: {"name": "", "bytes": 0.0, "us": 0.0})
    for r in rows:
        k = kern[r["ID"]]
        k["name"] = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", "")) * UNITS.get(r["Metric Unit"], 1.0)
        if r["Metric Name"].startswith("dram__bytes"):
            k["bytes"] += v
        elif r["Metric Name"] == "gpu__time_duration.sum":
            k["us"] += v
    return list(kern.values())


def main():
    d = Path(sys.argv[1])
    res = {}
    algo = {}
    for f in sorted(d.glob("iter_dram_*_*.csv")):
        m = re.match(r"iter_dram_(c\d)_(\w+)\.csv", f.name)
        if not m:
            continue
        cfg, sched = m.groups()
        ks = load(f)
        if not ks:
            continue
        upd = [k for k in ks if "mt_step_kernel" in k["name"]]
        rest = [k for k in ks if "mt_step_kernel" not in k["name"]]
        res[(cfg, sched)] = {
            "kernels": len(ks), "total_MB": sum(k["bytes"] for k in ks) / 1e6,
            "update_MB": sum(k["bytes"] for k in upd) / 1e6,
            "other_MB": sum(k["bytes"] for k in rest) / 1e6,
            "update_us": sum(k["us"] for k in upd), "total_us": sum(k["us"] for k in ks),
            "update_launches": len(upd)}
        log = f.with_suffix(".log")
        if log.exists():
            mm = re.search(r"update algorithmic bytes (\d+)", log.read_text(errors="replace"))
            if mm:
                algo[cfg] = int(mm.group(1)) / 1e6
    print("# Whole-iteration DRAM traffic per schedule (ncu, one iteration, --cache-control none)\n")
    print("Kernels serialised by the profiler (no side-stream overlap); each kernel sees the L2 "
          "state its predecessors left.  update = mt_step_kernel launches; algorithmic = the "
          "update's byte model (SURVEY.md §8(d)).\n")
    print("| config | schedule | kernels | total DRAM MB | other MB | update MB | update algorithmic MB "
          "| update DRAM / algorithmic | update launches | update kernel us | all kernels us |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for (cfg, sched), r in sorted(res.items()):
        a = algo.get(cfg)
        ratio = f"{r['update_MB'] / a:.3f}" if a else "-"
        print(f"| {cfg} | {sched} | {r['kernels']} | {r['total_MB']:.1f} | {r['other_MB']:.1f} | "
              f"{r['update_MB']:.1f} | {a if a is None else round(a, 1)} | {ratio} | "
              f"{r['update_launches']} | {r['update_us']:.1f} | {r['total_us']:.1f} |")
    base = {cfg: r["total_MB"] for (cfg, s), r in res.items() if s == "baseline"}
    print("\nTotal DRAM bytes relative to the unfused baseline of the same config:\n")
    for (cfg, sched), r in sorted(res.items()):
        if cfg in base and sched != "baseline":
            print(f"* {cfg} {sched}: {r['total_MB'] / base[cfg]:.4f} "
                  f"({r['total_MB'] - base[cfg]:+.1f} MB)")


if __name__ == "__main__":
    main()
