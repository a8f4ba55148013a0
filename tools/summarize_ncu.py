"""Summarise ncu artefacts from gpurun_out/ into profiles/ (run here, no GPU).

    python tools/summarize_ncu.py launches gpurun_out/launches.csv > profiles/rNN_launches.md
    python tools/summarize_ncu.py report gpurun_out/prof_vgg.ncu-rep "title" > profiles/rNN_x.md
"""

import collections
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[start]
    K, V, G = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
    agg = collections.defaultdict(list)
    mine = []
    for r in rows[start + 1:]:
        name = r[K]
        short = name.split("(")[0][:90]
        agg[short].append(float(r[V]))
        if "mt_step" in name or "sqnorm" in name or "clip_coef" in name:
            mine.append((name.split("<", 1)[-1][:70], r[G], float(r[V])))
    tot = sum(sum(v) for v in agg.values())
    print(f"# ncu launch list summary: `{path}`\n")
    print(f"{len(rows) - start - 1} launches, {tot / 1e3:.1f} us total device time "
          "(serialised, cold-cache replay: compare shares, not absolutes)\n")
    print("| kernel | launches | total us | share | avg us |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:20]:
        print(f"| `{k}` | {len(v)} | {sum(v) / 1e3:.1f} | {sum(v) / tot:.3f} | {sum(v) / len(v) / 1e3:.2f} |")
    if mine:
        t = sum(x[2] for x in mine)
        print(f"\n## liboptfuse_b200 kernels: {len(mine)} launches, {t / 1e3:.1f} us, "
              f"share {t / tot:.4f}, avg {t / len(mine) / 1e3:.2f} us\n")
        print("| kernel | grid | us |\n|---|---|---|")
        for n, g, v in mine[:40]:
            print(f"| `{n}` | {g} | {v / 1e3:.2f} |")


def _raw_rows(path):
    """Rows of ncu's raw page: from a .ncu-rep (needs ncu) or its CSV export."""
    if path.endswith(".csv"):
        return list(csv.reader(open(path)))
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(path, title):
    rows = _raw_rows(path)
    hdr, units = rows[0], rows[1]
    print(f"# {title}\n\nSource: `{path}` (`ncu --set full --clock-control none`)\n")
    idx = [(m, hdr.index(m)) for m in METRICS if m in hdr]
    kn = hdr.index("Kernel Name")
    for r in rows[2:]:
        print(f"## `{r[kn][:120]}`\n\n| metric | value | unit |\n|---|---|---|")
        for m, i in idx:
            print(f"| {m} | {r[i]} | {units[i]} |")
        print()


def traffic(path, key, out_json):
    """Average DRAM bytes (read + write) and duration per captured launch,
    merged into ``out_json`` under ``key`` (read by bench.py's roofline)."""
    import json
    import os
    rows = _raw_rows(path)
    hdr, units = rows[0], rows[1]

    def val(r, m):
        v = float(r[hdr.index(m)].replace(",", ""))
        u = units[hdr.index(m)]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1,
                 "usecond": 1, "msecond": 1e3, "nsecond": 1e-3}.get(u, 1)
        return v * scale
    recs = [(val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
             val(r, "gpu__time_duration.sum")) for r in rows[2:]]
    d = json.load(open(out_json)) if os.path.exists(out_json) else {}
    d[key] = {"launches": len(recs), "dram_bytes_per_launch": round(sum(b for b, _ in recs) / len(recs)),
              "gpu_time_us_per_launch": round(sum(t for _, t in recs) / len(recs), 3),
              "source": f"ncu --set full --clock-control none ({os.path.basename(path)})"}
    with open(out_json, "w") as fh:
        json.dump(d, fh, indent=1)
    print(json.dumps(d[key]))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[2])
