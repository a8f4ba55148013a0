# pass F: every table re-measured after the native-engine baseline launch
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python bench.py --extras c1,c3,c4,c5 --sweep 32,64,256,512 --extras-out gpurun_out/bench_extras_full.json > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo bench_full=$?; tail -1 gpurun_out/bench_full.log | cut -c1-300
timeout 1200 python bench.py --graphs 0 --standalone 0 --in-situ 0 --sweep 32,64 --extras-out gpurun_out/bench_extras_c2_eager.json > gpurun_out/bench_eager.log 2> gpurun_out/bench_eager.err; echo bench_eager=$?
timeout 2000 python bench.py --extras c5m --standalone 0 --in-situ 0 --extras-out gpurun_out/bench_extras_c5m.json > gpurun_out/bench_c5m.log 2> gpurun_out/bench_c5m.err; echo bench_c5m=$?
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_extras_c2_eager.json"))
for k, v in d["rows"].items(): print("c2eager", k, v["ms_per_step"], v["instances_ms"])
d = json.load(open("gpurun_out/bench_extras_c5m.json"))
for s, r in d["c5m"]["schedules"].items(): print("c5m", s, r["ms_per_step"], r.get("speedup_vs_ours_unfused", ""))
d = json.load(open("gpurun_out/bench_extras_full.json"))
for c in ("c1", "c3", "c4", "c5"):
    for s, r in d[c]["schedules"].items(): print(c, s, r["ms_per_step"], r.get("speedup_vs_ours_unfused", ""))
PY
