# A/B: update launches with programmatic dependent launch (OF_PDL=1) vs plain launches,
# on the headline + C1/C4 rows (alternating processes: base, pdl, base, pdl)
mkdir -p gpurun_out
for rep in 1 2; do for lib in base pdl; do
  OPTFUSE_B200_LIB=build/pdl/$lib.so timeout 1200 python bench.py --extras c1,c4 --standalone 0 --in-situ 0 --instances 3 \
    --extras-out gpurun_out/pdl_${lib}_$rep.json > gpurun_out/pdl_${lib}_$rep.log 2> gpurun_out/pdl_${lib}_$rep.err; echo $lib $rep rc=$?
done; done
python - <<'PY'
import json
for rep in (1, 2):
    for lib in ("base", "pdl"):
        d = json.load(open(f"gpurun_out/pdl_{lib}_{rep}.json"))
        row = {k: v["ms_per_step"] for k, v in d["rows"].items()}
        for c in ("c1", "c4"):
            for n, r in d[c]["schedules"].items():
                if n.startswith("graph:ours") or n.startswith("ours"):
                    row[f"{c}:{n}"] = r["ms_per_step"]
        print(lib, rep, json.dumps(row))
PY
