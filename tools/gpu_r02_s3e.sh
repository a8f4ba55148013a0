# round-2 session-3 pass E: final validation of the shipped code -- smoke, full GPU suite, default bench, consumer rows
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu.log | tail -8
( time timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err ) 2> gpurun_out/bench_time.txt; echo bench=$?; cat gpurun_out/bench_time.txt | grep real; tail -c 2200 gpurun_out/bench.log
timeout 600 python tools/wgrad_bench.py > gpurun_out/wgrad_bench.json 2> gpurun_out/wgrad_bench.err; echo wgrad_bench=$?
timeout 2400 python bench.py --extras c5m --standalone 0 --in-situ 0 --extras-out gpurun_out/bench_extras_c5m.json > gpurun_out/bench_c5m.log 2> gpurun_out/bench_c5m.err; echo bench_c5m=$?
python -c "
import json;d=json.load(open('gpurun_out/bench_extras_c5m.json'))
for s,r in d['c5m']['schedules'].items(): print('%-60s %8.3f %s'%(s,r['ms_per_step'],r.get('speedup_vs_ours_unfused','')))"
