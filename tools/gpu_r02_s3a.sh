# round-2 session-3 pass A: slot-space update kernel -- GPU suite, A/B against
# the round-1 kernel, BF contention at fp32, device timelines, default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu.log | tail -8
AB_REPS=1 timeout 1500 python tools/update_ab.py > gpurun_out/update_ab.log 2>&1; echo update_ab=$?; head -4 gpurun_out/update_ab.log
for c in c2 c3 c5; do timeout 600 python tools/device_timeline.py $c > gpurun_out/device_timeline_$c.json 2> gpurun_out/device_timeline_$c.err; echo timeline_$c=$?; head -9 gpurun_out/device_timeline_$c.json | tail -5; done
timeout 1500 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?; tail -c 2200 gpurun_out/bench.log; tail -3 gpurun_out/bench.err
for c in c3 c4 c5; do timeout 1200 python tools/bf_contention.py $c 3 > gpurun_out/bf_contention_$c.json 2> gpurun_out/bf_contention_$c.err; echo contention_$c=$?; python -c "
import json,sys; d=json.load(open('gpurun_out/bf_contention_$c.json'))
for k,v in list(d.values())[0].items(): print(k, v['median_ms'], v['vs_baseline'])" ; done
