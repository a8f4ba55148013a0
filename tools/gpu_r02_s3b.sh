# round-2 session-3 pass B: ncu evidence for the update kernel, sanitizers, contention, full extras
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python -m pytest -q -m gpu tests/test_consumer_fusion_gpu.py tests/test_kernels_gpu.py > gpurun_out/pytest_b.log 2>&1; echo pytest_b=$?; tail -2 gpurun_out/pytest_b.log
for c in c2 c3 c5; do timeout 600 python tools/device_timeline.py $c > gpurun_out/device_timeline_$c.json 2> gpurun_out/device_timeline_$c.err; echo timeline_$c=$?; head -9 gpurun_out/device_timeline_$c.json | tail -5; done
# launch list of the headline's timed region (headline arm only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --replay-mode application --nvtx --nvtx-include "timed" -c 3000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --headline-only --steps 4 --warmup 3 --instances 1 > gpurun_out/ncu_bench.log 2>&1; echo ncu_list=$?
# full sections of the update launches: in situ (bf buckets) and one pass over each parameter set
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt_step -s 15 -c 3 -o gpurun_out/prof_bf -f python tools/profile_kernels.py bf > gpurun_out/ncu_bf.log 2>&1; echo ncu_bf=$?
for w in c2full vgg bert r50mixed; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt_step -s 2 -c 1 -o gpurun_out/prof_$w -f python tools/profile_kernels.py $w > gpurun_out/ncu_$w.log 2>&1; echo ncu_$w=$?
done
for r in gpurun_out/prof_*.ncu-rep; do
  [ -f "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  ncu -i "$r" --page details --csv > "${r%.ncu-rep}.details.csv" 2>/dev/null
  ncu -i "$r" --page source --csv > "${r%.ncu-rep}.source.csv" 2>/dev/null
  rm -f "$r"
done
ls -la gpurun_out | tail -30
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_kernels.py > gpurun_out/sanitizer_$tool.log 2>&1; echo sanitizer_$tool=$?
  tail -2 gpurun_out/sanitizer_$tool.log
done
TORCH_CUDA_SANITIZER=1 timeout 900 python tools/csan_schedules.py > gpurun_out/csan.log 2>&1; echo csan=$?
tail -3 gpurun_out/csan.log
for c in c3 c4 c5; do timeout 1200 python tools/bf_contention.py $c 3 > gpurun_out/bf_contention_$c.json 2> gpurun_out/bf_contention_$c.err; echo contention_$c=$?; python -c "
import json,sys; d=json.load(open('gpurun_out/bf_contention_$c.json'))
for k,v in list(d.values())[0].items(): print(k, v['median_ms'], v['vs_baseline'])" ; done
if [ -z "${SKIP_EXTRAS}" ]; then
timeout 2400 python bench.py --extras c1,c3,c4,c5 --sweep 32,64,256,512 --extras-out gpurun_out/bench_extras_full.json > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo bench_full=$?
tail -c 1600 gpurun_out/bench_full.log; tail -3 gpurun_out/bench_full.err
fi
