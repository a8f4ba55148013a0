# GPU round trip: smoke, tests, bench, ncu launch list + full captures of the update kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -z "${SKIP_TESTS}" ]; then
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -q -m gpu --durations=15 --timeout 400 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed|Error" gpurun_out/pytest_gpu.log | tail -5
fi
if [ -z "${SKIP_BENCH}" ]; then
timeout 1500 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?
tail -c 400 gpurun_out/bench.log
fi
if [ -n "${NCU}" ]; then
  # launch list of the headline command (NVTX-selected timed region)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --replay-mode application --nvtx --nvtx-include "timed" -c 3000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --no-extras --steps 4 --warmup 3 --instances 1 > gpurun_out/ncu_bench.log 2>&1; echo ncu_list=$?
  # the same step eager (no CUDA graph): cuDNN's semi-persistent batch-norm kernel fails to
  # launch under the profiler when it is a graph node
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed" -c 3000 --csv \
    --log-file gpurun_out/launches_eager.csv python bench.py --no-extras --graphs 0 --steps 4 --warmup 3 --instances 1 > gpurun_out/ncu_bench_eager.log 2>&1; echo ncu_list_eager=$?
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt_step -s 15 -c 3 \
    -o gpurun_out/prof_bf -f python tools/profile_kernels.py bf > gpurun_out/ncu_bf.log 2>&1; echo ncu_bf=$?
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt_step -s 1 -c 1 \
    -o gpurun_out/prof_vgg -f python tools/profile_kernels.py vgg > gpurun_out/ncu_vgg.log 2>&1; echo ncu_vgg=$?
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt_step -s 1 -c 1 \
    -o gpurun_out/prof_bert -f python tools/profile_kernels.py bert > gpurun_out/ncu_bert.log 2>&1; echo ncu_bert=$?
fi
if [ -n "${NCU_MIXED}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt_step -s 1 -c 1 \
    -o gpurun_out/prof_r50mixed -f python tools/profile_kernels.py r50mixed > gpurun_out/ncu_r50mixed.log 2>&1; echo ncu_r50mixed=$?
fi
# raw-page CSV exports (small) instead of the .ncu-rep files (gpurun_out/ must stay < 64 MiB)
for r in gpurun_out/prof_*.ncu-rep; do
  [ -f "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  ncu -i "$r" --page details --csv > "${r%.ncu-rep}.details.csv" 2>/dev/null
  [ -n "${KEEP_REPS}" ] || rm -f "$r"
done
ls -la gpurun_out | tail -20
