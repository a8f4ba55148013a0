# GPU round trip: smoke, tests, bench (compact line + extras file), optional ncu passes
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -z "${SKIP_TESTS}" ]; then
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu --durations=15 --timeout 600 -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed|Error" gpurun_out/pytest_gpu.log | tail -5
fi
if [ -z "${SKIP_BENCH}" ]; then
timeout 1500 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$?
tail -c 2500 gpurun_out/bench.log
tail -3 gpurun_out/bench.err
fi
if [ -n "${NCU}" ]; then
  # launch list of the headline (NVTX-selected timed region, headline arm only)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --replay-mode application --nvtx --nvtx-include "timed" -c 3000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --headline-only --steps 4 --warmup 3 --instances 1 > gpurun_out/ncu_bench.log 2>&1; echo ncu_list=$?
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt_step -s 15 -c 3 \
    -o gpurun_out/prof_bf -f python tools/profile_kernels.py bf > gpurun_out/ncu_bf.log 2>&1; echo ncu_bf=$?
fi
# raw-page CSV exports (small) instead of the .ncu-rep files (gpurun_out/ must stay < 64 MiB)
for r in gpurun_out/prof_*.ncu-rep; do
  [ -f "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  ncu -i "$r" --page details --csv > "${r%.ncu-rep}.details.csv" 2>/dev/null
  [ -n "${KEEP_REPS}" ] || rm -f "$r"
done
ls -la gpurun_out | tail -20
