# one GPU round trip: build check, smoke, GPU tests, bench, ncu launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?
tail -3 gpurun_out/bench.log
if [ -n "${NCU}" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mt_step -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --no-extras --steps 3 --warmup 2 > gpurun_out/ncu_bench.log 2>&1; echo ncu=$?
fi
