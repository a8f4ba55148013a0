# GPU round trip: tests, bench, ncu launch list + full captures of the update kernel
mkdir -p gpurun_out
if [ -z "${SKIP_TESTS}" ]; then
timeout 900 python -m pytest tests -q -m gpu --durations=10 --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed" gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?
tail -c 600 gpurun_out/bench.log
if [ -n "${NCU}" ]; then
  # launch list of the headline command (skip the first 3000 launches: build, cudnn autotune, capture)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -c 3000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --no-extras --steps 4 --warmup 3 --instances 1 > gpurun_out/ncu_bench.log 2>&1; echo ncu_list=$?
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt_step -s 40 -c 3 \
    -o gpurun_out/prof_bf -f python tools/profile_kernels.py bf > gpurun_out/ncu_bf.log 2>&1; echo ncu_bf=$?
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt_step -s 1 -c 1 \
    -o gpurun_out/prof_vgg -f python tools/profile_kernels.py vgg > gpurun_out/ncu_vgg.log 2>&1; echo ncu_vgg=$?
fi
