# Round-2 evidence pass: new parity/race tests, compute-sanitizer, CSAN, full extras bench
mkdir -p gpurun_out
export OPTFUSE_PARITY_OUT=gpurun_out/r02_c1_parity.json
timeout 1200 python -m pytest -q -m gpu tests/test_race_guard_gpu.py tests/test_c1_parity_gpu.py \
  "tests/test_schedules_gpu.py::test_captured_forward_fusion_flush_between_replays_is_rejected" \
  "tests/test_schedules_gpu.py::test_captured_forward_fusion_clip_bitwise_vs_eager" \
  "tests/test_schedules_gpu.py::test_clip_f64_uses_the_double_factor" \
  tests/test_kernels_gpu.py -k "multicast or race or c1 or captured or clip or Race or parity or one_step or free_running or schedules_bitwise" \
  > gpurun_out/pytest_new.log 2>&1; echo pytest_new=$?
tail -3 gpurun_out/pytest_new.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_kernels.py > gpurun_out/sanitizer_$tool.log 2>&1; echo sanitizer_$tool=$?
  tail -2 gpurun_out/sanitizer_$tool.log
done
TORCH_CUDA_SANITIZER=1 timeout 900 python tools/csan_schedules.py > gpurun_out/csan.log 2>&1; echo csan=$?
tail -4 gpurun_out/csan.log
if [ -z "${SKIP_EXTRAS}" ]; then
timeout 2400 python bench.py --extras c1,c3,c4,c5 --sweep 32,64,256,512 --extras-out gpurun_out/bench_extras_full.json > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo bench_full=$?
tail -c 1600 gpurun_out/bench_full.log; tail -3 gpurun_out/bench_full.err
fi
