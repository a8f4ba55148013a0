mkdir -p gpurun_out
export OPTFUSE_PARITY_OUT=gpurun_out/r02_c1_parity.json
timeout 900 python -m pytest -q -m gpu tests/test_wgrad_fused_gpu.py -x > gpurun_out/pytest_wgrad.log 2>&1; echo wgrad=$?
tail -15 gpurun_out/pytest_wgrad.log
timeout 1200 python -m pytest -q -m gpu tests/test_c1_parity_gpu.py tests/test_race_guard_gpu.py > gpurun_out/pytest_c1.log 2>&1; echo c1=$?
tail -15 gpurun_out/pytest_c1.log
CONFIGS="c2 c3 c4 c5" timeout 2400 bash tools/iter_dram.sh
