mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --durations=30 --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -45 gpurun_out/pytest_gpu.log
