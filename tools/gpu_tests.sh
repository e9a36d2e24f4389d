# GPU tests (all, no -x; a hung test is reported and ends the run)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=20 --timeout=600 --timeout-method=thread ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -45 gpurun_out/pytest_gpu.log
