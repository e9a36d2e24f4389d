mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; grep -E "FAILED|passed|failed|Error" gpurun_out/pytest_gpu.log | head -20
