mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
for w in lircmop13-1m mw7-1m; do ENVSET=GMPEA_NO_RPACK=1 W=$w bash tools/gpu_ab_env.sh; done
