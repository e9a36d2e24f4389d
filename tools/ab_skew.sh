timeout 900 python -m pytest tests/test_skew_gpu.py tests/test_sharded_gpu.py -m gpu -q -x > gpurun_out/pytest_skew.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_skew.log
for W in lircmop13-1m mw7-1m wta-p10-100k dascmop9-1m; do ENVSET="GMPEA_SKEW=0" W=$W bash tools/gpu_ab_env.sh; done
