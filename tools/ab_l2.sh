bash tools/gpu_tests.sh
for W in lircmop13-1m mw7-1m; do ENVSET="GMPEA_L2_PERSIST=0" W=$W bash tools/gpu_ab_env.sh; done
