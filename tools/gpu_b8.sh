mkdir -p gpurun_out
for w in lircmop13-1m mw7-1m; do ENVSET=GMPEA_SEL_B8=1 W=$w bash tools/gpu_ab_env.sh; done
