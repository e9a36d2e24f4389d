# ncu captures of the headline workload at steady state (generation ~40):
# vary_eval and select with source attribution, plus the launch list
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"vary_eval|select_kernel" --launch-skip 80 --launch-count 2 \
    -o gpurun_out/prof_l13 -f python bench.py --steps 30 --warmup 30 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo full=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
