# end-of-round validation: GPU tests, smoke, headline bench + reference arm,
# steady-state ncu capture of the final build and its source attribution
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
for w in mw1-1m mw7-1m lircmop14-1m dascmop7-1m dascmop9-1m wta-p10-100k c1dtlz1-1m; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo $w=$?
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
ncu --set full --import-source on --clock-control none -k regex:"vary_eval|select_kernel|op1_kernel" --launch-skip 120 --launch-count 3 \
    -o gpurun_out/prof_final -f python bench.py --steps 40 --warmup 40 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo full=$?
for w in mw7-1m wta-p10-100k dascmop9-1m; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"vary_eval|select_kernel" --launch-skip 60 --launch-count 2 \
      -o gpurun_out/prof_$w -f python bench.py --workload $w --steps 20 --warmup 20 --no-cpu-baseline --no-extras > gpurun_out/ncu_$w.log 2>&1; echo full_$w=$?
done
