mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "das or DAS or operator_chain or reproduce" > gpurun_out/pytest_das.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_das.log
for w in dascmop7-1m dascmop9-1m; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo $w=$?; tail -1 gpurun_out/bench_$w.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['ms_per_step'], l['value']/1e9, l['roofline']['kernel_ms'], l['roofline']['frac'], l['clocks'])"
done
