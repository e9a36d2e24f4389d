timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b3.log 2>&1; echo bench=$?
tail -1 gpurun_out/b3.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['ms_per_step'], l['value']/1e9, l['roofline']['kernel_ms'], l['e2e']['value']/1e9)"
for w in mw1-1m mw7-1m wta-p10-100k; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workload $w > gpurun_out/bench_$w.log 2>&1; echo "$w rc=$?"; tail -1 gpurun_out/bench_$w.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['ms_per_step'], l['value']/1e9, l['roofline']['kernel_ms'])"; done
ncu --set full --clock-control none --import-source on -k regex:"vary_eval|select_kernel" -s 2 -c 2 -o gpurun_out/prof3 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1; echo ncu=$?
