timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --workload wta-p10-100k > gpurun_out/bench_wta.log 2>&1; tail -1 gpurun_out/bench_wta.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['ms_per_step'], l['value']/1e9, l['roofline']['kernel_ms'])"
