timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/sweep.py --sizes 1000,10000,100000,1000000 --out gpurun_out/sweep_fused.json > gpurun_out/sweep_fused.log 2>&1; echo sw=$?; cut -c1-150 gpurun_out/sweep_fused.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_l13.log 2>&1; tail -1 gpurun_out/bench_l13.log | python -c "import json,sys; l=json.loads(sys.stdin.read()); print(l['ms_per_step'], l['value']/1e9, l['roofline']['kernel_ms'], l['clocks'])"
