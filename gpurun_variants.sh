timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for mb in 4 6 8; do
  GMPEA_LIB=$PWD/paper_2509_19821_b200/libgmpea_b200_mb$mb.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mb$mb.log 2>&1
  echo "mb=$mb rc=$?"; python -c "
import json; l=json.loads(open('gpurun_out/bench_mb$mb.log').read().strip().splitlines()[-1]); print(l['ms_per_step'], l['value']/1e9, l['roofline']['kernel_ms'], l['e2e']['value']/1e9)"
done
for w in mw1-1m mw7-1m; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workload $w > gpurun_out/bench_$w.log 2>&1; echo "$w rc=$?"; python -c "
import json; l=json.loads(open('gpurun_out/bench_$w.log').read().strip().splitlines()[-1]); print(l['ms_per_step'], l['value']/1e9, l['roofline']['kernel_ms'])"; done
