mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for v in 0 1; do
  GMPEA_NO_PDL=$v timeout 300 python tools/sweep.py --sizes 1000,10000,100000,1000000 --out gpurun_out/sweep_pdl$v.json > gpurun_out/sweep_pdl$v.log 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/sweep_pdl$v.json'))
print('NO_PDL=$v', [(p['N'], round(p['ms_per_generation']*1000,2)) for p in d['points']])"
done
ENVSET=GMPEA_NO_PDL=1 W=lircmop13-1m bash tools/gpu_ab_env.sh
