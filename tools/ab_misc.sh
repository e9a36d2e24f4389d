timeout 900 python -m pytest tests -m gpu -q -x -k "wta or WTA" > gpurun_out/pytest_wta.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_wta.log
for W in wta-p10-100k; do
  for C in def 55 100; do
    if [ $C = def ]; then unset GMPEA_CARVEOUT; else export GMPEA_CARVEOUT=$C; fi
    python bench.py --workload $W --no-cpu-baseline --no-extras --steps 200 > gpurun_out/ab_c$C.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/ab_c$C.log').read().strip().splitlines()[-1]); print('$W carve $C', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['roofline']['kernel_ms'].items()})"
  done
done
