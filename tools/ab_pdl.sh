# A/B of programmatic dependent launch (GMPEA_PDL=0 turns it off) on one box:
# the N = 10^6 workloads through bench.py and the MW7 sweep sizes 10^3..10^6
mkdir -p gpurun_out
for w in ${WORKLOADS:-lircmop13-1m mw7-1m wta-p10-100k}; do
  for rep in 1 2; do for v in on off; do
    if [ $v = off ]; then export GMPEA_PDL=0; else unset GMPEA_PDL; fi
    python bench.py --workload $w --no-cpu-baseline --no-extras --steps 200 > gpurun_out/abpdl_$v.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/abpdl_$v.log').read().strip().splitlines()[-1]); print('$w pdl=$v', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['roofline']['kernel_ms'].items()}, d['replacement_rate'])"
  done; done
done
for v in on off; do
  if [ $v = off ]; then export GMPEA_PDL=0; else unset GMPEA_PDL; fi
  python tools/sweep.py --sizes 1000,10000,100000,1000000 --out gpurun_out/abpdl_sweep_$v.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/abpdl_sweep_$v.json')); print('sweep pdl=$v', [(r['N'], round(r['ms_per_generation'],4)) for r in (d['points'] if 'points' in d else d)])"
done
