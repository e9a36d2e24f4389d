# A/B of an env switch on the same library and box: ENV="NAME=VALUE" W=workload
mkdir -p gpurun_out
W=${W:-lircmop13-1m}
for rep in 1 2; do for v in base alt; do
  if [ $v = alt ]; then export $ENVSET; else unset ${ENVSET%%=*}; fi
  python bench.py --workload $W --no-cpu-baseline --steps 200 > gpurun_out/ab_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$W $v', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['roofline']['kernel_ms'].items()}, d['replacement_rate'])"
done; done
