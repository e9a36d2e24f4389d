#!/bin/bash
# A/B: alternate libraries on the same box; prints ms/step and vary ms
W=${W:-lircmop13-1m}
for rep in ${REPS:-1 2}; do for L in "$@"; do
  GMPEA_LIB=$PWD/ab/$L python bench.py --workload $W --no-cpu-baseline --no-extras --steps 200 > gpurun_out/ab_$L.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$L.log').read().strip().splitlines()[-1]); print('$W $L', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['roofline']['kernel_ms'].items()})"
done; done
