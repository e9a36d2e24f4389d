export PYTHONPATH=$PWD
mkdir -p gpurun_out
GMPEA_SELECT_WIN=0 python tools/bitident.py gpurun_out/bi_off.npz > gpurun_out/bi.log 2>&1
python tools/bitident.py gpurun_out/bi_on.npz >> gpurun_out/bi.log 2>&1
python tools/bitident.py --cmp gpurun_out/bi_off.npz gpurun_out/bi_on.npz >> gpurun_out/bi.log 2>&1
cat gpurun_out/bi.log; rm -f gpurun_out/bi_*.npz
for w in lircmop13-1m mw7-1m wta-p10-100k dascmop9-1m; do
  for rep in 1 2; do for v in on off; do
    if [ $v = off ]; then export GMPEA_SELECT_WIN=0; else unset GMPEA_SELECT_WIN; fi
    timeout 300 python bench.py --workload $w --no-cpu-baseline --no-extras --steps 200 > gpurun_out/abwin_$v.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/abwin_$v.log').read().strip().splitlines()[-1]); print('$w win=$v', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['roofline']['kernel_ms'].items()}, d['replacement_rate'])"
  done; done
done
unset GMPEA_SELECT_WIN
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
