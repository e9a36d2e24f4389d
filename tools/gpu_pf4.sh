mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; grep -E "^FAILED|passed|failed" gpurun_out/pytest_gpu.log | head -20
python tools/dbg_pf.py MW9 DASCMOP1 DASCMOP7 DASCMOP8 2>&1 | grep -v "^  "
W=mw7-1m REPS="1" bash ab/run.sh sel5b.so trig.so
W=dascmop7-1m REPS="1" bash ab/run.sh sel5b.so trig.so
