mkdir -p gpurun_out
W=mw7-1m REPS="1" bash ab/run.sh v8.so mw10.so
W=mw1-1m REPS="1" bash ab/run.sh v8.so mw10.so
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 1200 python tools/quality_budget.py --problems MW1,MW3,MW7,MW9,MW11,MW14,DASCMOP1,DASCMOP5,DASCMOP7,DASCMOP9 --out gpurun_out/quality_1s_mw_das.json > gpurun_out/quality.log 2>&1; echo q=$?; tail -3 gpurun_out/quality.log
