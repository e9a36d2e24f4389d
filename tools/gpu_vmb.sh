mkdir -p gpurun_out
for W in lircmop13-1m mw7-1m; do W=$W REPS="1 2" bash ab/run.sh v8.so v6.so v10.so; done
timeout 900 python tools/quality_budget.py --problems MW1,MW3,MW7,MW9,MW11,MW14,DASCMOP1,DASCMOP5,DASCMOP7,DASCMOP9 --out gpurun_out/quality_1s_mw_das.json > gpurun_out/quality.log 2>&1; echo q=$?; tail -5 gpurun_out/quality.log
