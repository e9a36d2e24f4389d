timeout 900 python -m pytest tests -m gpu -q -x -k "select or chain or headline or sharded or engine" > gpurun_out/pytest_sel.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_sel.log
for W in lircmop13-1m mw7-1m; do W=$W REPS="1 2" bash ab/run.sh sel_old.so s11.so s12.so s14.so s24.so; done
