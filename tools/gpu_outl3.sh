mkdir -p gpurun_out
for W in lircmop13-1m dascmop7-1m mw7-1m; do W=$W REPS="1 2" bash ab/run.sh before.so outl.so rare_only.so; done
