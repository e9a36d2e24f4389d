mkdir -p gpurun_out
for W in lircmop13-1m mw7-1m; do W=$W REPS="1 2" bash ab/run.sh sel4.so sel5.so sel6.so; done
