for W in lircmop13-1m mw7-1m c1dtlz1-1m; do W=$W REPS="1 2" bash ab/run.sh notma.so tma8.so; done
