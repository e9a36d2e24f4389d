for W in lircmop13-1m mw7-1m dascmop9-1m; do W=$W REPS="1 2" bash ab/run.sh pf0.so pf1.so pf2.so pf3.so; done
