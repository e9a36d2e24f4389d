for W in lircmop13-1m lircmop14-1m; do W=$W REPS="1 2" bash ab/run.sh v1.so hyb.so hyb2.so; done
