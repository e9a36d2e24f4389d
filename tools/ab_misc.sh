for W in lircmop13-1m lircmop14-1m; do W=$W REPS="1 2" bash ab/run.sh base.so de6.so de7.so de9.so; done
