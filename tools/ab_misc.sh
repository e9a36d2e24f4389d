for W in mw7-1m mw1-1m dascmop9-1m c1dtlz1-1m; do W=$W REPS="1 2" bash ab/run.sh base.so eu2.so eu3.so eu5.so; done
