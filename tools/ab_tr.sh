for W in lircmop13-1m mw7-1m dascmop9-1m c1dtlz1-1m wta-p10-100k lircmop14-1m; do W=$W REPS="1 2" bash ab/run.sh head.so trows.so; done
