for W in mw7-1m wta-p10-100k dascmop9-1m c1dtlz1-1m; do W=$W REPS="1 2" bash ab/run.sh sbx_old.so sbx_new.so sbx_fg.so; done
