for W in lircmop13-1m mw7-1m; do W=$W REPS="1 2" bash ab/run.sh base.so smb6.so smb8.so snbp8.so; done
W=wta-p10-100k REPS="1 2" bash ab/run.sh base.so seltree.so
