for W in lircmop13-1m lircmop14-1m; do W=$W REPS="1 2" bash ab/run.sh de_base.so de_gap8.so de_gap9.so de_gap10.so de_coin9.so; done
