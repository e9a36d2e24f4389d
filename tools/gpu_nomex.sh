mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for W in lircmop13-1m mw7-1m; do W=$W REPS="1 2" bash ab/run.sh cur2.so nomex.so; done
