mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_gpu.log
for W in lircmop13-1m mw7-1m; do W=$W REPS="1 2" bash ab/run.sh sel5.so sel5b.so; done
