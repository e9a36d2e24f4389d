timeout 900 python -m pytest tests -m gpu -q -x -k "wta or WTA or chain" > gpurun_out/pytest_wta.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_wta.log
W=wta-p10-100k REPS="1 2" bash ab/run.sh stage0.so stage1.so
