timeout 900 python tools/sweep.py > gpurun_out/sweep.log 2>&1; echo sweep=$?; tail -5 gpurun_out/sweep.log | cut -c1-200
timeout 1200 python tools/quality_budget.py --budget 1.0 --seeds 3 > gpurun_out/quality.log 2>&1; echo q=$?; tail -40 gpurun_out/quality.log
cp profiles/r01_sweep_mw7.json profiles/r01_quality_1s.json gpurun_out/ 2>/dev/null
