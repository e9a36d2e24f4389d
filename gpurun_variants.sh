timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/sweep.py --sizes 1000,10000,100000 --out gpurun_out/sweep_coop.json > gpurun_out/sweep_coop.log 2>&1; echo coop=$?; cut -c1-150 gpurun_out/sweep_coop.log
GMPEA_COOP_MAX_N=0 timeout 300 python tools/sweep.py --sizes 1000,10000,100000 --out gpurun_out/sweep_nocoop.json > gpurun_out/sweep_nocoop.log 2>&1; echo nocoop=$?; cut -c1-150 gpurun_out/sweep_nocoop.log
