# round-2 evidence runs: config 0, the MW7 sweep, the 1 s quality table
mkdir -p gpurun_out
python tools/mw_parity.py gpu --ref-json tests/golden/config0_mw1_ref.json --out gpurun_out/r02_config0_mw1.json > gpurun_out/config0.log 2>&1; echo config0=$?
python tools/sweep.py --out gpurun_out/r02_sweep_mw7.json > gpurun_out/sweep.log 2>&1; echo sweep=$?
python tools/quality_budget.py --seeds 3 --out gpurun_out/r02_quality_1s.json > gpurun_out/quality.log 2>&1; echo quality=$?
python tools/quality_budget.py --seeds 3 --problems MW1,MW3,MW7,MW9,MW11,MW14,DASCMOP1,DASCMOP5,DASCMOP7,DASCMOP9 --out gpurun_out/r02_quality_1s_mw_das.json > gpurun_out/quality2.log 2>&1; echo quality2=$?
python tools/quality_budget.py --seeds 3 --problems WTA-P10,WTA-P5 --out gpurun_out/r02_quality_1s_wta.json > gpurun_out/quality3.log 2>&1; echo quality3=$?
python -m pytest tests/test_gpu_parity.py -q -k config0 > gpurun_out/config0_test.log 2>&1; echo config0test=$?; tail -2 gpurun_out/config0_test.log
