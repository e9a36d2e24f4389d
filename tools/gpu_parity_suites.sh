# 30-seed statistical parity against the reference's own run_gmpea (draw schema v2)
mkdir -p gpurun_out
python tools/mw_parity.py gpu --out gpurun_out/r02_mw_parity.json > gpurun_out/mw_parity.log 2>&1; echo mw=$?
python tools/mw_parity.py gpu --ref-json tests/golden/das_ref_hv.json --out gpurun_out/r02_das_parity.json > gpurun_out/das_parity.log 2>&1; echo das=$?
python tools/mw_parity.py gpu --ref-json tests/golden/refsuite_ref_hv.json --out gpurun_out/r02_refsuite_parity.json > gpurun_out/refsuite.log 2>&1; echo ref=$?
python tools/mw_parity.py gpu --ref-json tests/golden/refsuite1e4_ref_hv.json --out gpurun_out/r02_refsuite1e4_parity.json > gpurun_out/refsuite1e4.log 2>&1; echo ref1e4=$?
