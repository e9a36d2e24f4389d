# the bench lines of the current build (profiles/r02/bench_*.jsonl)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
for w in mw1-1m mw7-1m lircmop14-1m dascmop7-1m dascmop9-1m wta-p10-100k c1dtlz1-1m; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo $w=$?
done
