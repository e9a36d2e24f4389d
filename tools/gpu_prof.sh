# ncu --set full captures of the steady-state generation kernels (one GPU,
# each after the same command ran clean without ncu), for profiles/
mkdir -p gpurun_out
TAG=${TAG:-r02}
for w in ${WORKLOADS:-lircmop13-1m mw7-1m wta-p10-100k}; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/pre_$w.log 2>&1 || { echo "$w failed"; continue; }
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${KREGEX:-vary_eval|select_kernel|op1_kernel}" \
      --launch-skip ${SKIP:-30} --launch-count ${COUNT:-3} -o gpurun_out/${TAG}_$w -f \
      python bench.py --workload $w --steps 20 --warmup 20 --no-cpu-baseline --no-extras > gpurun_out/ncu_$w.log 2>&1
  echo "$w ncu=$?"
done
