mkdir -p gpurun_out
WL=${1:-C3}
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${WL}.csv python bench.py --workload $WL --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench_${WL}.log 2>&1
echo "launch list rc=$?"
