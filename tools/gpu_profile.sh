# ncu evidence for bench.py's workload: launch list (cold, serialised) + one --set full capture of
# the top kernel. Never a multi-rank command. Numbers printed under ncu are NOT bench values.
mkdir -p gpurun_out
WL=${1:-C3}
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${WL}.csv python bench.py --workload $WL --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench_${WL}.log 2>&1
echo "launch list rc=$?"
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:k_rr_warp -s 8 -c 1 \
  -o gpurun_out/prof_rr_${WL} -f python bench.py --workload $WL --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${WL}.log 2>&1
echo "full rr rc=$?"
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:k_rr_giant -s 8 -c 1 \
  -o gpurun_out/prof_giant_${WL} -f python bench.py --workload $WL --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_giant_${WL}.log 2>&1
echo "full giant rc=$?"
ls -la gpurun_out
