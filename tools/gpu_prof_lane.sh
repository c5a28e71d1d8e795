mkdir -p gpurun_out
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on -k regex:k_rr_ic_lane -s 9 -c 1 \
  -o gpurun_out/prof_lane_C5 -f python bench.py --workload C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_lane.log 2>&1
echo "lane rc=$?"
