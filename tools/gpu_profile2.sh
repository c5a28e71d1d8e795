mkdir -p gpurun_out
WL=${1:-C3}
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:k_rr_warp -s 8 -c 1 \
  -o gpurun_out/prof2_rr_${WL} -f python bench.py --workload $WL --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu2_rr.log 2>&1
echo "rr rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none -k regex:k_philox_bench -s 1 -c 1 \
  -o gpurun_out/prof2_philox -f python bench.py --workload C1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu2_ph.log 2>&1
echo "philox rc=$?"
