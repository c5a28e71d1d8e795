# full ncu captures of one early and one late greedy step of the C3 selection (k_cover, k_argmax)
mkdir -p gpurun_out
WL=${1:-C3}
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_cover -s 202 -c 1 \
  -o gpurun_out/prof_cover_${WL} -f python bench.py --workload $WL --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cover.log 2>&1
echo "cover rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_argmax -s 230 -c 1 \
  -o gpurun_out/prof_argmax_${WL} -f python bench.py --workload $WL --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_argmax.log 2>&1
echo "argmax rc=$?"
