# warm per-launch durations of the selection kernels (ncu, caches NOT flushed between launches)
mkdir -p gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"k_cover|k_argmax" \
  --csv --log-file gpurun_out/sel_steps_${1:-C3}.csv python bench.py --workload ${1:-C3} --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/sel_steps.log 2>&1
echo "ncu rc=$?"
