# Bench lines of every BASELINE.json config (+ the geometric-skip variant measured in the same
# run for IC configs) and the BA density extremes, one B200.
mkdir -p gpurun_out
for w in C1 C2 C3 C4 C5; do
  python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/r02_bench_$w.json 2> gpurun_out/r02_bench_$w.err
done
for w in B2 B32; do
  python bench.py --workload $w --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/r02_bench_$w.json 2> gpurun_out/r02_bench_$w.err
done
