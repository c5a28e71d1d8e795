# Round evidence on one B200 (run from the repo root through gpurun): the full GPU test suite,
# bench lines of every workload (+ the geometric-skip variant measured in the same run for IC),
# the reference arm, ncu launch lists of C3/C5 IMM steps, and full captures of the hot kernels.
# Outputs land in gpurun_out/ (copied to profiles/ by hand, named per round).
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_final.log 2>&1
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1
for w in C1 C2 C4 C5; do
  python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
for w in B2 B32; do
  python bench.py --workload $w --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
for w in C3 C5; do
  timeout -s KILL 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 1 --warmup 1 \
    --no-e2e --no-cpu-baseline --no-variants > gpurun_out/ncu_launches_$w.log 2>&1
done
bash tools/ncu_kernel.sh k_rr_warp 3 C3 --no-variants
bash tools/ncu_kernel.sh k_cover 60 C3 --no-variants
bash tools/ncu_kernel.sh k_select_cta 1 C1 --no-variants
bash tools/ncu_kernel.sh k_set_ids 2 C5 --no-variants
