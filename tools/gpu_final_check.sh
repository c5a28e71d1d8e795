# Final check on one B200: GPU test suite, smoke, and the bench lines of BASELINE.md §4.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_final.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for w in C1 C2 C4 C5; do
  python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
