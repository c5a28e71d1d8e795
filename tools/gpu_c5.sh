mkdir -p gpurun_out
nproc; free -g | head -2
t0=$(date +%s)
GIM_TEST_C5=1 timeout -s KILL 1800 python -m pytest tests/test_gpu_parity.py -q -k "full_size_sampled and C5" -p no:cacheprovider > gpurun_out/c5_test.log 2>&1; echo "c5 test rc=$? ($(( $(date +%s) - t0 ))s)"; tail -3 gpurun_out/c5_test.log
timeout -s KILL 1800 python bench.py --workload C5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "c5 bench rc=$? ($(( $(date +%s) - t0 ))s)"; tail -2 gpurun_out/bench_C5.err
