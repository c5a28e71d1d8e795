# round-end evidence: smoke, default bench (e2e + cpu baseline), reference arm, other configs,
# ncu launch list + full captures of the top kernels on C3
mkdir -p gpurun_out
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
bash tools/gpu_bench_all.sh
timeout -s KILL 900 python bench.py --workload C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "C5 rc=$?"
timeout -s KILL 900 python bench.py --workload C3 --k 10 --rounds 5 --steps 3 --cpu-seconds 8 > gpurun_out/bench_C3_mrim.json 2> gpurun_out/bench_C3_mrim.err; echo "mrim rc=$?"
bash tools/gpu_profile.sh C3
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
