mkdir -p gpurun_out
timeout -s KILL 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "default rc=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference rc=$?"
timeout -s KILL 600 python bench.py --workload C4 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "C4 rc=$?"
timeout -s KILL 600 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo "C2 rc=$?"
timeout -s KILL 600 python bench.py --workload C1 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err; echo "C1 rc=$?"
