# full ncu capture (with source-level PC sampling) of one launch of kernel $1 after skipping $2 launches, workload $3
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s ${2:-0} -c 1 \
  -o gpurun_out/prof_$1 -f python bench.py --workload ${3:-C3} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$1.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/prof_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$1.csv 2>&1; echo "src rc=$?"
ncu -i gpurun_out/prof_$1.ncu-rep --page raw --csv > gpurun_out/raw_$1.csv 2>&1; echo "raw rc=$?"
