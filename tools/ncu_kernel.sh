# Full ncu capture (source-level sampling) of one launch of kernel regex $1 after skipping $2
# launches, on `bench.py --workload $3` plus any further bench arguments; exports the source and
# raw pages as CSV next to the report (read them here with tools/src_hot.py).
#   tools/ncu_kernel.sh k_skip_warp 2 C3 --skip
k=$1; s=${2:-0}; w=${3:-C3}; shift 3
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
  -o gpurun_out/prof_$k -f python bench.py --workload $w --steps 1 --warmup 1 --no-e2e --no-cpu-baseline "$@" \
  > gpurun_out/ncu_$k.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/prof_$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_$k.csv 2>&1
ncu -i gpurun_out/prof_$k.ncu-rep --page raw --csv > gpurun_out/raw_$k.csv 2>&1
ncu -i gpurun_out/prof_$k.ncu-rep --page details > gpurun_out/details_$k.txt 2>&1
