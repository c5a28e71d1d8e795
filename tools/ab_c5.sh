# A/B of build/libgim_*.so on C5 (graph generated once, cached under gpurun_out/ for the run)
mkdir -p gpurun_out
for f in build/libgim_*.so; do
  n=$(basename $f .so)
  GIM_LIB_PATH=$PWD/$f timeout -s KILL 900 python bench.py --workload C5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ab5_$n.json 2>gpurun_out/ab5_$n.err
  python -c "
import json
d=json.load(open('gpurun_out/ab5_$n.json')); ph=d['phase_ms_per_step']
print('$n', 'step %.2f ms'%d['ms_per_step'], {k: round(v,2) for k,v in ph.items()}, 'wall', d['step_wall_ms'])
" || tail -3 gpurun_out/ab5_$n.err
done
