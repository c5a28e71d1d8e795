# A/B tuning variants built under build/ (GIM_LIB_PATH), same bench workload
mkdir -p gpurun_out
WL=${1:-C3}
for f in build/libgim_*.so; do
  n=$(basename $f .so)
  GIM_LIB_PATH=$PWD/$f timeout -s KILL 300 python bench.py --workload $WL --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$n.json 2>gpurun_out/ab_$n.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/ab_$n.json'))
ph=d['phase_ms_per_step']; r=d['roofline']
print('$n', 'step %.2f ms'%d['ms_per_step'], 'rr %.2f giant %.2f store %.2f inv %.2f sel %.2f'%(ph['ms_rr'],ph['ms_giant'],ph['ms_store'],ph['ms_inv'],ph['ms_select']), 'Gcoin/s %.0f'%r['achieved'], 'giant_frac %.4f'%d['rr_stats']['giant_frac'], 'wall', d['step_wall_ms'])
" || tail -3 gpurun_out/ab_$n.err
done
