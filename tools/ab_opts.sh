# A/B of library options on the same build: tools/ab_opts.sh WL "OPT_A=0" "OPT_A=1" ...
mkdir -p gpurun_out
WL=$1; shift
for o in "$@"; do
  n=$(echo "$o" | tr '=' '_')
  timeout -s KILL 300 python bench.py --workload $WL --steps 6 --warmup 3 --no-e2e --no-cpu-baseline --opt $o > gpurun_out/abo_$n.json 2>gpurun_out/abo_$n.err
  python -c "
import json
d=json.load(open('gpurun_out/abo_$n.json')); ph=d['phase_ms_per_step']
print('$WL $o', 'step %.2f ms'%d['ms_per_step'], 'rr %.2f giant %.2f store %.2f inv %.2f sel %.2f'%(ph['ms_rr'],ph['ms_giant'],ph['ms_store'],ph['ms_inv'],ph['ms_select']), 'giant_frac %.4f coins/giant %.0f'%(d['rr_stats']['giant_frac'], d['rr_stats'].get('coins_per_giant_set', 0)), 'wall', d['step_wall_ms'])
" || tail -3 gpurun_out/abo_$n.err
done
