# A/B build/ variants on several workloads: bash tools/ab_multi.sh C3 C2 C5
mkdir -p gpurun_out
for wl in "$@"; do
for f in build/libgim_*.so; do
  n=$(basename $f .so)
  GIM_LIB_PATH=$PWD/$f timeout -s KILL 600 python bench.py --workload $wl --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ab_${wl}_$n.json 2>gpurun_out/ab_${wl}_$n.err
  python -c "
import json
d=json.load(open('gpurun_out/ab_${wl}_$n.json')); ph=d['phase_ms_per_step']
print('$wl $n', 'step %.2f'%d['ms_per_step'], ' '.join('%s %.2f'%(k[3:],v) for k,v in ph.items()))
" || tail -2 gpurun_out/ab_${wl}_$n.err
done; done
