# one iteration: parity tests + smoke + short bench + ncu capture of the dominant kernel
bash tools/gpu_check.sh > gpurun_out/check.log 2>&1
head -8 gpurun_out/check.log | cut -c1-300
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json')); ph=d['phase_ms_per_step']; r=d['roofline']
print('step %.2f ms'%d['ms_per_step'], {k: round(v,2) for k,v in ph.items()}, 'Gcoin/s %.0f'%r['achieved'], 'launches', d['gpu_launches'])
PY
WL=${1:-C3}
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_rr_warp -s 8 -c 1 \
  -o gpurun_out/prof_iter_rr -f python bench.py --workload $WL --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_iter.log 2>&1
echo "ncu rc=$?"
