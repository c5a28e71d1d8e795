# Round evidence on one B200: K-RR traffic captures (per-edge and skip contracts), the default
# bench line, the reference arm, and torchrun lines of every N > 1 exchange protocol driven
# through NCCL at N = 1 (--force-collectives).
set -x
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none -k regex:k_rr_warp -s 1 -c 1 -f \
  -o gpurun_out/traffic_coin python tools/traffic_capture.py C3 gpurun_out/traffic_coin.json \
  > gpurun_out/traffic_coin.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:'k_skip_(lane|warp)' -s 2 -c 2 -f \
  -o gpurun_out/traffic_skip python tools/traffic_capture.py C3 gpurun_out/traffic_skip.json --skip \
  > gpurun_out/traffic_skip.log 2>&1
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1
for proto in replicated allreduce reducescatter; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 2 --protocol $proto --force-collectives \
    --no-e2e --no-cpu-baseline --no-variants > gpurun_out/bench_proto_$proto.json 2> gpurun_out/bench_proto_$proto.err
done
