# per-kernel durations of the selection kernels for each build/libgim_*.so (ncu launch list)
mkdir -p gpurun_out
WL=${1:-C3}
for f in build/libgim_*.so; do
  n=$(basename $f .so)
  GIM_LIB_PATH=$PWD/$f timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cover|k_argmax|k_set_segs" --csv \
    --log-file gpurun_out/sel_$n.csv python bench.py --workload $WL --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python3 - "$n" <<'PY'
import csv, sys, collections
n = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/sel_{n}.csv")))
hdr = None; agg = collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); k = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", "")); u = d["Metric Unit"]
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(u, 1)
        agg[k].append(v)
for k, v in agg.items():
    print(n, k, "launches", len(v), "total_us %.0f" % sum(v), "avg_us %.2f" % (sum(v) / len(v)))
PY
done
