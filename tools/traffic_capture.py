"""DRAM traffic of ONE K-RR launch paired with that launch's algorithmic bytes (bench.py's
roofline.traffic). Run under ncu on the GPU box:

  ncu --set full --clock-control none -k regex:k_rr_warp -s 1 -c 1 -o gpurun_out/traffic \
      python tools/traffic_capture.py C3 gpurun_out/traffic_stats.json
  ncu ... -k regex:'k_skip_(lane|warp)' -s 2 -c 2 ... --skip     (both kernels of the call)

The script generates 2^20 RR sets twice (the first call warms allocations; the second, with
another seed, is the captured launch: one generation chunk = one k_rr_warp launch) and writes
that call's counters. tools/traffic_capture.py --merge then combines the ncu report's
dram__bytes_read/write and gpu__time_duration with the counters into profiles/ncu_traffic.json.
Algorithmic bytes per launch: 12 B per set (size + staging offset) + 12 B per
visited node (row-pointer pair + staging write) + 4 B per live in-edge (its source)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SETS = 1 << 20


def capture(key, out, skip):
    import gim_inputs as gi
    import paper_2009_07325_b200 as P
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    c = P.Gim(0)
    c.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme, p_uniform=w.p_uniform)
    if skip:
        c.set_option(P.OPT_SKIP, 1)
    c.generate_rr(SETS, 1)
    c.reset_stats()
    c.generate_rr(SETS, 2)                 # the captured launch (a new seed restarts the pool)
    st = c.stats()
    alg = 12 * st["rr_sets"] + 12 * st["rr_elements"] + 4 * st["live_edges"]
    json.dump({"workload": key, "skip": skip, "sets": st["rr_sets"], "elements": st["rr_elements"],
               "live": st["live_edges"], "coins": st["coins"], "giant_sets": st["giant_sets"],
               "alg_bytes": alg}, open(out, "w"), indent=1)


def merge(rep, stats_json, kernel):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    import csv
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    u = dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
             "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}
    dram = dur = 0.0
    kernels = []
    for vals in rows[2:]:                      # every captured launch of the call (lane + warp)
        d = dict(zip(hdr, vals))

        def num(name):
            return float(d[name].replace(",", "")) * scale.get(u[name], 1.0)
        dram += num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        dur += num("gpu__time_duration.sum")
        kernels.append(d.get("Kernel Name", ""))
    st = json.load(open(stats_json))
    key = f"{st['workload']}:{kernel}{':skip' if st['skip'] else ''}"
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tab = json.load(open(path)) if os.path.exists(path) else {}
    tab[key] = {"dram_bytes": dram, "launch_s": dur, "dram_gbs": dram / dur / 1e9, "launch_sets": st["sets"],
                "launch_elements": st["elements"], "launch_live": st["live"], "launch_coins": st["coins"],
                "alg_bytes": st["alg_bytes"], "sector_eff": st["alg_bytes"] / dram,
                "kernels": kernels,
                "source": "tools/traffic_capture.py: ncu --set full of the one k_rr launch of a 2^20-set "
                          "generate_rr call; counters of the same call"}
    json.dump(tab, open(path, "w"), indent=1)
    print(json.dumps(tab[key], indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "--merge":
        merge(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        capture(sys.argv[1], sys.argv[2], "--skip" in sys.argv)
