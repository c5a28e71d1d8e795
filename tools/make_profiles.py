"""Summarise ncu evidence from gpurun_out/ into profiles/ (committed, per round).

  python tools/make_profiles.py r01 C3

Reads gpurun_out/launches_<WL>.csv (ncu --metrics gpu__time_duration.sum launch list of
`bench.py --steps 1 --warmup 1`) and gpurun_out/prof_rr_<WL>.ncu-rep / prof_giant_<WL>.ncu-rep
(ncu --set full of one launch each), and writes:
  profiles/<round>_launches_<WL>.csv      the raw launch list
  profiles/<round>_launch_shares_<WL>.txt per-kernel totals and shares (cold, serialised)
  profiles/<round>_ncu_<kernel>_<WL>.txt  key metrics of the full capture
  profiles/ncu_traffic.json               bench-launch:* DRAM bytes per captured launch
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")
GO = os.path.join(ROOT, "gpurun_out")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__cycles_elapsed.avg.per_second",
]


def launch_shares(wl, rnd):
    src = os.path.join(GO, f"launches_{wl}.csv")
    shutil.copy(src, os.path.join(OUT, f"{rnd}_launches_{wl}.csv"))
    rows = list(csv.reader(open(src)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list of `python bench.py --workload {wl} --steps 1 --warmup 1` "
             f"(gpu__time_duration.sum, --clock-control none; cold caches, serialised launches:",
             "# compare SHARES, not absolutes). k_philox_bench is bench.py's ALU-roof microbenchmark.",
             f"{'kernel':44s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>10s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k:44s} {v[0]:8d} {v[1] / 1e3:10.3f} {v[1] / v[0]:10.1f} {v[1] / tot:6.3f}")
    no_bench = tot - sum(v[1] for k, v in agg.items() if k.startswith("k_philox_bench"))
    rr = sum(v[1] for k, v in agg.items() if k.startswith("k_rr_warp"))
    lines.append(f"# share of the hot path without the microbenchmark: k_rr_warp {rr / no_bench:.3f}")
    open(os.path.join(OUT, f"{rnd}_launch_shares_{wl}.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full_capture(rep, name, wl, rnd):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else name
    lines = [f"# ncu --set full --clock-control none --import-source on, one launch of {kname}",
             f"# workload {wl} (bench.py --steps 1 --warmup 1)"]
    rec = {}
    for key in KEYS:
        if key in hdr:
            i = hdr.index(key)
            lines.append(f"{key:64s} {vals[i]:>20s} {units[i]}")
            rec[key] = (vals[i], units[i])
    stall = [(h, vals[i]) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
             and not h.endswith("_not_issued")]
    stall = sorted(((h, float(v.replace(",", "") or 0)) for h, v in stall), key=lambda x: -x[1])
    tot = sum(v for _, v in stall) or 1
    lines.append("# warp-state samples (top):")
    for h, v in stall[:8]:
        lines.append(f"  {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {v / tot:6.3f}")
    open(os.path.join(OUT, f"{rnd}_ncu_{name}_{wl}.txt"), "w").write("\n".join(lines) + "\n")

    def as_bytes(v):
        x, u = v
        x = float(x.replace(",", ""))
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    traffic = as_bytes(rec["dram__bytes_read.sum"]) + as_bytes(rec["dram__bytes_write.sum"])
    return traffic


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    wl = sys.argv[2] if len(sys.argv) > 2 else "C3"
    os.makedirs(OUT, exist_ok=True)
    launch_shares(wl, rnd)
    tj = os.path.join(OUT, "ncu_traffic.json")
    traffic = json.load(open(tj)) if os.path.exists(tj) else {}
    for name, rep in [("k_rr_warp", f"prof_rr_{wl}.ncu-rep"), ("k_rr_giant", f"prof_giant_{wl}.ncu-rep"),
                      ("k_cover", f"prof_cover_{wl}.ncu-rep"), ("k_argmax", f"prof_argmax_{wl}.ncu-rep")]:
        p = os.path.join(GO, rep)
        if os.path.exists(p):
            traffic[f"bench-launch:{wl}:{name}"] = full_capture(p, name, wl, rnd)
    traffic["_note"] = ("bench-launch:* = DRAM read+write bytes of ONE captured launch (ncu --set full) "
                        "of the kernel inside bench.py --steps 1 --warmup 1; <WL>:k_rr_warp[:skip] = "
                        "tools/traffic_capture.py (one 2^20-set generate_rr call, paired with the same "
                        "call's algorithmic bytes; what bench.py reports)")
    json.dump(traffic, open(tj, "w"), indent=1)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
