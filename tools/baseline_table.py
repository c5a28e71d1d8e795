"""Print BASELINE.md §4's results table from the committed bench lines (profiles/r02_bench_<cfg>.json)
and the oracle goldens (tests/golden/imm_<cfg>.json)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {"C1": "C1 NetHEPT-shaped, IC-WC, k=50, ε=0.5", "C2": "C2 Epinions-shaped, IC-WC, k=50, ε=0.1",
         "C3": "C3 LJ-shaped, IC-WC, k=50, ε=0.1", "C4": "C4 LJ-shaped, LT-WC, k=50, ε=0.1",
         "C5": "C5 Twitter-shaped, IC p=0.01, k=100, ε=0.1"}
print("| Config | IMM time (resident) | RR sets per IMM | RR sets/s | phase split rr / giant / store / index / "
      "select (ms) | dominant-kernel roofline | e2e (graph upload + IMM) | geometric-skip variant (R31) | "
      "oracle full IMM (1 core) | seeds vs oracle |")
print("|---|---|---|---|---|---|---|---|---|---|")
for cfg, name in NAMES.items():
    d = json.load(open(os.path.join(ROOT, "profiles", f"r02_bench_{cfg}.json")))
    gd = json.load(open(os.path.join(ROOT, "tests", "golden", f"imm_{cfg}.json")))
    ph = d["phase_ms_per_step"]
    split = " / ".join(f"{ph[k]:.2f}" for k in ("ms_rr", "ms_giant", "ms_store", "ms_inv", "ms_select"))
    rf = d["roofline"]
    roof = f"{rf['achieved']:.0f} {rf['unit']} = {100 * rf['frac']:.1f}% ({rf['bound']})"
    e2e = f"{d['e2e']['ms_per_step']:.1f} ms" if d.get("e2e") else "—"
    sk = (d.get("variants") or {}).get("geometric_skip")
    skip = f"{sk['ms_per_step']:.1f} ms ({sk['phase_ms_per_step']['ms_rr']:.2f} ms sampling)" if sk else "— (LT)"
    print(f"| {name} | {d['ms_per_step']:.2f} ms | {d['rr_sets_per_step']:,} | {d['value'] / 1e6:.1f} M/s | {split} | "
          f"{roof} | {e2e} | {skip} | {gd['oracle_run']['imm_s']:.1f} s | bit-exact, full IMM (golden) |")
