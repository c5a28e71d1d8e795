"""Summarise gpurun_out/sweep_*.jsonl into profiles/<round>_sweeps.md (committed evidence).
  python tools/sweep_table.py r01"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rows(name):
    p = os.path.join(ROOT, "gpurun_out", f"sweep_{name}.jsonl")
    return [json.loads(x) for x in open(p)] if os.path.exists(p) else []


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    out = [f"# Parameter sweeps on one B200 (`python tools/sweep.py <name>`; bench.py, 3 timed IMM runs",
           "after 3 warm-ups, graph resident; `cpu` = the oracle's RR sets/s on one host core, bounded",
           "sample). Reproduces the *shape* of the paper's Figs. 4-7 (P:716-779) on synthetic inputs.", ""]
    for name, title in (("density", "Density sweep: Barabasi-Albert n = 10^6, IC-WC, k = 50, eps = 0.05 (P:754-779)"),
                        ("k", "k sweep, eps = 0.1 (P:744-748)"), ("eps", "eps sweep, C3, k = 50 (P:750)"),
                        ("mrim", "MRIM (CR-NAIMM, Table 3 settings k = 10 per round, T = 5, eps = 0.1; "
                                 "sets = MRIM sets of T reverse BFS each; P:790-822)")):
        rs = rows(name)
        if not rs:
            continue
        out += [f"## {title}", "",
                "| workload | k | eps | IMM ms | rounds | RR sets | RR sets/s | rr / giant / store / inv / select ms | mean set | coins/set | oracle RR sets/s | GPU/oracle |",
                "|---|---|---|---|---|---|---|---|---|---|---|---|"]
        for d in rs:
            if "error" in d:
                out.append(f"| {' '.join(d['point'])} | error: {d['error'][-80:]!r} |")
                continue
            c, ph, st = d["config"], d["phase_ms_per_step"], d["rr_stats"]
            cpu = d.get("cpu_baseline") or {}
            cv = cpu.get("value")
            out.append(f"| {c['workload'].split(':')[0]} | {c['k']} | {c['eps']} | {d['ms_per_step']:.2f} | {d['rounds']} | "
                       f"{d['rr_sets_per_step']:,} | {d['value'] / 1e6:.1f} M | "
                       f"{ph['ms_rr']:.2f} / {ph['ms_giant']:.2f} / {ph['ms_store']:.2f} / {ph['ms_inv']:.2f} / {ph['ms_select']:.2f} | "
                       f"{st['mean_len']:.1f} | {st['coins_per_set']:.0f} | "
                       f"{(f'{cv / 1e3:.1f} K' if cv else '—')} | {(f'{d['value'] / cv:.0f}x' if cv else '—')} |")
        out.append("")
    path = os.path.join(ROOT, "profiles", f"{rnd}_sweeps.md")
    open(path, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
