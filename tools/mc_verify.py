"""Monte-Carlo verification of IMM's seeds at full size (north_star: "Monte-Carlo-verified spread
within 1%"): GPU IMM, then the forward-MC spread of its seeds (gim_mc_spread) against
n * F_R'(S) on an independent RR pool R' (2^21 sets, another seed; reading R24). One JSON line
per workload to gpurun_out/mc_verify.jsonl.
  python tools/mc_verify.py C3 C5"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gim_inputs as gi  # noqa: E402
import paper_2009_07325_b200 as P  # noqa: E402


def main():
    out = open(os.path.join(ROOT, "gpurun_out", "mc_verify.jsonl"), "a")
    for key in [a for a in sys.argv[1:] if not a.startswith("--")]:
        w = gi.WORKLOADS[key]
        g = gi.workload_graph(key)
        c = P.Gim(0)
        c.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme, weights=g.weights, p_uniform=w.p_uniform)
        r = c.imm(w.k, w.eps, w.ell, w.rr_seed)
        T = 1 << (25 if key == "C5" else 21)   # C5: F ~ 0.9%, needs ~2^25 sets for a 0.3% RIS error
        c2 = P.Gim(0)
        c2.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme, weights=g.weights, p_uniform=w.p_uniform)
        c2.generate_rr(T, w.rr_seed + 1)
        ids, off, nodes = c2.rr_export(sort_each_set=False)
        member = np.isin(nodes, r.seeds)
        hit = np.zeros(T, dtype=bool)
        hit[np.repeat(np.arange(T), np.diff(off.astype(np.int64)))[member]] = True
        ris = g.n * hit.mean()
        ris_se = g.n * np.sqrt(hit.mean() * (1 - hit.mean()) / T)
        t0 = time.perf_counter()
        if "--host-lt" not in sys.argv or w.model == gi.IC:
            trials, mc_impl = 2000, "gpu gim_mc_spread"
            mean, se = c.mc_spread(r.seeds, trials, 17)
        else:   # LT with the oracle's forward MC on the host (single-threaded, bounded trials)
            import oracle
            trials, mc_impl = 400, "oracle og_mc_spread (host)"
            mean, se = oracle.Oracle(g, w.model, w.scheme, w.p_uniform).mc_spread(r.seeds, trials, 17)
        mc_s = time.perf_counter() - t0
        line = {"workload": key, "k": w.k, "eps": w.eps, "R_final": r.R_final,
                "spread_est_imm_pool": r.spread_est, "ris_independent_pool": ris, "ris_stderr": ris_se,
                "mc_impl": mc_impl, "mc_trials": trials, "mc_mean": mean, "mc_stderr": se, "mc_seconds_incl_out_csr": mc_s,
                "rel_diff_mc_vs_ris": abs(mean - ris) / mean}
        print(json.dumps(line), flush=True)
        out.write(json.dumps(line) + "\n")
        c.close()
        c2.close()


if __name__ == "__main__":
    main()
