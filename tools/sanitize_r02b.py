"""compute-sanitizer target for the late round-2 paths (run under memcheck / racecheck /
synccheck): IMM with the bounded greedy + first-step probe + lazily merged index segments (C1,
IC and LT, and MRIM), the single-CTA selection (incl. a truncated pool), the sort-based index
segments, the candidate argmax with its certificate failure + full-scan redo (k = n), the step
graphs, and multi-chunk generation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import gim_inputs as gi  # noqa: E402
import paper_2009_07325_b200 as P  # noqa: E402


def ctx(g, model, scheme, opts=None):
    c = P.Gim(0, torch_allocator=False)
    c.load_graph(g.n, g.row_ptr, g.src, model, scheme)
    for k, v in (opts or {}).items():
        c.set_option(k, v)
    return c


w = gi.WORKLOADS["C1"]
g = gi.workload_graph("C1")
for model in (gi.IC, gi.LT):
    for opts in ({}, {P.OPT_SELECT_CTA: 0}, {P.OPT_INV_SORT: 1, P.OPT_CHUNK: 4096},
                 {P.OPT_ARGMAX_CAND: 2, P.OPT_SELECT_CTA: 0}):
        c = ctx(g, model, w.scheme, opts)
        r = c.imm(w.k, w.eps, w.ell, w.rr_seed)
        print(model, opts, r.seeds[:3], r.sel_steps_i.tolist(), flush=True)
        c.close()
c = ctx(g, gi.IC, w.scheme, {P.OPT_ARGMAX_CAND: 2, P.OPT_SELECT_CTA: 0})
c.generate_rr(3001, 5)
print("k = n", c.select(g.n)[1][-3:], c.stats()["fused_fallbacks"], flush=True)
c.generate_rr(9000, 5)
c.generate_rr(6000, 5)                             # truncation: cut sets skipped by the cover
print("truncated", c.select(20)[0][:3], flush=True)
c.close()
c = ctx(g, gi.IC, w.scheme)
c.set_rounds(3)
r = c.imm(5, 0.5, 1.0, 3)
print("mrim", r.seeds[:3], r.sel_steps_i.tolist(), flush=True)
c.close()
