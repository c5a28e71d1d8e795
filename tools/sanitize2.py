"""compute-sanitizer driver for the round's new paths: MRIM generate/select (T=3), forward MC
(IC and LT), narrow giant CTAs, fresh-final IMM, persistent selection. Small sizes.
  compute-sanitizer --tool memcheck python tools/sanitize2.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gim_inputs as gi  # noqa: E402
import paper_2009_07325_b200 as P  # noqa: E402

w = gi.WORKLOADS["C1"]
g = gi.workload_graph("C1")
for model in (gi.IC, gi.LT):
    c = P.Gim(0, torch_allocator=False)
    c.load_graph(g.n, g.row_ptr, g.src, model, w.scheme)
    c.set_option(P.OPT_GIANT_NT, 128)
    c.set_option(P.OPT_QUEUE_CAP, 16)
    c.generate_rr(3000, w.rr_seed)
    s, gn, cov = c.select(10)
    print("model", model, "select", s[:4].tolist(), cov)
    print("mc", c.mc_spread(s, 50, 3))
    c.set_option(P.OPT_FRESH_FINAL, 1)
    c.set_option(P.OPT_SELECT_PERSISTENT, 1)
    r = c.imm(10, 0.5, 1.0, w.rr_seed)
    print("imm fresh+persistent", r.seeds[:4].tolist(), r.R_final)
    c.set_rounds(3)
    c.set_option(P.OPT_SELECT_PERSISTENT, 0)
    c.generate_rr(1000, w.rr_seed)
    s, gn, cov = c.select(5)
    print("mrim", s[:4].tolist(), cov)
    c.close()
print("done")
