import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys, numpy as np, gim_inputs as gi, paper_2009_07325_b200 as P
key = sys.argv[1] if len(sys.argv) > 1 else "C3"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
w = gi.WORKLOADS[key]; g = gi.workload_graph(key)
c = P.Gim(0, torch_allocator=False)
c.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme, p_uniform=w.p_uniform)
c.generate_rr(T, w.rr_seed)
print("generated", c.stats()["giant_sets"], "giants")
s, gn, cov = c.select(w.k)
print("selected", s[:5], cov)
