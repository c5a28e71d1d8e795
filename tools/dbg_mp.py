import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, gim_inputs as gi
import paper_2009_07325_b200 as P
key, T, k = "C2", 40009, 30
w = gi.WORKLOADS[key]; g = gi.workload_graph(key)
ref = P.Gim(0, torch_allocator=(sys.argv[1] == "1"))
ref.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme)
ref.generate_rr(T, w.rr_seed)
try:
    print(ref.select(k)[2])
except Exception as e:
    print("ERR", e)
