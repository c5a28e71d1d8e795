import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07325_b200 as P
c = P.Gim(0, torch_allocator=False)
for ch in (1, 4, 8):
    c.set_option(P.OPT_MB_CHAINS, ch)
    best = 0
    for _ in range(3):
        ms = c.microbench_philox(1 << 31)
        best = max(best, 4 * (1 << 31) / (ms / 1e3) / 1e9)
    print(f"chains {ch}: {best:.0f} Gcoin/s")
