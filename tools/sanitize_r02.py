"""compute-sanitizer target for the round-2 paths (run under memcheck / racecheck / synccheck):
geometric-skip kernels (lane, warp + spill tier, CTA giant), the shared-memory giant pass and its
hand-over, fused and cooperative selection, the node-sharded protocol at world 1 (host hooks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import gim_inputs as gi  # noqa: E402
import paper_2009_07325_b200 as P  # noqa: E402


def ctx(g, model, scheme, pu=0.0, opts=None):
    c = P.Gim(0, torch_allocator=False)
    c.load_graph(g.n, g.row_ptr, g.src, model, scheme, p_uniform=pu)
    for k, v in (opts or {}).items():
        c.set_option(k, v)
    return c


w = gi.WORKLOADS["C1"]
g = gi.workload_graph("C1")
leaves = 6000
edges = [(i, 0) for i in range(1, leaves + 1)] + [(leaves + 1 + i, leaves + 2 + i) for i in range(300)]
edges += [(leaves + 301, 0)]
star = gi.from_edges(leaves + 302, edges)
for opts in ({P.OPT_SKIP: 1}, {P.OPT_SKIP: 3, P.OPT_QUEUE_CAP: 16, P.OPT_SPILL: 64},
             {P.OPT_SKIP: 1, P.OPT_FORCE_GIANT: 1}, {P.OPT_GIANT_SHARED: 1, P.OPT_QUEUE_CAP: 16},
             {P.OPT_SELECT_FUSED: 2048}, {P.OPT_SELECT_COOP: 2048}, {P.OPT_SELECT_COOP: 1},
             {P.OPT_SKIP: 3, P.OPT_SKIP_LANE_CAP: 100}):
    c = ctx(g, w.model, w.scheme, opts=opts)
    c.generate_rr(6001, 7)
    print(opts, c.select(10)[0][:3], flush=True)
    c.close()
for model, scheme, pu in ((gi.IC, gi.W_UNIFORM, 0.9), (gi.LT, gi.W_WC, 0.0)):
    c = ctx(star, model, scheme, pu, {P.OPT_GIANT_SHARED: 1})
    c.generate_rr(1500, 3)
    print("star", model, c.select(3)[0], flush=True)
    c.close()
# node-sharded protocol at world 1 through device-side hooks (world 1: reduce-scatter = copy)
import torch  # noqa: E402


def view(ptr, count):
    class V:
        __cuda_array_interface__ = {"shape": (int(count),), "typestr": "<i4", "data": (int(ptr), False),
                                    "version": 3, "strides": None, "stream": None}
    return torch.as_tensor(V(), device="cuda")


def rs(send, recv, count, stream):
    with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
        view(recv, count).copy_(view(send, count))
    return 0


c = P.Gim(0, torch_allocator=False)
c.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme)
c.set_shard(0, 1)
c.set_allreduce(lambda ptr, count, stream: 0)           # world 1: SUM over one rank = identity
c.set_reducescatter(rs)
c.set_option(P.OPT_FORCE_COLLECTIVES, 1)
c.generate_rr(6001, 7)
print("rs", c.select(10)[0][:3], flush=True)
