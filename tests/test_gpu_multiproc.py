"""The real multi-process N > 1 path on one GPU: P processes (gloo process group, all on cuda:0),
each holding its RR-id slices, exchanging through the binding's torch.distributed callbacks —
the same callbacks that run NCCL on a multi-GPU node (their NCCL data plane is exercised by
tests/test_gpu_multirank.py::test_nccl_world1_protocols). Every rank must return the ORACLE's
seeds, gains and IMM, and hold exactly the oracle's RR sets of its slice (element by element)."""
import os
import socket

import numpy as np
import pytest

import gim_inputs as gi
import oracle

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, key, T, k, proto):
    import torch.distributed as dist
    import paper_2009_07325_b200 as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    c = P.Gim(0)
    c.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme)
    c.set_shard(rank, world)
    c.set_allreduce(P.torch_allreduce())
    if proto == "allgather":
        c.set_allgather(P.torch_allgather())
    elif proto == "reducescatter":
        c.set_reducescatter(P.torch_reducescatter())
    c.generate_rr(T, w.rr_seed)
    seeds, gains, cov = c.select(k)
    ids, off, nodes = c.rr_export(sort_each_set=True)
    r = c.imm(k, w.eps, w.ell, w.rr_seed)
    q.put((rank, seeds.tolist(), gains.tolist(), cov, ids, off, nodes, r.seeds.tolist(), r.R_final, r.LB))
    dist.destroy_process_group()


@pytest.mark.parametrize("proto", ["allreduce", "allgather", "reducescatter"])
@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_vs_oracle(world, proto):
    import torch.multiprocessing as mp
    import paper_2009_07325_b200 as P
    key, T, k = "C2", 40009, 30
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    o = oracle.Oracle(g, w.model, w.scheme)
    o.generate(T, w.rr_seed)
    ooff, onodes, _ = o.export()
    oseeds, ogains, ocov = o.select(k)
    oimm = oracle.Oracle(g, w.model, w.scheme).imm(k, w.eps, w.ell, w.rr_seed)
    import torch
    if torch.cuda.is_initialized():          # cached memory of earlier tests back to the device
        torch.cuda.empty_cache()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, key, T, k, proto)) for r in range(world)]
    [p.start() for p in procs]
    out = sorted([q.get(timeout=600) for _ in range(world)], key=lambda x: x[0])
    [p.join(120) for p in procs]
    for rank, seeds, gains, cov, ids, off, nodes, iseeds, R, LB in out:
        assert seeds == oseeds.tolist() and gains == ogains.tolist() and cov == ocov
        lo, hi = (0, T) if proto == "allgather" else P.shard_slice(0, T, rank, world)
        assert np.array_equal(ids, np.arange(lo, hi, dtype=np.uint64))
        assert np.array_equal(off - off[0], ooff[lo:hi + 1] - ooff[lo])
        assert np.array_equal(nodes[off[0]:off[-1]], onodes[ooff[lo]:ooff[hi]])   # element by element
        assert iseeds == oimm.seeds.tolist() and R == oimm.R_final
        assert abs(LB - oimm.LB) <= 1e-12 * oimm.LB
