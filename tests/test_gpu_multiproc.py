"""The real multi-process N > 1 path on one GPU: P processes (gloo process group, all on cuda:0)
each hold their RR-id slices and all-reduce counts / decrements through the binding's
torch.distributed callback; every rank must return the single-process seeds, gains and pool
slice (the library's NCCL path differs only in the backend of the same callback)."""
import os
import socket

import numpy as np
import pytest

import gim_inputs as gi

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, key, T, k, replicated=False):
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
    if replicated:
        c.set_allgather(P.torch_allgather())
    c.generate_rr(T, w.rr_seed)
    seeds, gains, cov = c.select(k)
    ids, off, nodes = c.rr_export()
    r = c.imm(k, w.eps, w.ell, w.rr_seed)
    q.put((rank, seeds.tolist(), gains.tolist(), cov, int(ids[0]) if len(ids) else -1, len(ids),
           int(np.sum(nodes.astype(np.uint64))), r.seeds.tolist(), r.R_final, r.LB))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_shards_equal_single(world):
    import torch.multiprocessing as mp
    import paper_2009_07325_b200 as P
    key, T, k = "C2", 40009, 30
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    ref = P.Gim(0)
    ref.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme)
    ref.generate_rr(T, w.rr_seed)
    rs, rg, rc = ref.select(k)
    _, roff, rnodes = ref.rr_export()
    rimm = ref.imm(k, w.eps, w.ell, w.rr_seed)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, key, T, k)) for r in range(world)]
    [p.start() for p in procs]
    out = sorted([q.get(timeout=600) for _ in range(world)])
    [p.join(120) for p in procs]
    for rank, seeds, gains, cov, id0, nids, nsum, iseeds, R, LB in out:
        assert seeds == rs.tolist() and gains == rg.tolist() and cov == rc
        lo, hi = P.shard_slice(0, T, rank, world)
        assert id0 == lo and nids == hi - lo
        assert nsum == int(np.sum(rnodes[roff[lo]:roff[hi]].astype(np.uint64)))
        assert iseeds == rimm.seeds.tolist() and R == rimm.R_final and LB == rimm.LB


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_replicated_pool_equals_single(world):
    """The replicated-pool protocol through torch.distributed (gloo, all ranks on cuda:0): each
    rank ends with the whole P = 1 pool and returns the P = 1 selection and IMM."""
    import torch.multiprocessing as mp
    import paper_2009_07325_b200 as P
    key, T, k = "C2", 40009, 30
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    ref = P.Gim(0)
    ref.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme)
    ref.generate_rr(T, w.rr_seed)
    rs, rg, rc = ref.select(k)
    _, roff, rnodes = ref.rr_export()
    rimm = ref.imm(k, w.eps, w.ell, w.rr_seed)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, key, T, k, True)) for r in range(world)]
    [p.start() for p in procs]
    out = sorted([q.get(timeout=600) for _ in range(world)])
    [p.join(120) for p in procs]
    for rank, seeds, gains, cov, id0, nids, nsum, iseeds, R, LB in out:
        assert seeds == rs.tolist() and gains == rg.tolist() and cov == rc
        assert id0 == 0 and nids == T
        assert nsum == int(np.sum(rnodes.astype(np.uint64)))
        assert iseeds == rimm.seeds.tolist() and R == rimm.R_final and LB == rimm.LB
