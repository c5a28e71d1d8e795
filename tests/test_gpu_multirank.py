"""The world > 1 exchange protocols on the CUDA path (include/gim.h),
compared with the ORACLE — never with another GPU run.

The paper is single-GPU (§4.2); the data-parallel split is this build's: RR-id
slices per rank against a replicated graph, and the counter-based greedy of §3.8
distributed three ways:
  * "allreduce"      dense count / per-step decrement SUM all-reduce (north_star's protocol);
  * "allgather"      replicated pool: each round's sets all-gathered, selection local;
  * "reducescatter"  node-sharded selection: shard counts reduce-scattered, per-step key
                     exchange, decrements reduce-scattered to the shard owners.
Every emulated rank (one context and one host thread per rank, collectives staged through host
memory) must return the oracle's seeds, gains and covered count (O7), hold exactly the oracle's
RR sets of its slice (or of the whole pool when replicated, O6), and reproduce the oracle's IMM
(Alg. 2). The NCCL data plane of the same callbacks is driven on one GPU by a world-1
NCCL process group with GIM_OPT_FORCE_COLLECTIVES (test_nccl_world1_protocols)."""
import os
import socket
import threading

import numpy as np
import pytest

import gim_inputs as gi
import oracle

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2009_07325_b200")


def _view(ptr, n, typestr):
    import torch

    class V:
        __cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                    "version": 3, "strides": None, "stream": None}
    return torch.as_tensor(V(), device="cuda")


class HostCollectives:
    """Host-staged collectives among Pn threads (one per emulated rank)."""

    def __init__(self, Pn):
        self.Pn = Pn
        self.bar = threading.Barrier(Pn)
        self.parts = [None] * Pn

    def _exchange(self, r, t):
        self.parts[r] = t
        self.bar.wait()
        allp = list(self.parts)
        self.bar.wait()
        return allp

    def allreduce(self, r):
        import torch

        def cb(ptr, count, stream):
            torch.cuda.ExternalStream(stream).synchronize()
            t = _view(ptr, count, "<i4")
            tot = sum(self._exchange(r, t.cpu()))
            t.copy_(tot.cuda())
            torch.cuda.synchronize()
            return 0
        return cb

    def allgather(self, r):
        import torch

        def cb(send, nbytes, recv, stream):
            torch.cuda.ExternalStream(stream).synchronize()
            allp = torch.cat(self._exchange(r, _view(send, nbytes, "|u1").cpu()))
            _view(recv, nbytes * self.Pn, "|u1").copy_(allp.cuda())
            torch.cuda.synchronize()
            return 0
        return cb

    def reducescatter(self, r):
        import torch

        def cb(send, recv, count, stream):
            torch.cuda.ExternalStream(stream).synchronize()
            tot = sum(self._exchange(r, _view(send, count * self.Pn, "<i4").cpu()))
            _view(recv, count, "<i4").copy_(tot[r * count:(r + 1) * count].cuda())
            torch.cuda.synchronize()
            return 0
        return cb


def _setup(c, proto, coll, r):
    c.set_allreduce(coll.allreduce(r))
    if proto == "allgather":
        c.set_allgather(coll.allgather(r))
    elif proto == "reducescatter":
        c.set_reducescatter(coll.reducescatter(r))


def _sorted_sets(off, nodes):
    return [np.sort(nodes[off[i]:off[i + 1]]) for i in range(len(off) - 1)]


def _check_slice(ids, off, nodes, ooff, onodes, lo, hi):
    assert np.array_equal(ids, np.arange(lo, hi, dtype=np.uint64))
    assert np.array_equal(off - off[0], ooff[lo:hi + 1] - ooff[lo]), "set sizes"
    got = _sorted_sets(off, nodes)
    for i in range(hi - lo):                                    # element by element
        assert np.array_equal(got[i], onodes[ooff[lo + i]:ooff[lo + i + 1]]), lo + i


@pytest.mark.parametrize("proto", ["allreduce", "allgather", "reducescatter"])
@pytest.mark.parametrize("Pn", [2, 3])
def test_protocol_emulation_vs_oracle(proto, Pn):
    w = gi.WORKLOADS["C2"]
    g = gi.workload_graph("C2")
    T, k = 30011, 30
    o = oracle.Oracle(g, w.model, w.scheme)
    o.generate(T, w.rr_seed)
    ooff, onodes, ocnt = o.export()
    oseeds, ogains, ocov = o.select(k)
    oimm = oracle.Oracle(g, w.model, w.scheme).imm(k, w.eps, w.ell, w.rr_seed)
    coll = HostCollectives(Pn)
    ctxs = []
    for r in range(Pn):
        c = P.Gim(0)
        c.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme)
        c.set_shard(r, Pn)
        _setup(c, proto, coll, r)
        ctxs.append(c)
    out = [None] * Pn

    def run(r):
        c = ctxs[r]
        for t in (1000, T):                                     # two rounds: two slices per rank
            c.generate_rr(t, w.rr_seed)
        sel = c.select(k)
        exp = c.rr_export(sort_each_set=True)
        cnt = c.counts_export()
        imm = c.imm(k, w.eps, w.ell, w.rr_seed)
        out[r] = (sel, exp, cnt, imm)

    th = [threading.Thread(target=run, args=(r,)) for r in range(Pn)]
    [t.start() for t in th]
    [t.join() for t in th]
    for r in range(Pn):
        (seeds, gains, cov), (ids, off, nodes), cnt, imm = out[r]
        assert seeds.tolist() == oseeds.tolist() and gains.tolist() == ogains.tolist() and cov == ocov
        if proto == "allgather":                                # the whole pool, global id order
            _check_slice(ids, off, nodes, ooff, onodes, 0, T)
            assert np.array_equal(cnt, ocnt)
        else:                                                   # this rank's slice of each round
            parts = [P.shard_slice(0, 1000, r, Pn), P.shard_slice(1000, T, r, Pn)]
            b = 0
            for lo, hi in parts:
                ln = hi - lo
                _check_slice(ids[b:b + ln], off[b:b + ln + 1], nodes, ooff, onodes, lo, hi)
                b += ln
        assert imm.seeds.tolist() == oimm.seeds.tolist() and imm.R_final == oimm.R_final
        assert imm.covered == oimm.cov and imm.rounds == oimm.rounds
        assert abs(imm.LB - oimm.LB) <= 1e-12 * oimm.LB


@pytest.mark.parametrize("proto", ["allreduce", "allgather"])
def test_mrim_protocol_emulation_vs_oracle(proto):
    """MRIM (R26-R28) under P = 2: whole MRIM sets per rank; the oracle's pair seeds and IMM."""
    w = gi.WORKLOADS["C1"]
    g = gi.workload_graph("C1")
    Tr, k, N = 3, 10, 4001
    o = oracle.Oracle(g, w.model, w.scheme)
    o.mrim_generate(N, Tr, w.rr_seed)
    oseeds, ogains, ocov = o.mrim_select(k)
    oimm = oracle.Oracle(g, w.model, w.scheme).mrim(k, Tr, w.eps, w.ell, w.rr_seed)
    Pn = 2
    coll = HostCollectives(Pn)
    out = [None] * Pn
    ctxs = []
    for r in range(Pn):
        c = P.Gim(0)
        c.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme)
        c.set_rounds(Tr)
        c.set_shard(r, Pn)
        _setup(c, proto, coll, r)
        ctxs.append(c)

    def run(r):
        c = ctxs[r]
        c.generate_rr(N, w.rr_seed)
        out[r] = (c.select(k), c.imm(k, w.eps, w.ell, w.rr_seed))

    th = [threading.Thread(target=run, args=(r,)) for r in range(Pn)]
    [t.start() for t in th]
    [t.join() for t in th]
    for r in range(Pn):
        (seeds, gains, cov), imm = out[r]
        assert seeds.tolist() == oseeds.tolist() and gains.tolist() == ogains.tolist() and cov == ocov
        assert imm.seeds.tolist() == oimm.seeds.tolist() and imm.R_final == oimm.R_final


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_world1_protocols():
    """The binding's NCCL callbacks (torch.distributed all_reduce / all_gather_into_tensor /
    reduce_scatter_tensor on the library's stream) driven for real: a world-1 NCCL process group
    with GIM_OPT_FORCE_COLLECTIVES runs each exchange protocol's code path; results equal the
    oracle's."""
    import torch
    import torch.distributed as dist
    if not dist.is_nccl_available():
        pytest.skip("no NCCL in this torch build")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        w = gi.WORKLOADS["C2"]
        g = gi.workload_graph("C2")
        T, k = 20011, 20
        o = oracle.Oracle(g, w.model, w.scheme)
        o.generate(T, w.rr_seed)
        oseeds, ogains, ocov = o.select(k)
        oimm = oracle.Oracle(g, w.model, w.scheme).imm(k, w.eps, w.ell, w.rr_seed)
        for proto in ("allreduce", "allgather", "reducescatter"):
            stream = torch.cuda.Stream(0)
            c = P.Gim(0, stream=stream.cuda_stream)
            c.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme)
            c.set_shard(0, 1)
            c.set_allreduce(P.torch_allreduce())
            if proto == "allgather":
                c.set_allgather(P.torch_allgather())
            elif proto == "reducescatter":
                c.set_reducescatter(P.torch_reducescatter())
            c.set_option(P.OPT_FORCE_COLLECTIVES, 1)
            c.reset_stats()
            c.generate_rr(T, w.rr_seed)
            seeds, gains, cov = c.select(k)
            assert c.stats()["allreduces"] > 0, proto             # the callbacks did run
            assert seeds.tolist() == oseeds.tolist() and gains.tolist() == ogains.tolist() and cov == ocov
            r = c.imm(k, w.eps, w.ell, w.rr_seed)
            assert r.seeds.tolist() == oimm.seeds.tolist() and r.R_final == oimm.R_final, proto
            c.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("proto", ["allreduce", "replicated", "reducescatter"])
def test_native_nccl_world1_protocols(proto):
    """The library's own NCCL communicator (gim_set_nccl: collectives issued by libgim on its
    stream, no Python per step) at world 1 with GIM_OPT_FORCE_COLLECTIVES: every protocol's code
    path runs through real NCCL collectives and the results equal the oracle's (the RR sets of the
    pool element by element, the selection, the full IMM)."""
    w = gi.WORKLOADS["C2"]
    g = gi.workload_graph("C2")
    T, k = 20011, 20
    o = oracle.Oracle(g, w.model, w.scheme)
    o.generate(T, w.rr_seed)
    ooff, onodes, _ = o.export()
    oseeds, ogains, ocov = o.select(k)
    oimm = oracle.Oracle(g, w.model, w.scheme).imm(k, w.eps, w.ell, w.rr_seed)
    c = P.Gim(0)
    c.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme)
    c.set_shard(0, 1)
    P.setup_nccl(c, 0, 1, proto)
    c.set_option(P.OPT_FORCE_COLLECTIVES, 1)
    c.reset_stats()
    c.generate_rr(T, w.rr_seed)
    ids, off, nodes = c.rr_export(sort_each_set=True)
    assert np.array_equal(off, ooff) and np.array_equal(nodes, onodes)
    seeds, gains, cov = c.select(k)
    assert c.stats()["allreduces"] > 0 or proto == "replicated"
    assert seeds.tolist() == oseeds.tolist() and gains.tolist() == ogains.tolist() and cov == ocov
    r = c.imm(k, w.eps, w.ell, w.rr_seed)
    assert r.seeds.tolist() == oimm.seeds.tolist() and r.R_final == oimm.R_final and r.LB == oimm.LB, proto
    c.close()


def test_native_nccl_errors():
    """gim_set_nccl validates its arguments before touching NCCL: rank / world must match
    gim_set_shard, the protocol must be 0..2, an id is required."""
    g = gi.workload_graph("C1")
    w = gi.WORKLOADS["C1"]
    c = P.Gim(0)
    c.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme)
    c.set_shard(0, 1)
    nid = P.nccl_unique_id()
    assert len(nid) == 128
    with pytest.raises(P.GimError, match="GIM_EINVAL"):
        c.set_nccl(nid, 0, 2, "allreduce")             # world differs from gim_set_shard
    with pytest.raises(KeyError):
        c.set_nccl(nid, 0, 1, "bogus")
    c.set_nccl(nid, 0, 1, "replicated")                # valid: a world-1 communicator
    c.close()
