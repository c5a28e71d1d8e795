"""Multi-process (world_size 2 and 3, gloo on CPU) tests of the N > 1 host logic: the collective
callback plumbing of the binding (all-reduce, all-gather, reduce-scatter), the RR-id slicing, and
HOST EMULATIONS of the library's exchange protocols — dense count/decrement all-reduce per greedy
step, node-sharded reduce-scatter selection, replicated-pool round all-gather — executed here on
oracle pools split by rank, which must reproduce the oracle's single-process selection / pool.
(The library's own implementation of the protocols is checked on the GPU against the oracle by
tests/test_gpu_multirank.py and tests/test_gpu_multiproc.py.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gim_inputs as gi


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_callback(rank, world, port, q):
    _init(rank, world, port)
    import paper_2009_07325_b200 as P
    fn = P.torch_allreduce(device="cpu")
    buf = np.arange(10, dtype=np.int32) * (rank + 1)
    rc = fn(buf.ctypes.data, len(buf), 0)
    q.put((rank, rc, buf.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_allreduce_callback_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker_callback, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in procs]
    out = [q.get(timeout=120) for _ in range(world)]
    [p.join(60) for p in procs]
    tot = sum(range(1, world + 1))
    for rank, rc, buf in out:
        assert rc == 0 and buf == [i * tot for i in range(10)]


def test_shard_slices_partition():
    from paper_2009_07325_b200 import shard_slice
    for a, b in [(0, 10), (5, 6), (100, 1000003), (7, 7)]:
        for world in (1, 2, 3, 8):
            parts = [shard_slice(a, b, r, world) for r in range(world)]
            assert parts[0][0] == a and parts[-1][1] == b
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))


def _sharded_select(rank, world, port, q, key, T, k):
    """The library's P > 1 selection protocol, on the oracle pool slices of this rank."""
    _init(rank, world, port)
    import oracle
    from paper_2009_07325_b200 import shard_slice
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    o = oracle.Oracle(g, w.model, w.scheme)
    o.generate(T, w.rr_seed)
    off, nodes, _ = o.export()
    lo, hi = shard_slice(0, T, rank, world)
    sets = [nodes[off[i]:off[i + 1]] for i in range(lo, hi)]
    local = np.zeros(g.n, dtype=np.int64)
    for s in sets:
        local[s] += 1
    cnt = torch.from_numpy(local.copy())
    dist.all_reduce(cnt)                                   # count: once per selection
    cnt = cnt.numpy()
    inv = {}
    for r, s in enumerate(sets):
        for v in s:
            inv.setdefault(int(v), []).append(r)
    covered = np.zeros(len(sets), dtype=bool)
    selected = np.zeros(g.n, dtype=bool)
    seeds, gains = [], []
    for _ in range(k):
        key_ = np.where(selected, -1, cnt)
        u = int(np.argmax(key_))                           # lowest id among maxima
        seeds.append(u)
        gains.append(int(cnt[u]))
        selected[u] = True
        dec = np.zeros(g.n, dtype=np.int64)
        for r in inv.get(u, []):
            if not covered[r]:
                covered[r] = True
                dec[sets[r]] += 1
        d = torch.from_numpy(dec)
        dist.all_reduce(d)                                  # decrement: once per step
        cnt = cnt - d.numpy()
    q.put((rank, seeds, gains))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_selection_protocol_equals_single(world):
    import oracle
    key, T, k = "C1", 20000, 20
    w = gi.WORKLOADS[key]
    o = oracle.Oracle(gi.workload_graph(key), w.model, w.scheme)
    o.generate(T, w.rr_seed)
    rs, rg, _ = o.select(k)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_sharded_select, args=(r, world, port, q, key, T, k)) for r in range(world)]
    [p.start() for p in procs]
    out = [q.get(timeout=300) for _ in range(world)]
    [p.join(60) for p in procs]
    for rank, seeds, gains in out:
        assert seeds == rs.tolist() and gains == rg.tolist()


def _worker_allgather(rank, world, port, q):
    _init(rank, world, port)
    import paper_2009_07325_b200 as P
    fn = P.torch_allgather(device="cpu")
    send = (np.arange(6, dtype=np.uint8) + 10 * rank)
    recv = np.zeros(6 * world, dtype=np.uint8)
    rc = fn(send.ctypes.data, send.nbytes, recv.ctypes.data, 0)
    q.put((rank, rc, recv.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_allgather_callback_gloo(world):
    """The replicated-pool protocol's all-gather callback (binding plumbing): every rank receives
    all ranks' bytes in rank order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker_allgather, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in procs]
    out = sorted(q.get(timeout=120) for _ in range(world))
    [p.join(60) for p in procs]
    want = [int(x) for r in range(world) for x in (np.arange(6) + 10 * r)]
    for rank, rc, recv in out:
        assert rc == 0 and recv == want


def _replicated_round_protocol(rank, world, port, q, T, key):
    """Host emulation of replicate_round (gim_api.cu) on oracle pools: each rank holds its slice of
    RR ids, exchanges element counts, all-gathers sizes and elements padded to the largest slice,
    and rebuilds the global pool in rank order."""
    _init(rank, world, port)
    import oracle
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    o = oracle.Oracle(g, w.model, w.scheme)
    o.generate(T, w.rr_seed)
    off, nodes, _ = o.export()
    lo, hi = rank * T // world, (rank + 1) * T // world
    sizes = np.diff(off[lo:hi + 1]).astype(np.uint32)
    elems = nodes[off[lo]:off[hi]].astype(np.uint32)
    L = torch.tensor([len(elems)], dtype=torch.int64)
    Ls = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(Ls, L)
    Ls = [int(x) for x in Ls]
    S = [(r + 1) * T // world - r * T // world for r in range(world)]
    maxL, maxS = max(Ls), max(S)
    ps = np.zeros(maxS, dtype=np.uint32); ps[:len(sizes)] = sizes
    pe = np.zeros(maxL, dtype=np.uint32); pe[:len(elems)] = elems
    gs = [torch.zeros(maxS, dtype=torch.int64) for _ in range(world)]
    ge = [torch.zeros(maxL, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gs, torch.from_numpy(ps.astype(np.int64)))
    dist.all_gather(ge, torch.from_numpy(pe.astype(np.int64)))
    all_sizes = np.concatenate([gs[r].numpy()[:S[r]] for r in range(world)])
    all_elems = np.concatenate([ge[r].numpy()[:Ls[r]] for r in range(world)])
    q.put((rank, np.array_equal(np.concatenate([[0], np.cumsum(all_sizes)]), off.astype(np.int64)),
           np.array_equal(all_elems, nodes.astype(np.int64))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_replicated_round_host_emulation(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_replicated_round_protocol, args=(r, world, port, q, 5003, "C1"))
             for r in range(world)]
    [p.start() for p in procs]
    out = sorted(q.get(timeout=300) for _ in range(world))
    [p.join(60) for p in procs]
    for rank, off_ok, elems_ok in out:
        assert off_ok and elems_ok, rank


def _worker_reducescatter(rank, world, port, q):
    _init(rank, world, port)
    import paper_2009_07325_b200 as P
    fn = P.torch_reducescatter(device="cpu")
    send = (np.arange(4 * world, dtype=np.int32) + 100 * rank)
    recv = np.zeros(4, dtype=np.int32)
    rc = fn(send.ctypes.data, recv.ctypes.data, 4, 0)
    q.put((rank, rc, recv.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_reducescatter_callback_gloo(world):
    """The node-sharded protocol's reduce-scatter callback: rank r receives the SUM over ranks of
    block r."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker_reducescatter, args=(r, world, port, q)) for r in range(world)]
    [p.start() for p in procs]
    out = sorted(q.get(timeout=120) for _ in range(world))
    [p.join(60) for p in procs]
    for rank, rc, recv in out:
        want = [sum(4 * rank + i + 100 * r for r in range(world)) for i in range(4)]
        assert rc == 0 and recv == want


def _node_sharded_select(rank, world, port, q, key, T, k):
    """Host emulation of select_launch_rs (gim_api.cu): node shards of ceil(n / world); counts
    reduce-scattered once; per step the shard argmax, the key exchange (one slot per rank, SUM),
    the local cover and the decrements reduce-scattered to the owners."""
    _init(rank, world, port)
    import oracle
    from paper_2009_07325_b200 import shard_slice
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    o = oracle.Oracle(g, w.model, w.scheme)
    o.generate(T, w.rr_seed)
    off, nodes, _ = o.export()
    lo, hi = shard_slice(0, T, rank, world)
    sets = [nodes[off[i]:off[i + 1]] for i in range(lo, hi)]
    n = g.n
    ns = -(-n // world)
    local = np.zeros(ns * world, dtype=np.int64)
    for s_ in sets:
        local[s_] += 1
    full = torch.from_numpy(local)
    dist.all_reduce(full)                                  # reduce-scatter = all-reduce + own block
    gshard = full.numpy()[rank * ns:(rank + 1) * ns].copy()
    valid = max(0, min(ns, n - rank * ns))
    inv = {}
    for r, s_ in enumerate(sets):
        for v in s_:
            inv.setdefault(int(v), []).append(r)
    covered = np.zeros(len(sets), dtype=bool)
    selected = np.zeros(ns, dtype=bool)
    seeds, gains = [], []
    for _ in range(k):
        key_ = 0
        if valid:
            c = np.where(selected[:valid], -1, gshard[:valid])
            i = int(np.argmax(c))                            # lowest id among maxima
            if c[i] >= 0:
                key_ = (int(c[i]) << 32) | (0xFFFFFFFF - (rank * ns + i))
        kx = torch.zeros(world, dtype=torch.int64)
        kx[rank] = key_
        dist.all_reduce(kx)                                  # key exchange: one slot per rank
        best = int(kx.max())
        u = 0xFFFFFFFF - (best & 0xFFFFFFFF)
        seeds.append(u)
        gains.append(best >> 32)
        if rank * ns <= u < rank * ns + valid:
            selected[u - rank * ns] = True
        dec = np.zeros(ns * world, dtype=np.int64)
        for r in inv.get(u, []):
            if not covered[r]:
                covered[r] = True
                dec[sets[r]] += 1
        d = torch.from_numpy(dec)
        dist.all_reduce(d)
        gshard -= d.numpy()[rank * ns:(rank + 1) * ns]
    q.put((rank, seeds, gains))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_node_sharded_protocol_host_emulation(world):
    import oracle
    key, T, k = "C1", 20000, 20
    w = gi.WORKLOADS[key]
    o = oracle.Oracle(gi.workload_graph(key), w.model, w.scheme)
    o.generate(T, w.rr_seed)
    rs, rg, _ = o.select(k)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_node_sharded_select, args=(r, world, port, q, key, T, k)) for r in range(world)]
    [p.start() for p in procs]
    out = [q.get(timeout=300) for _ in range(world)]
    [p.join(60) for p in procs]
    for rank, seeds, gains in out:
        assert seeds == rs.tolist() and gains == rg.tolist()
