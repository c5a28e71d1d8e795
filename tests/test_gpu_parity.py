"""Parity of the CUDA path (through the C ABI, libgim.so) with the oracle, element by element.

Bar: RR sets (sorted), offsets, ids, counts, seeds and gains bit-exact;
IMM doubles (lambda', lambda*, theta_i, LB, theta) within 1e-12 relative. Sizes: tiny graphs,
C1/C2 pools spanning many warps and a ragged tail, and C3/C4 at full size on sampled ids.
"""
import math
import os
import threading

import numpy as np
import pytest

import gim_inputs as gi
from tests.imm_trace import check_cov_trace, oracle_round_gains
import oracle

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2009_07325_b200")


def _ctx(g, model, scheme, p_uniform=0.0, opts=None):
    c = P.Gim(0)
    c.load_graph(g.n, g.row_ptr, g.src, model, scheme, weights=g.weights, p_uniform=p_uniform)
    for k, v in (opts or {}).items():
        c.set_option(k, v)
    return c


def _same_pool(c, o, T):
    ids, off, nodes = c.rr_export(sort_each_set=True)
    ooff, onodes, ocnt = o.export()
    assert len(ids) == T and np.array_equal(ids, np.arange(T, dtype=np.uint64))
    assert np.array_equal(off, ooff), "offsets"
    assert np.array_equal(nodes, onodes), "pool contents"
    assert np.array_equal(c.counts_export(o.n), ocnt), "counts"


def _variants(g):
    rng = np.random.default_rng(g.n)
    din = g.in_degree()
    dst = np.repeat(np.arange(g.n), din)
    w_ic = rng.choice([0.0, 0.2, 0.5, 1.0], size=g.m).astype(np.float32)
    w_lt = (rng.uniform(0.1, 1.0, size=g.m) / np.maximum(din[dst], 1)).astype(np.float32)
    return [("ic_wc", g, gi.IC, gi.W_WC, 0.0), ("ic_uni", g, gi.IC, gi.W_UNIFORM, 0.3),
            ("ic_exp", gi.with_weights(g, w_ic), gi.IC, gi.W_EXPLICIT, 0.0),
            ("lt_wc", g, gi.LT, gi.W_WC, 0.0), ("lt_exp", gi.with_weights(g, w_lt), gi.LT, gi.W_EXPLICIT, 0.0)]


def test_keyscheme_golden_diamond():
    import json, os
    gd = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "diamond_keyscheme.json")))
    d = gi.diamond()
    for case, g, model, scheme in [("ic_wc", d, gi.IC, gi.W_WC),
                                   ("ic_half", gi.with_weights(d, np.full(4, 0.5)), gi.IC, gi.W_EXPLICIT),
                                   ("lt_wc", d, gi.LT, gi.W_WC)]:
        c = _ctx(g, model, scheme)
        c.generate_rr(16, gd["seed"])
        ids, off, nodes = c.rr_export()
        sets = ["".join(str(int(v)) for v in nodes[off[i]:off[i + 1]]) for i in range(16)]
        assert sets == gd[case + "_sets"]
        assert c.counts_export(4).tolist() == gd[case + "_counts"]
        seeds, gains, cov = c.select(2)
        assert seeds.tolist() == gd[case + "_greedy_k2"]["seeds"]
        assert gains.tolist() == gd[case + "_greedy_k2"]["gains"]


@pytest.mark.parametrize("gname", ["diamond", "chain", "star", "cycle", "rand0", "rand1", "rand2"])
def test_pool_parity_tiny(gname):
    g = {"diamond": gi.diamond(), "chain": gi.chain(6), "star": gi.star_in(40),
         "cycle": gi.cycle_plus(), "rand0": gi.random_small(9, 30, 0),
         "rand1": gi.random_small(12, 60, 1), "rand2": gi.random_small(30, 200, 2)}[gname]
    for (name, gg, model, scheme, pu), lane in [(v, l) for v in _variants(g) for l in (0, 1)]:
        T = 3001                       # many warps + a ragged tail
        c = _ctx(gg, model, scheme, pu, opts={P.OPT_IC_LANE: lane})
        c.generate_rr(T, 4242)
        o = oracle.Oracle(gg, model, scheme, pu)
        o.generate(T, 4242)
        _same_pool(c, o, T)
        k = min(3, g.n)
        assert [x.tolist() if hasattr(x, "tolist") else x for x in c.select(k)] == \
               [x.tolist() if hasattr(x, "tolist") else x for x in o.select(k)], name


@pytest.mark.parametrize("opts", [{}, {P.OPT_FORCE_GIANT: 1}, {P.OPT_QUEUE_CAP: 4},
                                  {P.OPT_STAGING_CAP: 64}, {P.OPT_QUEUE_CAP: 32, P.OPT_STAGING_CAP: 1000},
                                  {P.OPT_IC_LANE: 1}, {P.OPT_IC_LANE: 1, P.OPT_STAGING_CAP: 64},
                                  {P.OPT_IC_LANE: 1, P.OPT_FORCE_GIANT: 1}, {P.OPT_IC_LANE: 1, P.OPT_QUEUE_CAP: 8},
                                  {P.OPT_FORCE_GIANT: 1, P.OPT_GIANT_NT: 128}, {P.OPT_QUEUE_CAP: 16, P.OPT_GIANT_NT: 128},
                                  {P.OPT_FORCE_GIANT: 1, P.OPT_GIANT_NT: 256},
                                  {P.OPT_SPILL: 0}, {P.OPT_QUEUE_CAP: 8, P.OPT_SPILL: 64},
                                  {P.OPT_QUEUE_CAP: 32, P.OPT_SPILL: 40, P.OPT_STAGING_CAP: 1000},
                                  {P.OPT_IC_LANE: 1, P.OPT_QUEUE_CAP: 4, P.OPT_SPILL: 16384},
                                  {P.OPT_GIANT_SHARED: 0}, {P.OPT_GIANT_SHARED: 0, P.OPT_FORCE_GIANT: 1},
                                  {P.OPT_GIANT_SHARED: 1, P.OPT_QUEUE_CAP: 16},
                                  {P.OPT_CHUNK: 4096}, {P.OPT_CHUNK: 1024, P.OPT_STAGING_CAP: 1000},
                                  {P.OPT_CHUNK: 4096, P.OPT_IC_LANE: 1}])
def test_pool_parity_C1_invariance(opts):
    """Same pool whatever the queue capacity, spill-tier capacity (sets beyond the shared queue
    continue in the warp's global queue + hash, beyond the spill cap in K-GIANT), forced
    fallback or staging retries."""
    w = gi.WORKLOADS["C1"]
    g = gi.workload_graph("C1")
    T = 40013
    c = _ctx(g, w.model, w.scheme, opts=opts)
    c.generate_rr(T, w.rr_seed)
    o = oracle.Oracle(g, w.model, w.scheme)
    o.generate(T, w.rr_seed)
    _same_pool(c, o, T)
    if opts.get(P.OPT_FORCE_GIANT):
        assert c.stats()["giant_sets"] == T


@pytest.mark.parametrize("graph,segs,cand,extra", [
    (1, 1, 1, {}), (0, 1, 2, {}), (1, 0, 1, {}), (1, 1, 0, {}), (1, 1, 2, {}),
    (1, 1, 1, {"OPT_INV_PASSES": 7}), (1, 0, 2, {"OPT_INV_PASSES": 3}),
    (0, 1, 1, {"OPT_INV_PASSES": 64})])
def test_pool_parity_C2_and_select(graph, segs, cand, extra):
    """k = 50 selection through the argmax/cover launches replayed from a CUDA graph (default:
    one conditional IF node per step; or a plain graph) and launched one by one; pool generated
    in several calls (several index segments), index scattered in 1..64 node-range passes."""
    w = gi.WORKLOADS["C2"]
    g = gi.workload_graph("C2")
    T = 30011
    opts = {P.OPT_SELECT_GRAPH: graph, P.OPT_INV_SEGMENTS: segs, P.OPT_ARGMAX_CAND: cand}
    opts.update({getattr(P, k): v for k, v in extra.items()})
    c = _ctx(g, w.model, w.scheme, opts=opts)
    for t in (1000, 7000, 7001, 20000):
        c.generate_rr(t, w.rr_seed)
    c.generate_rr(T, w.rr_seed)
    o = oracle.Oracle(g, w.model, w.scheme)
    o.generate(T, w.rr_seed)
    _same_pool(c, o, T)
    s, gns, cov = c.select(50)
    os_, ogn, ocov = o.select(50)
    assert np.array_equal(s, os_) and np.array_equal(gns, ogn) and cov == ocov
    s2, g2, c2 = c.select(50)                          # non-destructive (reading R9)
    assert np.array_equal(s2, s) and np.array_equal(g2, gns) and c2 == cov
    st = c.stats()
    assert st["coins"] == o.stats()["coins"] or st["giant_sets"] > 0   # aborted work is recounted
    assert st["rr_elements"] == len(o.export()[1])


@pytest.mark.parametrize("pdl", [0, 1])
def test_select_pdl_invariance(pdl):
    """Programmatic dependent launch of the argmax/cover chain (GIM_OPT_PDL) changes no result,
    with the CUDA-graph replay and with one-by-one launches."""
    w = gi.WORKLOADS["C2"]
    g = gi.workload_graph("C2")
    o = oracle.Oracle(g, w.model, w.scheme)
    o.generate(20011, w.rr_seed)
    ref = o.select(50)
    for graph in (1, 0):
        c = _ctx(g, w.model, w.scheme, opts={P.OPT_SELECT_GRAPH: graph})
        c.set_option(P.OPT_PDL, pdl)
        c.generate_rr(20011, w.rr_seed)
        s, gn, cov = c.select(50)
        assert np.array_equal(s, ref[0]) and np.array_equal(gn, ref[1]) and cov == ref[2]
    c.set_option(P.OPT_PDL, 1)


def test_extend_truncate_reseed():
    g = gi.random_small(40, 300, 5)
    c = _ctx(g, gi.IC, gi.W_WC)
    o = oracle.Oracle(g, gi.IC, gi.W_WC)
    for T, seed in [(1000, 1), (5000, 1), (777, 1), (4000, 1), (4000, 2), (0, 2), (10, 2)]:
        c.generate_rr(T, seed)
        o.generate(T, seed)
        _same_pool(c, o, T)


@pytest.mark.parametrize("graph,cand", [(1, 1), (0, 0), (1, 2)])
def test_select_zero_gain_and_k_eq_n(graph, cand):
    g = gi.diamond()
    c = _ctx(g, gi.LT, gi.W_WC, opts={P.OPT_SELECT_GRAPH: graph, P.OPT_ARGMAX_CAND: cand})
    c.generate_rr(16, 200907325)
    s, gns, cov = c.select(4)
    o = oracle.Oracle(g, gi.LT, gi.W_WC)
    o.generate(16, 200907325)
    os_, ogn, ocov = o.select(4)
    assert s.tolist() == os_.tolist() and gns.tolist() == ogn.tolist() and cov == ocov == 16


def test_errors():
    g = gi.diamond()
    c = P.Gim(0)
    with pytest.raises(P.GimError) as e:
        c.generate_rr(10, 1)
    assert e.value.status == 2                     # no graph
    with pytest.raises(P.GimError) as e:
        c.load_graph(4, np.array([0, 0, 1, 2, 4], np.uint64), np.array([0, 0, 2, 1], np.uint32), gi.IC, gi.W_WC)
    assert e.value.status == 1                     # row 3 not ascending
    with pytest.raises(P.GimError) as e:
        c.load_graph(2, np.array([0, 1, 1], np.uint64), np.array([0], np.uint32), gi.IC, gi.W_WC)
    assert e.value.status == 1                     # self-loop
    with pytest.raises(P.GimError) as e:
        c.load_graph(g.n, g.row_ptr, g.src, gi.LT, gi.W_EXPLICIT, weights=np.full(4, 0.6, np.float32))
    assert e.value.status == 6                     # LT in-weights of node 3 sum to 1.2
    c.load_graph(g.n, g.row_ptr, g.src, gi.IC, gi.W_WC)
    with pytest.raises(P.GimError) as e:
        c.select(1)
    assert e.value.status == 2                     # empty pool
    c.generate_rr(10, 1)
    for k in (0, 5):
        with pytest.raises(P.GimError) as e:
            c.select(k)
        assert e.value.status == 1
    with pytest.raises(P.GimError):
        c.imm(2, 0.0, 1.0, 1)
    g1 = gi.from_edges(1, [])
    c.load_graph(1, g1.row_ptr, g1.src, gi.IC, gi.W_WC)
    c.generate_rr(5, 3)
    ids, off, nodes = c.rr_export()
    assert off.tolist() == [0, 1, 2, 3, 4, 5] and c.counts_export(1).tolist() == [5]
    with pytest.raises(P.GimError) as e:
        c.imm(1, 0.1, 1.0, 1)
    assert e.value.status == 1                     # n = 1 (reading R25)


def _imm_parity(key, k=None, eps=None):
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    k = k or w.k
    eps = eps or w.eps
    c = _ctx(g, w.model, w.scheme, w.p_uniform)
    r = c.imm(k, eps, w.ell, w.rr_seed)
    o = oracle.Oracle(g, w.model, w.scheme, w.p_uniform)
    ro = o.imm(k, eps, w.ell, w.rr_seed)
    rel = lambda a, b: abs(a - b) <= 1e-12 * max(abs(b), 1e-300)
    assert rel(r.lambda_prime, ro.lambda_prime) and rel(r.lambda_star, ro.lambda_star)
    assert rel(r.ell_eff, ro.ell_eff) and rel(r.eps_prime, ro.eps_prime)
    assert r.rounds == ro.rounds
    assert all(rel(a, b) for a, b in zip(r.theta_i_real, ro.theta_i))
    assert np.array_equal(r.theta_i, ro.T_i)
    check_cov_trace(r, ro.T_i, ro.cov_i, g.n, ro.eps_prime, k,
                    oracle_round_gains(oracle.Oracle(g, w.model, w.scheme, w.p_uniform), ro.T_i, k, w.rr_seed))
    assert rel(r.LB, ro.LB) and rel(r.theta, ro.theta)
    assert r.R_final == ro.R_final and r.covered == ro.cov
    assert np.array_equal(r.seeds, ro.seeds), (r.seeds, ro.seeds)
    assert rel(r.spread_est, ro.spread_est)
    return r


def test_imm_parity_C1():
    _imm_parity("C1")


def test_imm_parity_C2():
    _imm_parity("C2")


def test_imm_parity_C1_LT():
    w = gi.WORKLOADS["C1"]
    g = gi.workload_graph("C1")
    c = _ctx(g, gi.LT, gi.W_WC)
    r = c.imm(w.k, w.eps, w.ell, w.rr_seed)
    o = oracle.Oracle(g, gi.LT, gi.W_WC)
    ro = o.imm(w.k, w.eps, w.ell, w.rr_seed)
    assert np.array_equal(r.seeds, ro.seeds) and r.R_final == ro.R_final and r.covered == ro.cov


def test_imm_parity_BA_small():
    """The paper's density workload family (Barabasi-Albert) at a size the oracle runs
    in a second: full IMM trace and seeds bit-exact (WC on an undirected graph is critical, so
    sets reach the giant path)."""
    g = gi.ba(20000, 8, 11)
    c = _ctx(g, gi.IC, gi.W_WC)
    r = c.imm(20, 0.3, 1.0, 5)
    ro = oracle.Oracle(g, gi.IC, gi.W_WC).imm(20, 0.3, 1.0, 5)
    assert r.rounds == ro.rounds and np.array_equal(r.theta_i, ro.T_i)
    check_cov_trace(r, ro.T_i, ro.cov_i, g.n, ro.eps_prime, 20,
                    oracle_round_gains(oracle.Oracle(g, gi.IC, gi.W_WC), ro.T_i, 20, 5))
    assert r.R_final == ro.R_final and r.covered == ro.cov
    assert np.array_equal(r.seeds, ro.seeds), (r.seeds, ro.seeds)


@pytest.mark.parametrize("key", ["C3", "C4", "B8", "B32", "C5"])
def test_full_size_sampled(key):
    """BASELINE.json full size: 2^21 RR sets in the launch configuration bench.py times; sampled
    ids recomputed one by one by the oracle; counts checked by the size-free identities."""
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    c = _ctx(g, w.model, w.scheme, w.p_uniform)
    T = 1 << 21
    c.generate_rr(T, w.rr_seed)
    ids, off, nodes = c.rr_export(sort_each_set=True)
    assert np.array_equal(ids, np.arange(T, dtype=np.uint64))
    o = oracle.Oracle(g, w.model, w.scheme, w.p_uniform)
    rng = np.random.default_rng(1)
    sample = np.concatenate([[0, 1, T - 1], rng.choice(T, 300, replace=False)])
    sizes = np.diff(off.astype(np.int64))
    sample = np.concatenate([sample, np.argsort(sizes)[-5:]])       # include the largest sets
    for i in sample:
        assert np.array_equal(nodes[off[i]:off[i + 1]], o.rr_set(w.rr_seed, int(i))), int(i)
    cnt = c.counts_export(g.n)
    assert int(cnt.sum()) == len(nodes)
    assert np.array_equal(np.bincount(nodes, minlength=g.n).astype(np.uint32), cnt)
    assert np.all(sizes >= 1)
    d = np.diff(nodes.astype(np.int64))
    starts = off[1:-1].astype(np.int64)
    mask = np.ones(len(d), dtype=bool)
    mask[starts - 1] = False
    assert np.all(d[mask] > 0)                                       # distinct members
    # NodeSelection at full size: graph replay == one-by-one launches; properties
    # that hold at any size: first pick is the lowest-id argmax of the counts, gains are
    # non-increasing (greedy on a coverage function), covered = #sets hit by the seeds.
    seeds, gains, cov = c.select(w.k)
    c.set_option(P.OPT_SELECT_GRAPH, 0)
    c.set_option(P.OPT_ARGMAX_CAND, 2)
    s2, g2, c2 = c.select(w.k)
    assert np.array_equal(seeds, s2) and np.array_equal(gains, g2) and cov == c2
    assert seeds[0] == int(np.argmax(cnt)) and gains[0] == int(cnt.max())
    assert np.all(np.diff(gains.astype(np.int64)) <= 0) and len(set(seeds.tolist())) == w.k
    hit = np.zeros(T, dtype=bool)
    set_of = np.repeat(np.arange(T), sizes)
    hit[set_of[np.isin(nodes, seeds)]] = True
    assert int(hit.sum()) == cov == int(gains.sum())


@pytest.mark.parametrize("key", ["C3", "C4"])
def test_imm_speculation_invariance(key):
    """gim_imm with the next round's RR ids sampled on a second stream while each round's
    NodeSelection runs (default) returns exactly what the sequential schedule returns."""
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    out = []
    for spec in (1, 0):
        c = _ctx(g, w.model, w.scheme, opts={P.OPT_SPECULATE: spec})
        out.append(c.imm(w.k, w.eps, w.ell, w.rr_seed))
        ids, off, nodes = c.rr_export(sort_each_set=False)
        assert len(ids) == out[-1].R_final
        c.close()
    a, b = out
    assert np.array_equal(a.seeds, b.seeds) and a.R_final == b.R_final and a.covered == b.covered
    assert a.LB == b.LB and a.theta == b.theta and a.rounds == b.rounds
    assert np.array_equal(a.theta_i, b.theta_i) and np.array_equal(a.cov_i, b.cov_i)


@pytest.mark.parametrize("key,rounds", [("C1", 1), ("C2", 1), ("C1", 3)])
def test_imm_fresh_final_parity(key, rounds):
    """Reading R29 (GIM_OPT_FRESH_FINAL): the final phase on a fresh pool of the second key —
    trace, R_final and seeds bit-exact against the oracle's fresh-final driver (IMM and MRIM)."""
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    k = w.k if rounds == 1 else 10
    c = _ctx(g, w.model, w.scheme, opts={P.OPT_FRESH_FINAL: 1})
    o = oracle.Oracle(g, w.model, w.scheme)
    o.set_fresh_final(True)
    if rounds > 1:
        c.set_rounds(rounds)
        ro = o.mrim(k, rounds, w.eps, w.ell, w.rr_seed)
    else:
        ro = o.imm(k, w.eps, w.ell, w.rr_seed)
    r = c.imm(k, w.eps, w.ell, w.rr_seed)
    rel = lambda a, b: abs(a - b) <= 1e-12 * max(abs(b), 1e-300)
    assert r.rounds == ro.rounds and np.array_equal(r.theta_i, ro.T_i)
    o2 = oracle.Oracle(g, w.model, w.scheme)
    check_cov_trace(r, ro.T_i, ro.cov_i, g.n, ro.eps_prime, k * rounds,
                    oracle_round_gains(o2, ro.T_i, k, w.rr_seed, mrim_T=rounds if rounds > 1 else None))
    assert rel(r.LB, ro.LB) and rel(r.theta, ro.theta)
    assert r.R_final == ro.R_final == math.ceil(ro.theta) and r.covered == ro.cov
    assert np.array_equal(r.seeds, ro.seeds)


@pytest.mark.parametrize("rounds", [1, 3])
def test_select_persistent_equals_oracle(rounds):
    """GIM_OPT_SELECT_PERSISTENT: the k greedy steps in one cooperative launch (grid barriers
    between argmax and cover) — seeds, gains and coverage bit-exact, standard and MRIM."""
    w = gi.WORKLOADS["C2"]
    g = gi.workload_graph("C2")
    N = 20011 if rounds == 1 else 5003
    k = 50 if rounds == 1 else 10
    c = _ctx(g, w.model, w.scheme, opts={P.OPT_SELECT_PERSISTENT: 1})
    c.set_rounds(rounds)
    c.generate_rr(N, w.rr_seed)
    o = oracle.Oracle(g, w.model, w.scheme)
    if rounds == 1:
        o.generate(N, w.rr_seed)
        ref = o.select(k)
    else:
        o.mrim_generate(N, rounds, w.rr_seed)
        ref = o.mrim_select(k)
    for _ in range(2):                                     # non-destructive, repeatable
        s, gn, cov = c.select(k)
        assert np.array_equal(s, ref[0]) and np.array_equal(gn, ref[1]) and cov == ref[2]
    r = c.imm(k, w.eps, w.ell, w.rr_seed)
    ro = o.imm(k, w.eps, w.ell, w.rr_seed) if rounds == 1 else o.mrim(k, rounds, w.eps, w.ell, w.rr_seed)
    assert np.array_equal(r.seeds, ro.seeds) and r.R_final == ro.R_final


@pytest.mark.parametrize("key", ["C1", "C2"])
def test_fused_selection_modes(key):
    """GIM_OPT_SELECT_FUSED (one launch per greedy step, candidate argmax certified by tau in the
    last CTA): every candidate cap — including caps so small that the certificate fails and the
    selection is redone unfused — gives the oracle's seeds and gains (O7, Alg. 7)."""
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    T = 50021
    o = oracle.Oracle(g, w.model, w.scheme, w.p_uniform)
    o.generate(T, w.rr_seed)
    os_, og, oc = o.select(w.k)
    for cap, graph in ((2048, 1), (2048, 0), (64, 1), (1, 1), (0, 1)):
        c = _ctx(g, w.model, w.scheme, w.p_uniform, {P.OPT_SELECT_FUSED: cap, P.OPT_SELECT_GRAPH: graph})
        c.generate_rr(T, w.rr_seed)
        c.reset_stats()
        s, gn, cv = c.select(w.k)
        assert np.array_equal(s, os_) and np.array_equal(gn, og) and cv == oc, cap
        if cap == 1:
            assert c.stats()["fused_fallbacks"] >= 1
        s2, g2, c2 = c.select(w.k)                  # non-destructive, graph replay
        assert np.array_equal(s2, os_) and np.array_equal(g2, og)
        c.close()


@pytest.mark.parametrize("model,scheme,pu", [(gi.IC, gi.W_UNIFORM, 0.9), (gi.IC, gi.W_WC, 0.0), (gi.LT, gi.W_WC, 0.0)])
def test_giant_shared_pass_handover(model, scheme, pu):
    """Giant sets beyond the shared-memory giant pass (4096 nodes) are handed to the global-bitmap
    pass and resumed there: an in-star of 20,000 leaves fed by a chain (IC uniform p = 0.9 gives
    ~18,000-node sets), plus long chains for WC/LT; pools bit-exact with the oracle under both
    giant modes and forced giant."""
    leaves = 20000
    edges = [(i, 0) for i in range(1, leaves + 1)] + [(leaves + 1 + i, leaves + 2 + i) for i in range(6000)]
    edges += [(leaves + 6001, 0)]
    g = gi.from_edges(leaves + 6002, edges)
    T = 3000
    o = oracle.Oracle(g, model, scheme, pu)
    o.generate(T, 9)
    for opts in ({}, {P.OPT_FORCE_GIANT: 1}, {P.OPT_GIANT_SHARED: 0}):
        c = _ctx(g, model, scheme, pu, opts)
        c.generate_rr(T, 9)
        _same_pool(c, o, T)
        c.close()


@pytest.mark.parametrize("key", ["C1", "C2"])
def test_coop_selection_modes(key):
    """GIM_OPT_SELECT_COOP (one cooperative launch, one grid barrier per greedy step, redundant
    candidate argmax per CTA, candidate-only decrement rings): the oracle's seeds and gains at
    every candidate cap, including caps that fail the certificate and rerun (O7, Alg. 7)."""
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    T = 50021
    o = oracle.Oracle(g, w.model, w.scheme, w.p_uniform)
    o.generate(T, w.rr_seed)
    os_, og, oc = o.select(w.k)
    for cap in (8192, 2048, 64, 1):
        c = _ctx(g, w.model, w.scheme, w.p_uniform, {P.OPT_SELECT_COOP: cap})
        c.generate_rr(T // 2, w.rr_seed)
        c.generate_rr(T, w.rr_seed)                       # two index segments
        c.reset_stats()
        for _ in range(2):                                # non-destructive, repeatable
            s, gn, cv = c.select(w.k)
            assert np.array_equal(s, os_) and np.array_equal(gn, og) and cv == oc, cap
        if cap == 1:
            assert c.stats()["fused_fallbacks"] >= 1
        c.close()


@pytest.mark.parametrize("key", ["C1", "C3", "C4"])
def test_coop_selection_imm_golden(key):
    """Full IMM with the cooperative selection equals the oracle's committed run."""
    import json
    gd = json.load(open(os.path.join(os.path.dirname(__file__), "golden", f"imm_{key}.json")))
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    c = _ctx(g, w.model, w.scheme, w.p_uniform, {P.OPT_SELECT_COOP: 4096})
    r = c.imm(w.k, w.eps, w.ell, w.rr_seed)
    assert r.seeds.tolist() == gd["seeds"] and r.R_final == gd["R_final"]
    check_cov_trace(r, gd["T_i"], gd["cov_i"], g.n, gd["eps_prime"], w.k)
    c.close()


@pytest.mark.parametrize("key,small", [("C1", 1), ("C1", 0), ("C2", 2), ("C2", 0)])
def test_select_small_cta_equals_oracle(key, small):
    """Single-launch selection — one CTA (C1, n <= 51,200) or a thread-block cluster with the counts
    in its CTAs' shared memories (C2: 2 CTAs, DSMEM atomics) — and the multi-CTA graph replay
    (small = 0) all equal the oracle (small = 2: GIM_OPT_SELECT_CLUSTER, off by default): a pool in
    several generate calls (several index segments),
    k = 50 and k = 200, a truncated pool (cut sets skipped), and the full IMM with its
    bounded-greedy trace."""
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    c = _ctx(g, w.model, w.scheme, opts={P.OPT_SELECT_CTA: min(small, 1), P.OPT_SELECT_CLUSTER: int(small == 2)})
    o = oracle.Oracle(g, w.model, w.scheme)
    for T in (5000, 12001, 40013):
        c.generate_rr(T, w.rr_seed)
    o.generate(40013, w.rr_seed)
    for k in (50, 200):
        s, gn, cov = c.select(k)
        os_, ogn, ocov = o.select(k)
        assert np.array_equal(s, os_) and np.array_equal(gn, ogn) and cov == ocov
    c.generate_rr(30011, w.rr_seed)                    # truncation: sets >= 30011 are cut
    o.generate(30011, w.rr_seed)
    s, gn, cov = c.select(50)
    os_, ogn, ocov = o.select(50)
    assert np.array_equal(s, os_) and np.array_equal(gn, ogn) and cov == ocov
    r = c.imm(w.k, w.eps, w.ell, w.rr_seed)
    ro = oracle.Oracle(g, w.model, w.scheme).imm(w.k, w.eps, w.ell, w.rr_seed)
    assert np.array_equal(r.seeds, ro.seeds) and r.R_final == ro.R_final and r.covered == ro.cov
    check_cov_trace(r, ro.T_i, ro.cov_i, g.n, ro.eps_prime, w.k,
                    oracle_round_gains(oracle.Oracle(g, w.model, w.scheme), ro.T_i, w.k, w.rr_seed))
    c.close()


@pytest.mark.parametrize("key", ["C1", "C2"])
def test_inv_sort_segments_equal_oracle(key):
    """Sort-based index segments (GIM_OPT_INV_SORT = 1; the default for n * 4 > 64 MB): selection
    over a pool built in several generate calls (several segments, one rebuilt after a
    truncation) and a full IMM equal the oracle."""
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    c = _ctx(g, w.model, w.scheme, opts={P.OPT_INV_SORT: 1})
    o = oracle.Oracle(g, w.model, w.scheme)
    for T in (3001, 9000, 30011):
        c.generate_rr(T, w.rr_seed)
    o.generate(30011, w.rr_seed)
    assert [x.tolist() if hasattr(x, "tolist") else x for x in c.select(50)] == \
           [x.tolist() if hasattr(x, "tolist") else x for x in o.select(50)]
    c.generate_rr(20000, w.rr_seed)
    c.generate_rr(25000, w.rr_seed)
    o.generate(25000, w.rr_seed)
    assert [x.tolist() if hasattr(x, "tolist") else x for x in c.select(50)] == \
           [x.tolist() if hasattr(x, "tolist") else x for x in o.select(50)]
    r = c.imm(w.k, w.eps, w.ell, w.rr_seed)
    ro = oracle.Oracle(g, w.model, w.scheme).imm(w.k, w.eps, w.ell, w.rr_seed)
    assert np.array_equal(r.seeds, ro.seeds) and r.R_final == ro.R_final and r.covered == ro.cov
    c.close()
