"""MRIM (multi-round IM, CR-NAIMM as gIM adapts it, §4.8; readings R26-R28) on the
CUDA path through the C ABI vs the oracle: pools of (node, round) pair ids, pair counts, the
per-round-budget selection and the full MRIM IMM trace, bit-exact (doubles within 1e-12)."""
import threading

import numpy as np
import pytest

import gim_inputs as gi
from tests.imm_trace import check_cov_trace, oracle_round_gains
import oracle
from tests.test_gpu_parity import _ctx, _variants

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2009_07325_b200")


def _mrim_pool_gpu(c, N, T):
    """GPU export (per-round sets i*T + t, sorted) regrouped into MRIM sets."""
    ids, off, nodes = c.rr_export(sort_each_set=True)
    assert np.array_equal(ids, np.arange(N * T, dtype=np.uint64))
    moff = off[::T].copy()                      # MRIM set i = the T consecutive round sets
    assert len(moff) == N + 1
    return moff, nodes


def _same_mrim_pool(c, o, N, T, n):
    moff, pairs = _mrim_pool_gpu(c, N, T)
    ooff, opairs, ocnt = o.mrim_export()
    assert np.array_equal(moff, ooff), "MRIM offsets"
    assert np.array_equal(pairs, opairs), "MRIM pair sets"
    assert np.array_equal(c.counts_export(n * T), ocnt), "pair counts"


@pytest.mark.parametrize("gname", ["diamond", "cycle", "rand1", "rand2"])
@pytest.mark.parametrize("T", [2, 5])
def test_mrim_pool_and_select_tiny(gname, T):
    g = {"diamond": gi.diamond(), "cycle": gi.cycle_plus(), "rand1": gi.random_small(12, 60, 1),
         "rand2": gi.random_small(30, 200, 2)}[gname]
    for name, gg, model, scheme, pu in _variants(g):
        N = 2003                                    # many warps, ragged tail, T*N not a multiple of 32
        c = _ctx(gg, model, scheme, pu)
        c.set_rounds(T)
        c.generate_rr(N, 777)
        o = oracle.Oracle(gg, model, scheme, pu)
        o.mrim_generate(N, T, 777)
        _same_mrim_pool(c, o, N, T, g.n)
        k = min(2, g.n)
        s, gn, cov = c.select(k)
        os_, ogn, ocov = o.mrim_select(k)
        assert np.array_equal(s, os_) and np.array_equal(gn, ogn) and cov == ocov, (name, s, os_)


@pytest.mark.parametrize("graph", [1, 0])
def test_mrim_pool_and_select_C2(graph):
    """Epinions-shaped graph (the dataset of the paper's Table 3 first row), k = 10, T = 5, pool
    grown in several calls (several index segments)."""
    w = gi.WORKLOADS["C2"]
    g = gi.workload_graph("C2")
    T, N, k = 5, 12007, 10
    c = _ctx(g, w.model, w.scheme, opts={P.OPT_SELECT_GRAPH: graph})
    c.set_rounds(T)
    for t in (500, 4001, N):
        c.generate_rr(t, w.rr_seed)
    o = oracle.Oracle(g, w.model, w.scheme)
    o.mrim_generate(N, T, w.rr_seed)
    _same_mrim_pool(c, o, N, T, g.n)
    s, gn, cov = c.select(k)
    os_, ogn, ocov = o.mrim_select(k)
    assert np.array_equal(s, os_) and np.array_equal(gn, ogn) and cov == ocov
    assert np.bincount(s // g.n, minlength=T).tolist() == [k] * T
    s2, g2, c2 = c.select(k)                                   # non-destructive
    assert np.array_equal(s2, s) and np.array_equal(g2, gn) and c2 == cov


def test_mrim_T1_equals_standard():
    w = gi.WORKLOADS["C1"]
    g = gi.workload_graph("C1")
    a = _ctx(g, w.model, w.scheme)
    b = _ctx(g, w.model, w.scheme)
    b.set_rounds(1)
    for c in (a, b):
        c.generate_rr(20011, w.rr_seed)
    ea, eb = a.rr_export(), b.rr_export()
    assert all(np.array_equal(x, y) for x, y in zip(ea, eb))
    assert all(np.array_equal(np.asarray(x), np.asarray(y)) for x, y in zip(a.select(50), b.select(50)))


def test_mrim_truncate_extend_reseed_and_errors():
    g = gi.random_small(40, 300, 5)
    c = _ctx(g, gi.IC, gi.W_WC)
    c.set_rounds(3)
    c.generate_rr(900, 9)
    c.generate_rr(300, 9)
    c.generate_rr(700, 9)
    o = oracle.Oracle(g, gi.IC, gi.W_WC)
    o.mrim_generate(700, 3, 9)
    _same_mrim_pool(c, o, 700, 3, g.n)
    s, gn, cov = c.select(4)
    os_, ogn, ocov = o.mrim_select(4)
    assert np.array_equal(s, os_) and np.array_equal(gn, ogn) and cov == ocov
    with pytest.raises(P.GimError):
        c.set_rounds(0)
    with pytest.raises(P.GimError):
        c.set_rounds(1 << 30)                                   # n * T >= 2^32 - 1


@pytest.mark.parametrize("key,model,k,T,eps", [("C1", gi.IC, 10, 5, 0.5), ("C1", gi.LT, 10, 5, 0.5),
                                               ("C1", gi.IC, 5, 3, 0.3)])
def test_mrim_imm_parity(key, model, k, T, eps):
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    c = _ctx(g, model, w.scheme)
    c.set_rounds(T)
    r = c.imm(k, eps, w.ell, w.rr_seed)
    o = oracle.Oracle(g, model, w.scheme)
    ro = o.mrim(k, T, eps, w.ell, w.rr_seed)
    rel = lambda a, b: abs(a - b) <= 1e-12 * max(abs(b), 1e-300)
    assert rel(r.lambda_prime, ro.lambda_prime) and rel(r.lambda_star, ro.lambda_star)
    assert r.rounds == ro.rounds and np.array_equal(r.theta_i, ro.T_i)
    check_cov_trace(r, ro.T_i, ro.cov_i, g.n, ro.eps_prime, k * T,
                    oracle_round_gains(oracle.Oracle(g, model, w.scheme), ro.T_i, k, w.rr_seed, mrim_T=T))
    assert rel(r.LB, ro.LB) and rel(r.theta, ro.theta)
    assert r.R_final == ro.R_final and r.covered == ro.cov
    assert np.array_equal(r.seeds, ro.seeds), (r.seeds, ro.seeds)
    assert rel(r.spread_est, ro.spread_est)


def test_mrim_full_size_sampled_C3():
    """LJ-shaped graph at full size, T = 5: sampled MRIM sets recomputed by the oracle, size-free
    identities on the pair counts, and the per-round budget of the selection."""
    w = gi.WORKLOADS["C3"]
    g = gi.workload_graph("C3")
    T, N, k = 5, 1 << 18, 10
    c = _ctx(g, w.model, w.scheme)
    c.set_rounds(T)
    c.generate_rr(N, w.rr_seed)
    moff, pairs = _mrim_pool_gpu(c, N, T)
    o = oracle.Oracle(g, w.model, w.scheme)
    rng = np.random.default_rng(3)
    sample = np.concatenate([[0, N - 1], rng.choice(N, 120, replace=False)])
    for i in sample:
        assert np.array_equal(pairs[moff[i]:moff[i + 1]], o.mrim_set(w.rr_seed, int(i), T)), int(i)
    cnt = c.counts_export(g.n * T)
    assert int(cnt.sum()) == len(pairs)
    assert np.array_equal(np.bincount(pairs, minlength=g.n * T).astype(np.uint32), cnt)
    s, gn, cov = c.select(k)
    assert np.bincount(s // g.n, minlength=T).tolist() == [k] * T
    assert s[0] == int(np.argmax(cnt)) and gn[0] == int(cnt.max())
    assert np.all(np.diff(gn.astype(np.int64)) <= 0)
    hit = np.zeros(N, dtype=bool)
    set_of = np.repeat(np.arange(N), np.diff(moff.astype(np.int64)))
    hit[set_of[np.isin(pairs, s)]] = True
    assert int(hit.sum()) == cov == int(gn.sum())
