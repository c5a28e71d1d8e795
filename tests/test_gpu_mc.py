"""Forward Monte-Carlo spread on the GPU (gim_mc_spread, csrc/mc.cu):
bit-exact against the oracle's og_mc_spread (same tag-11 Philox coins per out-slot, same
expressions for mean and standard error), then the north_star check at full size: the MC spread
of IMM's seeds within 1% of n * F_R'(S) on an independent RR pool (Eq. 3)."""
import os

import numpy as np
import pytest

import gim_inputs as gi
import oracle
from tests.test_gpu_parity import _ctx

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2009_07325_b200")


@pytest.mark.parametrize("scheme,pu", [(gi.W_WC, 0.0), (gi.W_UNIFORM, 0.3), (gi.W_EXPLICIT, 0.0)])
def test_mc_equals_oracle_tiny(scheme, pu):
    for g0 in (gi.diamond(), gi.cycle_plus(), gi.random_small(30, 200, 2), gi.random_small(12, 60, 1)):
        g = g0
        if scheme == gi.W_EXPLICIT:
            rng = np.random.default_rng(g.n)
            g = gi.with_weights(g0, rng.choice([0.0, 0.2, 0.5, 1.0], size=g0.m).astype(np.float32))
        c = _ctx(g, gi.IC, scheme, pu)
        o = oracle.Oracle(g, gi.IC, scheme, pu)
        for S in ([0], [1, 2], [0, 0, 3]):                       # duplicates activate once
            S = [s % g.n for s in S]
            mean, se = c.mc_spread(S, 4001, 99)
            om, ose = o.mc_spread(S, 4001, 99)
            assert mean == om and se == ose, (S, mean, om)


@pytest.mark.parametrize("key,k", [("C1", 50), ("C2", 10)])
def test_mc_equals_oracle_workloads(key, k):
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    c = _ctx(g, w.model, w.scheme)
    o = oracle.Oracle(g, w.model, w.scheme)
    c.generate_rr(20000, w.rr_seed)
    seeds, _, _ = c.select(k)
    mean, se, sizes = c.mc_spread(seeds, 3001, 7, return_sizes=True)
    om, ose = o.mc_spread(seeds, 3001, 7)
    assert mean == om and se == ose
    assert sizes.min() >= len(set(seeds.tolist())) and sizes.max() <= g.n


def _ris_estimate(c_pool, n, S, T):
    ids, off, nodes = c_pool.rr_export(sort_each_set=False)
    assert len(ids) == T
    member = np.isin(nodes, np.asarray(S, dtype=np.uint32))
    hit = np.zeros(T, dtype=bool)
    hit[np.repeat(np.arange(T), np.diff(off.astype(np.int64)))[member]] = True
    return n * hit.mean()


@pytest.mark.parametrize("key", ["C3", "C5"])
def test_mc_verified_spread_full_size(key):
    """north_star: Monte-Carlo-verified spread within 1% — IMM's seeds at BASELINE size, forward
    MC (2,000 instance graphs) vs n * F_R'(S) on an independent pool R' (2^21 sets, another seed;
    reading R24: the pool IMM selected on is biased upward)."""
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    c = _ctx(g, w.model, w.scheme, w.p_uniform)
    r = c.imm(w.k, w.eps, w.ell, w.rr_seed)
    T = 1 << (25 if key == "C5" else 21)      # C5: F ~ 0.9%, needs ~2^25 sets for a 0.3% RIS error
    c2 = _ctx(g, w.model, w.scheme, w.p_uniform)
    c2.generate_rr(T, w.rr_seed + 1)
    ris = _ris_estimate(c2, g.n, r.seeds, T)
    mean, se = c.mc_spread(r.seeds, 2000, 17)
    assert se / mean < 0.003, (mean, se)
    assert abs(mean - ris) / mean < 0.01, (mean, ris, r.spread_est)


@pytest.mark.parametrize("scheme", [gi.W_WC, gi.W_EXPLICIT])
def test_mc_lt_equals_oracle_tiny(scheme):
    """LT forward process (reading R30: exact threshold comparison) bit-exact with the oracle."""
    for g0 in (gi.diamond(), gi.cycle_plus(), gi.random_small(30, 200, 2), gi.random_small(12, 60, 1)):
        g = g0
        if scheme == gi.W_EXPLICIT:
            rng = np.random.default_rng(g.n)
            din = g0.in_degree()
            dst = np.repeat(np.arange(g0.n), din)
            g = gi.with_weights(g0, (rng.uniform(0.0, 1.0, size=g0.m) / np.maximum(din[dst], 1)).astype(np.float32))
        c = _ctx(g, gi.LT, scheme)
        o = oracle.Oracle(g, gi.LT, scheme)
        for S in ([0], [1, 2], [0, 0, 3]):
            S = [s % g.n for s in S]
            assert c.mc_spread(S, 4001, 99) == o.mc_spread(S, 4001, 99), S


def test_mc_lt_equals_oracle_C1():
    w = gi.WORKLOADS["C1"]
    g = gi.workload_graph("C1")
    c = _ctx(g, gi.LT, gi.W_WC)
    c.generate_rr(20000, w.rr_seed)
    seeds, _, _ = c.select(50)
    assert c.mc_spread(seeds, 2001, 5) == oracle.Oracle(g, gi.LT, gi.W_WC).mc_spread(seeds, 2001, 5)


def test_mc_lt_verified_spread_C4():
    """C4 (LT): forward MC of IMM's seeds within 1% of n * F_R'(S) on an independent pool."""
    w = gi.WORKLOADS["C4"]
    g = gi.workload_graph("C4")
    c = _ctx(g, w.model, w.scheme)
    r = c.imm(w.k, w.eps, w.ell, w.rr_seed)
    T = 1 << 21
    c2 = _ctx(g, w.model, w.scheme)
    c2.generate_rr(T, w.rr_seed + 1)
    ris = _ris_estimate(c2, g.n, r.seeds, T)
    mean, se = c.mc_spread(r.seeds, 2000, 17)
    assert se / mean < 0.004, (mean, se)
    assert abs(mean - ris) / mean < 0.01, (mean, ris, r.spread_est)


def test_mc_errors():
    g = gi.diamond()
    c = _ctx(g, gi.IC, gi.W_WC)
    with pytest.raises(P.GimError):
        c.mc_spread([7], 10, 1)                                  # seed out of range
