"""Pins of the oracle's geometric-skip contract (reading R31; oracle/gim_oracle.c
"R31"): the option replaces Alg. 3 l.18's per-edge coin by geometric gaps between live
in-edges where every in-edge of a node has the same probability (WC p = 1/d_in; uniform
p). What fixes it from outside the oracle:

* ``og_skip_ln`` against mpmath's natural log (relative error);
* the exact distribution of the gap, counted over all 2^32 Philox words (the gap is monotone in
  the word, so {r : gap(r) >= g} is a prefix found by bisection), against the geometric law
  Pr[gap >= g] = (1 - p)^g evaluated in mpmath;
* per-slot live rates, block boundaries and slot independence on a bipartite graph, against
  Bernoulli(p) per slot;
* the RIS estimator (Eq. 3) against exact enumeration of live-edge worlds;
* an independent pure-Python evaluation of the contract (its own Philox, exact fma via
  fractions) giving the same RR sets by brute-force reachability.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import gim_inputs as gi
import oracle
from tests.philox_ref import philox4x32_10
from tests.test_oracle_pins import (_check_estimator, _closure_reaching, _edge_list, _ic_worlds,
                                    _p_exact, _root_ref, _tiny_graphs)

mpmath = pytest.importorskip("mpmath")
mpmath.mp.dps = 40


def test_skip_ln_series_vs_mpmath():
    """The table entries' own log (the series form) against mpmath."""
    worst = 0.0
    for k in range(-75, 107):
        c = 1.0 + k / 256.0
        if k == 0:
            assert oracle.skip_ln_series(c) == 0.0
            continue
        ex = mpmath.log(mpmath.mpf(c))
        worst = max(worst, float(abs((mpmath.mpf(oracle.skip_ln_series(c)) - ex) / ex)))
    assert worst < 4e-16, worst


def test_skip_ln_vs_mpmath():
    rng = np.random.default_rng(7)
    xs = list(rng.uniform(0.0, 1.0, 3000)) + list(np.exp(rng.uniform(-24, 0.7, 3000)))
    xs += [(d - 1) / d for d in (2, 3, 7, 14, 100, 1023, 15000, 800000, 4_000_000_000)]
    xs += [1.0 - float(np.float32(p)) for p in (0.01, 0.3, 0.5, 0.999, 1e-6)]
    xs += [(r + 0.5) * 2.0 ** -32 for r in (0, 1, 2, 1000, 2**31, 2**32 - 1)]
    xs += [0.7071067811865475, 0.7071067811865476, 1.4142135623730951, 1.4142135623730954, 1.0, 2.0]
    worst = 0.0
    for x in xs:
        if x <= 0.0:
            continue
        ex = mpmath.log(mpmath.mpf(x))
        got = oracle.skip_ln(float(x))
        if ex == 0:
            assert got == 0.0
            continue
        worst = max(worst, float(abs((mpmath.mpf(got) - ex) / ex)))
    assert worst < 4e-16, worst


def _r_threshold(inv, g):
    """min r with gap(r) < g (gap is non-increasing in r); 2^32 if none."""
    lo, hi = 0, 1 << 32
    while lo < hi:
        mid = (lo + hi) // 2
        if oracle.skip_gap(inv, mid) < g:
            hi = mid
        else:
            lo = mid + 1
    return lo


_CASES = [("wc", d, None) for d in (2, 3, 7, 100, 1023, 15000, 10**6)] + \
         [("uni", None, p) for p in (0.01, 0.3, 0.5, 0.999)]


@pytest.mark.parametrize("case", _CASES, ids=lambda c: f"{c[0]}-{c[1] or c[2]}")
def test_gap_distribution_exact(case):
    kind, d, p = case
    if kind == "wc":
        inv = oracle.skip_inv(gi.W_WC, d)
        q = mpmath.mpf(d - 1) / d
    else:
        p32 = float(np.float32(p))
        inv = oracle.skip_inv(gi.W_UNIFORM, 1, p32)
        q = 1 - mpmath.mpf(p32)
    assert inv < 0
    # Pr[gap >= g] over all 2^32 words, at g where (1-p)^g spans 1 .. 1e-7
    gmax = float(mpmath.log(mpmath.mpf("1e-7")) / mpmath.log(q))
    grid = sorted(set([0, 1, 2, 3] + [int(gmax * f) for f in np.linspace(0.0, 1.0, 41)]))
    prev = 1 << 32
    for g in grid:
        rg = _r_threshold(inv, g)
        assert rg <= prev                                      # monotone counts
        prev = rg
        if 0 < rg < (1 << 32):                                 # the boundary really is a boundary
            assert oracle.skip_gap(inv, rg - 1) >= g > oracle.skip_gap(inv, rg)
        exact = q ** g
        assert abs(mpmath.mpf(rg) / 2**32 - exact) <= 2.0 ** -32 + 1e-13 * g, (g, rg / 2**32, float(exact))


def _bipartite(d, hubs):
    """Sources 0..d-1 (no in-edges) -> each of `hubs` hub nodes d..d+hubs-1."""
    n = d + hubs
    row_ptr = np.zeros(n + 1, dtype=np.uint64)
    row_ptr[d + 1:] = d * np.arange(1, hubs + 1, dtype=np.uint64)
    src = np.tile(np.arange(d, dtype=np.uint32), hubs)
    return gi.Graph(n=n, row_ptr=row_ptr, src=src, name=f"bip{d}x{hubs}")


def _hub_live_matrix(g, d, scheme, p, T, seed):
    o = oracle.Oracle(g, gi.IC, scheme, p)
    o.set_skip(True)
    o.generate(T, seed)
    off, nodes, _ = o.export()
    rows = []
    for i in range(T):
        s = nodes[off[i]:off[i + 1]]
        if s[-1] >= d:                                          # rooted at a hub
            m = np.zeros(d, dtype=bool)
            m[s[s < d]] = True
            rows.append(m)
    return np.array(rows)


def test_slot_rates_and_independence_uniform():
    d = 2100                                                    # blocks 1024 + 1024 + 52
    p = float(np.float32(0.3))
    g = _bipartite(d, d)
    L = _hub_live_matrix(g, d, gi.W_UNIFORM, 0.3, 8000, 11)
    N = len(L)
    assert N > 3500
    rate = L.mean(axis=0)
    z = (rate - p) / math.sqrt(p * (1 - p) / N)
    assert np.all(np.abs(z) < 5.0), np.abs(z).max()             # every slot, incl. block edges
    chi2 = float(np.sum(z ** 2))
    assert abs(chi2 - d) < 6 * math.sqrt(2 * d)
    for blk in ((0, 1024), (1024, 2048), (2048, 2100)):        # per-block totals
        tot = L[:, blk[0]:blk[1]].sum()
        n_ = N * (blk[1] - blk[0])
        assert abs(tot - n_ * p) < 5 * math.sqrt(n_ * p * (1 - p))
    # pairs: adjacent slots, across the block boundary, and far apart are independent
    for a, b in ((0, 1), (500, 501), (1023, 1024), (2047, 2048), (10, 2000)):
        both = float(np.mean(L[:, a] & L[:, b]))
        assert abs(both - p * p) < 5 * math.sqrt(p * p * (1 - p * p) / N), (a, b, both)
    # live count per hub set ~ Binomial(d, p)
    k = L.sum(axis=1)
    assert abs(k.mean() - d * p) < 5 * math.sqrt(d * p * (1 - p) / N)
    assert abs(k.var() / (d * p * (1 - p)) - 1.0) < 0.1


def test_slot_rates_wc():
    d = 1500                                                    # p = 1/1500, two blocks
    g = _bipartite(d, 3 * d)
    L = _hub_live_matrix(g, d, gi.W_WC, 0.0, 400000, 12)
    N = len(L)
    p = 1.0 / d
    k = L.sum(axis=1)
    assert abs(k.mean() - 1.0) < 5 * math.sqrt((1 - p) / N)     # E[live in-edges] = d * 1/d = 1
    assert abs(k.var() / (1 - p) - 1.0) < 0.05
    for blk in ((0, 1024), (1024, 1500)):
        tot = L[:, blk[0]:blk[1]].sum()
        n_ = N * (blk[1] - blk[0])
        assert abs(tot - n_ * p) < 5 * math.sqrt(n_ * p)


@pytest.mark.parametrize("scheme", [gi.W_WC, gi.W_UNIFORM])
def test_skip_estimator_vs_exact(scheme):
    """Eq. 3: n * Pr[S cap RR != {}] equals the exact spread over live-edge worlds."""
    for gg, seed in ((gi.diamond(), 41), (gi.cycle_plus(), 42), (gi.random_small(6, 10, 44), 43)):
        pu = 0.45 if scheme == gi.W_UNIFORM else 0.0
        o = oracle.Oracle(gg, gi.IC, scheme, pu)
        o.set_skip(True)
        _check_estimator(gg, o, list(_ic_worlds(gg, _p_exact(gg, scheme, pu))), seed, 30000,
                         [[0], [1, 2]])


# ---- independent pure-Python evaluation of the contract --------------------------------------
def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))      # one correctly rounded result


def _ln_series_ref(x):
    m, e = math.frexp(x)                                        # x = m 2^e, m in [0.5, 1)
    m, e = m * 2.0, e - 1                                       # m in [1, 2)
    if m > 1.4142135623730951:
        m, e = m * 0.5, e + 1
    y = (m - 1.0) / (m + 1.0)
    y2 = y * y
    s = 1.0 / 19.0
    for k in (17, 15, 13, 11, 9, 7, 5, 3):
        s = _fma(s, y2, 1.0 / k)
    s = _fma(s, y2, 1.0)
    return e * 6.93147180369123816490e-01 + (e * 1.90821492927058770002e-10 + (2.0 * y) * s)


_TAB = {k: (_ln_series_ref(1.0 + k / 256.0), 1.0 / (1.0 + k / 256.0)) for k in range(-75, 107)}


def _ln_ref(x):
    m, e = math.frexp(x)
    m, e = m * 2.0, e - 1
    if m > 1.4142135623730951:
        m, e = m * 0.5, e + 1
    k = math.floor((m - 1.0) * 256.0 + 0.5)
    L, R = _TAB[k]
    t = (m - (1.0 + k / 256.0)) * R
    s = 1.0 / 7.0
    for c in (-1.0 / 6.0, 1.0 / 5.0, -1.0 / 4.0, 1.0 / 3.0, -1.0 / 2.0, 1.0):
        s = _fma(s, t, c)
    return e * 6.93147180369123816490e-01 + (e * 1.90821492927058770002e-10 + (L + t * s))


def _skip_live_ref(g, scheme, pu, seed, rr_id):
    live = []
    for v in range(g.n):
        a, b = int(g.row_ptr[v]), int(g.row_ptr[v + 1])
        d = b - a
        if d == 0 or (scheme == gi.W_UNIFORM and pu == 0.0):
            continue
        q = (d - 1) / d if scheme == gi.W_WC else 1.0 - float(np.float32(pu))
        inv = 0.0 if q <= 0.0 else 1.0 / _ln_ref(q)
        for blk in range((d + 1023) // 1024):
            pos, end, j = blk * 1024, min(d, blk * 1024 + 1024), 0
            while pos < end:
                if inv != 0.0:
                    w = philox4x32_10([rr_id & 0xFFFFFFFF, 0x80000000 | blk, v, j >> 2],
                                      [seed & 0xFFFFFFFF, seed >> 32])[j & 3]
                    j += 1
                    gap = math.floor(_ln_ref((w + 0.5) * 2.0 ** -32) * inv)
                    if gap >= end - pos:
                        break
                    pos += gap
                live.append((int(g.src[a + pos]), v))
                pos += 1
    return live


def test_skip_words_and_gaps_match_reference():
    rng = np.random.default_rng(3)
    for _ in range(200):
        seed, rid = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**32))
        v, blk, j = int(rng.integers(0, 2**32)), int(rng.integers(0, 2**21)), int(rng.integers(0, 5000))
        w = philox4x32_10([rid, 0x80000000 | blk, v, j >> 2], [seed & 0xFFFFFFFF, seed >> 32])[j & 3]
        assert oracle.skip_word(seed, rid, v, blk, j) == w
        x = float(rng.uniform(1e-12, 1.5))
        assert oracle.skip_ln(x) == _ln_ref(x)
        assert oracle.skip_ln_series(x) == _ln_series_ref(x)


@pytest.mark.parametrize("scheme", [gi.W_WC, gi.W_UNIFORM])
def test_skip_rr_equals_bruteforce_reachability(scheme):
    seed = 987654321
    graphs = _tiny_graphs() + [_bipartite(1100, 3)]
    for gg in graphs:
        pu = 0.37 if scheme == gi.W_UNIFORM else 0.0
        o = oracle.Oracle(gg, gi.IC, scheme, pu)
        o.set_skip(True)
        ids = range(25) if gg.n < 100 else range(8)
        for i in ids:
            want = _closure_reaching(gg.n, _skip_live_ref(gg, scheme, pu, seed, i), _root_ref(seed, i, gg.n))
            assert o.rr_set(seed, i).tolist() == sorted(want), (gg.name, i)


def test_skip_option_errors_and_degenerate():
    d = gi.diamond()
    with pytest.raises(ValueError):
        oracle.Oracle(d, gi.LT, gi.W_WC).set_skip(True)
    with pytest.raises(ValueError):
        oracle.Oracle(gi.with_weights(d, np.full(4, 0.5)), gi.IC, gi.W_EXPLICIT).set_skip(True)
    # p = 0: only the root; p = 1: the whole reverse closure, no draws
    for pu, want in ((0.0, lambda r: [r]), (1.0, None)):
        o = oracle.Oracle(gi.chain(4), gi.IC, gi.W_UNIFORM, pu)
        o.set_skip(True)
        for i in range(10):
            r = _root_ref(5, i, 4)
            got = o.rr_set(5, i).tolist()
            assert got == (want(r) if want else list(range(r + 1)))
    assert oracle.skip_inv(gi.W_WC, 1) == 0.0 and oracle.skip_inv(gi.W_UNIFORM, 9, 1.0) == 0.0
