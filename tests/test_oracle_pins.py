"""Pins of the oracle (oracle/gim_oracle.c) against what the paper and mathematics fix.

Each test pins one oracle function to something other than itself:
known-answer vectors, exact enumeration of live-edge worlds (rational arithmetic), brute-force
reachability on the coin-defined instance graph, brute-force max coverage, and closed forms
evaluated in 40-digit arithmetic. A plausible mistake anywhere in the oracle (a dropped term, a
wrong sign or index, a transposed edge direction) fails at least one of them.
"""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import gim_inputs as gi
import oracle
from tests.philox_ref import keyed, philox4x32_10

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SEED = 200907325


# --------------------------------------------------------------------------------------
# O2: Philox4x32-10
# --------------------------------------------------------------------------------------
def _kat():
    rows = []
    for line in open(os.path.join(GOLD, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        x = [int(t, 16) for t in line.split()]
        rows.append((x[0:4], x[4:6], x[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,expect", _kat())
def test_philox_kat_oracle(ctr, key, expect):
    assert [int(v) for v in oracle.philox(ctr, key)] == expect


@pytest.mark.parametrize("ctr,key,expect", _kat())
def test_philox_kat_python_ref(ctr, key, expect):
    assert philox4x32_10(ctr, key) == expect


# --------------------------------------------------------------------------------------
# O2-O7 golden vectors (independent evaluation)
# --------------------------------------------------------------------------------------
def _gold():
    return json.load(open(os.path.join(GOLD, "diamond_keyscheme.json")))


def _sets_str(o, seed, T):
    return ["".join(str(int(v)) for v in o.rr_set(seed, i)) for i in range(T)]


def test_keyscheme_roots_and_coins():
    g = _gold()
    assert [oracle.root(g["seed"], i, 4) for i in range(16)] == g["roots_n4"]
    assert [format(oracle.coin(g["seed"], 0, e), "08x") for e in range(4)] == g["coins_id0_e0_3"]
    assert [oracle.root(g["seed"], i, 4847571) for i in range(4)] == g["roots_n4847571_id0_3"]
    assert [oracle.root(g["seed"], i, 41652230) for i in range(4)] == g["roots_n41652230_id0_3"]


@pytest.mark.parametrize("case", ["ic_wc", "ic_half", "lt_wc"])
def test_keyscheme_diamond_sets_counts_greedy(case):
    gd = _gold()
    d = gi.diamond()
    if case == "ic_wc":
        o = oracle.Oracle(d, gi.IC, gi.W_WC)
    elif case == "ic_half":
        o = oracle.Oracle(gi.with_weights(d, np.full(4, 0.5)), gi.IC, gi.W_EXPLICIT)
    else:
        o = oracle.Oracle(d, gi.LT, gi.W_WC)
    assert _sets_str(o, gd["seed"], 16) == gd[case + "_sets"]
    o.generate(16, gd["seed"])
    off, nodes, cnt = o.export()
    assert cnt.tolist() == gd[case + "_counts"]
    assert off.tolist() == [0] + list(np.cumsum([len(s) for s in gd[case + "_sets"]]))
    seeds, gains, cov = o.select(2)
    assert seeds.tolist() == gd[case + "_greedy_k2"]["seeds"]
    assert gains.tolist() == gd[case + "_greedy_k2"]["gains"]
    assert cov == sum(gains.tolist())


# --------------------------------------------------------------------------------------
# O3/O4/O5 vs brute-force reachability on the coin-defined instance graph.
# The instance graph g: edge e=(u,v) kept iff U < p_uv, with U = coin/2^32
# (reading R16). The RR set of root r is {u : u reaches r in g}. Computed here by
# transitive closure, with exact rational comparison — independent of the oracle's BFS and
# of its integer threshold arithmetic.
# --------------------------------------------------------------------------------------
def _edge_list(g):
    dst = np.repeat(np.arange(g.n), np.diff(g.row_ptr).astype(np.int64))
    return [(int(u), int(v)) for u, v in zip(g.src, dst)]


def _p_exact(g, scheme, p_uniform=0.0):
    din = g.in_degree()
    out = []
    for e, (u, v) in enumerate(_edge_list(g)):
        if scheme == gi.W_WC:
            out.append(Fraction(1, int(din[v])))
        elif scheme == gi.W_UNIFORM:
            out.append(Fraction(float(np.float32(p_uniform))))
        else:
            out.append(Fraction(float(g.weights[e])))
    return out


def _closure_reaching(n, live_edges, target):
    reach = [[False] * n for _ in range(n)]
    for i in range(n):
        reach[i][i] = True
    for u, v in live_edges:
        reach[u][v] = True
    for k in range(n):
        for i in range(n):
            if reach[i][k]:
                for j in range(n):
                    if reach[k][j]:
                        reach[i][j] = True
    return sorted(u for u in range(n) if reach[u][target])


def _root_ref(seed, rr_id, n):
    o = keyed(seed, rr_id, 1 << 63)
    u64 = o[0] | (o[1] << 32)
    return (u64 * n) >> 64          # floor(U * n) with U = u64 / 2^64 (reading R17)


def _ic_rr_bruteforce(g, p, seed, rr_id):
    live = []
    for e, (u, v) in enumerate(_edge_list(g)):
        coin = keyed(seed, rr_id, e >> 2)[e & 3]
        if Fraction(coin, 1 << 32) < p[e]:
            live.append((u, v))
    return _closure_reaching(g.n, live, _root_ref(seed, rr_id, g.n))


def _lt_rr_bruteforce(g, scheme, seed, rr_id):
    """LT live-edge world: every node v picks at most one in-edge, edge t with probability
    w_t, via the draw r = Philox(seed; id, 2^62|v).out[0] and the fixed-point
    half-open intervals of reading R18 (WC: exactly [t/d, (t+1)/d))."""
    live = []
    for v in range(g.n):
        a, b = int(g.row_ptr[v]), int(g.row_ptr[v + 1])
        d = b - a
        if d == 0:
            continue
        r = keyed(seed, rr_id, (1 << 62) | v)[0]
        pick = None
        if scheme == gi.W_WC:
            for t in range(d):
                if Fraction(t, d) <= Fraction(r, 1 << 32) < Fraction(t + 1, d):
                    pick = t
        else:
            acc = 0
            for t in range(d):
                lo = acc
                acc += math.floor(Fraction(float(g.weights[a + t])) * (1 << 32))
                if lo <= r < acc:
                    pick = t
        if pick is not None:
            live.append((int(g.src[a + pick]), v))
    return _closure_reaching(g.n, live, _root_ref(seed, rr_id, g.n))


def _tiny_graphs():
    out = [gi.diamond(), gi.chain(4), gi.cycle_plus(), gi.star_in(5)]
    for s in range(6):
        out.append(gi.random_small(7, 14, s))
    return out


@pytest.mark.parametrize("scheme", ["wc", "uniform", "explicit"])
def test_rr_ic_equals_bruteforce_reachability(scheme):
    rng = np.random.default_rng(7)
    for gidx, g in enumerate(_tiny_graphs()):
        if scheme == "wc":
            o, p = oracle.Oracle(g, gi.IC, gi.W_WC), _p_exact(g, gi.W_WC)
        elif scheme == "uniform":
            o, p = oracle.Oracle(g, gi.IC, gi.W_UNIFORM, 0.3), _p_exact(g, gi.W_UNIFORM, 0.3)
        else:
            w = rng.choice([0.0, 0.25, 0.5, 0.7, 1.0], size=g.m).astype(np.float32)
            gw = gi.with_weights(g, w)
            o, p = oracle.Oracle(gw, gi.IC, gi.W_EXPLICIT), _p_exact(gw, gi.W_EXPLICIT)
        seed = 1000 + gidx * 7919
        for i in range(60):
            assert o.rr_set(seed, i).tolist() == _ic_rr_bruteforce(g, p, seed, i), (g.name, i)


@pytest.mark.parametrize("scheme", ["wc", "explicit"])
def test_rr_lt_equals_bruteforce_reachability(scheme):
    rng = np.random.default_rng(11)
    for gidx, g in enumerate(_tiny_graphs()):
        if scheme == "wc":
            gg, o = g, oracle.Oracle(g, gi.LT, gi.W_WC)
        else:
            din = g.in_degree()
            dst = np.repeat(np.arange(g.n), din)
            w = (rng.uniform(0.2, 1.0, size=g.m) / np.maximum(din[dst], 1)).astype(np.float32)
            gg = gi.with_weights(g, w)
            o = oracle.Oracle(gg, gi.LT, gi.W_EXPLICIT)
        seed = 77 + gidx
        for i in range(60):
            assert o.rr_set(seed, i).tolist() == _lt_rr_bruteforce(gg, gi.W_WC if scheme == "wc"
                                                                    else gi.W_EXPLICIT, seed, i)


def test_rr_trivial_cases():
    # p=1 chain 0->1->2, root 2 -> {0,1,2}; p=0 -> {root} (SPEC.md S:136-137 ideas)
    c = gi.chain(3)
    o1 = oracle.Oracle(gi.with_weights(c, np.ones(2)), gi.IC, gi.W_EXPLICIT)
    o0 = oracle.Oracle(gi.with_weights(c, np.zeros(2)), gi.IC, gi.W_EXPLICIT)
    for i in range(50):
        r = oracle.root(5, i, 3)
        assert o1.rr_set(5, i).tolist() == list(range(r + 1))
        assert o0.rr_set(5, i).tolist() == [r]
    # single-node graph, T=5 -> offsets [0..5], count[0]=5
    g1 = gi.from_edges(1, [])
    o = oracle.Oracle(g1, gi.IC, gi.W_WC)
    o.generate(5, 3)
    off, nodes, cnt = o.export()
    assert off.tolist() == [0, 1, 2, 3, 4, 5] and cnt.tolist() == [5]


def test_generate_extend_truncate_reseed():
    g = gi.random_small(8, 20, 3)
    o = oracle.Oracle(g, gi.IC, gi.W_WC)
    o.generate(100, 9)
    full = o.export()
    o.generate(40, 9)
    part = o.export()
    assert part[0].tolist() == full[0][:41].tolist()
    o.generate(100, 9)
    again = o.export()
    assert all(np.array_equal(a, b) for a, b in zip(full, again))
    o.generate(100, 10)
    assert not np.array_equal(o.export()[1], full[1])
    # counts equal the recomputed histogram; sets ascending and distinct (O6)
    off, nodes, cnt = full
    assert np.array_equal(np.bincount(nodes, minlength=g.n), cnt)
    for i in range(100):
        s = nodes[off[i]:off[i + 1]]
        assert len(s) >= 1 and np.all(np.diff(s.astype(np.int64)) > 0)


def test_root_uniformity_chi2():
    n, T = 37, 40000
    h = np.bincount([oracle.root(123, i, n) for i in range(T)], minlength=n)
    chi2 = float(np.sum((h - T / n) ** 2 / (T / n)))
    assert chi2 < 70.0       # chi2_{36} 0.999 quantile ~ 67.985


def test_coin_threshold_frequencies():
    # live rate vs p in {1/2, 1/3, 1/7, 0.01} within 4 sigma (SURVEY.md §8(c) pins)
    T = 200000
    coins = np.array([oracle.coin(99, i // 50, i % 50) for i in range(T)], dtype=np.uint64)
    for p, rule in [(0.5, coins * 2 < 2**32), (1 / 3, coins * 3 < 2**32),
                    (1 / 7, coins * 7 < 2**32), (0.01, coins < math.ceil(float(np.float32(0.01)) * 2**32))]:
        f = float(np.mean(rule))
        assert abs(f - p) < 4 * math.sqrt(p * (1 - p) / T), (p, f)


# --------------------------------------------------------------------------------------
# Eq. 3 and the RR definition by exact enumeration of worlds
# --------------------------------------------------------------------------------------
def _ic_worlds(g, p):
    edges = _edge_list(g)
    for mask in range(1 << len(edges)):
        pr = Fraction(1)
        live = []
        for e, (u, v) in enumerate(edges):
            if mask >> e & 1:
                pr *= p[e]
                live.append((u, v))
            else:
                pr *= 1 - p[e]
        if pr:
            yield pr, live


def _lt_worlds(g, w):
    """Each node picks at most one in-edge, edge t with probability w_t, none w.p. 1-sum."""
    choices = []
    for v in range(g.n):
        a, b = int(g.row_ptr[v]), int(g.row_ptr[v + 1])
        opts = [(w[e], (int(g.src[e]), v)) for e in range(a, b)]
        opts.append((1 - sum(w[e] for e in range(a, b)), None))
        choices.append([o for o in opts if o[0]])
    for combo in itertools.product(*choices):
        pr = Fraction(1)
        live = []
        for q, ed in combo:
            pr *= q
            if ed is not None:
                live.append(ed)
        yield pr, live


def _forward_reach(n, live, S):
    adj = [[] for _ in range(n)]
    for u, v in live:
        adj[u].append(v)
    seen, st = set(S), list(S)
    while st:
        x = st.pop()
        for y in adj[x]:
            if y not in seen:
                seen.add(y)
                st.append(y)
    return seen


def exact_spread(g, worlds, S):
    """E[I(S)] = E[|R(S)|] over instance graphs."""
    return sum(pr * len(_forward_reach(g.n, live, S)) for pr, live in worlds)


def exact_ris(g, worlds, S):
    """n * Pr[S cap RR != {}] with a uniform root (right-hand side of Eq. 3)."""
    tot = Fraction(0)
    for pr, live in worlds:
        hit = sum(1 for r in range(g.n) if any(r in _forward_reach(g.n, live, [s]) for s in S))
        tot += pr * Fraction(hit, g.n)
    return g.n * tot


def test_enumeration_diamond_values():
    d = gi.diamond()
    half = [Fraction(1, 2)] * 4
    W = list(_ic_worlds(d, half))
    # Pr[0 in RR(3)] = 7/16 (re-derived)
    assert sum(pr for pr, live in W if 3 in _forward_reach(4, live, [0])) == Fraction(7, 16)
    assert exact_spread(d, W, [0]) == Fraction(39, 16)
    assert exact_spread(d, W, [1]) == Fraction(3, 2)
    assert exact_spread(d, W, [1, 2]) == Fraction(11, 4)
    assert exact_spread(d, W, [0, 3]) == 3
    Wwc = list(_ic_worlds(d, _p_exact(d, gi.W_WC)))
    assert exact_spread(d, Wwc, [0]) == Fraction(15, 4)
    assert exact_spread(d, Wwc, [1, 2]) == Fraction(11, 4)
    wlt = _p_exact(d, gi.W_WC)
    Wlt = list(_lt_worlds(d, wlt))
    assert exact_spread(d, Wlt, [0]) == 4 and exact_spread(d, Wlt, [1, 2]) == 3
    cp = gi.cycle_plus()
    Wc = list(_lt_worlds(cp, _p_exact(cp, gi.W_WC)))
    assert [exact_spread(cp, Wc, [s]) for s in range(4)] == [3, Fraction(5, 2), 2, Fraction(5, 2)]
    # Eq. 3 identity holds exactly on the definitions
    for S in ([0], [1, 2], [3]):
        assert exact_spread(d, W, S) == exact_ris(d, W, S)
        assert exact_spread(d, Wlt, S) == exact_ris(d, Wlt, S)


def _check_estimator(g, o, worlds, seed, T, sets_to_test):
    o.generate(T, seed)
    off, nodes, cnt = o.export()
    for S in sets_to_test:
        hit = 0
        for i in range(T):
            s = nodes[off[i]:off[i + 1]]
            if np.intersect1d(s, S).size:
                hit += 1
        f = hit / T
        ex = float(exact_spread(g, worlds, S)) / g.n
        se = math.sqrt(max(ex * (1 - ex), 1e-12) / T)
        assert abs(f - ex) < 4.5 * se + 1e-12, (S, f, ex)
    # root-marginal: count[u]/T vs (1/n) sum_v Pr[u reaches v]
    for u in range(g.n):
        ex = float(exact_spread(g, worlds, [u])) / g.n
        f = cnt[u] / T
        se = math.sqrt(max(ex * (1 - ex), 1e-12) / T)
        assert abs(f - ex) < 4.5 * se + 1e-12, (u, f, ex)


def test_ic_estimator_vs_exact():
    d = gi.diamond()
    o = oracle.Oracle(gi.with_weights(d, np.full(4, 0.5)), gi.IC, gi.W_EXPLICIT)
    _check_estimator(d, o, list(_ic_worlds(d, [Fraction(1, 2)] * 4)), 31, 40000,
                     [[0], [1, 2], [3], [0, 3]])
    g = gi.random_small(6, 10, 42)
    o = oracle.Oracle(g, gi.IC, gi.W_WC)
    _check_estimator(g, o, list(_ic_worlds(g, _p_exact(g, gi.W_WC))), 32, 40000, [[0], [2, 5]])


def test_lt_estimator_vs_exact():
    for g in (gi.diamond(), gi.cycle_plus(), gi.random_small(6, 10, 43)):
        o = oracle.Oracle(g, gi.LT, gi.W_WC)
        _check_estimator(g, o, list(_lt_worlds(g, _p_exact(g, gi.W_WC))), 33, 30000, [[0], [1, 2]])


def test_forward_mc_vs_exact():
    d = gi.diamond()
    for model, worlds in ((gi.IC, list(_ic_worlds(d, _p_exact(d, gi.W_WC)))),
                          (gi.LT, list(_lt_worlds(d, _p_exact(d, gi.W_WC))))):
        o = oracle.Oracle(d, model, gi.W_WC)
        for S in ([0], [1, 2], [1]):
            mean, se = o.mc_spread(S, 40000, 5)
            assert abs(mean - float(exact_spread(d, worlds, S))) < 4.5 * se + 1e-9


def _mc_cases():
    """og_mc_spread's non-WC branches (IC uniform, IC explicit, LT explicit) on the diamond and the
    cycle-plus-tail graph. Weights differ per in-slot so that a wrong slot index, a swapped
    source/destination or a dropped weight moves the exact spread by far more than 4.5 standard
    errors at 40,000 trials."""
    d, cy = gi.diamond(), gi.cycle_plus()
    # diamond in-slots: e0 0->1, e1 0->2, e2 1->3, e3 2->3; cycle_plus: e0 2->0, e1 3->0, e2 0->1, e3 1->2
    return [
        ("ic_uni_diamond", d, gi.IC, gi.W_UNIFORM, 0.3),
        ("ic_uni_cycle", cy, gi.IC, gi.W_UNIFORM, 0.55),
        ("ic_exp_diamond", gi.with_weights(d, [0.9, 0.2, 0.6, 0.1]), gi.IC, gi.W_EXPLICIT, 0.0),
        ("ic_exp_cycle", gi.with_weights(cy, [0.7, 0.25, 0.5, 0.95]), gi.IC, gi.W_EXPLICIT, 0.0),
        ("lt_exp_diamond", gi.with_weights(d, [0.9, 0.2, 0.6, 0.3]), gi.LT, gi.W_EXPLICIT, 0.0),
        ("lt_exp_cycle", gi.with_weights(cy, [0.45, 0.35, 0.8, 0.6]), gi.LT, gi.W_EXPLICIT, 0.0),
    ]


@pytest.mark.parametrize("case", _mc_cases(), ids=lambda c: c[0])
def test_forward_mc_vs_exact_weight_schemes(case):
    """Forward MC (IC P:118-122; LT Eq. 1 P:127-131 with the exact thresholds of reading R30)
    against the exact spread over all live-edge worlds (IC: each edge live w.p. p_e; LT: each node
    keeps at most one in-edge, edge t w.p. w_t — the live-edge view of LT)."""
    _, g, model, scheme, pu = case
    p = _p_exact(g, scheme, pu)
    worlds = list(_ic_worlds(g, p)) if model == gi.IC else list(_lt_worlds(g, p))
    o = oracle.Oracle(g, model, scheme, pu)
    for S in ([0], [1], [2], [3], [1, 2]):
        exact = float(exact_spread(g, worlds, S))
        mean, se = o.mc_spread(S, 40000, 17)
        assert abs(mean - exact) < 4.5 * se + 1e-9, (S, mean, exact, se)


# --------------------------------------------------------------------------------------
# O7: NodeSelection vs brute force
# --------------------------------------------------------------------------------------
def _pool(sets):
    off = np.concatenate([[0], np.cumsum([len(s) for s in sets])]).astype(np.uint64)
    nodes = np.concatenate([np.sort(np.asarray(s, dtype=np.uint32)) for s in sets]) if sets else \
        np.zeros(0, dtype=np.uint32)
    return off, nodes


def test_select_spec_examples():
    # {1,2},{2,3},{3}, k=1 -> 2
    seeds, gains, cov = oracle.select_pool(4, *_pool([[1, 2], [2, 3], [3]]), k=1)
    assert seeds.tolist() == [2] and gains.tolist() == [2]
    # occur [3,5,5] -> node 1: sets realising counts 3,5,5
    sets = [[0, 1, 2]] * 3 + [[1, 2]] * 2
    seeds, gains, _ = oracle.select_pool(3, *_pool(sets), k=1)
    assert seeds.tolist() == [1] and gains.tolist() == [5]
    # retire 2 over {1,2},{2,3},{2} -> all zero; the next pick is the lowest unselected id
    seeds, gains, cov = oracle.select_pool(4, *_pool([[1, 2], [2, 3], [2]]), k=2)
    assert seeds.tolist() == [2, 0] and gains.tolist() == [3, 0] and cov == 3


def _coverage(sets, S):
    S = set(S)
    return sum(1 for s in sets if S.intersection(s))


@pytest.mark.parametrize("trial", range(25))
def test_select_greedy_bruteforce(trial):
    rng = np.random.default_rng(trial)
    n = int(rng.integers(3, 10))
    nsets = int(rng.integers(1, 20))
    sets = [sorted(rng.choice(n, size=int(rng.integers(1, n + 1)), replace=False).tolist())
            for _ in range(nsets)]
    k = int(rng.integers(1, n + 1))
    seeds, gains, cov = oracle.select_pool(n, *_pool(sets), k=k)
    chosen = []
    for j in range(k):
        base = _coverage(sets, chosen)
        marg = [(_coverage(sets, chosen + [v]) - base) if v not in chosen else -1 for v in range(n)]
        best = max(marg)
        u = marg.index(best)                 # lowest id among ties (R10)
        assert seeds[j] == u and gains[j] == best, (j, seeds, gains, marg)
        chosen.append(u)
    assert cov == _coverage(sets, chosen)
    opt = max(_coverage(sets, c) for c in itertools.combinations(range(n), k))
    assert cov >= (1 - 1 / math.e) * opt - 1e-9     # greedy max-cover guarantee


# --------------------------------------------------------------------------------------
# O8: IMM constants vs 40-digit closed forms (mpmath), invariants, and the driver
# --------------------------------------------------------------------------------------
def _mp_constants(n, k, eps, ell):
    import mpmath as mp
    mp.mp.dps = 40
    n_, eps_ = mp.mpf(n), mp.mpf(eps)
    ell_eff = mp.mpf(ell) * (1 + mp.log(2) / mp.log(n_))
    epsp = mp.sqrt(2) * eps_
    lnC = mp.log(mp.binomial(n, k))
    lam_p = (2 + mp.mpf(2) / 3 * epsp) * (lnC + ell_eff * mp.log(n_) + mp.log(mp.log(n_, 2))) * n_ / epsp ** 2
    a = mp.sqrt(ell_eff * mp.log(n_) + mp.log(2))
    b = mp.sqrt((1 - 1 / mp.e) * (lnC + ell_eff * mp.log(n_) + mp.log(2)))
    lam_s = 2 * n_ * ((1 - 1 / mp.e) * a + b) ** 2 / eps_ ** 2
    return dict(ell_eff=ell_eff, eps_prime=epsp, lnC=lnC, lambda_prime=lam_p, alpha=a, beta=b,
                lambda_star=lam_s)


@pytest.mark.parametrize("n,k,eps", [(1000, 10, 0.1), (15233, 50, 0.5), (75879, 50, 0.1),
                                     (4847571, 50, 0.1), (41652230, 100, 0.1), (8, 2, 0.1),
                                     (2, 1, 0.3), (10, 10, 0.2)])
def test_imm_constants_mpmath(n, k, eps):
    got = oracle.imm_constants(n, k, eps, 1.0)
    ref = _mp_constants(n, k, eps, 1.0)
    for key in got:
        r = float(ref[key])
        assert abs(got[key] - r) <= 1e-12 * max(abs(r), 1e-300), key


def test_imm_constants_survey_values_and_invariants():
    c = oracle.imm_constants(1000, 10, 0.1, 1.0)
    assert abs(c["lnC"] - 53.927997037888276) < 1e-12 * 54
    assert abs(c["lambda_prime"] - 6683694.0621400805) < 1e-12 * 6.7e6
    assert abs(c["lambda_star"] - 13096023.335691445) < 1e-12 * 1.3e7
    assert abs(oracle.imm_constants(10, 2, 0.1)["lnC"] - math.log(45)) < 1e-12
    c2 = oracle.imm_constants(1000, 10, 0.05, 1.0)
    assert abs(c2["lambda_star"] / c["lambda_star"] - 4.0) < 1e-12      # eps^-2 scaling
    for bad in [(1, 1, 0.1), (10, 0, 0.1), (10, 11, 0.1), (10, 2, 0.0), (10, 2, 1.0)]:
        with pytest.raises(ValueError):
            oracle.imm_constants(*bad)
    # LB plug-in of SPEC.md S:250: n=100, F=0.6, eps=0.1 -> 52.566039414
    assert abs(100 * 0.6 / (1 + math.sqrt(2) * 0.1) - 52.566039414) < 1e-8


def test_imm_driver_trace():
    g = gi.workload_graph("C1")
    w = gi.WORKLOADS["C1"]
    o = oracle.Oracle(g, w.model, w.scheme)
    r = o.imm(w.k, w.eps, w.ell, w.rr_seed)
    c = oracle.imm_constants(g.n, w.k, w.eps, w.ell)
    assert r.lambda_prime == c["lambda_prime"] and r.lambda_star == c["lambda_star"]
    x = [g.n / 2.0 ** i for i in range(1, r.rounds + 1)]
    for i in range(r.rounds):
        assert r.theta_i[i] == c["lambda_prime"] / x[i]
        assert r.T_i[i] == math.ceil(r.theta_i[i])
        passed = (g.n * float(r.cov_i[i])) / float(r.T_i[i]) >= (1 + c["eps_prime"]) * x[i]
        assert passed == (i == r.rounds - 1 and r.LB > 1.0)
    assert 1.0 <= r.LB <= g.n
    assert r.theta == c["lambda_star"] / r.LB
    assert r.R_final == max(int(r.T_i[-1]), math.ceil(r.theta))
    assert len(set(r.seeds.tolist())) == w.k
    assert np.all(np.diff(r.gains.astype(np.int64)) <= 0)     # greedy gains non-increasing
    assert r.cov == int(r.gains.sum())
    assert abs(r.spread_est - g.n * r.cov / r.R_final) < 1e-9 * g.n


@pytest.mark.slow
def test_imm_guarantee_tiny_graphs():
    """(1-1/e-eps) * OPT with probability >= 1 - 1/n^ell (SPEC.md S:505 idea), exact spreads."""
    ok = 0
    runs = 40
    for t in range(runs):
        g = gi.random_small(8, 10, 500 + t)
        p = _p_exact(g, gi.W_WC)
        W = list(_ic_worlds(g, p))
        spreads = {S: exact_spread(g, W, list(S)) for S in itertools.combinations(range(8), 2)}
        opt = max(spreads.values())
        o = oracle.Oracle(g, gi.IC, gi.W_WC)
        r = o.imm(2, 0.1, 1.0, 900 + t)
        got = spreads[tuple(sorted(r.seeds.tolist()))]
        ok += got >= (1 - 1 / math.e - 0.1) * opt
    assert ok >= runs - 2


@pytest.mark.slow
def test_mc_spread_vs_ris_estimate_C1():
    """Forward MC spread of IMM's seeds within 1% of n*F_R'(S) on an independent pool."""
    g = gi.workload_graph("C1")
    w = gi.WORKLOADS["C1"]
    o = oracle.Oracle(g, w.model, w.scheme)
    r = o.imm(w.k, w.eps, w.ell, w.rr_seed)
    o2 = oracle.Oracle(g, w.model, w.scheme)
    T = 200000
    o2.generate(T, w.rr_seed + 1)
    off, nodes, _ = o2.export()
    S = np.sort(r.seeds)
    hit = np.zeros(T, dtype=bool)
    member = np.isin(nodes, S)
    idx = np.repeat(np.arange(T), np.diff(off).astype(np.int64))
    hit[idx[member]] = True
    ris = g.n * hit.mean()
    mean, se = o.mc_spread(r.seeds, 20000, 17)
    assert se / mean < 0.003
    assert abs(mean - ris) / mean < 0.01, (mean, ris)


def test_imm_fresh_final_pool_C1():
    """R29 (SURVEY R8's NEXT variant, Chen 2018 [EXT]): with a fresh final pool the estimation
    trace is IMM's unchanged, and the final seeds are exactly NodeSelection over the
    ceil(lambda*/LB) sets of the second key — recomputed here by composing the pinned og_generate
    and og_select, not by the driver."""
    g = gi.workload_graph("C1")
    w = gi.WORKLOADS["C1"]
    o = oracle.Oracle(g, w.model, w.scheme)
    r = o.imm(w.k, w.eps, w.ell, w.rr_seed)
    o.set_fresh_final(True)
    f = o.imm(w.k, w.eps, w.ell, w.rr_seed)
    assert (f.rounds, f.LB, f.theta) == (r.rounds, r.LB, r.theta)
    assert np.array_equal(f.T_i, r.T_i) and np.array_equal(f.cov_i, r.cov_i)
    T = math.ceil(f.theta)
    assert f.R_final == T
    o2 = oracle.Oracle(g, w.model, w.scheme)
    o2.generate(T, w.rr_seed ^ 0x9E3779B97F4A7C15)
    s, gn, cov = o2.select(w.k)
    assert np.array_equal(f.seeds, s) and np.array_equal(f.gains, gn) and f.cov == cov
    assert abs(f.spread_est - g.n * cov / T) < 1e-9 * g.n
    # the fresh pool shares no set with the estimation pool's key: its estimate is not biased by
    # the selection (R24) — both estimates agree within a few percent on C1
    assert abs(f.spread_est - r.spread_est) / r.spread_est < 0.05
