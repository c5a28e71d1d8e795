"""Pins of the oracle's MRIM functions (multi-round IM, CR-NAIMM as gIM adapts it, §4.8
P:818-822; readings R26-R28 in DESIGN.md §3) against things other than the oracle itself:
  * the T = 1 reduction to the pinned standard pipeline (RR sets, counts, selection, IMM);
  * brute-force reachability of every round's live-edge world with an independent Python
    Philox (tests/philox_ref.py) and the shared root of P:820;
  * exact enumeration of the independent rounds' live-edge worlds: the MRIM objective
    E[#nodes influenced at least once] equals n * Pr[S cap MRR != {}] exactly, and the
    sampler hits it within 4.5 sigma (a dropped round key, i.e. identical rounds, fails it);
  * brute-force greedy with per-round budgets, the partition-matroid greedy bound 1/2 * OPT;
  * ln C(nT, kT) closed forms in mpmath and the driver's trace identities.
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

import gim_inputs as gi
import oracle
from tests.philox_ref import keyed
from tests.test_oracle_pins import (_closure_reaching, _edge_list, _forward_reach, _ic_worlds,
                                    _lt_worlds, _p_exact, _root_ref, _tiny_graphs)

SEED = 200907325


def _pool_sets(off, nodes):
    return [nodes[off[i]:off[i + 1]].tolist() for i in range(len(off) - 1)]


# ---- T = 1 reduction ------------------------------------------------------------------------
@pytest.mark.parametrize("model,scheme", [(gi.IC, gi.W_WC), (gi.IC, gi.W_EXPLICIT), (gi.LT, gi.W_WC)])
def test_mrim_T1_equals_standard_pool_and_selection(model, scheme):
    for g in _tiny_graphs()[:6]:
        if scheme == gi.W_EXPLICIT:
            g = gi.with_weights(g, np.full(g.m, 0.5 if model == gi.IC else 0.3, dtype=np.float32))
        o = oracle.Oracle(g, model, scheme)
        o.generate(700, SEED)
        off, nodes, cnt = o.export()
        o.mrim_generate(700, 1, SEED)
        moff, mpairs, mcnt = o.mrim_export()
        assert np.array_equal(off, moff) and np.array_equal(nodes, mpairs) and np.array_equal(cnt, mcnt)
        k = min(3, g.n)
        assert [a.tolist() if hasattr(a, "tolist") else a for a in o.select(k)] == \
            [a.tolist() if hasattr(a, "tolist") else a for a in o.mrim_select(k)]


def test_mrim_T1_imm_equals_imm_C1():
    g = gi.workload_graph("C1")
    w = gi.WORKLOADS["C1"]
    o = oracle.Oracle(g, w.model, w.scheme)
    r = o.imm(w.k, w.eps, w.ell, w.rr_seed)
    m = o.mrim(w.k, 1, w.eps, w.ell, w.rr_seed)
    assert m.seeds.tolist() == r.seeds.tolist() and m.gains.tolist() == r.gains.tolist()
    assert (m.LB, m.theta, m.R_final, m.rounds, m.cov) == (r.LB, r.theta, r.R_final, r.rounds, r.cov)


# ---- R26: MRIM sets vs brute-force reachability ----------------------------------------------
def _ic_bf(g, p, seed, coin_id, root):
    live = []
    for e, (u, v) in enumerate(_edge_list(g)):
        coin = keyed(seed, coin_id, e >> 2)[e & 3]
        if Fraction(coin, 1 << 32) < p[e]:
            live.append((u, v))
    return _closure_reaching(g.n, live, root)


def _lt_bf_wc(g, seed, coin_id, root):
    live = []
    for v in range(g.n):
        a, b = int(g.row_ptr[v]), int(g.row_ptr[v + 1])
        if b == a:
            continue
        r = keyed(seed, coin_id, (1 << 62) | v)[0]
        t = (r * (b - a)) >> 32                      # the t with t/d <= r/2^32 < (t+1)/d
        live.append((int(g.src[a + t]), v))
    return _closure_reaching(g.n, live, root)


@pytest.mark.parametrize("model", [gi.IC, gi.LT])
@pytest.mark.parametrize("T", [2, 3, 5])
def test_mrim_sets_equal_bruteforce(model, T):
    for g in _tiny_graphs():
        o = oracle.Oracle(g, model, gi.W_WC)
        N = 40
        o.mrim_generate(N, T, SEED)
        off, pairs, cnt = o.mrim_export()
        p = _p_exact(g, gi.W_WC)
        for i in range(N):
            root = _root_ref(SEED, i, g.n)                # one random node per MRIM set
            want = []
            for t in range(T):
                coin_id = i * T + t
                nodes = _ic_bf(g, p, SEED, coin_id, root) if model == gi.IC else _lt_bf_wc(g, SEED, coin_id, root)
                want += [t * g.n + u for u in nodes]
            assert pairs[off[i]:off[i + 1]].tolist() == sorted(want), (i, t)
        assert np.array_equal(cnt, np.bincount(pairs.astype(np.int64), minlength=g.n * T))


def test_mrim_set_alone_equals_pool():
    g = gi.random_small(9, 30, 0)
    o = oracle.Oracle(g, gi.IC, gi.W_WC)
    o.mrim_generate(50, 4, SEED)
    off, pairs, _ = o.mrim_export()
    for i in range(50):
        assert o.mrim_set(SEED, i, 4).tolist() == pairs[off[i]:off[i + 1]].tolist()


def test_mrim_extend_truncate_reseed():
    g = gi.random_small(7, 14, 3)
    o = oracle.Oracle(g, gi.IC, gi.W_WC)
    o.mrim_generate(90, 3, SEED)
    full = o.mrim_export()
    o.mrim_generate(40, 3, SEED)
    o.mrim_generate(90, 3, SEED)                          # truncate then extend == direct
    again = o.mrim_export()
    assert all(np.array_equal(a, b) for a, b in zip(full, again))
    o.mrim_generate(90, 3, SEED + 1)
    assert not np.array_equal(o.mrim_export()[1], full[1])


# ---- R26 + Eq. 3 analog: exact enumeration of independent rounds ----------------------------
def _reach_prob(g, worlds, nodes, root):
    return sum(pr for pr, live in worlds if root in _forward_reach(g.n, live, nodes))


def exact_mrim_objective(g, worlds, S_by_round):
    """E[#nodes influenced in at least one round], rounds independent."""
    tot = Fraction(0)
    for v in range(g.n):
        miss = Fraction(1)
        for S in S_by_round:
            miss *= 1 - (_reach_prob(g, worlds, S, v) if S else 0)
        tot += 1 - miss
    return tot


def exact_mrim_ris(g, worlds, S_by_round):
    """n * Pr[S cap MRR != {}], MRR from a uniform root shared by the rounds (R26)."""
    T = len(S_by_round)
    tot = Fraction(0)
    for root in range(g.n):
        # enumerate the T independent worlds jointly (tiny graphs only)
        hit = Fraction(0)
        for combo in itertools.product(worlds, repeat=T):
            pr = Fraction(1)
            covered = False
            for t, (p_t, live) in enumerate(combo):
                pr *= p_t
                if S_by_round[t] and any(root in _forward_reach(g.n, live, [s]) for s in S_by_round[t]):
                    covered = True
            if covered:
                hit += pr
        tot += Fraction(1, g.n) * hit
    return g.n * tot


def test_mrim_objective_identity_exact():
    d = gi.diamond()
    W = list(_ic_worlds(d, [Fraction(1, 2)] * 4))
    for S in ([[0], [0]], [[1], [2]], [[0], []], [[3], [1, 2]]):
        assert exact_mrim_objective(d, W, S) == exact_mrim_ris(d, W, S)
    # two rounds with the same seed beat one round: 1 - (1 - p)^2 per node, not p
    one = exact_mrim_objective(d, W, [[0]])
    two = exact_mrim_objective(d, W, [[0], [0]])
    assert one == Fraction(39, 16) and two > one


@pytest.mark.parametrize("model", [gi.IC, gi.LT])
def test_mrim_estimator_vs_exact(model):
    d = gi.diamond()
    if model == gi.IC:
        g = gi.with_weights(d, np.full(4, 0.5, dtype=np.float32))
        o = oracle.Oracle(g, gi.IC, gi.W_EXPLICIT)
        W = list(_ic_worlds(d, [Fraction(1, 2)] * 4))
    else:
        o = oracle.Oracle(d, gi.LT, gi.W_WC)
        W = list(_lt_worlds(d, _p_exact(d, gi.W_WC)))
    T, N = 2, 40000
    o.mrim_generate(N, T, 77)
    off, pairs, cnt = o.mrim_export()
    sets = _pool_sets(off, pairs)
    for S in ([[0], [0]], [[1], [2]], [[3], []], [[1, 2], [0]]):
        Sp = {t * d.n + u for t in range(T) for u in S[t]}
        f = sum(1 for s in sets if Sp.intersection(s)) / N
        ex = float(exact_mrim_objective(d, W, S)) / d.n
        se = math.sqrt(max(ex * (1 - ex), 1e-12) / N)
        assert abs(f - ex) < 4.5 * se, (S, f, ex)
    # pair marginals: count[(u, t)] / N vs (1/n) sum_v Pr[u reaches v], every round
    for t in range(T):
        for u in range(d.n):
            ex = float(sum(_reach_prob(d, W, [u], v) for v in range(d.n))) / d.n
            f = cnt[t * d.n + u] / N
            se = math.sqrt(max(ex * (1 - ex), 1e-12) / N)
            assert abs(f - ex) < 4.5 * se, (t, u, f, ex)


# ---- R27: selection vs brute force ----------------------------------------------------------
def _cov(sets, S):
    S = set(S)
    return sum(1 for s in sets if S.intersection(s))


@pytest.mark.parametrize("trial", range(25))
def test_mrim_select_bruteforce(trial):
    rng = np.random.default_rng(1000 + trial)
    n = int(rng.integers(2, 6))
    T = int(rng.integers(1, 4))
    k = int(rng.integers(1, n + 1))
    nsets = int(rng.integers(1, 16))
    sets = [sorted(rng.choice(n * T, size=int(rng.integers(1, n * T + 1)), replace=False).tolist())
            for _ in range(nsets)]
    off = np.concatenate([[0], np.cumsum([len(s) for s in sets])]).astype(np.uint64)
    pairs = np.concatenate([np.asarray(s, dtype=np.uint32) for s in sets])
    picks, gains, cov = oracle.mrim_select_pool(n, T, off, pairs, k)
    chosen = []
    for j in range(k * T):
        full = {t for t in range(T) if sum(1 for c in chosen if c // n == t) >= k}
        base = _cov(sets, chosen)
        marg = [(_cov(sets, chosen + [v]) - base) if (v not in chosen and v // n not in full) else -1
                for v in range(n * T)]
        best = max(marg)
        u = marg.index(best)                          # lowest pair id among ties (R27)
        assert picks[j] == u and gains[j] == best, (j, picks, gains, marg)
        chosen.append(u)
    assert [sum(1 for c in chosen if c // n == t) for t in range(T)] == [k] * T
    assert cov == _cov(sets, chosen)
    # greedy over a partition matroid: >= 1/2 of the best per-round assignment
    opt = max(_cov(sets, sum(c, ())) for c in itertools.product(
        *[[tuple(t * n + u for u in comb) for comb in itertools.combinations(range(n), k)] for t in range(T)]))
    assert 2 * cov >= opt


# ---- R28: constants and the driver ----------------------------------------------------------
def _mp_lnC(N, K):
    import mpmath as mp
    mp.mp.dps = 40
    return mp.log(mp.binomial(N, K))


@pytest.mark.parametrize("n,k,T,eps", [(75879, 10, 5, 0.1), (15233, 10, 5, 0.5), (1000, 3, 2, 0.2),
                                       (4847571, 10, 5, 0.1)])
def test_mrim_constants_mpmath(n, k, T, eps):
    import mpmath as mp
    mp.mp.dps = 40
    got = oracle.mrim_constants(n, k, T, eps, 1.0)
    n_, eps_ = mp.mpf(n), mp.mpf(eps)
    ell_eff = 1 + mp.log(2) / mp.log(n_)
    epsp = mp.sqrt(2) * eps_
    lnC = _mp_lnC(n * T, k * T)
    lam_p = (2 + mp.mpf(2) / 3 * epsp) * (lnC + ell_eff * mp.log(n_) + mp.log(mp.log(n_, 2))) * n_ / epsp ** 2
    a = mp.sqrt(ell_eff * mp.log(n_) + mp.log(2))
    b = mp.sqrt((1 - 1 / mp.e) * (lnC + ell_eff * mp.log(n_) + mp.log(2)))
    lam_s = 2 * n_ * ((1 - 1 / mp.e) * a + b) ** 2 / eps_ ** 2
    for key, ref in (("lnC", lnC), ("lambda_prime", lam_p), ("lambda_star", lam_s), ("ell_eff", ell_eff)):
        assert abs(got[key] - float(ref)) <= 1e-12 * abs(float(ref)), key
    assert oracle.mrim_constants(n, k, 1, eps) == oracle.imm_constants(n, k, eps)


def test_mrim_driver_trace_C1():
    g = gi.workload_graph("C1")
    w = gi.WORKLOADS["C1"]
    k, T = 10, 5
    o = oracle.Oracle(g, w.model, w.scheme)
    r = o.mrim(k, T, w.eps, w.ell, w.rr_seed)
    c = oracle.mrim_constants(g.n, k, T, w.eps, w.ell)
    assert r.lambda_prime == c["lambda_prime"] and r.lambda_star == c["lambda_star"]
    x = [g.n / 2.0 ** i for i in range(1, r.rounds + 1)]
    for i in range(r.rounds):
        assert r.theta_i[i] == c["lambda_prime"] / x[i]
        assert r.T_i[i] == math.ceil(r.theta_i[i])
        passed = (g.n * float(r.cov_i[i])) / float(r.T_i[i]) >= (1 + c["eps_prime"]) * x[i]
        assert passed == (i == r.rounds - 1 and r.LB > 1.0)
    assert r.theta == c["lambda_star"] / r.LB
    assert r.R_final == max(int(r.T_i[-1]), math.ceil(r.theta))
    rounds = r.seeds // g.n
    assert np.bincount(rounds, minlength=T).tolist() == [k] * T      # k seeds per round
    assert len(set(r.seeds.tolist())) == k * T
    assert r.cov == int(r.gains.sum()) and np.all(np.diff(r.gains.astype(np.int64)) <= 0)
