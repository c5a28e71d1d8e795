"""CPU pins of the bounded greedy that gim_imm runs in its estimation rounds (include/gim.h
GIM_OPT_IMM_EARLY_EXIT). The claim: with gains g_0 >= g_1 >= ... of
the greedy (max coverage is submodular and counts only decrease, Alg. 7), the final
covered count is at most cov_j + (k - j) g_j after the argmax of any step j, so once that bound
is below c* — the smallest covered count passing Alg. 2 l.7 (reading R7) — the round's
test fails whatever the rest of the greedy picks, and stopping changes nothing IMM returns.

Checked here on the oracle's own rounds (plain Alg. 2, all k steps): the premise (gains never
increase), the bound at every step, the minimality of c*, and that every round the rule would
stop is a round the oracle's test fails — IMM and MRIM, several graphs and epsilons.
"""
import numpy as np
import pytest

import gim_inputs as gi
import oracle
from tests.imm_trace import cstar, oracle_round_gains, passes


def _check_rounds(g, n, ro, gains_of, picks):
    stops = 0
    for i in range(ro.rounds):
        g_i = [int(v) for v in gains_of(i)]
        assert len(g_i) == picks and sum(g_i) == int(ro.cov_i[i])
        assert all(a >= b for a, b in zip(g_i, g_i[1:])), "greedy gains must never increase"
        T = int(ro.T_i[i])
        x = n / 2.0 ** (i + 1)
        cs = cstar(n, T, ro.eps_prime, x)
        if 0 < cs <= T:
            assert passes(n, cs, T, ro.eps_prime, x) and not passes(n, cs - 1, T, ro.eps_prime, x)
        for j in range(picks):
            assert int(ro.cov_i[i]) <= sum(g_i[:j]) + (picks - j) * g_i[j]
        stop = next((j for j in range(picks) if sum(g_i[:j]) + (picks - j) * g_i[j] < cs), None)
        if stop is not None:
            stops += 1
            assert not passes(n, int(ro.cov_i[i]), T, ro.eps_prime, x), f"round {i + 1} passes but would stop"
        else:
            # never stopped: nothing to check beyond the bound; a passing round never stops
            pass
        if passes(n, int(ro.cov_i[i]), T, ro.eps_prime, x):
            assert stop is None
    return stops


@pytest.mark.parametrize("key,k,eps", [("C1", 50, 0.5), ("C1", 10, 0.3), ("C1", 50, 0.2)])
def test_bounded_greedy_imm_rounds(key, k, eps):
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    ro = oracle.Oracle(g, w.model, w.scheme).imm(k, eps, w.ell, w.rr_seed)
    o2 = oracle.Oracle(g, w.model, w.scheme)
    stops = _check_rounds(g, g.n, ro, oracle_round_gains(o2, ro.T_i, k, w.rr_seed), k)
    assert ro.rounds == 1 or stops >= 1     # the rule does fire on the failing rounds of C1


@pytest.mark.parametrize("seed", [3, 7])
def test_bounded_greedy_ba_and_lt(seed):
    g = gi.ba(3000, 4, seed)
    for model in (gi.IC, gi.LT):
        ro = oracle.Oracle(g, model, gi.W_WC).imm(8, 0.4, 1.0, seed)
        _check_rounds(g, g.n, ro, oracle_round_gains(oracle.Oracle(g, model, gi.W_WC), ro.T_i, 8, seed), 8)


def test_bounded_greedy_mrim_rounds():
    w = gi.WORKLOADS["C1"]
    g = gi.workload_graph("C1")
    k, T = 5, 3
    ro = oracle.Oracle(g, gi.IC, w.scheme).mrim(k, T, 0.5, w.ell, w.rr_seed)
    o2 = oracle.Oracle(g, gi.IC, w.scheme)
    _check_rounds(g, g.n, ro, oracle_round_gains(o2, ro.T_i, k, w.rr_seed, mrim_T=T), k * T)


def test_cstar_edges():
    # c* is the least passing count; nothing passes -> R + 1; everything passes -> 0
    assert cstar(100, 10, 0.1, 1e9) == 11
    assert cstar(100, 10, 0.1, 0.0) == 0
    for R in (1, 7, 1000, 123457):
        for x in (0.5, 3.0, 50.0):
            c = cstar(1000, R, 0.2, x)
            assert (c == R + 1) or passes(1000, c, R, 0.2, x)
            assert c == 0 or not passes(1000, c - 1, R, 0.2, x)
