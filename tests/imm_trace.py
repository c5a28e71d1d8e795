"""Comparison of gim_imm's round trace with the oracle's, bounded greedy included.

gim_imm stops an estimation round's selection early (GIM_OPT_IMM_EARLY_EXIT, include/gim.h
gim_imm_result.sel_steps_i) once the greedy's bound cov_j + (picks - j) * gain_j — gains never
increase — falls below c*, the smallest covered count that passes the round's test (Alg. 2 l.7,
PAPER.md P:225; reading R7). The oracle (plain Alg. 2) always runs all picks, so:

* a round whose selection ran all picks must report the oracle's cov_i exactly;
* a stopped round must be one the oracle's test fails, and its partial coverage is at most the
  oracle's; given the oracle's own per-step gains of that round (``round_gains``), the partial
  coverage equals the sum of the first sel_steps gains and the stop happened at exactly the first
  step whose bound is below c* (computed here in the same double arithmetic as the library).
"""


def passes(n, cov, R, eps_prime, x):
    return (n * float(cov)) / float(R) >= (1.0 + eps_prime) * x


def cstar(n, R, eps_prime, x):
    lo, hi = 0, R + 1
    while lo < hi:
        mid = (lo + hi) // 2
        if passes(n, mid, R, eps_prime, x):
            hi = mid
        else:
            lo = mid + 1
    return lo


def check_cov_trace(r, T_i, cov_i, n, eps_prime, picks, round_gains=None):
    T_i = [int(t) for t in T_i]
    cov_i = [int(c) for c in cov_i]
    assert len(r.cov_i) == len(cov_i) and len(r.sel_steps_i) == len(cov_i)
    stopped = 0
    for i in range(len(cov_i)):
        steps = int(r.sel_steps_i[i])
        x = n / 2.0 ** (i + 1)
        if steps == picks:
            assert int(r.cov_i[i]) == cov_i[i], (i, int(r.cov_i[i]), cov_i[i])
            continue
        stopped += 1
        assert 1 <= steps < picks, (i, steps, picks)
        assert not passes(n, cov_i[i], T_i[i], eps_prime, x), "a passing round was cut short"
        assert int(r.cov_i[i]) <= cov_i[i]
        if round_gains is not None:
            g = [int(v) for v in round_gains(i)]
            assert sum(g) == cov_i[i]
            assert int(r.cov_i[i]) == sum(g[:steps]), (i, steps, int(r.cov_i[i]), g[:steps])
            cs = cstar(n, T_i[i], eps_prime, x)
            bound = lambda j: sum(g[:j]) + (picks - j) * g[j]
            first = next(j for j in range(picks) if bound(j) < cs)
            assert steps == first + 1, (i, steps, first)
    return stopped


def oracle_round_gains(o, T_i, k, seed, mrim_T=None):
    """Per-step gains of round i's full selection on the oracle ``o`` (its pool is regenerated)."""
    def gains(i):
        if mrim_T:
            o.mrim_generate(int(T_i[i]), mrim_T, seed)
            return o.mrim_select(k)[1]
        o.generate(int(T_i[i]), seed)
        return o.select(k)[1]
    return gains
