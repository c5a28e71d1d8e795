"""Full-IMM parity at BASELINE.json's full sizes: ``gim_imm`` (through the C ABI) against the
oracle's committed run, ``tests/golden/imm_<cfg>.json`` (written by tools/oracle_golden.py,
which calls only ``oracle/`` and ``gim_inputs/``).

This is the north_star target "bit-exact seed sets versus the CPU oracle on all five configs":
gIM's solution is IMM's (§4.3), and the whole Alg. 2 trace is
compared — rounds, T_i, cov_i and R_final exactly; the doubles (lambda', lambda*, theta_i, LB,
theta, spread) within 1e-12 relative; the final seeds and per-step gains bit-exact; the final
count vector by its sha256 and the pool by its length.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import gim_inputs as gi
from tests.imm_trace import check_cov_trace

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2009_07325_b200")

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).view(np.uint8).tobytes())
    return h.hexdigest()


def _rel(a, b):
    return abs(a - b) <= 1e-12 * max(abs(b), 1e-300)


@pytest.mark.parametrize("key,early,chunk", [("C1", 1, 0), ("C2", 1, 0), ("C3", 1, 0), ("C4", 1, 0), ("C5", 1, 0),
                                             ("C1", 0, 0), ("C3", 0, 0), ("C3", 1, 1 << 18), ("C5", 1, 1 << 22),
                                             ("C3", 2, 0), ("C5", 2, 0)])
def test_imm_golden(key, early, chunk):
    """early = 1: the default bounded greedy in the estimation rounds (stopped rounds checked by
    tests/imm_trace.py); early = 0: every round's k steps, cov_i exactly as the oracle's; early = 2:
    lookahead sampling forced one round ahead (its drop path runs when a round needs selection). chunk:
    RR ids per generation chunk (0 = the default 2^25; small chunks: every round in several)."""
    gd = json.load(open(os.path.join(GOLDEN, f"imm_{key}.json")))
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    assert _sha(g.row_ptr, g.src) == gd["graph_sha256"], "input generator drifted from the golden's graph"
    c = P.Gim(0)
    try:
        c.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme, p_uniform=w.p_uniform)
        c.set_option(P.OPT_IMM_EARLY_EXIT, min(early, 1))
        c.set_option(P.OPT_IMM_LOOKAHEAD, 2 if early == 2 else 1)
        c.set_option(P.OPT_CHUNK, chunk)
        r = c.imm(w.k, w.eps, w.ell, w.rr_seed)
        assert _rel(r.ell_eff, gd["ell_eff"]) and _rel(r.eps_prime, gd["eps_prime"])
        assert _rel(r.lambda_prime, gd["lambda_prime"]) and _rel(r.lambda_star, gd["lambda_star"])
        assert r.rounds == gd["rounds"]
        assert r.theta_i.tolist() == gd["T_i"]
        stopped = check_cov_trace(r, gd["T_i"], gd["cov_i"], g.n, gd["eps_prime"], w.k)
        if not early:
            assert stopped == 0 and r.cov_i.tolist() == gd["cov_i"]
        if early == 2 and key == "C3":
            assert c.stats()["lookahead_drops"] >= 1      # round 3 needed its selection
        assert all(_rel(a, b) for a, b in zip(r.theta_i_real.tolist(), gd["theta_i"]))
        assert _rel(r.LB, gd["LB"]) and _rel(r.theta, gd["theta"])
        assert r.R_final == gd["R_final"] and r.covered == gd["cov"]
        assert r.seeds.tolist() == gd["seeds"], (r.seeds.tolist()[:10], gd["seeds"][:10])
        assert _rel(r.spread_est, gd["spread_est"])
        # the final pool itself: length and the count vector (Occur) by hash
        ns, pl = c.pool_size()
        assert ns == gd["R_final"] and pl == gd["pool_len"]
        assert _sha(c.counts_export()) == gd["count_sha256"]
        # per-step marginal gains of the final selection (non-destructive, R9)
        seeds, gains, cov = c.select(w.k)
        assert seeds.tolist() == gd["seeds"] and gains.tolist() == gd["gains"] and cov == gd["cov"]
    finally:
        c.close()
