"""The committed full-IMM goldens (tests/golden/imm_<cfg>.json, written by tools/oracle_golden.py
from ``oracle/`` only) checked on the CPU: C1 and C2 are re-run and must reproduce the file
exactly; every file must satisfy the identities Alg. 2 and the greedy
(Alg. 1 l.6-10) impose, and carry IMM's constants as the (mpmath-pinned) oracle
computes them."""
import json
import math
import os

import numpy as np
import pytest

import gim_inputs as gi
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
KEYS = ["C1", "C2", "C3", "C4", "C5"]


def _load(key):
    return json.load(open(os.path.join(GOLDEN, f"imm_{key}.json")))


@pytest.mark.parametrize("key", KEYS)
def test_golden_identities(key):
    gd = _load(key)
    w = gi.WORKLOADS[key]
    assert (gd["n"], gd["m"], gd["k"], gd["eps"], gd["ell"], gd["rr_seed"]) == (w.n, w.m, w.k, w.eps, w.ell, w.rr_seed)
    c = oracle.imm_constants(w.n, w.k, w.eps, w.ell)
    for name in ("ell_eff", "eps_prime", "lambda_prime", "lambda_star"):
        assert gd[name] == c[name], name
    n, r = gd["n"], gd["rounds"]
    assert 1 <= r <= int(math.floor(math.log2(n))) - 1
    for i in range(r):
        x = n / 2.0 ** (i + 1)
        assert gd["theta_i"][i] == c["lambda_prime"] / x                  # theta_i = lambda'/x_i
        assert gd["T_i"][i] == math.ceil(gd["theta_i"][i])                # R4
        passed = (n * gd["cov_i"][i]) / gd["T_i"][i] >= (1.0 + c["eps_prime"]) * x
        if i < r - 1:
            assert not passed                                             # no earlier break
        elif passed:
            assert gd["LB"] == (n * gd["cov_i"][i]) / gd["T_i"][i] / (1.0 + c["eps_prime"])
        else:                                                             # R6: loop bound reached
            assert r == int(math.floor(math.log2(n))) - 1 and gd["LB"] == 1.0
    assert gd["theta"] == c["lambda_star"] / gd["LB"]
    assert gd["R_final"] == max(gd["T_i"][-1], math.ceil(gd["theta"]))
    seeds, gains = gd["seeds"], gd["gains"]
    assert len(seeds) == w.k and len(set(seeds)) == w.k and all(0 <= s < n for s in seeds)
    assert sum(gains) == gd["cov"] <= gd["R_final"]
    assert all(a >= b for a, b in zip(gains, gains[1:]))                # coverage is submodular
    assert gd["spread_est"] == n * gd["cov"] / gd["R_final"]
    assert gd["pool_len"] >= gd["R_final"]                              # every set holds its root


@pytest.mark.parametrize("key", ["C1", "C2"])
def test_golden_reproduced_by_oracle(key):
    gd = _load(key)
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    import hashlib
    h = hashlib.sha256()
    for a in (g.row_ptr, g.src):
        h.update(np.ascontiguousarray(a).view(np.uint8).tobytes())
    assert h.hexdigest() == gd["graph_sha256"]
    r = oracle.Oracle(g, w.model, w.scheme, w.p_uniform).imm(w.k, w.eps, w.ell, w.rr_seed)
    assert r.seeds.tolist() == gd["seeds"] and r.gains.tolist() == gd["gains"]
    assert r.T_i.tolist() == gd["T_i"] and r.cov_i.tolist() == gd["cov_i"] and r.R_final == gd["R_final"]
    assert r.LB == gd["LB"] and r.theta == gd["theta"]
