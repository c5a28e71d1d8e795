"""Parity of the geometric-skip contract (reading R31, GIM_OPT_SKIP) on the CUDA path
(k_skip_lane / k_skip_warp / k_skip_giant, csrc/skip.cu) against the oracle's skip mirror
(og_set_skip, pinned in tests/test_oracle_skip.py): RR sets, counts, seeds, gains and the IMM
trace bit-exact, under every launch mode (lane-first, warp-only, forced giant, tiny queues) and
at full size on sampled ids."""
import json
import os

import numpy as np
import pytest

import gim_inputs as gi
from tests.imm_trace import check_cov_trace
import oracle

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2009_07325_b200")

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _ctx(g, scheme, p_uniform=0.0, mode=1, opts=None):
    c = P.Gim(0)
    c.load_graph(g.n, g.row_ptr, g.src, gi.IC, scheme, p_uniform=p_uniform)
    c.set_option(P.OPT_SKIP, 1)
    if mode != 1:
        c.set_option(P.OPT_SKIP, mode)          # 2: warp kernel only, 3: lane kernel first
    for k, v in (opts or {}).items():
        c.set_option(k, v)
    return c


def _oracle(g, scheme, p_uniform=0.0):
    o = oracle.Oracle(g, gi.IC, scheme, p_uniform)
    o.set_skip(True)
    return o


def _same_pool(c, o, T):
    ids, off, nodes = c.rr_export(sort_each_set=True)
    ooff, onodes, ocnt = o.export()
    assert len(ids) == T and np.array_equal(ids, np.arange(T, dtype=np.uint64))
    assert np.array_equal(off, ooff), "offsets"
    assert np.array_equal(nodes, onodes), "pool contents"
    assert np.array_equal(c.counts_export(), ocnt), "counts"


def _bipartite(d, hubs):
    n = d + hubs
    row_ptr = np.zeros(n + 1, dtype=np.uint64)
    row_ptr[d + 1:] = d * np.arange(1, hubs + 1, dtype=np.uint64)
    src = np.tile(np.arange(d, dtype=np.uint32), hubs)
    return gi.Graph(n=n, row_ptr=row_ptr, src=src, name=f"bip{d}x{hubs}")


MODES = {"auto": (1, {}), "warp": (2, {}), "lane": (3, {}), "giant": (1, {P.OPT_FORCE_GIANT: 1}),
         "q4": (2, {P.OPT_QUEUE_CAP: 4}), "q32_lane": (3, {P.OPT_QUEUE_CAP: 32}),
         "staging": (3, {P.OPT_STAGING_CAP: 64}), "lane512": (3, {P.OPT_SKIP_LANE_CAP: 512}),
         "lane8": (3, {P.OPT_SKIP_LANE_CAP: 8}), "lane40_q4": (3, {P.OPT_SKIP_LANE_CAP: 40, P.OPT_QUEUE_CAP: 4})}


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("scheme", [gi.W_WC, gi.W_UNIFORM])
def test_skip_tiny_graphs(mode, scheme):
    m, opts = MODES[mode]
    graphs = [gi.diamond(), gi.chain(5), gi.cycle_plus(), gi.star_in(40)] + \
             [gi.random_small(9, 30, s) for s in range(3)] + [_bipartite(2100, 6)]
    pu = 0.35 if scheme == gi.W_UNIFORM else 0.0
    for g in graphs:
        T = 3001
        c = _ctx(g, scheme, pu, m, opts)
        c.generate_rr(T, 77)
        o = _oracle(g, scheme, pu)
        o.generate(T, 77)
        _same_pool(c, o, T)
        k = min(3, g.n)
        s, gn, cv = c.select(k)
        os_, og, oc = o.select(k)
        assert np.array_equal(s, os_) and np.array_equal(gn, og) and cv == oc
        c.close()


def test_skip_tiers_big_sets():
    """Sets beyond the shared queue (spill tier) and beyond the spill tier (giant restart): an
    in-star of 20,000 leaves plus a chain feeding the hub, uniform p = 0.9."""
    leaves = 20000
    edges = [(i, 0) for i in range(1, leaves + 1)] + [(leaves + 1 + i, leaves + 2 + i) for i in range(300)]
    edges += [(leaves + 301, 0)]
    g = gi.from_edges(leaves + 302, edges)
    T = 4000
    for m, cap in ((1, 2048), (2, 16384), (3, 600), (3, 16384)):
        c = _ctx(g, gi.W_UNIFORM, 0.9, m, {P.OPT_SPILL: cap})
        c.generate_rr(T, 3)
        o = _oracle(g, gi.W_UNIFORM, 0.9)
        o.generate(T, 3)
        _same_pool(c, o, T)
        c.close()


@pytest.mark.parametrize("key", ["C1", "C2"])
@pytest.mark.parametrize("mode", ["auto", "warp", "lane", "giant", "q32_lane", "lane512", "lane8"])
def test_skip_pool_configs(key, mode):
    m, opts = MODES[mode]
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    T = 40013
    c = _ctx(g, w.scheme, w.p_uniform, m, opts)
    c.generate_rr(T // 3, w.rr_seed)                    # grown in two calls
    c.generate_rr(T, w.rr_seed)
    o = _oracle(g, w.scheme, w.p_uniform)
    o.generate(T, w.rr_seed)
    _same_pool(c, o, T)
    s, gn, cv = c.select(w.k)
    os_, og, oc = o.select(w.k)
    assert np.array_equal(s, os_) and np.array_equal(gn, og) and cv == oc
    c.close()


def test_skip_uniform_C5_shaped_small():
    """Uniform p = 0.01 (C5's weights) on a graph with hubs of > 1024 in-edges: blocks, hubs and
    tiny sets together."""
    g = gi.plg(50000, 1500000, 2.3, 0.0, 40000.0, 9)
    T = 100003
    for m in (1, 3):
        c = _ctx(g, gi.W_UNIFORM, 0.01, m)
        c.generate_rr(T, 5)
        o = _oracle(g, gi.W_UNIFORM, 0.01)
        o.generate(T, 5)
        _same_pool(c, o, T)
        c.close()


def _rel(a, b):
    return abs(a - b) <= 1e-12 * max(abs(b), 1e-300)


@pytest.mark.parametrize("key", ["C1", "C2", "C3", "C5"])
def test_skip_imm_golden(key):
    """Full IMM under the skip contract against the oracle's committed run
    (tests/golden/imm_<cfg>_skip.json, tools/oracle_golden.py --skip)."""
    path = os.path.join(GOLDEN, f"imm_{key}_skip.json")
    gd = json.load(open(path))
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    c = _ctx(g, w.scheme, w.p_uniform)
    r = c.imm(w.k, w.eps, w.ell, w.rr_seed)
    assert r.rounds == gd["rounds"] and r.theta_i.tolist() == gd["T_i"]
    check_cov_trace(r, gd["T_i"], gd["cov_i"], g.n, gd["eps_prime"], w.k)
    assert _rel(r.LB, gd["LB"]) and _rel(r.theta, gd["theta"])
    assert r.R_final == gd["R_final"] and r.covered == gd["cov"]
    assert r.seeds.tolist() == gd["seeds"]
    ns, pl = c.pool_size()
    assert pl == gd["pool_len"]
    seeds, gains, cov = c.select(w.k)
    assert gains.tolist() == gd["gains"]
    c.close()


@pytest.mark.parametrize("key", ["C3", "C5"])
def test_skip_full_size_sampled(key):
    w = gi.WORKLOADS[key]
    g = gi.workload_graph(key)
    c = _ctx(g, w.scheme, w.p_uniform)
    T = 1 << 21
    c.generate_rr(T, w.rr_seed)
    ids, off, nodes = c.rr_export(sort_each_set=True)
    o = _oracle(g, w.scheme, w.p_uniform)
    rng = np.random.default_rng(2)
    sizes = np.diff(off.astype(np.int64))
    sample = np.concatenate([[0, 1, T - 1], rng.choice(T, 300, replace=False), np.argsort(sizes)[-5:]])
    for i in sample:
        assert np.array_equal(nodes[off[i]:off[i + 1]], o.rr_set(w.rr_seed, int(i))), int(i)
    cnt = c.counts_export()
    assert np.array_equal(np.bincount(nodes, minlength=g.n).astype(np.uint32), cnt)
    c.close()


def test_skip_mrim_C1():
    w = gi.WORKLOADS["C1"]
    g = gi.workload_graph("C1")
    c = _ctx(g, w.scheme)
    c.set_rounds(3)
    r = c.imm(10, 0.5, 1.0, w.rr_seed)
    o = _oracle(g, w.scheme)
    ro = o.mrim(10, 3, 0.5, 1.0, w.rr_seed)
    assert r.R_final == ro.R_final and np.array_equal(r.seeds, ro.seeds) and r.covered == ro.cov


def test_skip_option_errors():
    d = gi.diamond()
    c = P.Gim(0)
    c.load_graph(d.n, d.row_ptr, d.src, gi.LT, gi.W_WC)
    with pytest.raises(P.GimError) as e:
        c.set_option(P.OPT_SKIP, 1)
    assert e.value.status == 1
    c.close()
