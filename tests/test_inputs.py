"""The seeded input generator: determinism, canonical in-CSR invariants, exact edge count."""
import numpy as np

import gim_inputs as gi


def test_plg_deterministic_and_canonical():
    a = gi.plg(5000, 40000, 2.3, 0.5, 500.0, 9)
    b = gi.plg(5000, 40000, 2.3, 0.5, 500.0, 9)
    c = gi.plg(5000, 40000, 2.3, 0.5, 500.0, 10)
    a.validate()
    assert a.m == 40000
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.src, b.src)
    assert not np.array_equal(a.src, c.src)


def test_workload_shapes():
    for key in ("C1", "C2"):
        w = gi.WORKLOADS[key]
        g = gi.workload_graph(key)
        g.validate()
        assert (g.n, g.m) == (w.n, w.m)
        s = gi.stats(g)
        assert s["max_in"] > 10 * s["mean_deg"]     # heavy-tailed in-degrees


def test_symmetric_shape_C1():
    g = gi.workload_graph("C1")
    dst = np.repeat(np.arange(g.n), np.diff(g.row_ptr).astype(np.int64))
    fwd = set(zip(g.src.tolist(), dst.tolist()))
    recip = sum((v, u) in fwd for u, v in fwd) / len(fwd)
    assert recip > 0.99                              # rho = 1 (undirected collaboration shape)


def test_from_edges_canonical():
    g = gi.from_edges(3, [(0, 1), (0, 2), (1, 2), (1, 2), (2, 2)])
    assert g.row_ptr.tolist() == [0, 0, 1, 3] and g.src.tolist() == [0, 0, 1]


def test_gcsr_roundtrip(tmp_path):
    g = gi.workload_graph("C1")
    p = str(tmp_path / "c1.gcsr")
    gi.save_gcsr(g, p)
    h = gi.load_gcsr(p)
    assert h.n == g.n and np.array_equal(h.row_ptr, g.row_ptr) and np.array_equal(h.src, g.src)
    assert h.meta["graph_seed"] == 1
