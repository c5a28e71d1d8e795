"""Seeded synthetic inputs shared by the oracle (``oracle/``) and the CUDA path.

This module holds none of the method's arithmetic (no Philox, no coin thresholds, no
influence probabilities, no IMM formulas). It produces graphs as canonical in-CSR arrays
(reading R15) and the parameter table of the five workloads
of BASELINE.json. Weighted-cascade weights p_uv = 1/d_in(v) (PAPER.md
P:602-603, §4.2) are *implicit*: each side derives them from ``row_ptr`` on its own.
"""
from __future__ import annotations

import ctypes
import dataclasses
import functools
import json
import os
import subprocess
from typing import Iterable, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libplg.so")

IC, LT = 0, 1                      # diffusion model (§2.2)
W_EXPLICIT, W_WC, W_UNIFORM = 0, 1, 2  # weight scheme


@dataclasses.dataclass
class Graph:
    """Canonical in-CSR: row v lists the sources u of edges u->v, strictly ascending, no
    self-loops (PAPER.md P:293-296 CSR, read as the in-CSR per DESIGN.md reading R14/R15)."""

    n: int
    row_ptr: np.ndarray            # uint64[n+1]
    src: np.ndarray                # uint32[m]
    weights: Optional[np.ndarray] = None   # float32[m], only for the explicit scheme
    name: str = ""
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.src.shape[0])

    def in_degree(self) -> np.ndarray:
        return np.diff(self.row_ptr).astype(np.int64)

    def out_degree(self) -> np.ndarray:
        return np.bincount(self.src.astype(np.int64), minlength=self.n).astype(np.int64)

    def validate(self) -> None:
        rp, s = self.row_ptr, self.src
        assert rp.dtype == np.uint64 and s.dtype == np.uint32
        assert rp.shape == (self.n + 1,) and int(rp[0]) == 0 and int(rp[-1]) == self.m
        assert np.all(np.diff(rp.astype(np.int64)) >= 0)
        if self.m:
            assert int(s.max()) < self.n
            dst = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(rp).astype(np.int64))
            assert not np.any(dst == s.astype(np.int64)), "self-loop"
            same_row = dst[1:] == dst[:-1]
            assert np.all(s[1:][same_row].astype(np.int64) > s[:-1][same_row].astype(np.int64)), \
                "rows must be strictly ascending"
        if self.weights is not None:
            assert self.weights.dtype == np.float32 and self.weights.shape == (self.m,)


def from_edges(n: int, edges: Iterable[Tuple[int, int]],
               weights: Optional[Sequence[float]] = None, name: str = "") -> Graph:
    """Canonical in-CSR from a directed edge list u->v: self-loops dropped, duplicates keep
    the first occurrence (SPEC.md S:56 idea), sources ascending within each row."""
    e = np.asarray(list(edges), dtype=np.int64).reshape(-1, 2)
    w = None if weights is None else np.asarray(list(weights), dtype=np.float32)
    if e.size:
        assert e.min() >= 0 and e.max() < n
    keep = e[:, 0] != e[:, 1]
    e = e[keep]
    if w is not None:
        w = w[keep]
    key = e[:, 1] * n + e[:, 0]
    _, first = np.unique(key, return_index=True)     # sorted by (dst, src); first occurrence
    e = e[first]
    if w is not None:
        w = w[first]
    row_ptr = np.zeros(n + 1, dtype=np.uint64)
    np.add.at(row_ptr, e[:, 1] + 1, 1)
    row_ptr = np.cumsum(row_ptr).astype(np.uint64)
    g = Graph(n=n, row_ptr=row_ptr, src=e[:, 0].astype(np.uint32),
              weights=None if w is None else w.astype(np.float32), name=name)
    g.validate()
    return g


# ---------------------------------------------------------------------------------------
# Tiny fixture graphs (SURVEY.md §8(c) pins)
# ---------------------------------------------------------------------------------------
def diamond() -> Graph:
    """0->1, 0->2, 1->3, 2->3 (SPEC.md S:138 idea; SURVEY.md §8(c) golden vectors)."""
    return from_edges(4, [(0, 1), (0, 2), (1, 3), (2, 3)], name="diamond")


def chain(n: int = 3) -> Graph:
    return from_edges(n, [(i, i + 1) for i in range(n - 1)], name=f"chain{n}")


def star_in(leaves: int) -> Graph:
    """Leaves 1..leaves all point at hub 0: the hub's RR set under p=1 is the whole graph."""
    return from_edges(leaves + 1, [(i, 0) for i in range(1, leaves + 1)], name=f"star{leaves}")


def cycle_plus() -> Graph:
    """0->1->2->0 plus 3->0 (SURVEY.md §8(c) LT pin)."""
    return from_edges(4, [(0, 1), (1, 2), (2, 0), (3, 0)], name="cycle_plus")


def random_small(n: int, m: int, seed: int) -> Graph:
    """Uniform random simple digraph with exactly min(m, n(n-1)) edges (tiny test inputs)."""
    rng = np.random.default_rng(seed)
    pairs = [(u, v) for u in range(n) for v in range(n) if u != v]
    m = min(m, len(pairs))
    pick = rng.choice(len(pairs), size=m, replace=False)
    return from_edges(n, [pairs[i] for i in pick], name=f"rand{n}_{m}_{seed}")


def with_weights(g: Graph, w: np.ndarray) -> Graph:
    return dataclasses.replace(g, weights=np.asarray(w, dtype=np.float32))


# ---------------------------------------------------------------------------------------
# Synthetic power-law generator (C++, libplg.so)
# ---------------------------------------------------------------------------------------
def build_lib(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "plg.cpp")):
        subprocess.check_call(["g++", "-O3", "-std=c++17", "-fopenmp", "-shared", "-fPIC",
                               os.path.join(_HERE, "plg.cpp"), "-o", _LIB_PATH])
    return _LIB_PATH


@functools.lru_cache(maxsize=1)
def _lib():
    lib = ctypes.CDLL(build_lib())
    lib.ba_generate.restype = ctypes.c_int
    lib.ba_generate.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
    lib.plg_set_threads.restype = None
    lib.plg_set_threads.argtypes = [ctypes.c_int]
    lib.plg_generate.restype = ctypes.c_int
    lib.plg_generate.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                                 ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.POINTER(ctypes.c_double)]
    return lib


def set_threads(k: int) -> None:
    """OpenMP threads used by the generator (its output is independent of the thread count)."""
    _lib().plg_set_threads(int(k))


def plg(n: int, m: int, gamma: float, rho: float, d_cap: float, graph_seed: int,
        name: str = "") -> Graph:
    """Directed Chung-Lu power-law graph, canonical in-CSR."""
    row_ptr = np.empty(n + 1, dtype=np.uint64)
    src = np.empty(m, dtype=np.uint32)
    i0 = ctypes.c_double(0.0)
    rc = _lib().plg_generate(n, m, gamma, rho, d_cap, graph_seed,
                             row_ptr.ctypes.data, src.ctypes.data, ctypes.byref(i0))
    if rc != 0:
        raise RuntimeError(f"plg_generate failed rc={rc}")
    return Graph(n=n, row_ptr=row_ptr, src=src, name=name,
                 meta=dict(generator="plg", n=n, m=m, gamma=gamma, rho=rho, d_cap=d_cap,
                           graph_seed=graph_seed, i0=i0.value))


def ba_edges(n: int, r: int, r0: int) -> int:
    """Directed edge count of the BA graph: both directions of r0(r0-1)/2 + r(n - r0) edges."""
    return 2 * (r0 * (r0 - 1) // 2 + r * (n - r0))


def ba(n: int, r: int, graph_seed: int, r0: int = 0, name: str = "") -> Graph:
    """Barabasi-Albert scale-free graph of the paper's density experiment: clique of
    r0 (default r + 1) nodes, each later node attaches to r distinct degree-proportional
    targets; undirected, stored as both directed edges (canonical in-CSR)."""
    r0 = r0 or r + 1
    m = ba_edges(n, r, r0)
    row_ptr = np.empty(n + 1, dtype=np.uint64)
    src = np.empty(m, dtype=np.uint32)
    rc = _lib().ba_generate(n, r, r0, graph_seed, m, row_ptr.ctypes.data, src.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"ba_generate failed rc={rc}")
    return Graph(n=n, row_ptr=row_ptr, src=src, name=name,
                 meta=dict(generator="ba", n=n, m=m, r=r, r0=r0, graph_seed=graph_seed))


def stats(g: Graph) -> dict:
    """n, m, degree summary and the reverse-branching factor R0."""
    din, dout = g.in_degree(), g.out_degree()
    m = max(g.m, 1)
    return dict(n=g.n, m=g.m, max_in=int(din.max()), max_out=int(dout.max()),
                mean_deg=g.m / g.n, frac_din0=float(np.mean(din == 0)),
                R0_wc=float(np.sum(dout * (din > 0)) / m),
                R0_uniform_per_p=float(np.sum(dout * din) / m))


# ---------------------------------------------------------------------------------------
# Workload table (BASELINE.json configs)
# ---------------------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Workload:
    key: str
    desc: str
    n: int
    m: int
    gamma: float
    rho: float
    d_cap: float
    graph_seed: int
    model: int
    scheme: int
    p_uniform: float
    k: int
    eps: float
    ell: float = 1.0
    rr_seed: int = 200907325
    gen: str = "plg"       # "plg" (Chung-Lu, configs C1-C5) or "ba" (Barabasi-Albert, r = ba_r)
    ba_r: int = 0


WORKLOADS = {
    "C1": Workload("C1", "NetHEPT-shaped (15,233 / 58,892), IC-WC, k=50, eps=0.5",
                   15233, 58892, 2.3, 1.0, 300.0, 1, IC, W_WC, 0.0, 50, 0.5),
    "C2": Workload("C2", "Epinions-shaped (75,879 / 508,837), IC-WC, k=50, eps=0.1",
                   75879, 508837, 2.3, 0.4, 3000.0, 2, IC, W_WC, 0.0, 50, 0.1),
    "C3": Workload("C3", "LiveJournal-shaped (4,847,571 / 68,993,773), IC-WC, k=50, eps=0.1",
                   4847571, 68993773, 2.3, 0.7, 15000.0, 3, IC, W_WC, 0.0, 50, 0.1),
    "C4": Workload("C4", "LiveJournal-shaped (4,847,571 / 68,993,773), LT-WC, k=50, eps=0.1",
                   4847571, 68993773, 2.3, 0.7, 15000.0, 3, LT, W_WC, 0.0, 50, 0.1),
    "C5": Workload("C5", "Twitter-shaped (41,652,230 / 1,468,365,182), IC p=0.01, k=100, eps=0.1",
                   41652230, 1468365182, 2.3, 0.0, 800000.0, 5, IC, W_UNIFORM, 0.01, 100, 0.1),
}


# The paper's density sweep (§4.6): BA graphs, n = 10^6, r = 2..32, IC-WC, k = 50,
# eps = 0.05. Not a BASELINE.json config: bench lines only.
for _r in (2, 4, 8, 16, 32):
    WORKLOADS[f"B{_r}"] = Workload(
        f"B{_r}", f"Barabasi-Albert n=10^6, r={_r} (undirected, both directions), IC-WC, k=50, eps=0.05",
        1000000, ba_edges(1000000, _r, _r + 1), 0.0, 1.0, 0.0, 100 + _r, IC, W_WC, 0.0, 50, 0.05,
        gen="ba", ba_r=_r)


@functools.lru_cache(maxsize=4)
def workload_graph(key: str) -> Graph:
    w = WORKLOADS[key]
    if w.gen == "ba":
        return ba(w.n, w.ba_r, w.graph_seed, name=f"{key}-graph")
    return plg(w.n, w.m, w.gamma, w.rho, w.d_cap, w.graph_seed, name=f"{key}-graph")


# ---------------------------------------------------------------------------------------
# GCSR binary file (SURVEY.md §8(d) "File format")
# ---------------------------------------------------------------------------------------
def save_gcsr(g: Graph, path: str) -> None:
    with open(path, "wb") as f:
        f.write(b"GCSR" + bytes([1]))
        f.write(np.array([g.n, g.m], dtype="<u8").tobytes())
        f.write(g.row_ptr.astype("<u8").tobytes())
        f.write(g.src.astype("<u4").tobytes())
        f.write(json.dumps(g.meta).encode())


def load_gcsr(path: str) -> Graph:
    with open(path, "rb") as f:
        buf = f.read()
    assert buf[:4] == b"GCSR" and buf[4] == 1
    n, m = np.frombuffer(buf, dtype="<u8", count=2, offset=5)
    n, m = int(n), int(m)
    off = 5 + 16
    row_ptr = np.frombuffer(buf, dtype="<u8", count=n + 1, offset=off).copy()
    off += 8 * (n + 1)
    src = np.frombuffer(buf, dtype="<u4", count=m, offset=off).copy()
    off += 4 * m
    meta = json.loads(buf[off:].decode() or "{}")
    return Graph(n=n, row_ptr=row_ptr, src=src, meta=meta, name=os.path.basename(path))
