"""ctypes wrapper of the parity oracle (``oracle/gim_oracle.c``).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The product path
(``paper_2009_07325_b200``) never imports it, and this package never imports the product.
"""
from __future__ import annotations

import ctypes
import dataclasses
import functools
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gim_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_p = ctypes.c_void_p
_u32, _u64, _dbl, _int = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double, ctypes.c_int


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_DEFAULT_SOURCE", "-ffp-contract=off",
                               "-fno-fast-math", "-fPIC", "-shared", _SRC, "-o", _LIB, "-lm"])
    return _LIB


@functools.lru_cache(maxsize=1)
def _lib():
    lib = ctypes.CDLL(build())
    sig = {
        "og_philox": (None, [_p, _p, _p]),
        "og_root": (_u32, [_u64, _u64, _u32]),
        "og_coin": (_u32, [_u64, _u64, _u64]),
        "og_lt_draw": (_u32, [_u64, _u64, _u32]),
        "og_create": (_p, [_u32, _u64, _p, _p, _p, _int, _int, ctypes.c_float]),
        "og_destroy": (None, [_p]),
        "og_rr_set": (_u32, [_p, _u64, _u64, _p]),
        "og_generate": (_int, [_p, _u64, _u64]),
        "og_num_sets": (_u64, [_p]),
        "og_pool_len": (_u64, [_p]),
        "og_export": (None, [_p, _p, _p, _p]),
        "og_stats": (None, [_p, _p]),
        "og_select_pool": (_int, [_u32, _u64, _p, _p, _p, _u32, _p, _p, _p]),
        "og_select": (_int, [_p, _u32, _p, _p, _p]),
        "og_imm_constants": (_int, [_u32, _u32, _dbl, _dbl, _p]),
        "og_imm": (_int, [_p, _u32, _dbl, _dbl, _u64, _p, _p, _p, _p, _p, _p, _p]),
        "og_mc_spread": (_int, [_p, _p, _u32, _u64, _u64, _p, _p]),
        "og_mrim_generate": (_int, [_p, _u64, _u32, _u64]),
        "og_set_fresh_final": (None, [_p, _int]),
        "og_set_skip": (_int, [_p, _int]),
        "og_skip_ln": (_dbl, [_dbl]),
        "og_skip_ln_series": (_dbl, [_dbl]),
        "og_skip_inv": (_dbl, [_int, _u64, ctypes.c_float]),
        "og_skip_gap": (_dbl, [_dbl, _u32]),
        "og_skip_word": (_u32, [_u64, _u64, _u32, _u32, _u32]),
        "og_mrim_num_sets": (_u64, [_p]),
        "og_mrim_set": (_u32, [_p, _u64, _u64, _u32, _p]),
        "og_mrim_pool_len": (_u64, [_p]),
        "og_mrim_export": (None, [_p, _p, _p, _p]),
        "og_mrim_select_pool": (_int, [_u32, _u32, _u64, _p, _p, _p, _u32, _p, _p, _p]),
        "og_mrim_select": (_int, [_p, _u32, _p, _p, _p]),
        "og_mrim_constants": (_int, [_u32, _u32, _u32, _dbl, _dbl, _p]),
        "og_mrim": (_int, [_p, _u32, _u32, _dbl, _dbl, _u64, _p, _p, _p, _p, _p, _p, _p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


# --- RNG key scheme (O2, O3) -------------------------------------------------------------
def philox(ctr: Sequence[int], key: Sequence[int]) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    _lib().og_philox(_ptr(c), _ptr(k), _ptr(o))
    return o


def root(seed: int, rr_id: int, n: int) -> int:
    return int(_lib().og_root(seed, rr_id, n))


def coin(seed: int, rr_id: int, e: int) -> int:
    return int(_lib().og_coin(seed, rr_id, e))


def lt_draw(seed: int, rr_id: int, v: int) -> int:
    return int(_lib().og_lt_draw(seed, rr_id, v))


# --- R31 geometric-skip contract (oracle/gim_oracle.c "R31") -----------------------------
def skip_ln(x: float) -> float:
    return float(_lib().og_skip_ln(x))


def skip_ln_series(x: float) -> float:
    return float(_lib().og_skip_ln_series(x))


def skip_inv(scheme: int, d: int, p_uniform: float = 0.0) -> float:
    return float(_lib().og_skip_inv(scheme, d, p_uniform))


def skip_gap(inv: float, r: int) -> float:
    return float(_lib().og_skip_gap(inv, r))


def skip_word(seed: int, rr_id: int, v: int, block: int, j: int) -> int:
    return int(_lib().og_skip_word(seed, rr_id, v, block, j))


def imm_constants(n: int, k: int, eps: float, ell: float = 1.0) -> dict:
    out = np.zeros(7, dtype=np.float64)
    rc = _lib().og_imm_constants(n, k, eps, ell, _ptr(out))
    if rc:
        raise ValueError("invalid IMM parameters")
    return dict(zip(["ell_eff", "eps_prime", "lnC", "lambda_prime", "alpha", "beta",
                     "lambda_star"], out.tolist()))


def mrim_constants(n: int, k: int, T: int, eps: float, ell: float = 1.0) -> dict:
    """R28: IMM's constants with ln C(n*T, k*T) for ln C(n, k)."""
    out = np.zeros(7, dtype=np.float64)
    rc = _lib().og_mrim_constants(n, k, T, eps, ell, _ptr(out))
    if rc:
        raise ValueError("invalid MRIM parameters")
    return dict(zip(["ell_eff", "eps_prime", "lnC", "lambda_prime", "alpha", "beta",
                     "lambda_star"], out.tolist()))


def mrim_select_pool(n: int, T: int, offsets: np.ndarray, pairs: np.ndarray, k: int,
                     count: Optional[np.ndarray] = None):
    """R27 on an explicit system of ascending pair sets (pair id = t*n + u). Returns
    (picks, gains, cov) with k*T picks (pair ids) in pick order."""
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    pairs = np.ascontiguousarray(pairs, dtype=np.uint32)
    if count is None:
        count = np.bincount(pairs.astype(np.int64), minlength=n * T).astype(np.uint32)
    count = np.ascontiguousarray(count, dtype=np.uint32)
    seeds = np.zeros(k * T, dtype=np.uint32)
    gains = np.zeros(k * T, dtype=np.uint64)
    cov = np.zeros(1, dtype=np.uint64)
    rc = _lib().og_mrim_select_pool(n, T, len(offsets) - 1, _ptr(offsets), _ptr(pairs) if len(pairs) else None,
                                    _ptr(count), k, _ptr(seeds), _ptr(gains), _ptr(cov))
    if rc:
        raise ValueError(f"og_mrim_select_pool rc={rc}")
    return seeds, gains, int(cov[0])


def select_pool(n: int, offsets: np.ndarray, nodes: np.ndarray, k: int,
                count: Optional[np.ndarray] = None):
    """O7 on an explicit set system (sets ascending). Returns (seeds, gains, cov)."""
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    nodes = np.ascontiguousarray(nodes, dtype=np.uint32)
    if count is None:
        count = np.bincount(nodes.astype(np.int64), minlength=n).astype(np.uint32)
    count = np.ascontiguousarray(count, dtype=np.uint32)
    seeds = np.zeros(k, dtype=np.uint32)
    gains = np.zeros(k, dtype=np.uint64)
    cov = np.zeros(1, dtype=np.uint64)
    rc = _lib().og_select_pool(n, len(offsets) - 1, _ptr(offsets), _ptr(nodes) if len(nodes) else None,
                               _ptr(count), k, _ptr(seeds), _ptr(gains), _ptr(cov))
    if rc:
        raise ValueError(f"og_select_pool rc={rc}")
    return seeds, gains, int(cov[0])


@dataclasses.dataclass
class ImmResult:
    seeds: np.ndarray
    gains: np.ndarray
    LB: float
    theta: float
    spread_est: float
    ell_eff: float
    eps_prime: float
    lambda_prime: float
    lambda_star: float
    rounds: int
    R_final: int
    cov: int
    theta_i: np.ndarray
    T_i: np.ndarray
    cov_i: np.ndarray


class Oracle:
    """One oracle context: a copy of the graph (O1) plus the RR pool (O6)."""

    def __init__(self, g, model: int, scheme: int, p_uniform: float = 0.0):
        self.n, self.m = g.n, g.m
        w = None
        if scheme == 0:
            assert g.weights is not None
            w = np.ascontiguousarray(g.weights, dtype=np.float32)
        rp = np.ascontiguousarray(g.row_ptr, dtype=np.uint64)
        src = np.ascontiguousarray(g.src, dtype=np.uint32)
        self._h = _lib().og_create(g.n, g.m, _ptr(rp), _ptr(src) if g.m else None, _ptr(w),
                                   model, scheme, p_uniform)
        if not self._h:
            raise ValueError("og_create failed")
        self._buf = np.zeros(max(g.n, 1), dtype=np.uint32)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib().og_destroy(h)
            self._h = None

    def rr_set(self, seed: int, rr_id: int) -> np.ndarray:
        ln = _lib().og_rr_set(self._h, seed, rr_id, _ptr(self._buf))
        return self._buf[:ln].copy()

    def generate(self, T: int, seed: int) -> None:
        _lib().og_generate(self._h, T, seed)

    @property
    def num_sets(self) -> int:
        return int(_lib().og_num_sets(self._h))

    @property
    def pool_len(self) -> int:
        return int(_lib().og_pool_len(self._h))

    def export(self):
        ns, pl = self.num_sets, self.pool_len
        off = np.zeros(ns + 1, dtype=np.uint64)
        nodes = np.zeros(max(pl, 1), dtype=np.uint32)
        cnt = np.zeros(self.n, dtype=np.uint32)
        _lib().og_export(self._h, _ptr(off), _ptr(nodes), _ptr(cnt))
        return off, nodes[:pl], cnt

    def stats(self) -> dict:
        o = np.zeros(2, dtype=np.uint64)
        _lib().og_stats(self._h, _ptr(o))
        return dict(coins=int(o[0]), live=int(o[1]))

    def select(self, k: int):
        seeds = np.zeros(k, dtype=np.uint32)
        gains = np.zeros(k, dtype=np.uint64)
        cov = np.zeros(1, dtype=np.uint64)
        rc = _lib().og_select(self._h, k, _ptr(seeds), _ptr(gains), _ptr(cov))
        if rc:
            raise ValueError(f"og_select rc={rc}")
        return seeds, gains, int(cov[0])

    def imm(self, k: int, eps: float, ell: float, seed: int) -> ImmResult:
        seeds = np.zeros(k, dtype=np.uint32)
        gains = np.zeros(k, dtype=np.uint64)
        dres = np.zeros(7, dtype=np.float64)
        th = np.zeros(64, dtype=np.float64)
        T = np.zeros(64, dtype=np.uint64)
        cv = np.zeros(64, dtype=np.uint64)
        u = np.zeros(3, dtype=np.uint64)
        rc = _lib().og_imm(self._h, k, eps, ell, seed, _ptr(seeds), _ptr(gains), _ptr(dres),
                           _ptr(th), _ptr(T), _ptr(cv), _ptr(u))
        if rc:
            raise ValueError("og_imm: invalid parameters")
        r = int(u[0])
        return ImmResult(seeds=seeds, gains=gains, LB=dres[0], theta=dres[1], spread_est=dres[2],
                         ell_eff=dres[3], eps_prime=dres[4], lambda_prime=dres[5],
                         lambda_star=dres[6], rounds=r, R_final=int(u[1]), cov=int(u[2]),
                         theta_i=th[:r].copy(), T_i=T[:r].copy(), cov_i=cv[:r].copy())

    def mc_spread(self, S: Sequence[int], trials: int, mc_seed: int):
        s = np.ascontiguousarray(S, dtype=np.uint32)
        mean, se = ctypes.c_double(), ctypes.c_double()
        _lib().og_mc_spread(self._h, _ptr(s), len(s), trials, mc_seed, ctypes.byref(mean),
                            ctypes.byref(se))
        return mean.value, se.value

    def set_skip(self, on: bool) -> None:
        """R31: live in-edges by geometric gaps (IC with WC or uniform weights); pool restarts."""
        if _lib().og_set_skip(self._h, int(bool(on))):
            raise ValueError("the skip contract needs IC with WC or uniform weights")

    def set_fresh_final(self, on: bool) -> None:
        """R29: IMM's final phase on a fresh pool (key seed ^ 0x9E3779B97F4A7C15)."""
        _lib().og_set_fresh_final(self._h, int(bool(on)))

    # ---- MRIM (R26-R28; oracle/gim_oracle.c "MRIM") ----------------------------------------
    def mrim_generate(self, N: int, T: int, seed: int) -> None:
        if _lib().og_mrim_generate(self._h, N, T, seed):
            raise ValueError("og_mrim_generate: invalid T")
        self._T_mr = T

    def mrim_set(self, seed: int, i: int, T: int) -> np.ndarray:
        buf = np.zeros(self.n * T, dtype=np.uint32)
        ln = _lib().og_mrim_set(self._h, seed, i, T, _ptr(buf))
        return buf[:ln].copy()

    def mrim_export(self):
        ns = int(_lib().og_mrim_num_sets(self._h))
        pl = int(_lib().og_mrim_pool_len(self._h))
        T = self._mrim_T
        off = np.zeros(ns + 1, dtype=np.uint64)
        pairs = np.zeros(max(pl, 1), dtype=np.uint32)
        cnt = np.zeros(self.n * T, dtype=np.uint32)
        _lib().og_mrim_export(self._h, _ptr(off), _ptr(pairs), _ptr(cnt))
        return off, pairs[:pl], cnt

    def mrim_select(self, k: int):
        T = self._mrim_T
        seeds = np.zeros(k * T, dtype=np.uint32)
        gains = np.zeros(k * T, dtype=np.uint64)
        cov = np.zeros(1, dtype=np.uint64)
        rc = _lib().og_mrim_select(self._h, k, _ptr(seeds), _ptr(gains), _ptr(cov))
        if rc:
            raise ValueError(f"og_mrim_select rc={rc}")
        return seeds, gains, int(cov[0])

    def mrim(self, k: int, T: int, eps: float, ell: float, seed: int) -> ImmResult:
        seeds = np.zeros(k * T, dtype=np.uint32)
        gains = np.zeros(k * T, dtype=np.uint64)
        dres = np.zeros(7, dtype=np.float64)
        th = np.zeros(64, dtype=np.float64)
        TT = np.zeros(64, dtype=np.uint64)
        cv = np.zeros(64, dtype=np.uint64)
        u = np.zeros(3, dtype=np.uint64)
        self._T_mr = T
        rc = _lib().og_mrim(self._h, k, T, eps, ell, seed, _ptr(seeds), _ptr(gains), _ptr(dres),
                            _ptr(th), _ptr(TT), _ptr(cv), _ptr(u))
        if rc:
            raise ValueError("og_mrim: invalid parameters")
        r = int(u[0])
        return ImmResult(seeds=seeds, gains=gains, LB=dres[0], theta=dres[1], spread_est=dres[2],
                         ell_eff=dres[3], eps_prime=dres[4], lambda_prime=dres[5],
                         lambda_star=dres[6], rounds=r, R_final=int(u[1]), cov=int(u[2]),
                         theta_i=th[:r].copy(), T_i=TT[:r].copy(), cov_i=cv[:r].copy())

    @property
    def _mrim_T(self) -> int:
        return int(self._T_mr) if hasattr(self, "_T_mr") else 1
