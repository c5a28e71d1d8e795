"""Thin Python binding of libgim.so (include/gim.h) — argument marshalling only.

Every step of the hot path (RR sampling, storage, inverted index, NodeSelection, the IMM
driver) runs inside libgim.so; this module only converts arrays and calls the C ABI. PyTorch is
used for plumbing: device memory (the caching allocator backs every library allocation), the
CUDA stream, and torch.distributed process groups for the selection all-reduce.

Method names follow the C names without the ``gim_`` prefix (``gim_load_graph`` ->
``Gim.load_graph`` ...). There is no fallback: if libgim.so is missing or no CUDA device is
present, construction raises.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Callable, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GIM_LIB_PATH") or os.path.join(_HERE, "libgim.so")

GIM_OK, GIM_EINVAL, GIM_ESTATE, GIM_ENOMEM, GIM_ECUDA, GIM_ECOLL, GIM_ELTWEIGHT = range(7)
IC, LT = 0, 1
W_EXPLICIT, W_WC, W_UNIFORM = 0, 1, 2
OPT_FORCE_GIANT, OPT_QUEUE_CAP, OPT_PROFILE, OPT_STAGING_CAP, OPT_SELECT_GRAPH, OPT_INV_SEGMENTS, OPT_ARGMAX_CAND, OPT_IC_LANE, OPT_SPECULATE, OPT_MB_CHAINS, OPT_PDL, OPT_GIANT_NT, OPT_FRESH_FINAL, OPT_SELECT_PERSISTENT, OPT_SKIP, OPT_SPILL, OPT_SELECT_FUSED, OPT_FUSED_CTAS, OPT_FORCE_COLLECTIVES, OPT_GIANT_SHARED, OPT_SKIP_LANE_CAP, OPT_SELECT_COOP, OPT_IMM_EARLY_EXIT, OPT_INV_PASSES, OPT_L2_PERSIST, OPT_SELECT_CTA, OPT_INV_SORT, OPT_CHUNK, OPT_SELECT_CLUSTER, OPT_IMM_LOOKAHEAD = 1, 2, 3, 4, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23, 24, 26, 27, 28, 29, 30, 31, 32

_STATUS = {0: "GIM_OK", 1: "GIM_EINVAL", 2: "GIM_ESTATE", 3: "GIM_ENOMEM", 4: "GIM_ECUDA",
           5: "GIM_ECOLL", 6: "GIM_ELTWEIGHT"}

_p, _u32, _u64, _i32, _i64, _dbl = (ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64,
                                    ctypes.c_int, ctypes.c_int64, ctypes.c_double)

ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, _p, _u64, _p, _p)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, _p, _u64, _p, _p, _p)
REDUCESCATTER_FN = ctypes.CFUNCTYPE(ctypes.c_int, _p, _p, _u64, _p, _p)
ALLOC_FN = ctypes.CFUNCTYPE(_p, _u64, _p, _p)
FREE_FN = ctypes.CFUNCTYPE(None, _p, _p, _p)


class ImmResultC(ctypes.Structure):
    _fields_ = [("ell_eff", _dbl), ("eps_prime", _dbl), ("lambda_prime", _dbl),
                ("lambda_star", _dbl), ("LB", _dbl), ("theta", _dbl), ("rounds", _u32),
                ("theta_i", _u64 * 64), ("cov_i", _u64 * 64), ("theta_i_real", _dbl * 64),
                ("R_final", _u64), ("covered", _u64), ("spread_est", _dbl), ("sel_steps_i", _u32 * 64)]


class StatsC(ctypes.Structure):
    _fields_ = [("launches", _u64), ("rr_sets", _u64), ("rr_elements", _u64),
                ("giant_sets", _u64), ("coins", _u64), ("live_edges", _u64), ("coins_giant", _u64),
                ("live_giant", _u64), ("selects", _u64),
                ("allreduces", _u64), ("ms_rr", _dbl), ("ms_giant", _dbl), ("ms_store", _dbl),
                ("ms_inv", _dbl), ("ms_select", _dbl), ("n_rr_launches", _u64),
                ("n_giant_launches", _u64), ("n_syncs", _u64), ("n_allocs", _u64),
                ("host_ms_sync", _dbl), ("host_ms_api", _dbl), ("fused_fallbacks", _u64),
                ("probe_stops", _u64), ("lookahead_drops", _u64)]


# name -> (restype, argtypes); exactly the functions declared in include/gim.h
SIGNATURES = {
    "gim_create": (_i32, [_i32, _p, ctypes.POINTER(_p)]),
    "gim_destroy": (None, [_p]),
    "gim_last_error": (ctypes.c_char_p, [_p]),
    "gim_load_graph": (_i32, [_p, _u32, _u64, _p, _p, _p, _i32, _i32, ctypes.c_float]),
    "gim_set_shard": (_i32, [_p, _i32, _i32]),
    "gim_set_allreduce": (_i32, [_p, ALLREDUCE_FN, _p]),
    "gim_set_allgather": (_i32, [_p, ALLGATHER_FN, _p]),
    "gim_set_reducescatter": (_i32, [_p, REDUCESCATTER_FN, _p]),
    "gim_nccl_unique_id": (_i32, [_p]),
    "gim_set_nccl": (_i32, [_p, _p, _i32, _i32, _i32]),
    "gim_set_allocator": (_i32, [_p, ALLOC_FN, FREE_FN, _p]),
    "gim_generate_rr": (_i32, [_p, _u64, _u64]),
    "gim_select": (_i32, [_p, _u32, _p, _p, _p]),
    "gim_imm": (_i32, [_p, _u32, _dbl, _dbl, _u64, _p, ctypes.POINTER(ImmResultC)]),
    "gim_rr_export": (_i32, [_p, _p, _p, _p, _p, _p, _i32]),
    "gim_counts_export": (_i32, [_p, _p]),
    "gim_set_option": (_i32, [_p, _i32, _i64]),
    "gim_get_stats": (_i32, [_p, ctypes.POINTER(StatsC)]),
    "gim_reset_stats": (_i32, [_p]),
    "gim_microbench_philox": (_i32, [_p, _u64, ctypes.POINTER(_dbl)]),
    "gim_set_rounds": (_i32, [_p, _u32]),
    "gim_mc_spread": (_i32, [_p, _p, _u32, _u64, _u64, ctypes.POINTER(_dbl), ctypes.POINTER(_dbl), _p]),
}

_lib_handle = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libgim.so (raises if it is missing — there is no fallback path)."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(path):
            raise RuntimeError(f"libgim.so not built ({path}); run `make` / __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(lib, name)
            f.restype, f.argtypes = res, args
        _lib_handle = lib
    return _lib_handle


class GimError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


@dataclasses.dataclass
class ImmResult:
    seeds: np.ndarray
    ell_eff: float
    eps_prime: float
    lambda_prime: float
    lambda_star: float
    LB: float
    theta: float
    rounds: int
    theta_i: np.ndarray
    theta_i_real: np.ndarray
    cov_i: np.ndarray
    R_final: int
    covered: int
    spread_est: float
    sel_steps_i: np.ndarray = None   # greedy steps run per round (< k: bounded-greedy early exit)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


class Gim:
    """One libgim context (one device, one stream)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None, torch_allocator: bool = True):
        self._lib = load_library()
        self._keep = []
        h = _p()
        st = self._lib.gim_create(device, stream, ctypes.byref(h))
        if st != GIM_OK:
            raise GimError(st, "gim_create failed (no usable CUDA device?)")
        self._h = h
        self.device = device
        self.rounds = 1                      # MRIM rounds T (gim_set_rounds)
        self.n = 0                           # nodes of the loaded graph
        if torch_allocator:
            self._use_torch_allocator(device)

    # -- plumbing -------------------------------------------------------------------------
    def _check(self, st: int):
        if st != GIM_OK:
            raise GimError(st, self._lib.gim_last_error(self._h).decode())

    def _use_torch_allocator(self, device: int):
        import torch

        def _alloc(nbytes, stream, user):
            try:
                return torch.cuda.caching_allocator_alloc(int(nbytes), device, int(stream or 0))
            except Exception:
                return None

        def _free(ptr, stream, user):
            if torch is not None and getattr(torch, "cuda", None) is not None:   # interpreter teardown
                torch.cuda.caching_allocator_delete(ptr)

        a, f = ALLOC_FN(_alloc), FREE_FN(_free)
        self._keep += [a, f]
        self._check(self._lib.gim_set_allocator(self._h, a, f, None))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.gim_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- C ABI ----------------------------------------------------------------------------
    def load_graph(self, n: int, row_ptr: np.ndarray, src: np.ndarray, model: int, scheme: int,
                   weights: Optional[np.ndarray] = None, p_uniform: float = 0.0):
        rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
        s = np.ascontiguousarray(src, dtype=np.uint32)
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float32)
        self._check(self._lib.gim_load_graph(self._h, n, len(s), _ptr(rp), _ptr(s) if len(s) else None,
                                             _ptr(w), model, scheme, p_uniform))
        self.n = n

    def set_shard(self, rank: int, world: int):
        self._check(self._lib.gim_set_shard(self._h, rank, world))

    def set_allreduce(self, fn: Callable[[int, int, int], int]):
        """fn(dev_ptr, count_int32, cuda_stream) -> 0 on success (in-place SUM)."""
        cb = ALLREDUCE_FN(lambda buf, count, stream, user: int(fn(buf, count, stream or 0)))
        self._keep.append(cb)
        self._check(self._lib.gim_set_allreduce(self._h, cb, None))

    def set_allgather(self, fn: Callable[[int, int, int, int], int]):
        """fn(send_ptr, nbytes, recv_ptr, cuda_stream) -> 0: all-gather of nbytes per rank into
        recv (world * nbytes, rank order). Switches world > 1 to the replicated-pool protocol."""
        cb = ALLGATHER_FN(lambda snd, nb, rcv, stream, user: int(fn(snd, nb, rcv, stream or 0)))
        self._keep.append(cb)
        self._check(self._lib.gim_set_allgather(self._h, cb, None))

    def set_nccl(self, nccl_id: bytes, rank: int, world: int, protocol: str = "allreduce"):
        """Native NCCL exchange (include/gim.h gim_set_nccl): the library creates its own NCCL
        communicator from the 128-byte id (same on every rank, see nccl_unique_id / setup_nccl)
        and issues the protocol's collectives on its stream itself; collective over the world."""
        proto = {"allreduce": 0, "replicated": 1, "reducescatter": 2}[protocol]
        buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        self._check(self._lib.gim_set_nccl(self._h, buf, rank, world, proto))

    def set_reducescatter(self, fn: Callable[[int, int, int, int], int]):
        """fn(send_ptr, recv_ptr, recv_count_int32, cuda_stream) -> 0: SUM reduce-scatter of int32
        (this rank's block of the sum). With set_allreduce (and no all-gather), world > 1
        selection runs the node-sharded protocol (include/gim.h gim_set_reducescatter)."""
        cb = REDUCESCATTER_FN(lambda snd, rcv, cnt, stream, user: int(fn(snd, rcv, cnt, stream or 0)))
        self._keep.append(cb)
        self._check(self._lib.gim_set_reducescatter(self._h, cb, None))

    def generate_rr(self, theta: int, seed: int):
        self._check(self._lib.gim_generate_rr(self._h, theta, seed))

    def set_rounds(self, rounds: int):
        """MRIM mode (readings R26-R28): T rounds; select/imm then return k*T pair ids t*n + u."""
        self._check(self._lib.gim_set_rounds(self._h, rounds))
        self.rounds = rounds

    def mc_spread(self, seeds, trials: int, mc_seed: int, return_sizes: bool = False):
        """Forward Monte-Carlo spread of `seeds` under IC (gim_mc_spread): (mean, stderr[, sizes])."""
        s = np.ascontiguousarray(seeds, dtype=np.uint32)
        mean, se = _dbl(), _dbl()
        sizes = np.zeros(trials, dtype=np.uint32) if return_sizes else None
        self._check(self._lib.gim_mc_spread(self._h, _ptr(s), len(s), trials, mc_seed, ctypes.byref(mean),
                                            ctypes.byref(se), _ptr(sizes)))
        return (mean.value, se.value, sizes) if return_sizes else (mean.value, se.value)

    def select(self, k: int):
        seeds = np.zeros(k * self.rounds, dtype=np.uint32)
        gains = np.zeros(k * self.rounds, dtype=np.uint64)
        cov = np.zeros(1, dtype=np.uint64)
        self._check(self._lib.gim_select(self._h, k, _ptr(seeds), _ptr(gains), _ptr(cov)))
        return seeds, gains, int(cov[0])

    def imm(self, k: int, eps: float, ell: float, seed: int) -> ImmResult:
        seeds = np.zeros(k * self.rounds, dtype=np.uint32)
        r = ImmResultC()
        self._check(self._lib.gim_imm(self._h, k, eps, ell, seed, _ptr(seeds), ctypes.byref(r)))
        nr = int(r.rounds)
        return ImmResult(seeds=seeds, ell_eff=r.ell_eff, eps_prime=r.eps_prime,
                         lambda_prime=r.lambda_prime, lambda_star=r.lambda_star, LB=r.LB,
                         theta=r.theta, rounds=nr, theta_i=np.array(r.theta_i[:nr], dtype=np.uint64),
                         theta_i_real=np.array(r.theta_i_real[:nr]),
                         cov_i=np.array(r.cov_i[:nr], dtype=np.uint64), R_final=int(r.R_final),
                         covered=int(r.covered), spread_est=r.spread_est,
                         sel_steps_i=np.array(r.sel_steps_i[:nr], dtype=np.uint32))

    def rr_export(self, sort_each_set: bool = True):
        ns, pl = _u64(), _u64()
        self._check(self._lib.gim_rr_export(self._h, ctypes.byref(ns), ctypes.byref(pl), None, None,
                                            None, 0))
        ids = np.zeros(max(ns.value, 1), dtype=np.uint64)
        off = np.zeros(ns.value + 1, dtype=np.uint64)
        nodes = np.zeros(max(pl.value, 1), dtype=np.uint32)
        self._check(self._lib.gim_rr_export(self._h, ctypes.byref(ns), ctypes.byref(pl), _ptr(ids),
                                            _ptr(off), _ptr(nodes), int(sort_each_set)))
        return ids[:ns.value], off, nodes[:pl.value]

    def pool_size(self):
        """(n_sets, pool_len) of this rank's pool (gim_rr_export size query)."""
        ns, pl = _u64(), _u64()
        self._check(self._lib.gim_rr_export(self._h, ctypes.byref(ns), ctypes.byref(pl), None, None,
                                            None, 0))
        return int(ns.value), int(pl.value)

    def rr_offsets(self) -> np.ndarray:
        """offsets[n_sets + 1] of this rank's pool only (gim_rr_export without the members)."""
        ns, pl = _u64(), _u64()
        self._check(self._lib.gim_rr_export(self._h, ctypes.byref(ns), ctypes.byref(pl), None, None,
                                            None, 0))
        off = np.zeros(ns.value + 1, dtype=np.uint64)
        self._check(self._lib.gim_rr_export(self._h, ctypes.byref(ns), ctypes.byref(pl), None,
                                            _ptr(off), None, 0))
        return off

    def counts_export(self, n: int = 0) -> np.ndarray:
        """count_total: n * rounds entries (MRIM pair counts when rounds > 1). The buffer is
        sized by the binding from the loaded graph and the rounds; ``n`` is only checked."""
        want = self.n * self.rounds
        if n and n not in (self.n, want):
            raise ValueError(f"counts_export: n={n} does not match the loaded graph ({self.n} x {self.rounds})")
        out = np.zeros(max(want, 1), dtype=np.uint32)
        self._check(self._lib.gim_counts_export(self._h, _ptr(out)))
        return out[:want]

    def set_option(self, opt: int, value: int):
        self._check(self._lib.gim_set_option(self._h, opt, value))

    def stats(self) -> dict:
        s = StatsC()
        self._check(self._lib.gim_get_stats(self._h, ctypes.byref(s)))
        return {name: getattr(s, name) for name, _ in StatsC._fields_}

    def reset_stats(self):
        self._check(self._lib.gim_reset_stats(self._h))

    def microbench_philox(self, groups: int) -> float:
        ms = _dbl()
        self._check(self._lib.gim_microbench_philox(self._h, groups, ctypes.byref(ms)))
        return ms.value


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (include/gim.h gim_nccl_unique_id)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    st = lib.gim_nccl_unique_id(buf)
    if st != GIM_OK:
        raise GimError(st, "ncclGetUniqueId failed (libnccl.so.2 not loadable?)")
    return buf.raw


def setup_nccl(ctx: "Gim", rank: int, world: int, protocol: str = "allreduce", group=None):
    """Rank 0 draws the NCCL id, torch.distributed broadcasts it (any backend), every rank then
    hands it to ctx.set_nccl: from there on the library runs its own NCCL collectives."""
    nid = nccl_unique_id() if rank == 0 else bytes(128)
    if world > 1:
        import torch.distributed as dist
        obj = [nid]
        dist.broadcast_object_list(obj, src=0, group=group)
        nid = obj[0]
    ctx.set_nccl(nid, rank, world, protocol)


def torch_allreduce(group=None, device: str = "cuda"):
    """all-reduce callback for Gim.set_allreduce: wraps the library's int32 buffer as a torch
    tensor and runs torch.distributed.all_reduce (SUM) ordered on the library's stream (NCCL over
    NVLink when the group's backend is nccl). device="cpu" wraps a host pointer instead (used by
    the multi-process gloo tests of this plumbing)."""
    import torch
    import torch.distributed as dist

    def fn(ptr: int, count: int, stream: int) -> int:
        if device == "cpu":
            arr = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_int32)), shape=(int(count),))
            dist.all_reduce(torch.from_numpy(arr), op=dist.ReduceOp.SUM, group=group)
            return 0

        class _View:
            __cuda_array_interface__ = {"shape": (int(count),), "typestr": "<i4",
                                        "data": (int(ptr), False), "version": 3, "strides": None,
                                        "stream": None}
        t = torch.as_tensor(_View(), device="cuda")
        s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            if dist.get_backend(group) == "gloo":     # functional testing: stage through host
                h = t.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return 0

    return fn


def torch_allgather(group=None, device: str = "cuda"):
    """all-gather callback for Gim.set_allgather: torch.distributed.all_gather_into_tensor of the
    library's device bytes, ordered on the library's stream (NCCL over NVLink for an nccl group;
    a gloo group stages through host memory, for functional tests). device="cpu" wraps host
    pointers instead (the multi-process gloo tests of this plumbing)."""
    import torch
    import torch.distributed as dist

    if device == "cpu":
        def fn_cpu(send: int, nbytes: int, recv: int, stream: int) -> int:
            world = dist.get_world_size(group)
            u8 = ctypes.POINTER(ctypes.c_uint8)
            src = np.ctypeslib.as_array(ctypes.cast(send, u8), shape=(int(nbytes),))
            dst = np.ctypeslib.as_array(ctypes.cast(recv, u8), shape=(int(nbytes) * world,))
            parts = [torch.empty(int(nbytes), dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(src.copy()), group=group)
            dst[:] = torch.cat(parts).numpy()
            return 0
        return fn_cpu

    def view(ptr, nbytes):
        class _View:
            __cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                        "data": (int(ptr), False), "version": 3, "strides": None,
                                        "stream": None}
        return torch.as_tensor(_View(), device="cuda")

    def fn(send: int, nbytes: int, recv: int, stream: int) -> int:
        world = dist.get_world_size(group)
        src = view(send, nbytes)
        dst = view(recv, nbytes * world)
        s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            if dist.get_backend(group) == "gloo":
                parts = [torch.empty(int(nbytes), dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(parts, src.cpu(), group=group)
                dst.copy_(torch.cat(parts).to(dst.device))
            else:
                dist.all_gather_into_tensor(dst, src, group=group)
        return 0

    return fn


def torch_reducescatter(group=None, device: str = "cuda"):
    """reduce-scatter callback for Gim.set_reducescatter: torch.distributed.reduce_scatter_tensor
    (SUM) of the library's int32 device buffers, ordered on the library's stream (NCCL over
    NVLink for an nccl group; a gloo group stages through host memory with an all-reduce, for
    functional tests). device="cpu" wraps host pointers (the multi-process gloo tests)."""
    import torch
    import torch.distributed as dist

    def host(ptr, count):
        return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_int32)), shape=(int(count),))

    if device == "cpu":
        def fn_cpu(send: int, recv: int, count: int, stream: int) -> int:
            world, rank = dist.get_world_size(group), dist.get_rank(group)
            full = torch.from_numpy(host(send, count * world).copy())
            dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
            host(recv, count)[:] = full[rank * count:(rank + 1) * count].numpy()
            return 0
        return fn_cpu

    def view(ptr, count):
        class _View:
            __cuda_array_interface__ = {"shape": (int(count),), "typestr": "<i4",
                                        "data": (int(ptr), False), "version": 3, "strides": None,
                                        "stream": None}
        return torch.as_tensor(_View(), device="cuda")

    def fn(send: int, recv: int, count: int, stream: int) -> int:
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        src = view(send, count * world)
        dst = view(recv, count)
        s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            if dist.get_backend(group) == "gloo":
                h = src.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
                dst.copy_(h[rank * count:(rank + 1) * count].to(dst.device))
            else:
                dist.reduce_scatter_tensor(dst, src, op=dist.ReduceOp.SUM, group=group)
        return 0

    return fn


def shard_slice(a: int, b: int, rank: int, world: int):
    """This rank's contiguous slice of RR ids [a, b) (include/gim.h gim_set_shard)."""
    ln = b - a
    return a + ln * rank // world, a + ln * (rank + 1) // world
