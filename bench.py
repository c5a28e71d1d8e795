#!/usr/bin/env python
"""bench.py — RR sets/s & IMM time of the gIM/IMM hot path on B200 (BASELINE.json metric).

One step = one full IMM run (gim_imm: every Alg. 2 round of RR sampling + NodeSelection, then
theta = lambda*/LB, the final sampling and the final NodeSelection) on the workload named by
--workload (default C3: LiveJournal-shaped synthetic graph, IC weighted cascade, k=50,
eps=0.1, ell=1), with the graph resident in HBM. value = RR sets generated (global R_final,
summed over steps) / device time of the K timed steps (max over ranks). Every rank holds the
replicated graph and generates its contiguous slice of every RR-id range (weak-by-ids
sharding, "scaling": "strong" since the per-job work is fixed); selection all-reduces counts
over NCCL.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gim|reference] [--workload C3]

--impl reference times the oracle (oracle/, single-threaded C, as it stands) on a bounded
sample of the same workload on the host cores.
"""
import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gim_inputs as gi  # noqa: E402

METRIC = "RR sets/s & IMM time (k=50, ε=0.1) at 1/2/4/8 B200; HBM GB/s vs peak"
UNIT = "RR sets/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gim", choices=["gim", "reference"])
    ap.add_argument("--workload", default="C3", choices=sorted(gi.WORKLOADS))
    ap.add_argument("--k", type=int, default=0, help="override the workload's k (parameter sweeps)")
    ap.add_argument("--eps", type=float, default=0.0, help="override the workload's eps (parameter sweeps)")
    ap.add_argument("--rounds", type=int, default=1,
                    help="MRIM rounds T (CR-NAIMM, §4.8; readings R26-R28): value counts MRIM sets/s")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--opt", action="append", default=[], help="library option NAME=VALUE (ablations)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo + --same-device: functional multi-rank test on 1 GPU)")
    ap.add_argument("--same-device", action="store_true", help="all ranks on cuda:0 (functional testing)")
    ap.add_argument("--torch-collectives", action="store_true",
                    help="exchange through torch.distributed callbacks instead of the library's own NCCL communicator")
    ap.add_argument("--skip", action="store_true",
                    help="geometric-skip RNG contract (reading R31, GIM_OPT_SKIP) instead of one coin per in-edge")
    ap.add_argument("--protocol", default="replicated", choices=["replicated", "allreduce", "reducescatter"],
                    help="N > 1 exchange: replicated pool (all-gather per round), dense per-step "
                         "all-reduce (north_star), or node-sharded reduce-scatter selection")
    ap.add_argument("--dense-exchange", action="store_true", help="alias of --protocol allreduce")
    ap.add_argument("--force-collectives", action="store_true",
                    help="run the --protocol exchange even at N = 1 (drives the NCCL callbacks on one GPU)")
    ap.add_argument("--no-variants", action="store_true", help="skip the geometric-skip variant measurement")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def unit_of(args):
    return UNIT if args.rounds == 1 else "MRIM sets/s"


PROTO_DESC = {"replicated": "each round's sets all-gathered, NodeSelection replicated",
              "allreduce": "count all-reduce + per-step decrement all-reduce",
              "reducescatter": "node-sharded selection: counts/decrements reduce-scattered, per-step key exchange"}


def config_of(w, world, rounds=1, protocol="replicated", force=False):
    mr = {} if rounds == 1 else {"mrim_rounds": rounds,
                                 "mrim": f"CR-NAIMM (§4.8): k={w.k} seeds per round, T={rounds} rounds"}
    return {"workload": f"{w.key}: {w.desc}", **mr, "n": w.n, "m": w.m, "k": w.k, "eps": w.eps,
            "ell": w.ell, "model": "IC" if w.model == gi.IC else "LT",
            "weights": {gi.W_WC: "weighted cascade 1/d_in", gi.W_UNIFORM: f"uniform p={w.p_uniform}",
                        gi.W_EXPLICIT: "explicit"}[w.scheme],
            "generator": (f"barabasi-albert r={w.ba_r} r0={w.ba_r + 1} graph_seed={w.graph_seed}" if w.gen == "ba"
                          else f"plg gamma={w.gamma} rho={w.rho} d_cap={w.d_cap} graph_seed={w.graph_seed}"),
            "rr_seed": w.rr_seed,
            "parallelism": f"dp{world} (RR-id slices sampled per rank, replicated graph"
                           + (f"; {protocol}: {PROTO_DESC[protocol]})" if world > 1 or force else ")"),
            "l2": "inputs larger than L2 (the graph's CSR exceeds the 126 MB L2)" if w.m > 30_000_000
            else "graph is L2-resident (no flush between steps)"}


# ------------------------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ------------------------------------------------------------------------------------------
class Clocks:
    """Samples SM clock and clock-event (throttle) reasons through NVML every 5 ms in a
    background thread while the timed region runs (falls back to nothing if NVML is absent)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index):
        import threading
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.005)

    def stop(self):
        if self.nv is None:
            return None
        self._stop.set()
        self.t.join(timeout=2)
        if not self.samples:
            return None
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml 5 ms"}


# ------------------------------------------------------------------------------------------
# reference arm: the oracle on the host cores
# ------------------------------------------------------------------------------------------
def host_cpu():
    """CPU model and core count of this host (lscpu), for the baseline's context."""
    model = "unknown"
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def golden_imm_time(key, skip=False):
    """The oracle's FULL single-core IMM run on this workload (the paper's baseline protocol,
    single-core IMM), recorded by tools/oracle_golden.py with its CPU model
    and pinned core in tests/golden/imm_<key>.json — measured on the build host, not in this run."""
    path = os.path.join(ROOT, "tests", "golden", f"imm_{key}{'_skip' if skip else ''}.json")
    if not os.path.exists(path):
        return None
    gd = json.load(open(path))
    o = gd.get("oracle_run", {})
    return {"kind": "oracle full IMM", "imm_s": o.get("imm_s"), "rr_sets": gd.get("R_final"),
            "rr_sets_per_s": o.get("rr_sets_per_s"), "cpu_model": o.get("cpu_model"), "nproc": o.get("nproc"),
            "taskset_core": o.get("taskset_core"), "where": "build host (tools/oracle_golden.py), not this run"}


def oracle_sample(w, g, seconds, k, rounds=1, skip=False):
    """Oracle RR generation (ids 0..T-1, grown in chunks until `seconds` elapse) followed by one
    NodeSelection (k) over that sample; returns (sets, wall seconds). rounds > 1: MRIM sets."""
    import oracle
    o = oracle.Oracle(g, w.model, w.scheme, w.p_uniform)
    if skip:
        o.set_skip(True)
    t0 = time.perf_counter()
    T, chunk = 0, max(2000 // rounds, 200)
    while time.perf_counter() - t0 < seconds:
        T += chunk
        if rounds > 1:
            o.mrim_generate(T, rounds, w.rr_seed)
        else:
            o.generate(T, w.rr_seed)
    if rounds > 1:
        o.mrim_select(k)
    else:
        o.select(k)
    return T, time.perf_counter() - t0


def run_reference(args, w):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    g = gi.workload_graph(w.key)
    core = sorted(os.sched_getaffinity(0))[-1]
    os.sched_setaffinity(0, {core})                           # the oracle is single-threaded: one core
    per_step = max(1.0, min(10.0, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample(w, g, per_step / 4, w.k, args.rounds)
    tot_sets, tot_s = 0, 0.0
    for _ in range(args.steps):
        T, s = oracle_sample(w, g, per_step, w.k, args.rounds)
        tot_sets += T
        tot_s += s
    v = tot_sets / tot_s
    unit = unit_of(args)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": unit, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_s / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": config_of(w, 1, args.rounds),
            "cpu_baseline": {"value": v, "unit": unit, "cores": 1, "kind": "oracle",
                             "sample": f"per step: oracle RR sets of ids 0..T-1 for ~{per_step:.1f}s, "
                                       f"then one k={w.k} NodeSelection over them",
                             **host_cpu(), "taskset_core": core, "full_imm": golden_imm_time(w.key)},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------
def alu_peak_gcoins(sm_mhz, sms=148):
    """ALU roof of IC sampling: one Philox4x32-10 = 20 IMAD.WIDE.U32, which issue
    only to the FMA-heavy pipe at 4 cycles per warp instruction (16 lanes x a 64-bit result; the
    32-bit IMAD rate of B300_MICROARCH.md "Pipe rates" is rt_SMSP = 2). 80 cycles per warp-Philox
    per SM sub-partition, 4 SMSPs -> 1.6 Philox = 6.4 coins per cycle per SM. ncu evidence:
    profiles/r01_ncu_k_philox_bench.txt (fmaheavy 82% busy, ALU 49%, issue 56%)."""
    return 6.4 * sms * sm_mhz * 1e6 / 1e9


def load_profile_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


def run_gim(args, w):
    import torch
    import torch.distributed as dist
    import paper_2009_07325_b200 as P

    world, rank, local = dist_env()
    if args.same_device:
        local = 0
    pg = world > 1 or args.force_collectives
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"          # no version banner on stdout: one JSON line only
    if pg:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    if world > 1:   # torchrun pins OMP_NUM_THREADS=1: give each rank its share of the host cores
        gi.set_threads(max(1, (os.cpu_count() or 1) // int(os.environ.get("LOCAL_WORLD_SIZE", world))))
    g = gi.workload_graph(w.key)
    stream = torch.cuda.Stream(local)
    ctx = P.Gim(local, stream=stream.cuda_stream)
    ctx.load_graph(g.n, g.row_ptr, g.src, w.model, w.scheme, weights=g.weights, p_uniform=w.p_uniform)
    if args.rounds > 1:
        ctx.set_rounds(args.rounds)
    exchange = {"kind": "none"}

    def hooks(cx):
        if world > 1 or args.force_collectives:
            cx.set_shard(rank, world)
            native = not args.torch_collectives and args.backend == "nccl"
            if native:
                try:          # the library's own NCCL communicator (gim_set_nccl): no Python per step
                    P.setup_nccl(cx, rank, world, args.protocol)
                    exchange["kind"] = "native NCCL (gim_set_nccl)"
                except Exception as ex:   # noqa: BLE001 — fall back to the torch.distributed callbacks
                    exchange["fallback"] = str(ex)[:120]
                    native = False
            if not native:
                cx.set_allreduce(P.torch_allreduce())
                if args.protocol == "replicated":      # no per-step collectives
                    cx.set_allgather(P.torch_allgather())
                elif args.protocol == "reducescatter":
                    cx.set_reducescatter(P.torch_reducescatter())
                exchange["kind"] = "torch.distributed callbacks"
            if args.force_collectives:
                cx.set_option(P.OPT_FORCE_COLLECTIVES, 1)
    hooks(ctx)
    if args.skip:
        ctx.set_option(P.OPT_SKIP, 1)
    for o in args.opt:
        name, val = o.split("=")
        ctx.set_option(getattr(P, name), int(val))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if args.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(args.warmup, 0)):
        ctx.imm(w.k, w.eps, w.ell, w.rr_seed)
    ctx.reset_stats()
    barrier()
    torch.cuda.synchronize()
    clk = Clocks(local) if rank == 0 else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    results, step_wall = [], []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        results.append(ctx.imm(w.k, w.eps, w.ell, w.rr_seed))
        step_wall.append(1000 * (time.perf_counter() - t0))
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop() if clk else None
    ms = max_over_ranks(e0.elapsed_time(e1))
    st_timed = ctx.stats()          # launches / syncs / allocations of the timed region
    total_sets = sum(r.R_final for r in results)
    # per-kernel-class event timing (GIM_OPT_PROFILE) adds a record per launch class, so the
    # phase split and the roofline come from a separate profiled pass of the same K steps
    ctx.set_option(P.OPT_PROFILE, 1)
    ctx.reset_stats()
    for _ in range(args.steps):
        ctx.imm(w.k, w.eps, w.ell, w.rr_seed)
    torch.cuda.synchronize()
    st = ctx.stats()
    ctx.set_option(P.OPT_PROFILE, 0)
    value = total_sets / (ms / 1000.0)
    r0 = results[-1]

    # RR-set size distribution of the last IMM run's pool, outside the timing
    sizes = np.diff(ctx.rr_offsets().astype(np.int64))
    size_q = ({"p50": int(np.percentile(sizes, 50)), "p99": int(np.percentile(sizes, 99)),
               "max": int(sizes.max())} if len(sizes) else None)

    # ---- dominant kernel roofline: K-RR (warp-per-RR sampling), ALU-bound by Philox ----------
    rr_ms = st["ms_rr"]
    n_rr = max(st["n_rr_launches"], 1)
    coins = st["coins"]
    sm_max = (clocks or {}).get("sm_max_mhz") or 1965.0
    peak = alu_peak_gcoins(sm_max)
    achieved = coins / (rr_ms / 1000.0) / 1e9 if rr_ms > 0 else 0.0
    # algorithmic bytes of K-RR: 12 B per set (size+offset) + 8 B row_ptr pair and 4 B staging
    # write per visited node + 4 B src per live in-edge (coins are drawn before any load)
    warp_elems = st["rr_elements"]
    alg_bytes = 12 * st["rr_sets"] + 12 * warp_elems + 4 * st["live_edges"]
    tr = load_profile_traffic().get(f"{w.key}:k_rr_warp{':skip' if args.skip else ''}")
    tr = tr if isinstance(tr, dict) else None
    mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = mp.get("hbm_gbs", 6650.0)
    measured_philox = None
    try:
        groups = 1 << 30
        mb_ms = ctx.microbench_philox(groups)
        measured_philox = 4 * groups / (mb_ms / 1000.0) / 1e9
    except Exception:
        pass
    alg_gbs = alg_bytes / (rr_ms / 1000.0) / 1e9 if rr_ms > 0 else 0.0
    if w.model == gi.IC:
        head = {"kernel": "k_rr_warp (K-IC warp-per-RR sampling)", "bound": "alu", "achieved": achieved,
                "peak": peak, "unit": "Gcoin/s", "frac": achieved / peak if peak else None}
    else:   # LT: one draw per visited node, dependent loads -> reported against HBM
        head = {"kernel": "k_rr_warp (K-LT reverse walk)", "bound": "hbm", "achieved": alg_gbs,
                "peak": hbm_peak, "unit": "GB/s", "frac": alg_gbs / hbm_peak}
    roofline = {
        **head,
        "traffic": tr["dram_bytes"] if tr else None,
        "traffic_launch_sets": tr["launch_sets"] if tr else None,
        "traffic_launch_alg_bytes": tr["alg_bytes"] if tr else None,
        "sector_eff": tr["sector_eff"] if tr else None,
        "dram_gbs": tr["dram_gbs"] if tr else None,
        "traffic_note": ("dram__bytes_read+write of ONE k_rr_warp launch (a 2^20-set generate_rr call, "
                         "tools/traffic_capture.py, profiles/ncu_traffic.json) against the algorithmic bytes "
                         "of the same launch; sector_eff = algorithmic / DRAM bytes") if tr else None,
        "per_launch_ms": rr_ms / n_rr, "launches": n_rr,
        "coins_per_launch": coins / n_rr,
        "peak_basis": f"derived: 6.4 coins/cycle/SM x 148 SMs x {sm_max:.0f} MHz (Philox4x32-10 = 20 IMAD.WIDE.U32, 4 cycles each on the FMA-heavy pipe)",
        "philox_microbench_gcoins": measured_philox,
        "frac_of_microbench": (achieved / measured_philox) if measured_philox else None,
        "algorithmic_gbs": alg_gbs,
        "hbm_peak_gbs": hbm_peak,
        "hbm_frac": alg_gbs / hbm_peak,
        "hbm_peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy)" if mp else "fallback 6.65 TB/s",
    }
    phases = {"ms_rr": st["ms_rr"] / args.steps, "ms_giant": st["ms_giant"] / args.steps,
              "ms_store": st["ms_store"] / args.steps, "ms_inv": st["ms_inv"] / args.steps,
              "ms_select": st["ms_select"] / args.steps}
    gen_ms = st["ms_rr"] + st["ms_giant"] + st["ms_store"]

    # ---- the geometric-skip contract (reading R31) on the same graph and launch shape -------
    variants = None
    if (not args.skip and not args.no_variants and w.model == gi.IC and w.scheme != gi.W_EXPLICIT
            and args.rounds == 1):
        ctx.set_option(P.OPT_SKIP, 1)
        for _ in range(max(args.warmup, 0)):
            ctx.imm(w.k, w.eps, w.ell, w.rr_seed)
        ctx.reset_stats()
        barrier()
        torch.cuda.synchronize()
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0.record(stream)
        vres = [ctx.imm(w.k, w.eps, w.ell, w.rr_seed) for _ in range(args.steps)]
        v1.record(stream)
        torch.cuda.synchronize()
        barrier()
        vms = max_over_ranks(v0.elapsed_time(v1))
        ctx.set_option(P.OPT_PROFILE, 1)            # phase split from a profiled pass
        ctx.reset_stats()
        for _ in range(args.steps):
            ctx.imm(w.k, w.eps, w.ell, w.rr_seed)
        torch.cuda.synchronize()
        vst = ctx.stats()
        ctx.set_option(P.OPT_PROFILE, 0)
        v_rr_ms = vst["ms_rr"] + vst["ms_giant"]
        # algorithmic bytes: 12 B per set + per visited node 8 B row pointers, 8 B tabulated
        # 1/ln(1-p) and 4 B staging write + 4 B per live in-edge; the draws are ~2 per node
        v_alg = 12 * vst["rr_sets"] + 20 * vst["rr_elements"] + 4 * (vst["live_edges"] + vst["live_giant"])
        v_gbs = v_alg / (v_rr_ms / 1000.0) / 1e9 if v_rr_ms > 0 else 0.0
        vtr = load_profile_traffic().get(f"{w.key}:k_rr_warp:skip")
        variants = {"geometric_skip": {
            "rng": "reading R31 (GIM_OPT_SKIP): live in-edges drawn as geometric gaps; bit-exact vs the "
                   "oracle's skip mirror (tests/test_gpu_skip.py), same distribution of RR sets",
            "value": sum(r.R_final for r in vres) / (vms / 1000.0), "unit": unit_of(args),
            "ms_per_step": vms / args.steps,
            "phase_ms_per_step": {k_: vst[k_] / args.steps for k_ in ("ms_rr", "ms_giant", "ms_store", "ms_inv",
                                                                      "ms_select")},
            "draws_per_set": (vst["coins"] + vst["coins_giant"]) / max(vst["rr_sets"], 1),
            "seeds_head": vres[-1].seeds[:8].tolist(),
            "roofline": {"kernel": "k_skip_lane + k_skip_warp (+ k_skip_giant): dependent row-pointer / "
                                   "source loads per BFS level", "bound": "hbm", "achieved": v_gbs,
                         "peak": hbm_peak, "unit": "GB/s", "frac": v_gbs / hbm_peak,
                         "traffic": vtr.get("dram_bytes") if isinstance(vtr, dict) else None,
                         "sector_eff": vtr.get("sector_eff") if isinstance(vtr, dict) else None}}}
        ctx.set_option(P.OPT_SKIP, 0)

    # ---- end to end through the public API with host buffers -------------------------------
    e2e = None
    if not args.no_e2e:
        rp_h = torch.from_numpy(g.row_ptr).pin_memory()
        src_h = torch.from_numpy(g.src).pin_memory()
        ctx2 = P.Gim(local, stream=stream.cuda_stream)
        if args.skip:
            ctx2.set_option(P.OPT_SKIP, 1)
        if args.rounds > 1:
            ctx2.set_rounds(args.rounds)
        hooks(ctx2)
        def e2e_step():
            ctx2.load_graph(g.n, rp_h.numpy(), src_h.numpy(), w.model, w.scheme, weights=g.weights,
                            p_uniform=w.p_uniform)
            if world > 1 or args.force_collectives:
                ctx2.set_shard(rank, world)
            return ctx2.imm(w.k, w.eps, w.ell, w.rr_seed)
        for _ in range(max(args.warmup, 1)):
            e2e_step()
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        e2e_sets = 0
        for _ in range(args.steps):
            r = e2e_step()
            e2e_sets += r.R_final
        f1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms2 = max_over_ranks(f0.elapsed_time(f1))
        e2e = {"value": e2e_sets / (ms2 / 1000.0), "unit": unit_of(args),
               "h2d_bytes_per_step": int(g.row_ptr.nbytes + g.src.nbytes),
               "d2h_bytes_per_step": int((4 * w.k + 8 * w.k * (r.rounds + 1)) * args.rounds),
               "ms_per_step": ms2 / args.steps,
               "note": "per step: gim_load_graph (H2D of the in-CSR from pinned host buffers + on-device validation) + gim_imm + seeds D2H"}
        ctx2.close()

    # ---- CPU baseline: the oracle on a bounded sample (rank 0, N=1 only) --------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        core = sorted(os.sched_getaffinity(0))[-1]
        old_aff = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {core})                       # one pinned host core
        try:
            T, s = oracle_sample(w, g, args.cpu_seconds, w.k, args.rounds, skip=args.skip)
        finally:
            os.sched_setaffinity(0, old_aff)
        cpu = {"value": T / s, "unit": unit_of(args), "cores": 1, "kind": "oracle",
               "sample": f"oracle {'MRIM' if args.rounds > 1 else 'RR'} sets of ids 0..{T - 1} ({s:.1f}s) + one "
                         f"k={w.k} NodeSelection over them, single-threaded C"
                         + (" (geometric-skip contract, R31)" if args.skip else ""),
               **host_cpu(), "taskset_core": core, "full_imm": golden_imm_time(w.key, args.skip)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": unit_of(args), "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
                "config": {**config_of(w, world, args.rounds, args.protocol, args.force_collectives),
                           "rng": ("geometric-skip contract (reading R31, GIM_OPT_SKIP)" if args.skip else
                                   "Philox4x32-10 coin per in-edge slot (reading R16, north_star)"),
                           **({"exchange": exchange} if exchange["kind"] != "none" else {})},
                "imm_time_s": ms / args.steps / 1000.0,
                "rr_sets_per_step": r0.R_final, "theta": r0.theta, "LB": r0.LB, "rounds": r0.rounds,
                "spread_est": r0.spread_est,
                "rr_gen_sets_per_s": (st["rr_sets"] * world) / (gen_ms / 1000.0) if gen_ms > 0 else None,
                "phase_ms_per_step": phases,
                "rr_stats": {"mean_len": st["rr_elements"] / max(st["rr_sets"], 1),
                             "coins_per_set": (st["coins"] + st["coins_giant"]) / max(st["rr_sets"], 1),
                             "giant_frac": st["giant_sets"] / max(st["rr_sets"], 1),
                             "coins_per_giant_set": st["coins_giant"] / max(st["giant_sets"], 1),
                             "size_quantiles": size_q},
                "gpu_launches": st_timed["launches"],
                "step_wall_ms": [round(x, 3) for x in step_wall],
                "host": {"api_ms_per_step": st_timed["host_ms_api"] / args.steps,
                         "sync_ms_per_step": st_timed["host_ms_sync"] / args.steps,
                         "syncs_per_step": st_timed["n_syncs"] / args.steps,
                         "allocs_in_timed_region": st_timed["n_allocs"]},
                "phase_split_note": ("phase_ms_per_step, rr_stats and roofline come from a second, profiled "
                                     "pass of the same K steps (GIM_OPT_PROFILE events); value and "
                                     "ms_per_step from the unprofiled timed region"),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
                "variants": variants,
                "seeds_head": r0.seeds[:8].tolist()}
        print(json.dumps(line), flush=True)
    ctx.close()
    if pg:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.dense_exchange:
        args.protocol = "allreduce"
    w = gi.WORKLOADS[args.workload]
    if args.k or args.eps:      # sweep point: same graph, other (k, eps); named in config
        w = dataclasses.replace(w, k=args.k or w.k, eps=args.eps or w.eps,
                                desc=f"{w.desc} [sweep: k={args.k or w.k}, eps={args.eps or w.eps}]")
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_gim(args, w)


if __name__ == "__main__":
    main()
