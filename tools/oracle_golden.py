"""Write the full-IMM goldens tests/golden/imm_<cfg>.json by running the ORACLE only.

Every stored value comes from ``oracle/`` (the plain single-threaded C IMM, SURVEY.md §8(c)
O1-O9) on the seeded input of ``gim_inputs/`` — nothing here imports or calls the CUDA path.
The GPU suite (tests/test_gpu_golden.py) regenerates the same graph on the box, checks its
hash against ``graph_sha256`` and compares ``gim_imm`` with these values bit for bit (doubles
to 1e-12 relative): the north_star target "bit-exact seed sets versus the CPU oracle on all
five configs" (§4.3: IMM's and gIM's solutions are the same; Alg. 2
P:211-236 for the trace).

The oracle run is also the full single-core IMM time of the paper's baseline protocol
(single-core IMM), recorded with the CPU model and the pinned core.

    python tools/oracle_golden.py C3 [C4 C5 ...] [--core 0] [--fresh-final] [--skip]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gim_inputs as gi  # noqa: E402
import oracle  # noqa: E402


def sha256(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).view(np.uint8).tobytes())
    return h.hexdigest()


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def run(key: str, core: int, fresh_final: bool, skip: bool = False) -> dict:
    w = gi.WORKLOADS[key]
    t0 = time.time()
    g = gi.workload_graph(key)
    t_graph = time.time() - t0
    graph_hash = sha256(g.row_ptr, g.src)
    os.sched_setaffinity(0, {core})
    o = oracle.Oracle(g, w.model, w.scheme, w.p_uniform)
    o.set_fresh_final(fresh_final)
    if skip:
        o.set_skip(True)
    t0 = time.perf_counter()
    r = o.imm(w.k, w.eps, w.ell, w.rr_seed)
    t_imm = time.perf_counter() - t0
    os.sched_setaffinity(0, set(range(os.cpu_count())))
    _, _, cnt = o.export()
    st = o.stats()
    out = dict(
        config=key, desc=w.desc, n=g.n, m=g.m, model=w.model, scheme=w.scheme,
        p_uniform=w.p_uniform, k=w.k, eps=w.eps, ell=w.ell, rr_seed=w.rr_seed,
        fresh_final=fresh_final, skip=skip, graph_sha256=graph_hash,
        seeds=r.seeds.tolist(), gains=[int(x) for x in r.gains], cov=r.cov, R_final=r.R_final,
        rounds=r.rounds, T_i=[int(x) for x in r.T_i], cov_i=[int(x) for x in r.cov_i],
        theta_i=r.theta_i.tolist(), LB=r.LB, theta=r.theta, spread_est=r.spread_est,
        ell_eff=r.ell_eff, eps_prime=r.eps_prime, lambda_prime=r.lambda_prime,
        lambda_star=r.lambda_star,
        pool_len=int(o.pool_len), count_sha256=sha256(cnt), coins=st["coins"], live=st["live"],
        oracle_run=dict(imm_s=t_imm, graph_gen_s=t_graph, cores=1, taskset_core=core,
                        cpu_model=cpu_model(), nproc=os.cpu_count(), host=platform.node(),
                        rr_sets_per_s=r.R_final / t_imm,
                        note="oracle/gim_oracle.c og_imm, one pinned core (sched_setaffinity)"),
    )
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--core", type=int, default=0)
    ap.add_argument("--fresh-final", action="store_true")
    ap.add_argument("--skip", action="store_true", help="geometric-skip RNG contract (reading R31)")
    ap.add_argument("--out-dir", default=os.path.join(ROOT, "tests", "golden"))
    a = ap.parse_args()
    for key in a.configs:
        res = run(key, a.core, a.fresh_final, a.skip)
        name = f"imm_{key}{'_fresh' if a.fresh_final else ''}{'_skip' if a.skip else ''}.json"
        with open(os.path.join(a.out_dir, name), "w") as f:
            json.dump(res, f, indent=1)
        print(f"{key}: R={res['R_final']} seeds[:5]={res['seeds'][:5]} "
              f"imm {res['oracle_run']['imm_s']:.1f}s", flush=True)


if __name__ == "__main__":
    main()
