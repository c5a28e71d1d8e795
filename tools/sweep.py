"""Parameter sweeps on the built path (the shape of the paper's
Figs. 4-7): runs bench.py once per point on the GPU box and appends its JSON line to
gpurun_out/sweep_<name>.jsonl.

  python tools/sweep.py density      # BA n=10^6, r = 2..32, k=50, eps=0.05
  python tools/sweep.py k            # C3 (IC) and C4 (LT), k = 1..200, eps=0.1
  python tools/sweep.py eps          # C3, eps = 0.05..0.5, k=50
  python tools/sweep.py mrim         # MRIM k=10, T=5, eps=0.1 on C2/C3/C4 (Table 3)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
POINTS = {
    "density": [["--workload", f"B{r}", "--cpu-seconds", "8"] for r in (2, 4, 8, 16, 32)],
    "k": [["--workload", wl, "--k", str(k), "--no-cpu-baseline"]
          for wl in ("C3", "C4") for k in (1, 10, 25, 50, 100, 200)],
    "eps": [["--workload", "C3", "--eps", str(e), "--no-cpu-baseline"] for e in (0.05, 0.1, 0.2, 0.3, 0.5)],
    # MRIM (CR-NAIMM, §4.8 Table 3 settings: k = 10, T = 5, eps = 0.1)
    "mrim": [["--workload", "C2", "--k", "10", "--rounds", "5", "--cpu-seconds", "8"],
             ["--workload", "C3", "--k", "10", "--rounds", "5", "--cpu-seconds", "8"],
             ["--workload", "C4", "--k", "10", "--rounds", "5", "--no-cpu-baseline"]],
}


def main():
    name = sys.argv[1]
    out = os.path.join(ROOT, "gpurun_out", f"sweep_{name}.jsonl")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        for pt in POINTS[name]:
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3", "--no-e2e"] + pt
            p = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
            line = p.stdout.strip().splitlines()[-1] if p.returncode == 0 and p.stdout.strip() else \
                json.dumps({"error": p.stderr[-400:], "point": pt})
            f.write(line + "\n")
            f.flush()
            print(" ".join(pt), "->", line[:160], flush=True)


if __name__ == "__main__":
    main()
