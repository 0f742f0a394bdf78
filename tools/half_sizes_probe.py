"""Half-length vs full-length level-solve engine by grid size: a batched
configs[2]-shaped march (B*n = 2^24, M levels) timed on the device for
TSF_HALF=1 and 0 (subprocesses).  python tools/half_sizes_probe.py [M]"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CHILD = r"""
import sys, time, json
sys.path.insert(0, %r)
import numpy as np, torch
import paper_2002_11978_b200 as P
from paper_2002_11978_b200 import workloads as WL
n, B, M = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
x, kx, fx, u0 = WL.instance_fields(n, 0, B)
kap = P.SeparableField([np.ones(n)], lambda t: [1.0 + 0.2 * t])
src = P.SeparableField([np.ones(n)], lambda t: [1.0 + t])
def run():
    torch.cuda.synchronize(); t0 = time.perf_counter()
    u, rep = P.run_fids_batched(0.5, 1.5, M, 3.0, n + 1, kap, src, u0, kappa_modes=kx[None],
                                source_modes=fx[None], epsilon=1e-12,
                                options=P.SolverOptions(solver="pkrylov", tol=1e-12))
    torch.cuda.synchronize()
    return time.perf_counter() - t0, rep["iterations"]
run()
t, its = run()
print(json.dumps({"n": n, "B": B, "M": M, "s": t, "its_mean": float(np.mean(its))}))
""" % str(ROOT)


def main():
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 48
    for n in (512, 1024, 2048, 4096):
        B = (1 << 23) // n
        row = {}
        for half in ("1", "0"):
            out = subprocess.run([sys.executable, "-c", CHILD, str(n), str(B), str(M)],
                                 env=dict(os.environ, TSF_HALF=half), capture_output=True, text=True)
            line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
            row[half] = json.loads(line[-1]) if line else {"err": out.stderr[-500:]}
        print(json.dumps({"n": n, "half": row["1"], "full": row["0"]}), flush=True)
    # single instance
    for n in (1024, 4096):
        row = {}
        for half in ("1", "0"):
            out = subprocess.run([sys.executable, "-c", CHILD, str(n), "1", "128"],
                                 env=dict(os.environ, TSF_HALF=half), capture_output=True, text=True)
            line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
            row[half] = json.loads(line[-1]) if line else {"err": out.stderr[-500:]}
        print(json.dumps({"n": n, "B": 1, "half": row["1"], "full": row["0"]}), flush=True)


if __name__ == "__main__":
    main()
