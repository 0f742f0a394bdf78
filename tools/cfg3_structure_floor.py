"""configs[3] iteration-count floor under a second transform STRUCTURE (CPU).

The committed cfg3 floor swaps numpy's FFT for scipy's, whose complex inverse
is bit-identical to numpy's, so it understates the spread a different correct
engine sees.  This runs the reference's control flow
(oracle/) at n = 2^20, M = 256 with the device engines' transform structures
emulated in numpy (tools/half_probe.py: `eng` = even/odd channels of
length-n transforms with the Strang spectrum reuse, `half` = the half-length
structure) and compares per-level iterations with the reference's own run
(tests/golden/cfg3.npz).  Writes tests/golden/cfg3_structure_floor.json.

    python tools/cfg3_structure_floor.py [levels]
"""
import json
import math
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np
from scipy.special import gammaln

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import oracle as O  # noqa: E402
from half_probe import Engine  # noqa: E402


def march(args):
    kind, M_run = args
    n, M, gamma, alpha = 1 << 20, 256, 0.7, 1.2
    N = n + 1
    r = (2 - gamma) / gamma
    t, tau = O.graded_mesh(M, r, 1.0)
    col, h, _ = O.ifl_column(alpha, 1 + alpha / 2, 1.0, N)
    _, sym = O.toeplitz_symbol(col)
    lam = O.strang_eigs(col)
    G = math.exp(gammaln(1 - gamma))
    s, w = O.soe_build(gamma, 1e-12, (1.0 / M) ** r, 1.0)
    x = -1.0 + (2.0 / N) * np.arange(1, N)
    eng = Engine(kind, "numpy", sym, n)
    W = np.zeros((s.size, n))
    up = (1.0 - x * x) ** 2
    its = np.zeros(M_run, dtype=int)
    for m in range(1, M_run + 1):
        amm = O.last_l1_weight(tau[m - 1], gamma)
        shift = amm / G
        kap = 1.0 + 0.5 * np.sin(np.pi * x) * np.exp(-t[m])
        f = (1.0 + t[m]) * np.sin(np.pi * x)
        rhs = f + (amm * up - O.soe_history_term(W, s, w, tau[m - 1])) / G
        total = shift + float(kap.mean()) * lam
        u, out = O.bicgstab(lambda q: shift * q + kap * eng.mv(q), lambda q: eng.pc(q, total),
                            rhs, tol=1e-12)
        its[m - 1] = out.iterations
        O.soe_push(W, s, u - up, tau[m - 1])
        up = u
        if m % 16 == 0:
            print(kind, m, its[m - 16:m].tolist(), flush=True)
    return kind, its


def main():
    M_run = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    ref = np.load(ROOT / "tests" / "golden" / "cfg3.npz")["its"][:M_run]
    out = {}
    with ProcessPoolExecutor(max_workers=2) as ex:
        for kind, its in ex.map(march, [("eng", M_run), ("half", M_run)]):
            d = its - ref
            out[kind] = {"levels": M_run, "within1": float(np.mean(np.abs(d) <= 1)),
                         "within2": float(np.mean(np.abs(d) <= 2)), "mean_d": float(d.mean()),
                         "max_abs_d": int(np.abs(d).max())}
            print(kind, out[kind], flush=True)
    (ROOT / "tests" / "golden" / "cfg3_structure_floor.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
