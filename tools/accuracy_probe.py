"""Accuracy probe: device matvec / preconditioner vs exact long-double
results, next to numpy pocketfft's own error (the reference engine)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
from tsf_testlib import golden
import oracle as O
import paper_2002_11978_b200 as P

def exact_toeplitz(col, v):
    n = col.size
    c = col.astype(np.longdouble); x = v.astype(np.longdouble)
    idx = np.abs(np.arange(n)[:, None] - np.arange(n)[None, :])
    return (c[idx] @ x)

def exact_circ_solve(total, v):
    n = v.size
    k = np.arange(n)
    ang = (2 * np.pi * np.outer(k, k) % (2*np.pi)).astype(np.longdouble) if False else None
    two_pi = np.longdouble(2) * np.longdouble(np.pi)
    kk = (np.outer(k, k) % n).astype(np.longdouble)
    Wc = np.cos(two_pi * kk / n); Ws = np.sin(two_pi * kk / n)
    x = v.astype(np.longdouble)
    Fr = Wc @ x; Fi = -(Ws @ x)
    t = total.astype(np.longdouble)
    Fr /= t; Fi /= t
    return (Wc @ Fr - Ws @ Fi) / n   # real part of inverse

g = golden("linalg")
for i in range(8):
    col, v = g[f"tp{i}_col"], g[f"tp{i}_v"]
    n = col.size
    if n > 4096: continue
    ex = exact_toeplitz(col, v)
    scale = float(np.max(np.abs(ex)))
    e_np = float(np.max(np.abs(g[f"tp{i}_Av"] - ex))) / scale
    gpu = P.toeplitz_matvec(P.build_toeplitz(col), v)
    e_gpu = float(np.max(np.abs(gpu - ex))) / scale
    line = f"n={n:5d} matvec  numpy {e_np:.2e}  gpu {e_gpu:.2e}"
    if n & (n - 1) == 0 and n >= 16:
        tot = g[f"tp{i}_total"]
        exs = exact_circ_solve(tot, v)
        sc = float(np.max(np.abs(exs)))
        e_np2 = float(np.max(np.abs(g[f"tp{i}_Pinv_v"] - exs))) / sc
        p = P.build_preconditioner(col, g[f"tp{i}_shift"][0], float(g[f"tp{i}_kappa"].mean()))
        e_gpu2 = float(np.max(np.abs(P.precond_solve(p, v) - exs))) / sc
        line += f" | precond numpy {e_np2:.2e} gpu {e_gpu2:.2e}"
    print(line, flush=True)
