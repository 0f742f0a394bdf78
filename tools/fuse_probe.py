"""SOE modes of the batched march must give bit-identical results:
TSF_FUSE_SOE=0 (standalone k_soe_push_rhs per level) and 1 (the solve
kernels' thread-streamed epilogue).  Prints max |du| and iteration
mismatches per configuration.  (A bulk-copy streamed epilogue, mode 2, was
built, bit-identical, and measured slower: DESIGN.md §3.4.)"""
import os
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import paper_2002_11978_b200 as P


def run(n, B, M, mode, seed=3):
    os.environ["TSF_FUSE_SOE"] = mode
    N = n + 1
    rng = np.random.default_rng(seed)
    x = -1.0 + (2.0 / N) * np.arange(1, N)
    kx = np.exp(0.3 * rng.standard_normal((B, 1)) * np.sin(np.pi * x)[None, :])
    fx = rng.standard_normal((B, 1)) * np.sin(np.pi * x)[None, :]
    u0 = (1 - x * x) ** 2 * rng.uniform(0.5, 2.0, (B, 1))
    kap = P.SeparableField([np.ones(n)], lambda t: [1.0 + 0.2 * t])
    src = P.SeparableField([np.ones(n)], lambda t: [1.0 + t])
    uB, rep = P.run_fids_batched(0.5, 1.5, M, 3.0, N, kap, src, u0, kappa_modes=kx[None],
                                 source_modes=fx[None], epsilon=1e-12,
                                 options=P.SolverOptions(solver="pkrylov", tol=1e-12))
    return np.asarray(uB), np.asarray(rep["iterations"])


ok = True
for n, B, M in [(4096, 48, 12), (1024, 40, 16), (256, 33, 20), (64, 9, 10)]:
    u0, i0 = run(n, B, M, "0")
    for mode in ("1",):
        u, i = run(n, B, M, mode)
        d = float(np.max(np.abs(u - u0)))
        im = int(np.sum(i != i0))
        ok &= d == 0.0 and im == 0
        print(f"n={n} B={B} M={M} mode={mode}: max|du|={d:.3e} iteration mismatches={im}", flush=True)
os.environ["TSF_FUSE_SOE"] = "0"
print("fuse_probe", "OK" if ok else "MISMATCH")
