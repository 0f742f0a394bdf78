"""Debug probe: batched march vs single-instance oracle runs (per-instance errors)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import oracle as O
import paper_2002_11978_b200 as P

n, M, gam, a = int(sys.argv[1]) if len(sys.argv) > 1 else 256, 24, 0.5, 1.5
B = int(sys.argv[2]) if len(sys.argv) > 2 else 5
N = n + 1
rng = np.random.default_rng(7)
x = -1.0 + (2.0 / N) * np.arange(1, N)
kx = np.exp(0.3 * rng.standard_normal((B, 1)) * np.sin(np.pi * x)[None, :])
fx = rng.standard_normal((B, 1)) * np.sin(np.pi * x)[None, :]
u0 = (1 - x * x) ** 2 * rng.uniform(0.5, 2.0, (B, 1))
kap = P.SeparableField([np.ones(n)], lambda t: [1.0 + 0.2 * t])
src = P.SeparableField([np.ones(n)], lambda t: [1.0 + t])
uB, rep = P.run_fids_batched(gam, a, M, 3.0, N, kap, src, u0, kappa_modes=kx[None],
                             source_modes=fx[None], epsilon=1e-12,
                             options=P.SolverOptions(solver="pkrylov", tol=1e-12))
for b in range(B):
    rec = O.fids_march(gam, a, 1.0, 1.0, M, 3.0, N, lambda xx, t, b=b: kx[b] * (1.0 + 0.2 * t),
                       lambda xx, t, b=b: fx[b] * (1.0 + t), lambda xx, b=b: u0[b],
                       epsilon=1e-12, tol=1e-12)
    e = np.linalg.norm(uB[b] - rec.hist[-1]) / np.linalg.norm(rec.hist[-1])
    print(b, "%.2e" % e, rep["iterations"][:, b].tolist()[:12], rec.iterations.tolist()[:12])
