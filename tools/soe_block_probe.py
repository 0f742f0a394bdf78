"""Blocked SOE schedule (TSF_SOE_BLOCK=K) against the per-level one
(TSF_SOE_BLOCK=1) on batched marches: final W (bit-identical expected),
solution difference and iteration mismatches per configuration."""
import os
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np
import paper_2002_11978_b200 as P
from paper_2002_11978_b200.scheme import FidsMarch  # noqa: F401


def run(n, B, M, K, seed=3):
    os.environ["TSF_SOE_BLOCK"] = str(K)
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


for n, B, M in [(4096, 48, 40), (1024, 40, 37), (256, 33, 20), (64, 9, 10)]:
    u1, i1 = run(n, B, M, 1)
    for K in (2, 8, 16):
        u, i = run(n, B, M, K)
        d = float(np.max(np.linalg.norm(u - u1, axis=1) / np.linalg.norm(u1, axis=1)))
        im = int(np.sum(i != i1))
        big = int(np.sum(np.abs(i - i1) > 1))
        print(f"n={n} B={B} M={M} K={K}: max rel-l2 {d:.2e}, iteration mismatches {im}/{i.size} "
              f"(|d|>1: {big}), mean d {float(np.mean(i - i1)):+.4f}", flush=True)
os.environ["TSF_SOE_BLOCK"] = "8"
