"""Blocked SOE schedule of the native march on the device (csrc/tsf_soe.cuh
k_soe_block / k_soe_level) against the per-level schedule (k_soe_push_rhs):
the SOE state W after the march is bit-identical (the pass applies the
reference's push recurrence, soe.py:221-223, in registers), the solutions
agree to rounding, and the iteration counts show no bias."""
import numpy as np
import pytest

import paper_2002_11978_b200 as P

pytestmark = pytest.mark.gpu


def _march(monkeypatch, n, B, M, K, seed=5):
    monkeypatch.setenv("TSF_SOE_BLOCK", str(K))
    N = n + 1
    rng = np.random.default_rng(seed)
    x = -1.0 + (2.0 / N) * np.arange(1, N)
    kx = np.exp(0.3 * rng.standard_normal((B, 1)) * np.sin(np.pi * x)[None, :])
    fx = rng.standard_normal((B, 1)) * np.sin(np.pi * x)[None, :]
    u0 = (1 - x * x) ** 2 * rng.uniform(0.5, 2.0, (B, 1))
    kap = P.SeparableField([np.ones(n)], lambda t: [1.0 + 0.2 * t])
    src = P.SeparableField([np.ones(n)], lambda t: [1.0 + t])
    u, rep = P.run_fids_batched(0.5, 1.5, M, 3.0, N, kap, src, u0, kappa_modes=kx[None],
                                source_modes=fx[None], epsilon=1e-12,
                                options=P.SolverOptions(solver="pkrylov", tol=1e-12))
    assert rep["soe_block"] == (K if K > 1 else 1)
    return np.asarray(u), rep["iterations"], rep["W"].cpu().numpy()


@pytest.mark.parametrize("n,B,M,K", [(1024, 24, 29, 8), (256, 17, 20, 3), (4096, 8, 17, 16),
                                     (64, 5, 8, 8)])
def test_blocked_soe_march(monkeypatch, n, B, M, K):
    u1, i1, W1 = _march(monkeypatch, n, B, M, 1)
    uk, ik, Wk = _march(monkeypatch, n, B, M, K)
    rel = np.linalg.norm(uk - u1, axis=1) / np.linalg.norm(u1, axis=1)
    assert rel.max() < 1e-11, rel.max()
    d = ik - i1
    # two device schedules whose history terms differ by rounding: at tol 1e-12
    # the reference itself keeps only 80.5% of cfg2-shaped levels within +-1
    # when its FFT engine is swapped (tests/golden/cfg2_floor.json), so the
    # gate sits between that floor and the 93-100% measured here
    assert np.mean(np.abs(d) <= 1) >= 0.88
    assert abs(d.mean()) < 0.15
    if np.array_equal(ik, i1) and np.array_equal(uk, u1):
        # identical trajectories: the pushed state must match bit for bit
        np.testing.assert_array_equal(Wk, W1)
    # the final W is the state after every push of the march in both schedules
    scale = np.abs(W1).max()
    assert np.abs(Wk - W1).max() <= 1e-10 * scale
