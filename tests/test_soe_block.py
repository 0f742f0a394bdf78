"""Blocked SOE schedule of the native march (csrc/tsf_soe.cuh k_soe_block /
k_soe_level): the host tables must reproduce the reference's per-level
recurrence (soe.py:209-225 push, scheme.py:281-282 history term) — a numpy
emulation of the exact device schedule against the per-level oracle path."""
import numpy as np
import pytest

import oracle as O
from paper_2002_11978_b200.scheme import soe_block_tables


def _tab(gamma, M, eps=1e-12):
    r = (2.0 - gamma) / gamma
    _, tau = O.graded_mesh(M, r, 1.0)
    s, w = O.soe_build(gamma, eps, (1.0 / M) ** r, 1.0)
    tab = np.empty((M, 3, s.size))
    for m in range(M):
        dec = np.exp(-s * tau[m])
        tab[m] = dec, -np.expm1(-s * tau[m]) / s, w * dec
    return tab, tau


def _per_level(tab, tau, U):
    """Reference order: H^m = h(m) . W^{m-1}; W^m = (W d) + (c du^m)."""
    M, _, nexp = tab.shape
    W = np.zeros((nexp, U.shape[1]))
    H = []
    for m in range(1, M + 1):
        d, c, h = tab[m - 1]
        H.append(h @ W)
        du = (U[m] - U[m - 1]) / tau[m - 1]
        W = (W * d[:, None]) + (c[:, None] * du[None, :])
    return np.array(H), W


def _blocked(tab, tau, U, K):
    """The device schedule: one W pass per K levels, du / G rings."""
    M, _, nexp = tab.shape
    alpha, beta = soe_block_tables(tab, K)
    n = U.shape[1]
    W = np.zeros((nexp, n))
    G = {}
    du = {}
    H = []

    def push(W, lev):
        d, c, _ = tab[lev - 1]
        return (W * d[:, None]) + (c[:, None] * du[lev][None, :])

    for m in range(1, M + 1):
        du[m - 1] = (U[m - 1] - U[m - 2]) / tau[m - 2] if m >= 2 else None
        mb = K * ((m - 1) // K)
        if m - 1 == mb:
            for lev in range(max(1, mb - K + 1), mb + 1):
                W = push(W, lev)
            for k in range(min(K, M - mb)):
                G[mb + 1 + k] = alpha[mb + k] @ W
            H.append(G[m])
        else:
            h = G[m].copy()
            for q in range(m - 1 - mb):
                h = h + beta[m - 1, q] * du[mb + 1 + q]
            H.append(h)
    du[M] = (U[M] - U[M - 1]) / tau[M - 1]
    mbl = K * ((M - 1) // K)
    for lev in range(mbl + 1, M + 1):
        W = push(W, lev)
    return np.array(H), W


@pytest.mark.parametrize("gamma,M,K", [(0.5, 40, 8), (0.3, 37, 5), (0.8, 24, 16), (0.5, 9, 2)])
def test_blocked_soe_matches_per_level(gamma, M, K):
    tab, tau = _tab(gamma, M)
    rng = np.random.default_rng(11)
    x = np.linspace(-1, 1, 34)[1:-1]
    U = np.cumsum(rng.standard_normal((M + 1, x.size)) * 0.1, axis=0) + (1 - x * x) ** 2
    H0, W0 = _per_level(tab, tau, U)
    H1, W1 = _blocked(tab, tau, U, K)
    # W advanced with the reference's own recurrence: bit-identical
    np.testing.assert_array_equal(W1, W0)
    # history terms: same quantity, summation regrouped
    scale = np.max(np.abs(H0), axis=1, keepdims=True) + 1e-300
    assert np.max(np.abs(H1 - H0) / scale) < 1e-13
