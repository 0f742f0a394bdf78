"""CPU experiment: does pairing two instances into one complex transform
(z = x_a 2^-ea + i x_b 2^-eb) change the reference's BiCGSTAB iteration
counts more than swapping pocketfft for scipy.fft does?

Matvec: the symbol S is shared by the instances, so IFFT(S FFT(pad z)) =
A x_a + i A x_b exactly.  Strang solve: the filters differ per instance
(kappa_bar), so the spectrum step uses the two-for-one split
Y_k = ((F_a+F_b)/2) Z_k + ((F_a-F_b)/2) conj(Z_{-k}).

Usage: python tools/pair_probe.py [n] [M] [pairs]
"""
import math
import sys
from pathlib import Path

import numpy as np
import scipy.fft as sfft
from scipy.special import gammaln

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import oracle as O  # noqa: E402
from paper_2002_11978_b200 import workloads as WL  # noqa: E402


def pow2_scale(v):
    m = float(np.max(np.abs(v)))
    if m == 0.0:
        return 1.0
    return math.ldexp(1.0, -math.frexp(m)[1])


def make_backend(kind, sym, n):
    fft, ifft = (sfft.fft, sfft.ifft) if kind == "scipy" else (np.fft.fft, np.fft.ifft)
    L = sym.size

    def mv(X, act):  # X [2,n] -> A X rows
        if kind in ("numpy", "scipy", "pair_pc"):
            Y = np.zeros_like(X)
            for i in range(2):
                if act[i]:
                    z = np.zeros(L, dtype=complex)
                    z[:n] = X[i]
                    Y[i] = ifft(sym * fft(z))[:n].real
            return Y
        sc = [pow2_scale(X[i]) if (act[i] and kind != "pair_noscale") else 1.0 for i in range(2)]
        z = np.zeros(L, dtype=complex)
        z[:n] = X[0] * sc[0] * act[0] + 1j * X[1] * sc[1] * act[1]
        y = ifft(sym * fft(z))[:n]
        return np.stack([y.real / sc[0], y.imag / sc[1]])

    def pc(X, totals, act):
        if kind in ("numpy", "scipy", "pair_mv"):
            Y = np.zeros_like(X)
            for i in range(2):
                if act[i]:
                    Y[i] = ifft(fft(X[i]) / totals[i]).real
            return Y
        sc = [pow2_scale(X[i]) if (act[i] and kind != "pair_noscale") else 1.0 for i in range(2)]
        z = X[0] * sc[0] * act[0] + 1j * X[1] * sc[1] * act[1]
        Z = fft(z)
        Fa = 1.0 / totals[0]
        Fb = 1.0 / totals[1]
        Fa = 0.5 * (Fa + np.roll(Fa[::-1], 1))
        Fb = 0.5 * (Fb + np.roll(Fb[::-1], 1))
        Zm = np.conj(np.roll(Z[::-1], 1))
        Y = 0.5 * (Fa + Fb) * Z + 0.5 * (Fa - Fb) * Zm
        y = ifft(Y)
        return np.stack([y.real / sc[0], y.imag / sc[1]])

    return mv, pc


def bicg2(mv, pc, shift, kap, totals, b, tol):
    """Two lock-stepped BiCGSTABs (krylov.py:88-153 control flow per row)."""
    n = b.shape[1]
    x = np.zeros_like(b)
    r = b.copy()
    r0 = b.copy()
    nb = np.linalg.norm(b, axis=1)
    its = np.zeros(2, dtype=int)
    done = nb == 0.0
    rho = np.ones(2); alpha = np.ones(2); omega = np.ones(2)
    v = np.zeros_like(b); p = np.zeros_like(b)
    it = 0
    while not done.all():
        it += 1
        act = ~done
        for i in range(2):
            if act[i]:
                rn = r0[i] @ r[i]
                if it == 1:
                    p[i] = r[i]
                else:
                    beta = (rn / rho[i]) * (alpha[i] / omega[i])
                    p[i] = r[i] + beta * (p[i] - omega[i] * v[i])
                bicg2.rn[i] = rn
        ph = pc(p, totals, act)
        v = np.where(act[:, None], shift * ph + kap * mv(ph, act), v)
        s = np.zeros_like(b)
        act2 = act.copy()
        for i in range(2):
            if act[i]:
                alpha[i] = bicg2.rn[i] / (r0[i] @ v[i])
                s[i] = r[i] - alpha[i] * v[i]
                if np.linalg.norm(s[i]) / nb[i] < tol:
                    x[i] += alpha[i] * ph[i]
                    its[i] = it
                    done[i] = True
                    act2[i] = False
        if not act2.any():
            break
        sh = pc(s, totals, act2)
        t = shift * sh + kap * mv(sh, act2)
        for i in range(2):
            if act2[i]:
                omega[i] = (t[i] @ s[i]) / (t[i] @ t[i])
                x[i] += alpha[i] * ph[i] + omega[i] * sh[i]
                r[i] = s[i] - omega[i] * t[i]
                rho[i] = bicg2.rn[i]
                if np.linalg.norm(r[i]) / nb[i] < tol:
                    its[i] = it
                    done[i] = True
    return x, its


bicg2.rn = np.zeros(2)


def march(kind, n, M, b0, gamma=0.5, alpha=1.5, tol=1e-12):
    N = n + 1
    r = (2 - gamma) / gamma
    t, tau = O.graded_mesh(M, r, 1.0)
    col, h, _ = O.ifl_column(alpha, 1 + alpha / 2, 1.0, N)
    _, sym = O.toeplitz_symbol(col)
    lam = O.strang_eigs(col)
    G = math.exp(gammaln(1 - gamma))
    s, w = O.soe_build(gamma, 1e-12, (1.0 / M) ** r, 1.0)
    x, kx, fx, u0 = WL.instance_fields(n, b0, 2)
    mv, pc = make_backend(kind, sym, n)
    W = [np.zeros((s.size, n)) for _ in range(2)]
    up = u0.copy()
    its = np.zeros((M, 2), dtype=int)
    for m in range(1, M + 1):
        amm = O.last_l1_weight(tau[m - 1], gamma)
        shift = amm / G
        kap = kx * WL.kappa_t(t[m])
        f = fx * WL.source_t(t[m])
        rhs = np.stack([f[i] + (amm * up[i] - O.soe_history_term(W[i], s, w, tau[m - 1])) / G
                        for i in range(2)])
        totals = [shift + float(kap[i].mean()) * lam for i in range(2)]
        u, its[m - 1] = bicg2(mv, pc, shift, kap, totals, rhs, tol)
        for i in range(2):
            O.soe_push(W[i], s, u[i] - up[i], tau[m - 1])
        up = u
    return up, its


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    pairs = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    kinds = sys.argv[4].split(",") if len(sys.argv) > 4 else ["scipy", "pair", "pair_noscale"]
    res = {k: [] for k in ["numpy"] + kinds}
    for p in range(pairs):
        for k in res:
            res[k].append(march(k, n, M, 2 * p))
    ref_u = np.concatenate([u for u, _ in res["numpy"]])
    ref_i = np.concatenate([i for _, i in res["numpy"]], axis=1)
    print(f"n={n} M={M} pairs={pairs} ref mean its {ref_i.mean():.3f}")
    for k in kinds:
        u = np.concatenate([u for u, _ in res[k]])
        i = np.concatenate([i for _, i in res[k]], axis=1)
        d = i - ref_i
        e = max(np.linalg.norm(u[j] - ref_u[j]) / np.linalg.norm(ref_u[j]) for j in range(len(u)))
        print(f"{k:13s} within1 {np.mean(np.abs(d) <= 1):.4f} mean {d.mean():+.4f} "
              f"exact {np.mean(d == 0):.3f} uM rel-l2 {e:.2e}")


if __name__ == "__main__":
    main()
