"""CPU experiment: iteration-count parity of a HALF-LENGTH transform engine.

Every transform of a level solve works on real data (or on the odd bins of a
real sequence), so each can run as ONE complex transform of half the length:

* Strang solve, forward: z_j = p_{2j} + i p_{2j+1}, FFT_{n/2}, split step;
  inverse: pre-step, IFFT_{n/2}, outputs (q_{2j}, q_{2j+1}).
* Toeplitz product, even bins: the stored Strang spectrum (as the device
  engine does), inverse as above.
* odd bins: X_{4m+1} = FFT_{n/2}[W_L^j (x_j - i x_{j+n/2})]_m exactly (the
  bins 4m+3 are the conjugate mirrors), inverse
  g = IFFT_{n/2}(Y_{4m+1}); y_j = Re(conj(w_j) g_j), y_{j+n/2} = -Im(conj(w_j) g_j).

Kinds: numpy (the reference's arithmetic), eng (the device engine's present
structure: even/odd channels of length-n complex transforms, Strang spectrum
reuse), half (the above).  The sub-transform backend is numpy pocketfft or
`ld` (long-double scipy.fft rounded once), which isolates the structure.

    python tools/half_probe.py [n] [M] [instances] [kinds] [backend]
"""
import math
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np
import scipy.fft as sfft
from scipy.special import gammaln

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import oracle as O  # noqa: E402
from paper_2002_11978_b200 import workloads as WL  # noqa: E402


def _subfft(backend):
    if backend == "ld":
        f = lambda z: sfft.fft(z.astype(np.clongdouble)).astype(complex)  # noqa: E731
        g = lambda z: sfft.ifft(z.astype(np.clongdouble)).astype(complex)  # noqa: E731
        return f, g
    return np.fft.fft, np.fft.ifft


def _twid(L, cnt):
    j = np.arange(cnt, dtype=np.longdouble)
    a = -2 * np.pi * j / np.longdouble(L)
    return (np.cos(a) + 1j * np.sin(a)).astype(complex)


class Engine:
    def __init__(self, kind, backend, sym, n):
        self.kind, self.n = kind, n
        self.fft, self.ifft = _subfft(backend)
        self.sym = sym.real.copy()
        L = sym.size
        assert L == 2 * n
        self.L = L
        self.wL = _twid(L, n)           # W_L^j, j < n
        self.wn = _twid(n, n // 2 + 1)  # W_n^k, k <= n/2
        self.last = None
        self.Q = None

    # ---- Strang solve ----
    def pc(self, p, total):
        n = self.n
        F = 1.0 / total
        F = 0.5 * (F + np.roll(F[::-1], 1))
        if self.kind == "numpy":
            return np.fft.ifft(np.fft.fft(p) / total).real
        if self.kind == "eng":
            Q = self.fft(p.astype(complex)) * F
            q = self.ifft(Q).real
            self.Q = 0.5 * (Q + np.conj(np.roll(Q[::-1], 1)))  # Herm part = FFT(q)
            self.last = q
            return q
        # half: packed forward
        h = n // 2
        z = p[0::2] + 1j * p[1::2]
        Z = self.fft(z)
        Zx = np.concatenate([Z, Z[:1]])           # Z_{h} = Z_0
        Zm = np.conj(Zx[::-1])                    # conj Z_{h-k}, k = 0..h
        E = 0.5 * (Zx + Zm)
        Od = -0.5j * (Zx - Zm)
        P = E + self.wn * Od                      # k = 0..h
        Q = P * F[:h + 1]
        Q[0] = Q[0].real
        Q[h] = Q[h].real
        self.Q = Q
        q = self._packed_inverse(Q)
        self.last = q
        return q

    def _packed_inverse(self, Q):
        """real q (length n) from the half spectrum Q_0..Q_{n/2}."""
        n = self.n
        h = n // 2
        Qm = np.conj(Q[::-1])                     # conj Q_{h-k}
        Ep = Q + Qm
        Op = np.conj(self.wn) * (Q - Qm)
        Zp = 0.5 * (Ep + 1j * Op)[:h]
        z = self.ifft(Zp)
        q = np.empty(n)
        q[0::2] = z.real
        q[1::2] = z.imag
        return q

    # ---- Toeplitz product ----
    def mv(self, x):
        n, L = self.n, self.L
        if self.kind == "numpy":
            z = np.zeros(L, dtype=complex)
            z[:n] = x
            return np.fft.ifft(self.sym * np.fft.fft(z))[:n].real
        reuse = self.last is not None and x is self.last
        if self.kind == "eng":
            if reuse:
                Xe = self.Q
            else:
                Xe = self.fft(x.astype(complex))
            ye = self.ifft(self.sym[0::2] * Xe)
            Xo = self.fft(x * self.wL)
            yo = self.ifft(self.sym[1::2] * Xo)
            return 0.5 * (ye.real + (np.conj(self.wL) * yo).real)
        h = n // 2
        if reuse:
            Qe = self.Q
        else:
            Qe = self.fft(x.astype(complex))[:h + 1]
        ye = self._packed_inverse(Qe * self.sym[0:n + 1:2])
        z = self.wL[:h] * (x[:h] - 1j * x[h:])
        X41 = self.fft(z)                          # bins 4m+1, m < h
        g = self.ifft(X41 * self.sym[1::4])        # (1/h) sum
        c = np.conj(self.wL[:h]) * g
        yo = np.concatenate([c.real, -c.imag])     # = (1/h) Re sum_m ... ; want (2/L)*h*...
        # y = (1/L)[n ye + 2 h yo_unnorm/h...]: ye carries 1/n, g carries 1/h
        return 0.5 * ye + 0.5 * yo


def march(args):
    kind, backend, n, M, b0, gamma, alpha, tol = args
    N = n + 1
    r = (2 - gamma) / gamma
    t, tau = O.graded_mesh(M, r, 1.0)
    col, h, _ = O.ifl_column(alpha, 1 + alpha / 2, 1.0, N)
    _, sym = O.toeplitz_symbol(col)
    lam = O.strang_eigs(col)
    G = math.exp(gammaln(1 - gamma))
    s, w = O.soe_build(gamma, 1e-12, (1.0 / M) ** r, 1.0)
    x, kx, fx, u0 = WL.instance_fields(n, b0, 1)
    kx, fx, up = kx[0], fx[0], u0[0].copy()
    eng = Engine(kind, backend, sym, n)
    W = np.zeros((s.size, n))
    its = np.zeros(M, dtype=int)
    for m in range(1, M + 1):
        amm = O.last_l1_weight(tau[m - 1], gamma)
        shift = amm / G
        kap = kx * WL.kappa_t(t[m])
        f = fx * WL.source_t(t[m])
        rhs = f + (amm * up - O.soe_history_term(W, s, w, tau[m - 1])) / G
        total = shift + float(kap.mean()) * lam
        u, out = O.bicgstab(lambda q: shift * q + kap * eng.mv(q), lambda q: eng.pc(q, total),
                            rhs, tol=tol)
        its[m - 1] = out.iterations
        O.soe_push(W, s, u - up, tau[m - 1])
        up = u
    return up, its


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    cnt = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    kinds = sys.argv[4].split(",") if len(sys.argv) > 4 else ["eng", "half"]
    backend = sys.argv[5] if len(sys.argv) > 5 else "numpy"
    jobs = [(k, backend if k != "numpy" else "numpy", n, M, b, 0.5, 1.5, 1e-12)
            for k in ["numpy"] + kinds for b in range(cnt)]
    with ProcessPoolExecutor(max_workers=8) as ex:
        res = list(ex.map(march, jobs))
    by = {}
    for (k, *_), r in zip(jobs, res):
        by.setdefault(k, []).append(r)
    ref_i = np.stack([i for _, i in by["numpy"]])
    ref_u = np.stack([u for u, _ in by["numpy"]])
    print(f"n={n} M={M} instances={cnt} backend={backend} ref mean its {ref_i.mean():.3f}")
    for k in kinds:
        i = np.stack([i for _, i in by[k]])
        u = np.stack([u for u, _ in by[k]])
        d = i - ref_i
        e = max(np.linalg.norm(u[j] - ref_u[j]) / np.linalg.norm(ref_u[j]) for j in range(cnt))
        print(f"{k:8s} within1 {np.mean(np.abs(d) <= 1):.4f} mean {d.mean():+.4f} "
              f"exact {np.mean(d == 0):.3f} max|d| {np.abs(d).max()} uM rel-l2 {e:.2e}")


if __name__ == "__main__":
    main()
