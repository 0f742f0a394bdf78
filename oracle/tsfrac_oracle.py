"""CPU oracle: a plain-numpy restatement of the reference FIDS per-step path.

TEST INFRASTRUCTURE ONLY.  The product package never imports this module;
tests, `__graft_entry__.smoke()` and bench.py's CPU arms do.

Every function cites the reference file:line it restates (paths relative to
`/root/reference/pkg/src/tsfrac/`).  The arithmetic follows the reference
operation by operation (same numpy FFT engine, same expression order) so
that, with OPENBLAS_NUM_THREADS=1, the oracle reproduces the reference's
outputs bit-for-bit on the golden vectors in `tests/golden/`; the pin is
`tests/test_oracle_golden.py`.

Third-party arithmetic the reference relies on (not vendored, lower-bound
pins only in `pkg/pyproject.toml:10-13`): numpy pocketfft (np.fft), OpenBLAS
(dot / GEMV), scipy.special.gammaln.  Versions used to pin: numpy 2.3.5,
scipy 1.18.1, OpenBLAS 0.3.30.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
from scipy.special import gammaln

__all__ = [
    "graded_mesh", "l1_weight_row", "last_l1_weight", "ifl_column",
    "normalization_constant", "soe_build", "SoeError", "toeplitz_symbol",
    "toeplitz_apply", "strang_column", "strang_eigs", "precond_apply",
    "bicgstab", "cg", "KrylovOutcome", "soe_push", "soe_history_term",
    "fids_march", "FidsRecord", "fids_step", "embed_length", "dids_march",
]


# --------------------------------------------------------------------------
# mesh.py
# --------------------------------------------------------------------------

def graded_mesh(M: int, r: float, T: float):
    """t_m = (m/M)^r T and tau = diff(t).  mesh.py:37-50."""
    if M < 1 or r < 1.0 or T <= 0.0:
        raise ValueError("graded_mesh needs M >= 1, r >= 1, T > 0")
    t = (np.arange(M + 1, dtype=float) / M) ** r * T
    return t, np.diff(t)


def last_l1_weight(tau_m: float, gamma: float) -> float:
    """a_m^{(m)} = tau_m^{-gamma}/(1-gamma).  scheme.py:101-102, mesh.py:79."""
    return tau_m ** (-gamma) / (1.0 - gamma)


def l1_weight_row(t: np.ndarray, tau: np.ndarray, gamma: float, m: int):
    """L1 weights a_1..a_m at level m (expm1/log1p form).  mesh.py:53-80."""
    tm = t[m]
    g1 = 1.0 - gamma
    a = np.empty(m)
    if m > 1:
        left = tm - t[:m - 1]
        right = tm - t[1:m]
        a[:-1] = (np.exp(g1 * np.log(right))
                  * np.expm1(g1 * np.log1p((left - right) / right))
                  / (tau[:m - 1] * g1))
    a[-1] = tau[m - 1] ** (-gamma) / g1
    return a


# --------------------------------------------------------------------------
# ifl.py
# --------------------------------------------------------------------------

def normalization_constant(alpha: float) -> float:
    """c_{1,alpha}.  ifl.py:48-57."""
    return (2.0 ** (alpha - 1.0) * alpha
            * math.exp(gammaln((alpha + 1.0) / 2.0) - gammaln(1.0 - alpha / 2.0))
            / math.sqrt(math.pi))


def _compensated(values) -> float:
    """Kahan summation in the reference's order.  ifl.py:60-70."""
    acc = 0.0
    comp = 0.0
    for v in values:
        y = v - comp
        nxt = acc + y
        comp = (nxt - acc) - y
        acc = nxt
    return acc


def ifl_column(alpha: float, mu: float, l: float, N: int):
    """First column of the IFL Toeplitz matrix A (order N-1).  ifl.py:73-115.

    Returns (col, h, scale).
    """
    if not (0.0 < alpha < 2.0 and alpha < mu <= 2.0 and N >= 3 and l > 0.0):
        raise ValueError("ifl_column: bad (alpha, mu, l, N)")
    nu = mu - alpha
    kmu = 2 if mu == 2.0 else 1
    h = 2.0 * l / N
    scale = normalization_constant(alpha) / (nu * h ** alpha)
    ell = np.arange(2.0, N)
    series = ((ell + 1.0) ** nu - (ell - 1.0) ** nu) / ell ** mu
    diag = (_compensated(series)
            + (N ** nu - (N - 1.0) ** nu) / N ** mu
            + (2.0 ** nu + kmu - 1.0)
            + 2.0 * nu / (alpha * N ** alpha))
    col = np.empty(N - 1)
    col[0] = scale * diag
    col[1] = -scale * (2.0 ** nu + kmu - 1.0) / 2.0
    k = np.arange(2.0, N - 1)
    col[2:] = -scale * ((k + 1.0) ** nu - (k - 1.0) ** nu) / (2.0 * k ** mu)
    return col, h, scale


# --------------------------------------------------------------------------
# soe.py
# --------------------------------------------------------------------------

class SoeError(RuntimeError):
    """Mirror of SoeConstructionError.  soe.py:48-49."""


def _lattice_h(gamma: float, target: float) -> float:
    """Fixed-point solve for the log-lattice step.  soe.py:90-105."""
    lg = gammaln(gamma)
    y = 20.0
    for _ in range(60):
        y = (2.0 / math.pi) * (math.log(8.0 * math.sqrt(2.0 * math.pi))
                               + (gamma - 0.5) * math.log(max(y, 1.0))
                               - lg - math.log(target))
    return 2.0 * math.pi / y


def _lattice(gamma, eps, delta, T, h):
    """Collapsed-left-tail midpoint lattice.  soe.py:108-133."""
    lg = gammaln(gamma)
    inv_g = math.exp(-lg)
    a = (eps * gamma * math.exp(lg) / (4.0 * T * T)) ** (1.0 / (gamma + 2.0))
    j0 = math.floor(math.log(a) / h - 0.5)
    u0 = (j0 + 0.5) * h
    m0 = h * inv_g * math.exp(gamma * u0) / (1.0 - math.exp(-gamma * h))
    m1 = (h * inv_g * math.exp((gamma + 1.0) * u0)
          / (1.0 - math.exp(-(gamma + 1.0) * h)))
    s_list, w_list = [m1 / m0], [m0]
    j = j0 + 1
    while True:
        u = (j + 0.5) * h
        s = math.exp(u)
        w = h * math.exp(gamma * u) * inv_g
        s_list.append(s)
        w_list.append(w)
        if s * delta > gamma + 1.0 and w * math.exp(-min(s * delta, 700.0)) < eps / 32.0:
            break
        j += 1
        if len(s_list) > 100_000:
            raise SoeError("right tail of the lattice does not terminate")
    return np.array(s_list), np.array(w_list)


def _soe_ok(gamma, s, w, eps, delta, T, n_grid=4096) -> bool:
    """A-posteriori check on a log grid.  soe.py:136-142."""
    t = np.logspace(math.log10(delta), math.log10(T), n_grid)
    ker = t ** (-gamma)
    err = np.abs(ker - np.exp(-np.outer(t, s)) @ w)
    return bool(np.all(err <= np.maximum(eps, 4.0 * np.finfo(float).eps * ker)))


def soe_build(gamma: float, eps: float, delta: float, T: float, cap: int = 256):
    """SOE nodes/weights for t^{-gamma} on [delta, T].  soe.py:145-184."""
    if not 0.0 < gamma < 1.0:
        raise ValueError("gamma must lie in (0, 1)")
    if eps <= 0.0:
        raise ValueError("epsilon must be > 0")
    if not 0.0 < delta < T:
        raise SoeError("need 0 < delta < T")
    h = _lattice_h(gamma, eps * delta ** gamma / 4.0)
    for _ in range(6):
        s, w = _lattice(gamma, eps, delta, T, h)
        if s.size > cap:
            raise SoeError(f"needs {s.size} exponentials, cap is {cap}")
        if _soe_ok(gamma, s, w, eps, delta, T):
            return s, w
        h *= 0.85
    raise SoeError("validation failed")


def soe_push(W: np.ndarray, s: np.ndarray, du: np.ndarray, tau: float) -> None:
    """In-place W_j <- e^{-s_j tau} W_j + (-expm1(-s_j tau)/s_j) du/tau.

    soe.py:209-225 (same two-statement order: scale, then add the outer).
    """
    W *= np.exp(-s * tau)[:, None]
    W += np.outer(-np.expm1(-s * tau) / s, du / tau)


def soe_history_term(W: np.ndarray, s: np.ndarray, w: np.ndarray, tau: float):
    """H = (w * e^{-s tau}) @ W.  scheme.py:281-282 (== soe.py:245)."""
    return (w * np.exp(-s * tau)) @ W


# --------------------------------------------------------------------------
# toeplitz.py
# --------------------------------------------------------------------------

def embed_length(n: int) -> int:
    """Smallest power of two >= 2n-1.  toeplitz.py:39-41."""
    L = 1
    while L < max(2 * n - 1, 1):
        L *= 2
    return L


def toeplitz_symbol(col: np.ndarray):
    """(L, FFT_L of the even circulant embedding).  toeplitz.py:34-48."""
    col = np.asarray(col, dtype=float)
    n = col.size
    L = embed_length(n)
    e = np.zeros(L)
    e[:n] = col
    if n > 1:
        e[L - n + 1:] = col[1:][::-1]
    return L, np.fft.fft(e)


def toeplitz_apply(symbol: np.ndarray, v: np.ndarray) -> np.ndarray:
    """A v = Re(IFFT(S * FFT(pad v)))[:n].  toeplitz.py:51-63."""
    n = v.size
    z = np.zeros(symbol.size, dtype=complex)
    z[:n] = v
    return np.fft.ifft(symbol * np.fft.fft(z))[:n].real


def strang_column(col: np.ndarray) -> np.ndarray:
    """Strang circulant first column.  toeplitz.py:66-80."""
    col = np.asarray(col, dtype=float)
    n = col.size
    if n < 2:
        raise ValueError("need n >= 2")
    N = n + 1
    return np.concatenate([col[:(N + 1) // 2], col[1:N // 2][::-1]])


def strang_eigs(col: np.ndarray) -> np.ndarray:
    """lambda = Re FFT_n(c_S).  toeplitz.py:114-116."""
    return np.fft.fft(strang_column(col)).real


def precond_apply(total: np.ndarray, v: np.ndarray) -> np.ndarray:
    """P^{-1} v = Re IFFT(FFT(v)/total).  toeplitz.py:131-136."""
    return np.fft.ifft(np.fft.fft(v) / total).real


# --------------------------------------------------------------------------
# krylov.py
# --------------------------------------------------------------------------

@dataclass
class KrylovOutcome:
    iterations: int
    relres: float
    converged: bool
    breakdown: Optional[str] = None


def bicgstab(apply: Callable, psolve: Optional[Callable], b: np.ndarray,
             tol: float = 1e-10, max_iters: Optional[int] = None):
    """Right-preconditioned BiCGSTAB, x0 = 0.  krylov.py:88-153.

    Control flow (iteration counting, early ||s|| exit, exact-zero breakdown
    tests) follows the reference statement by statement.
    """
    b = np.asarray(b, dtype=float)
    n = b.size
    max_iters = 10 * n if max_iters is None else max_iters
    ps = (lambda q: q) if psolve is None else psolve
    x = np.zeros(n)
    r = b.copy()
    r0 = b.copy()
    nb = float(np.linalg.norm(r0))
    if nb == 0.0:
        return x, KrylovOutcome(0, 0.0, True)
    rho = alpha = omega = 1.0
    v = np.zeros(n)
    p = np.zeros(n)
    for it in range(1, max_iters + 1):
        rho_new = float(r0 @ r)
        if rho_new == 0.0:
            return x, KrylovOutcome(it, float(np.linalg.norm(r)) / nb, False, "rho vanished")
        if it == 1:
            p[:] = r
        else:
            beta = (rho_new / rho) * (alpha / omega)
            p = r + beta * (p - omega * v)
        ph = ps(p)
        v = apply(ph)
        den = float(r0 @ v)
        if den == 0.0:
            return x, KrylovOutcome(it, float(np.linalg.norm(r)) / nb, False, "r0.v vanished")
        alpha = rho_new / den
        s = r - alpha * v
        if float(np.linalg.norm(s)) / nb < tol:
            x += alpha * ph
            return x, KrylovOutcome(it, float(np.linalg.norm(s)) / nb, True)
        sh = ps(s)
        t = apply(sh)
        tt = float(t @ t)
        if tt == 0.0:
            return x, KrylovOutcome(it, float(np.linalg.norm(s)) / nb, False,
                                    "omega denominator vanished")
        omega = float(t @ s) / tt
        x += alpha * ph + omega * sh
        r = s - omega * t
        rho = rho_new
        rel = float(np.linalg.norm(r)) / nb
        if rel < tol:
            return x, KrylovOutcome(it, rel, True)
        if omega == 0.0:
            return x, KrylovOutcome(it, rel, False, "omega vanished")
    return x, KrylovOutcome(max_iters, float(np.linalg.norm(r)) / nb, False)


def cg(apply: Callable, psolve: Optional[Callable], b: np.ndarray,
       tol: float = 1e-10, max_iters: Optional[int] = None):
    """Preconditioned CG, x0 = 0.  krylov.py:43-85."""
    b = np.asarray(b, dtype=float)
    n = b.size
    max_iters = 10 * n if max_iters is None else max_iters
    ps = (lambda q: q) if psolve is None else psolve
    x = np.zeros(n)
    r = b.copy()
    nb = float(np.linalg.norm(r))
    if nb == 0.0:
        return x, KrylovOutcome(0, 0.0, True)
    z = ps(r)
    p = z.copy()
    rz = float(r @ z)
    for it in range(1, max_iters + 1):
        q = apply(p)
        curv = float(p @ q)
        if curv <= 0.0:
            return x, KrylovOutcome(it, float(np.linalg.norm(r)) / nb, False,
                                    "non-positive curvature")
        a = rz / curv
        x += a * p
        r -= a * q
        rel = float(np.linalg.norm(r)) / nb
        if rel < tol:
            return x, KrylovOutcome(it, rel, True)
        z = ps(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, KrylovOutcome(max_iters, float(np.linalg.norm(r)) / nb, False)


# --------------------------------------------------------------------------
# scheme.py  (FIDS, pkrylov / krylov branches)
# --------------------------------------------------------------------------

def fids_step(u_prev, W, s, w, tau_m, gamma, g1mg, kappa, f, symbol, lam,
              tol, max_iters=None, precondition=True, use_cg=False):
    """One FIDS level (scheme.py:277-291): RHS, Krylov solve, SOE push.

    Mutates W.  Returns (u, rhs, KrylovOutcome).
    """
    a_mm = last_l1_weight(tau_m, gamma)
    H = soe_history_term(W, s, w, tau_m)
    rhs = f + (a_mm * u_prev - H) / g1mg
    shift = a_mm / g1mg

    def apply(q):
        return shift * q + kappa * toeplitz_apply(symbol, q)

    psolve = None
    if precondition:
        total = shift + float(kappa.mean()) * lam
        if np.any(total <= 0.0):
            raise RuntimeError("preconditioner has a non-positive eigenvalue")
        psolve = lambda q: precond_apply(total, q)  # noqa: E731
    solver = cg if use_cg else bicgstab
    u, out = solver(apply, psolve, rhs, tol=tol, max_iters=max_iters)
    if not out.converged:
        raise RuntimeError(f"Krylov solve did not converge: {out}")
    soe_push(W, s, u - u_prev, tau_m)
    return u, rhs, out


@dataclass
class FidsRecord:
    hist: np.ndarray          # (M+1, n) or (n,) when keep_history is False
    iterations: np.ndarray    # (M,)
    relres: np.ndarray        # (M,)
    nodes: np.ndarray
    weights: np.ndarray


def fids_march(gamma, alpha, l, T, M, r, N, kappa_fn, source_fn, initial_fn,
               epsilon=1e-10, mu=None, tol=1e-10, max_iters=None,
               precondition=True, use_cg=False, keep_history=True):
    """run_fids restated (scheme.py:236-303), Krylov branches only.

    `N` is the reference's interval count (n = N-1 unknowns).
    """
    t, tau = graded_mesh(M, r, T)
    mu = 1.0 + alpha / 2.0 if mu is None else mu
    col, h, _ = ifl_column(alpha, mu, l, N)
    x = -l + h * np.arange(1, N)
    _, symbol = toeplitz_symbol(col)
    lam = strang_eigs(col)
    g1mg = math.exp(gammaln(1.0 - gamma))
    s, w = soe_build(gamma, epsilon, (1.0 / M) ** r * T, T)
    n = N - 1
    u_prev = np.asarray(initial_fn(x), dtype=float)
    W = np.zeros((s.size, n))
    hist = np.empty((M + 1, n)) if keep_history else None
    if keep_history:
        hist[0] = u_prev
    its = np.zeros(M, dtype=np.int64)
    rel = np.zeros(M)
    for m in range(1, M + 1):
        tm = t[m]
        kappa = np.broadcast_to(np.asarray(kappa_fn(x, tm), dtype=float), x.shape).copy()
        if np.any(kappa <= 0.0):
            raise ValueError(f"kappa must be positive on the grid at t={tm}")
        f = np.asarray(source_fn(x, tm), dtype=float)
        u, _, out = fids_step(u_prev, W, s, w, tau[m - 1], gamma, g1mg, kappa, f,
                              symbol, lam, tol, max_iters, precondition, use_cg)
        its[m - 1] = out.iterations
        rel[m - 1] = out.relres
        u_prev = u
        if keep_history:
            hist[m] = u
    return FidsRecord(hist if keep_history else u_prev, its, rel, s, w)


# --------------------------------------------------------------------------
# scheme.py  (DIDS, Krylov branches)
# --------------------------------------------------------------------------

def dids_march(gamma, alpha, l, T, M, r, N, kappa_fn, source_fn, initial_fn,
               mu=None, tol=1e-10, max_iters=None, precondition=True, use_cg=False):
    """run_dids restated (scheme.py:184-233), Krylov branches only.

    History term at level m (scheme.py:213-216):
        rhs = f + (a[0]/G) u^0 ;  rhs += (diff(a) @ hist[1:m]) / G   (m > 1)
    with a = l1_weights(mesh, gamma, m).a (mesh.py:53-80); the level system
    is the one run_fids solves, with shift = a[-1]/G (scheme.py:218-219).
    Returns a FidsRecord (nodes/weights empty: DIDS has no SOE).
    """
    t, tau = graded_mesh(M, r, T)
    mu = 1.0 + alpha / 2.0 if mu is None else mu
    col, h, _ = ifl_column(alpha, mu, l, N)
    x = -l + h * np.arange(1, N)
    _, symbol = toeplitz_symbol(col)
    lam = strang_eigs(col)
    g1mg = math.exp(gammaln(1.0 - gamma))
    n = N - 1
    hist = np.empty((M + 1, n))
    hist[0] = initial_fn(x)
    its = np.zeros(M, dtype=np.int64)
    rel = np.zeros(M)
    for m in range(1, M + 1):
        a = l1_weight_row(t, tau, gamma, m)
        tm = t[m]
        kappa = np.broadcast_to(np.asarray(kappa_fn(x, tm), dtype=float), x.shape).copy()
        if np.any(kappa <= 0.0):
            raise ValueError(f"kappa must be positive on the grid at t={tm}")
        rhs = np.asarray(source_fn(x, tm), dtype=float) + (a[0] / g1mg) * hist[0]
        if m > 1:
            rhs += (np.diff(a) @ hist[1:m]) / g1mg
        shift = a[-1] / g1mg

        def apply(q, shift=shift, kappa=kappa):
            return shift * q + kappa * toeplitz_apply(symbol, q)

        psolve = None
        if precondition:
            total = shift + float(kappa.mean()) * lam
            if np.any(total <= 0.0):
                raise RuntimeError("preconditioner has a non-positive eigenvalue")
            psolve = lambda q, total=total: precond_apply(total, q)  # noqa: E731
        solver = cg if use_cg else bicgstab
        u, out = solver(apply, psolve, rhs, tol=tol, max_iters=max_iters)
        if not out.converged:
            raise RuntimeError(f"Krylov solve did not converge: {out}")
        its[m - 1] = out.iterations
        rel[m - 1] = out.relres
        hist[m] = u
    return FidsRecord(hist, its, rel, np.empty(0), np.empty(0))
