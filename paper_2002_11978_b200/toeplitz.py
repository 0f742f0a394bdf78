"""Toeplitz operator and Strang circulant preconditioner on the B200.

Mirror of tsfrac.toeplitz (toeplitz.py:21-136).  The symbol and the Strang
eigenvalues are host setup (one numpy FFT each, as in the reference, so
they are bit-identical to it); `toeplitz_matvec` and `precond_solve` run the
sm_100a FFT filter kernels through the C ABI (n <= 4096: one CTA per
instance, csrc/tsf_filters.cuh; larger powers of two: the four-step engine,
csrc/tsf_large.cuh).  Inputs may be numpy arrays (copied) or torch CUDA tensors [n] or
[B, n] (zero-copy, batched).
"""

from __future__ import annotations

import hashlib
import os
from collections import OrderedDict
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _arrays, _native


def embed_length(n: int) -> int:
    """Smallest power of two >= 2n-1 (toeplitz.py:39-41)."""
    L = 1
    while L < max(2 * n - 1, 1):
        L *= 2
    return L


def _even_embedding(col: np.ndarray, L: int) -> np.ndarray:
    n = col.size
    e = np.zeros(L)
    e[:n] = col
    if n > 1:
        e[L - n + 1:] = col[1:][::-1]
    return e


def _is_pow2(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


# Plan cache, least recently used first.  A plan keeps its Krylov workspaces
# (sized to the largest batch it ran) and cached graphs, so the cache is
# bounded: evicted plans are freed once no operator holds them.
_plans: "OrderedDict[tuple, _native.Plan]" = OrderedDict()
PLAN_CACHE_SIZE = int(os.environ.get("TSF_PLAN_CACHE", "8"))


def clear_plans() -> None:
    """Drop every cached plan (device memory is released with the last reference)."""
    _plans.clear()


def plan_for(first_col: np.ndarray, device: int = 0, lam: Optional[np.ndarray] = None,
             spectrum: Optional[np.ndarray] = None, private: bool = False) -> _native.Plan:
    """Cached device plan for a Toeplitz first column (symbol + Strang tables).

    private=True returns a fresh, uncached plan: its workspaces, solve
    graphs and instance counters are not shared, so marches holding private
    plans can run concurrently on different streams."""
    col = np.ascontiguousarray(first_col, dtype=np.float64)
    n = col.size
    L_ref = embed_length(n)
    L = max(L_ref, 32)
    pc_ok = _is_pow2(n) and n >= 16 and L == 2 * n
    if lam is None and pc_ok:
        lam = np.fft.fft(strang_first_column(col)).real
    if not pc_ok:
        lam = None
    key = (n, device, hashlib.sha1(col.tobytes()).hexdigest(),
           None if lam is None else hashlib.sha1(np.ascontiguousarray(lam).tobytes()).hexdigest())
    pl = None if private else _plans.get(key)
    if pl is not None:
        _plans.move_to_end(key)
    if pl is None:
        if spectrum is not None and L == L_ref:
            sym = np.ascontiguousarray(np.real(spectrum))
        else:
            sym = np.fft.fft(_even_embedding(col, L)).real
        pl = _native.Plan(n, L, sym, lam, device)
        if not private:
            _plans[key] = pl
            while len(_plans) > max(1, PLAN_CACHE_SIZE):
                _plans.popitem(last=False)
    return pl


@dataclass(frozen=True)
class ToeplitzOperator:
    """Matrix-free symmetric Toeplitz operator (toeplitz.py:21-31)."""

    n: int
    first_col: np.ndarray
    embed_len: int
    spectrum_embed: np.ndarray
    device: int = 0
    _plan: Optional[_native.Plan] = field(default=None, compare=False, repr=False)

    @property
    def plan(self) -> _native.Plan:
        if self._plan is None:   # built once per operator (hashing + host setup)
            object.__setattr__(self, "_plan",
                               plan_for(self.first_col, self.device, spectrum=self.spectrum_embed))
        return self._plan

    def matvec(self, v):
        return toeplitz_matvec(self, v)


def build_toeplitz(first_col, device: int = 0) -> ToeplitzOperator:
    """toeplitz.py:34-48: pow2 embedding L >= 2n-1 and its spectrum (host setup)."""
    col = np.asarray(first_col, dtype=float)
    n = col.size
    if n < 1:
        raise ValueError("first column must be nonempty")
    L = embed_length(n)
    spec = np.fft.fft(_even_embedding(col, L))
    return ToeplitzOperator(n=n, first_col=col, embed_len=L, spectrum_embed=spec,
                            device=device)


def _batched(v, n: int, device: int):
    t, as_np = _arrays.to_device(v, device)
    if t.shape[-1] != n or t.dim() not in (1, 2):
        raise ValueError(f"vector has shape {tuple(t.shape)}, operator order is {n}")
    return t, as_np


def toeplitz_matvec(op: ToeplitzOperator, v, kappa=None, shift: float = 0.0):
    """A v via the circulant embedding on the device (toeplitz.py:51-63).

    With `kappa` given returns shift*v + kappa*(A v) (scheme.py:129-130).
    """
    torch = _native.torch_mod()
    x, as_np = _batched(v, op.n, op.device)
    B = 1 if x.dim() == 1 else x.shape[0]
    y = torch.empty_like(x)
    k = None
    if kappa is not None:
        k, _ = _batched(kappa, op.n, op.device)
        if k.shape != x.shape:
            k = k.expand_as(x).contiguous()
    _native.check(_native.load().tsf_toeplitz_matvec(
        op.plan.handle, B, x.data_ptr(), y.data_ptr(), _native.ptr(k), float(shift),
        _native.stream_ptr(device=x.device)))
    return _arrays.back(y, as_np)


def strang_first_column(first_col) -> np.ndarray:
    """c_S = [a_1..a_{floor((N+1)/2)}, a_{floor(N/2)}..a_2], N = n+1 (toeplitz.py:66-80)."""
    col = np.asarray(first_col, dtype=float)
    n = col.size
    if n < 2:
        raise ValueError(f"need n >= 2, got {n}")
    N = n + 1
    return np.concatenate([col[: (N + 1) // 2], col[1: N // 2][::-1]])


class PreconditionerError(RuntimeError):
    """Circulant preconditioner not positive definite (toeplitz.py:83-84)."""


@dataclass(frozen=True)
class CirculantPreconditioner:
    """P = shift I + kappa_bar s(A) (toeplitz.py:87-98)."""

    n: int
    shift: float
    kappa_bar: float
    lam: np.ndarray
    total_eigs: np.ndarray
    first_col: Optional[np.ndarray] = field(default=None, compare=False, repr=False)
    device: int = 0

    _plan: Optional[_native.Plan] = field(default=None, compare=False, repr=False)

    def solve(self, v):
        return precond_solve(self, v)

    @property
    def strang_native(self) -> bool:
        """Power-of-two n >= 16: the plan carries the Strang tables and the
        fused level-solve kernels apply P^{-1} themselves."""
        return _is_pow2(self.n) and self.n >= 16

    @property
    def plan(self) -> _native.Plan:
        if self._plan is None:   # built once per preconditioner
            if not self.strang_native:
                pl = self._circulant_plan()
            elif self.first_col is not None:
                pl = plan_for(self.first_col, self.device, lam=self.lam)
            else:
                # bare spectrum: a plan whose "lam" is the given eigenvalue array
                pl = plan_for(np.zeros(self.n), self.device, lam=self.lam)
            object.__setattr__(self, "_plan", pl)
        return self._plan

    def _circulant_plan(self) -> _native.Plan:
        """Any n: P^{-1} = circ(c), c = IFFT_n(1/total) real and even, and a
        symmetric circulant is the symmetric Toeplitz matrix with first column
        c — applied by the same device Toeplitz engine through its pow2
        embedding (in exact arithmetic identical to the reference's
        Re IFFT(FFT(v)/total), toeplitz.py:131-136)."""
        c = np.fft.ifft(1.0 / self.total_eigs).real
        c = 0.5 * (c + np.roll(c[::-1], 1))          # c_j = c_{n-j} exactly
        L = max(embed_length(self.n), 32)
        sym = np.fft.fft(_even_embedding(c, L)).real
        return _native.Plan(self.n, L, sym, None, self.device)


def build_preconditioner(d, shift: float, kappa_bar: float, device: int = 0
                         ) -> CirculantPreconditioner:
    """Strang preconditioner with the reference's checks (toeplitz.py:101-128)."""
    if shift <= 0.0:
        raise ValueError(f"shift must be > 0, got {shift}")
    if kappa_bar <= 0.0:
        raise ValueError(f"kappa_bar must be > 0, got {kappa_bar}")
    col = d.first_col if hasattr(d, "first_col") else np.asarray(d, dtype=float)
    spec = np.fft.fft(strang_first_column(col))
    lam = spec.real
    resid = np.abs(spec.imag).max()
    if resid > 1e-10 * max(np.abs(lam).max(), 1e-300):
        raise PreconditionerError(
            f"Strang spectrum is not numerically real (residual {resid:g})")
    total = shift + kappa_bar * lam
    if np.any(total <= 0.0):
        raise PreconditionerError("preconditioner has a non-positive eigenvalue")
    return CirculantPreconditioner(n=lam.size, shift=float(shift), kappa_bar=float(kappa_bar),
                                   lam=lam, total_eigs=total,
                                   first_col=np.asarray(col, dtype=float), device=device)


def precond_solve(p: CirculantPreconditioner, v):
    """P^{-1} v = IFFT(FFT(v)/total) on the device (toeplitz.py:131-136)."""
    torch = _native.torch_mod()
    x, as_np = _batched(v, p.n, p.device)
    B = 1 if x.dim() == 1 else x.shape[0]
    z = torch.empty_like(x)
    if not p.strang_native:
        # circ(c) applied as a symmetric Toeplitz product (_circulant_plan)
        _native.check(_native.load().tsf_toeplitz_matvec(
            p.plan.handle, B, x.data_ptr(), z.data_ptr(), None, 0.0,
            _native.stream_ptr(device=x.device)))
        return _arrays.back(z, as_np)
    _native.check(_native.load().tsf_precond_solve(
        p.plan.handle, B, x.data_ptr(), z.data_ptr(), float(p.shift), float(p.kappa_bar), None,
        _native.stream_ptr(device=x.device)))
    return _arrays.back(z, as_np)
