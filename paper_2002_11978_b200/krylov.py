"""Krylov level solvers on the B200 (mirror of tsfrac.krylov, krylov.py:19-171).

`solve_bicgstab` / `solve_cg` on a `LevelOperator` (the structured level
system shift*I + diag(kappa) A of scheme.py:129-130) run the whole solve in
one sm_100a kernel per instance (csrc/tsf_kernels.cuh, k_krylov_solve):
the FFT matvec, the Strang preconditioner, the dots/norms and the scalar
control flow (iteration counting, early ||s|| exit, exact-zero breakdown
tests) all stay on the device.  Batched right-hand sides [B, n] solve B
independent systems at once.

For an arbitrary `MatrixFreeOperator` whose `apply` works on torch CUDA
tensors, a generic device loop restates the same algorithm with torch
vector ops (not a hot path; used for the reference's dense-operator tests).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Union

import numpy as np

from . import _arrays, _native


@dataclass(frozen=True)
class MatrixFreeOperator:
    """Dimension plus the action v -> M v (krylov.py:19-24)."""

    n: int
    apply: Callable


@dataclass(frozen=True)
class KrylovReport:
    """krylov.py:27-32."""

    iterations: int
    final_relative_residual: float
    converged: bool
    breakdown: Optional[str] = None


class LevelOperator(MatrixFreeOperator):
    """shift*I + diag(kappa) A with A a ToeplitzOperator (scheme.py:129-132)."""

    def __init__(self, toeplitz, shift: float, kappa):
        object.__setattr__(self, "toeplitz", toeplitz)
        object.__setattr__(self, "shift", float(shift))
        object.__setattr__(self, "kappa", kappa)
        object.__setattr__(self, "n", toeplitz.n)
        object.__setattr__(self, "apply", self._apply)

    def _apply(self, v):
        from .toeplitz import toeplitz_matvec
        return toeplitz_matvec(self.toeplitz, v, kappa=self.kappa, shift=self.shift)


def _reports(iters, relres, status) -> List[KrylovReport]:
    out = []
    for it, rr, st in zip(iters.tolist(), relres.tolist(), status.tolist()):
        out.append(KrylovReport(int(it), float(rr), st == _native.ST_OK,
                                _native.BREAKDOWN.get(int(st))))
    return out


def _device_solve(op: LevelOperator, precond, rhs, tol, max_iters, method):
    torch = _native.torch_mod()
    from .toeplitz import CirculantPreconditioner
    dev = op.toeplitz.device
    b, as_np = _arrays.to_device(rhs, dev)
    if b.shape[-1] != op.n or b.dim() not in (1, 2):
        raise ValueError(f"rhs has shape {tuple(b.shape)}, operator order is {op.n}")
    B = 1 if b.dim() == 1 else b.shape[0]
    kap, _ = _arrays.to_device(op.kappa, dev)
    if kap.shape != b.shape:
        kap = kap.expand_as(b).contiguous()
    pc = 0
    kbar = 0.0
    if precond is not None:
        if not isinstance(precond, CirculantPreconditioner):
            raise TypeError("device solve supports the Strang CirculantPreconditioner or None")
        if precond.n != op.n:
            raise ValueError("preconditioner order differs from the operator")
        pc = 1 if precond.strang_native else 2
        kbar = float(precond.kappa_bar)
    x = torch.empty_like(b)
    iters = torch.empty(B, dtype=torch.int32, device=b.device)
    relres = torch.empty(B, dtype=torch.float64, device=b.device)
    status = torch.empty(B, dtype=torch.int32, device=b.device)
    plan = op.toeplitz.plan
    if pc == 2:
        tab = torch.from_numpy(_circ_spectrum(precond, plan.L)).to(b.device)
        _native.check(_native.load().tsf_krylov_solve_circ(
            plan.handle, B, method, b.data_ptr(), x.data_ptr(), kap.data_ptr(), op.shift,
            tab.data_ptr(), 0, float(tol), int(max_iters) if max_iters is not None else 0,
            iters.data_ptr(), relres.data_ptr(), status.data_ptr(),
            _native.stream_ptr(device=b.device)))
        reps = _reports(iters.cpu(), relres.cpu(), status.cpu())
        xs = _arrays.back(x, as_np)
        return (xs, reps[0]) if b.dim() == 1 else (xs, reps)
    if pc and not plan.has_precond:
        raise NotImplementedError(
            f"device Strang preconditioner needs a power-of-two n >= 16 (got n={op.n})")
    _native.check(_native.load().tsf_krylov_solve(
        plan.handle, B, method, pc, b.data_ptr(), x.data_ptr(), kap.data_ptr(), op.shift,
        kbar, float(tol), int(max_iters) if max_iters is not None else 0, iters.data_ptr(),
        relres.data_ptr(), status.data_ptr(), _native.stream_ptr(device=b.device)))
    reps = _reports(iters.cpu(), relres.cpu(), status.cpu())
    xs = _arrays.back(x, as_np)
    return (xs, reps[0]) if b.dim() == 1 else (xs, reps)


def _psolve_of(precond):
    if precond is None:
        return lambda v: v
    if hasattr(precond, "solve"):
        return precond.solve
    return precond


def _caller_convention(fn, device_native: bool):
    """A user operator / preconditioner callable in the caller's convention:
    the package's own device operators (LevelOperator, the Strang
    CirculantPreconditioner) and callers that pass torch tensors get device
    tensors; a caller that passed numpy gets numpy in and numpy out, as the
    reference's callables do (krylov.py:19-24, 35-40) — e.g. the reference's
    dense test operators `lambda v: A @ v`."""
    if device_native:
        return lambda v: _arrays.to_device(fn(v))[0]
    return lambda v: _arrays.to_device(np.asarray(fn(v.detach().cpu().numpy()), dtype=float))[0]


def _native_parts(op, precond, as_np: bool):
    from .toeplitz import CirculantPreconditioner
    op_native = isinstance(op, LevelOperator) or not as_np
    pc_native = precond is None or isinstance(precond, CirculantPreconditioner) or not as_np
    return op_native, pc_native


def _generic_bicgstab(op, precond, rhs, tol, max_iters):
    torch = _native.torch_mod()
    b, as_np = _arrays.to_device(rhs)
    n = op.n
    if b.shape != (n,):
        raise ValueError(f"rhs has shape {tuple(b.shape)}, operator order is {n}")
    max_iters = max_iters if max_iters is not None else 10 * n
    ps = _psolve_of(precond)
    op_native, pc_native = _native_parts(op, precond, as_np)
    ap = _caller_convention(op.apply, op_native)
    pss = _caller_convention(ps, pc_native)
    x = torch.zeros_like(b)
    r = b.clone()
    r0 = b.clone()
    nrm0 = float(torch.linalg.norm(r0))
    if nrm0 == 0.0:
        return _arrays.back(x, as_np), KrylovReport(0, 0.0, True)
    rho = alpha = omega = 1.0
    v = torch.zeros_like(b)
    p = torch.zeros_like(b)
    for it in range(1, max_iters + 1):
        rho_new = float(r0 @ r)
        if rho_new == 0.0:
            return _arrays.back(x, as_np), KrylovReport(
                it, float(torch.linalg.norm(r)) / nrm0, False, "rho vanished")
        if it == 1:
            p = r.clone()
        else:
            beta = (rho_new / rho) * (alpha / omega)
            p = r + beta * (p - omega * v)
        ph = pss(p)
        v = ap(ph)
        den = float(r0 @ v)
        if den == 0.0:
            return _arrays.back(x, as_np), KrylovReport(
                it, float(torch.linalg.norm(r)) / nrm0, False, "r0.v vanished")
        alpha = rho_new / den
        s = r - alpha * v
        sn = float(torch.linalg.norm(s)) / nrm0
        if sn < tol:
            x += alpha * ph
            return _arrays.back(x, as_np), KrylovReport(it, sn, True)
        sh = pss(s)
        t = ap(sh)
        tt = float(t @ t)
        if tt == 0.0:
            return _arrays.back(x, as_np), KrylovReport(it, sn, False,
                                                        "omega denominator vanished")
        omega = float(t @ s) / tt
        x += alpha * ph + omega * sh
        r = s - omega * t
        rho = rho_new
        rel = float(torch.linalg.norm(r)) / nrm0
        if rel < tol:
            return _arrays.back(x, as_np), KrylovReport(it, rel, True)
        if omega == 0.0:
            return _arrays.back(x, as_np), KrylovReport(it, rel, False, "omega vanished")
    return _arrays.back(x, as_np), KrylovReport(
        max_iters, float(torch.linalg.norm(r)) / nrm0, False)


def _generic_cg(op, precond, rhs, tol, max_iters):
    torch = _native.torch_mod()
    b, as_np = _arrays.to_device(rhs)
    n = op.n
    if b.shape != (n,):
        raise ValueError(f"rhs has shape {tuple(b.shape)}, operator order is {n}")
    max_iters = max_iters if max_iters is not None else 10 * n
    ps = _psolve_of(precond)
    op_native, pc_native = _native_parts(op, precond, as_np)
    ap = _caller_convention(op.apply, op_native)
    pss = _caller_convention(ps, pc_native)
    x = torch.zeros_like(b)
    r = b.clone()
    nrm0 = float(torch.linalg.norm(r))
    if nrm0 == 0.0:
        return _arrays.back(x, as_np), KrylovReport(0, 0.0, True)
    z = pss(r)
    p = z.clone()
    rz = float(r @ z)
    for it in range(1, max_iters + 1):
        q = ap(p)
        curv = float(p @ q)
        if curv <= 0.0:
            return _arrays.back(x, as_np), KrylovReport(
                it, float(torch.linalg.norm(r)) / nrm0, False, "non-positive curvature")
        a = rz / curv
        x += a * p
        r -= a * q
        rel = float(torch.linalg.norm(r)) / nrm0
        if rel < tol:
            return _arrays.back(x, as_np), KrylovReport(it, rel, True)
        z = pss(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return _arrays.back(x, as_np), KrylovReport(
        max_iters, float(torch.linalg.norm(r)) / nrm0, False)


def _fused_ok(op, precond) -> bool:
    """The fused level-solve kernels take a LevelOperator with no or a
    power-of-two Strang preconditioner BUILT FOR THIS OPERATOR: the kernels
    form P from the operator's own shift, the plan's Strang eigenvalues and
    the preconditioner's kappa_bar, so a preconditioner with another shift
    or another eigenvalue array (a hand-made CirculantPreconditioner, as in
    pkg/tests/test_toeplitz.py:163-164) takes the device-vector loop below,
    whose P^{-1} is exactly that preconditioner's.  Anything else (non-pow2 n
    with the Strang preconditioner, user callables) runs that loop too; its
    operator and preconditioner applications are still the sm_100a Toeplitz
    kernels."""
    if not isinstance(op, LevelOperator):
        return False
    if precond is None:
        return True
    from .toeplitz import CirculantPreconditioner
    if not isinstance(precond, CirculantPreconditioner) or precond.n != op.n:
        return False
    if not precond.strang_native:
        # non-power-of-two n: the circulant-column preconditioner inside the
        # fused kernels (tsf_krylov_solve_circ) uses THIS preconditioner's
        # eigenvalues, so any shift / lam is honoured; single-CTA engine only
        return op.n <= 4096
    if float(precond.shift) != float(op.shift):
        return False
    return precond.plan is op.toeplitz.plan or _same_strang(precond, op)


def _circ_spectrum(precond, L: int):
    """(S_2k, S_2k+1)/L of the length-L embedding of the circulant column
    c = Re IFFT_n(1/total) (symmetrised: c_j = c_{n-j}), even part of the
    symbol in extended precision — the table tsf_krylov_solve_circ takes.
    Cached on the preconditioner."""
    cached = getattr(precond, "_circ_tab", None)
    if cached is not None and cached[0] == L:
        return cached[1]
    from .toeplitz import _even_embedding
    c = np.fft.ifft(1.0 / np.asarray(precond.total_eigs, dtype=float)).real
    c = 0.5 * (c + np.roll(c[::-1], 1))
    sym = np.fft.fft(_even_embedding(c, L)).real.astype(np.longdouble)
    ev = (0.5 * (sym + np.roll(sym[::-1], 1)) / L).astype(np.float64)
    tab = np.ascontiguousarray(np.stack([ev[0::2], ev[1::2]], axis=1))   # [L/2, 2]
    object.__setattr__(precond, "_circ_tab", (L, tab))
    return tab


def _same_strang(precond, op) -> bool:
    """The preconditioner's eigenvalues are the operator plan's (same Strang
    column), so the fused kernels' P equals the preconditioner."""
    from .toeplitz import strang_first_column
    col = getattr(op.toeplitz, "first_col", None)
    if col is None or getattr(precond, "first_col", None) is None:
        return False
    if not np.array_equal(np.asarray(precond.first_col), np.asarray(col)):
        return False
    lam = np.fft.fft(strang_first_column(np.asarray(col, dtype=float))).real
    return np.array_equal(np.asarray(precond.lam), lam)


def _zero_iteration_report(rhs, max_iters):
    """max_iters <= 0 (krylov.py:105-116 with an empty loop): zero RHS ->
    (0, 0.0, converged); otherwise (max_iters, ||r0||/||r0|| = 1, not converged)."""
    torch = _native.torch_mod()
    b, as_np = _arrays.to_device(rhs)
    x = torch.zeros_like(b)
    if b.dim() == 1:
        nrm = float(torch.linalg.norm(b))
        rep = (KrylovReport(0, 0.0, True) if nrm == 0.0
               else KrylovReport(int(max_iters), 1.0, False))
        return _arrays.back(x, as_np), rep
    nrms = torch.linalg.norm(b, dim=1).cpu().tolist()
    reps = [KrylovReport(0, 0.0, True) if v == 0.0 else KrylovReport(int(max_iters), 1.0, False)
            for v in nrms]
    return _arrays.back(x, as_np), reps


def solve_bicgstab(op: MatrixFreeOperator, precond, rhs, tol: float = 1e-10,
                   max_iters: Optional[int] = None):
    """Right-preconditioned BiCGSTAB, x0 = 0 (krylov.py:88-153)."""
    if max_iters is not None and max_iters <= 0:
        return _zero_iteration_report(rhs, max_iters)
    if _fused_ok(op, precond):
        return _device_solve(op, precond, rhs, tol, max_iters, method=0)
    return _generic_bicgstab(op, precond, rhs, tol, max_iters)


def solve_cg(op: MatrixFreeOperator, precond, rhs, tol: float = 1e-10,
             max_iters: Optional[int] = None):
    """Preconditioned CG, x0 = 0 (krylov.py:43-85)."""
    if max_iters is not None and max_iters <= 0:
        return _zero_iteration_report(rhs, max_iters)
    if _fused_ok(op, precond):
        return _device_solve(op, precond, rhs, tol, max_iters, method=1)
    return _generic_cg(op, precond, rhs, tol, max_iters)


DENSE_SOLVE_CAP = 2048


def solve_dense(matrix, rhs):
    """Dense LU on the device (krylov.py:156-171; out of the FIDS hot path)."""
    torch = _native.torch_mod()
    A, as_np = _arrays.to_device(matrix)
    b, _ = _arrays.to_device(rhs)
    n = A.shape[0]
    if A.shape != (n, n) or b.shape != (n,):
        raise ValueError("matrix/rhs shapes are inconsistent")
    if n > DENSE_SOLVE_CAP:
        raise ValueError(f"dense solve capped at {DENSE_SOLVE_CAP}, got {n}")
    x, info = torch.linalg.solve_ex(A, b)
    if int(info) != 0:
        raise ValueError("matrix is singular")
    return _arrays.back(x, as_np)
