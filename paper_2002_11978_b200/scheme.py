"""FIDS time march on the B200 (mirror of tsfrac.scheme, scheme.py:36-303).

`run_fids` keeps the reference's signature, argument meaning, return types
and errors.  Host setup (mesh, IFL column, SOE, per-level scalars and SOE
coefficient rows) is computed with numpy exactly as the reference does; the
march itself runs natively (`tsf_fids_march`, csrc/tsf_abi.cu): per level
one fused SOE-push + history-term + RHS kernel and one fused level-solve
kernel (kappa, kappa_bar, preconditioner check, full BiCGSTAB/CG), with no
host round trip until the end of the run.

Coefficients: arbitrary callables kappa(x, t) / source(x, t) are tabulated
on the host at every level (the reference evaluates them per level too,
scheme.py:156-160,283) and uploaded once; a `SeparableField` instead keeps
only its spatial modes on the device and evaluates sum_q mode_q(x) c_q(t)
per level inside the kernels (bit-identical to the same numpy expression).

`run_fids_batched` runs B independent instances (per-instance modes and
initial data) in one march — the configs[2] workload.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np
from scipy.special import gammaln

from . import _arrays, _native
from .ifl import IflDiscretization, build_ifl
from .mesh import GradedMesh, build_mesh, l1_weights
from .soe import SoeApproximation, build_soe
from .toeplitz import PreconditionerError, build_toeplitz, plan_for

DIRECT_THRESHOLD = 128


@dataclass(frozen=True)
class ProblemSpec:
    """scheme.py:39-51."""

    gamma: float
    alpha: float
    l: float
    T: float
    kappa: Callable
    source: Callable
    initial: Callable
    exact: Optional[Callable] = None
    kappa_x_independent: bool = False


@dataclass(frozen=True)
class SolverOptions:
    """scheme.py:54-59."""

    solver: str = "auto"
    tol: float = 1e-10
    max_iters: Optional[int] = None
    direct_threshold: int = DIRECT_THRESHOLD


@dataclass(frozen=True)
class TimeStepSystem:
    shift: float
    kappa_diag: object
    ifl: IflDiscretization
    rhs: object


@dataclass
class SolveReport:
    """scheme.py:72-82 (+ per-level iteration counts, which the reference drops)."""

    err_inf: Optional[float]
    err_2: Optional[float]
    rates: Optional[tuple] = None
    avg_iterations: float = 0.0
    wall_time: float = 0.0
    scheme_tag: str = ""
    solver_tag: str = ""
    history_ops: np.ndarray = field(default=None)
    history_memory_values: int = 0
    iterations: Optional[np.ndarray] = None
    relres: Optional[np.ndarray] = None


class SeparableField:
    """g(x, t) = sum_q mode_q(x) * c_q(t): the device-evaluable coefficient form.

    `modes` are arrays over the interior grid (or callables of x); `coef(t)`
    returns the q coefficients.  Calling the object evaluates
    ((mode_0 c_0) + mode_1 c_1) + ... left to right, which is also exactly
    what the kernels compute (no FMA contraction), so e.g. the configs[0]
    diffusivity 1 + 0.5 sin(pi x) e^{-t} == SeparableField([1, 0.5 sin(pi x)],
    lambda t: [1.0, exp(-t)]) matches numpy bit for bit.
    """

    def __init__(self, modes: Sequence, coef: Callable[[float], Sequence[float]]):
        if not 1 <= len(modes) <= 4:
            raise ValueError("a SeparableField needs 1..4 modes")
        self.modes = list(modes)
        self.coef = coef

    def mode_values(self, x: np.ndarray) -> np.ndarray:
        rows = []
        for m in self.modes:
            v = m(x) if callable(m) else m
            rows.append(np.broadcast_to(np.asarray(v, dtype=float), np.shape(x)))
        return np.stack(rows)

    def __call__(self, x, t):
        vals = self.mode_values(np.asarray(x, dtype=float))
        c = [float(v) for v in self.coef(t)]
        acc = np.zeros(vals.shape[1:])
        for q in range(vals.shape[0]):
            acc = acc + vals[q] * c[q]
        return acc


def select_solver(N: int, options: SolverOptions = SolverOptions()) -> str:
    """scheme.py:94-98."""
    if options.solver != "auto":
        return options.solver
    return "direct" if N - 1 <= options.direct_threshold else "pkrylov"


def _last_weight(tau_m: float, gamma: float) -> float:
    return tau_m ** (-gamma) / (1.0 - gamma)


def _setup(spec: ProblemSpec, M: int, r: float, N: int, mu: Optional[float]):
    if N < 3:
        raise ValueError(f"N must be >= 3, got {N}")
    mesh = build_mesh(M, r, spec.T)
    mu = 1.0 + spec.alpha / 2.0 if mu is None else mu
    disc = build_ifl(spec.alpha, mu, spec.l, N)
    return mesh, disc, disc.interior_points()


def _kappa_at(spec: ProblemSpec, x: np.ndarray, t: float) -> np.ndarray:
    k = np.broadcast_to(np.asarray(spec.kappa(x, t), dtype=float), x.shape).copy()
    if np.any(k <= 0.0):
        raise ValueError(f"kappa must be positive on the grid at t={t}")
    return k


# ---------------------------------------------------------------- march core
@dataclass
class _FieldDev:
    nmodes: int
    modes: object          # torch tensor (keeps memory alive)
    q_stride: int
    b_stride: int
    t_stride: int
    coef: np.ndarray       # host [M+1, nmodes]

    def as_c(self) -> _native.Field:
        return _native.Field(self.nmodes, self.modes.data_ptr() if self.modes is not None else None,
                             self.q_stride, self.b_stride, self.t_stride,
                             self.coef.ctypes.data if self.coef is not None else None)


def _field_separable(f: SeparableField, x: np.ndarray, t: np.ndarray, B: int,
                     per_instance: Optional[np.ndarray], dev) -> _FieldDev:
    torch = _native.torch_mod()
    n = x.size
    if per_instance is not None:      # [Q, B, n]
        vals = np.ascontiguousarray(per_instance, dtype=np.float64)
        Q = vals.shape[0]
        b_stride = n
    else:
        vals = np.ascontiguousarray(f.mode_values(x))
        Q = vals.shape[0]
        b_stride = 0
    coef = np.ascontiguousarray(
        np.array([[float(c) for c in f.coef(tm)] for tm in t], dtype=np.float64))
    if coef.shape[1] != Q:
        raise ValueError("SeparableField.coef(t) must return one value per mode")
    mt = torch.from_numpy(vals).to(dev)
    return _FieldDev(Q, mt, vals[0].size if per_instance is not None else n, b_stride, 0, coef)


def _field_tabulated(tab: np.ndarray, B: int, n: int, M: int, dev) -> _FieldDev:
    """tab [M+1, B, n] (level 0 unused) -> one mode, coef 1, t_stride = B n."""
    torch = _native.torch_mod()
    mt = torch.from_numpy(np.ascontiguousarray(tab, dtype=np.float64)).to(dev)
    coef = np.ones((M + 1, 1))
    return _FieldDev(1, mt, 0, n, B * n, coef)


@dataclass
class MarchResult:
    u_final: object        # torch [B, n]
    hist: Optional[object]  # torch [(M+1), hist_B, n]
    iterations: np.ndarray  # [M, B]
    relres: np.ndarray      # [M, B]
    status: np.ndarray      # [M, B]
    W: object               # torch [B, nexp, n]


def _soe_block_default(B: int, n: int) -> int:
    """Levels per W pass of the march's blocked SOE schedule.

    TSF_SOE_BLOCK overrides (0 or 1: one W pass per level).  By default the
    schedule is blocked (K = 8) on both engines: on the single-CTA engine
    batches make the SOE pass a large share of a level (configs[2]: 16%), and
    since the half-length four-step engine the per-level pass
    was 10% of a configs[3] level (0.29 of 2.80 ms; blocked: 0.06 ms).  The
    choice does not depend on B, so an instance's result does not depend on
    the batch it is in."""
    env = os.environ.get("TSF_SOE_BLOCK")
    if env is not None:
        k = int(env)
        return k if 2 <= k <= 16 else 1
    return 8


def soe_block_tables(tab: np.ndarray, K: int):
    """Host tables of the blocked SOE schedule (csrc/tsf_soe.cuh k_soe_block).

    tab[m-1] = (d(m), c(m), h(m)) are level m's decay e^{-s tau_m}, push
    coefficient -expm1(-s tau_m)/s and history weight w e^{-s tau_m}, i.e. the
    factors of history_push (soe.py:221-223) and of the history term
    (scheme.py:281-282).  For level m in the block with base mb = K floor((m-1)/K):
      alpha_j(m)   = h_j(m) prod_{l=mb+1}^{m-1} d_j(l)
      beta(m, i)   = sum_j h_j(m) prod_{l=i+1}^{m-1} d_j(l) c_j(i),  mb < i < m
    so that H^m = sum_j alpha_j(m) W_j^{mb} + sum_i beta(m, i) du^i exactly in
    real arithmetic (products and sums in extended precision, rounded once)."""
    M, _, nexp = tab.shape
    ld = np.longdouble
    dec, cf, hc = tab[:, 0].astype(ld), tab[:, 1].astype(ld), tab[:, 2].astype(ld)
    alpha = np.empty((M, nexp))
    beta = np.zeros((M, 16))
    for m in range(1, M + 1):
        mb = K * ((m - 1) // K)
        # Q_i = prod_{l=i+1}^{m-1} d(l) for i = m-1 down to mb
        Q = np.ones(nexp, dtype=ld)
        for i in range(m - 1, mb - 1, -1):
            if i > mb:
                beta[m - 1, i - mb - 1] = float(np.sum(hc[m - 1] * Q * cf[i - 1]))
            if i >= mb + 1:
                Q = Q * dec[i - 1]
        alpha[m - 1] = (hc[m - 1] * Q).astype(np.float64)
    return alpha, beta


class FidsMarch:
    """Device state + native driver for a batch of FIDS instances sharing
    (gamma, alpha, l, T, M, r, N, SOE).  Reusable: `reset()` then `run()`."""

    def __init__(self, gamma, alpha, l, T, M, r, N, soe: SoeApproximation, method: int,
                 precond: int, tol: float, max_iters: Optional[int], B: int,
                 kappa: _FieldDev, source: _FieldDev, u0, hist_B: int = 0, device: int = 0,
                 mu: Optional[float] = None, private_plan: bool = False,
                 soe_block: Optional[int] = None):
        torch = _native.torch_mod()
        self.dev = torch.device(f"cuda:{device}")
        self.mesh = build_mesh(M, r, T)
        mu = 1.0 + alpha / 2.0 if mu is None else mu
        self.disc = build_ifl(alpha, mu, l, N)
        self.n = N - 1
        self.B, self.M = int(B), int(M)
        self.gamma = gamma
        self.soe = soe
        self.method, self.precond = int(method), int(precond)
        self.tol = float(tol)
        self.max_iters = int(max_iters) if max_iters is not None else 10 * self.n
        self.G = math.exp(gammaln(1.0 - gamma))
        op = build_toeplitz(self.disc.first_col, device=device)
        self.plan = plan_for(self.disc.first_col, device, spectrum=op.spectrum_embed,
                             private=private_plan)
        if self.precond and not self.plan.has_precond:
            raise NotImplementedError(
                f"device Strang preconditioner needs a power-of-two n >= 16 (got n={self.n})")
        tau = self.mesh.tau
        a_mm = np.array([_last_weight(float(tau[m]), gamma) for m in range(M)])
        self.a_mm = a_mm
        self.shift = a_mm / self.G
        self.tau = np.ascontiguousarray(tau, dtype=np.float64)
        s, w = soe.nodes, soe.weights
        tab = np.empty((M, 3, s.size))
        for m in range(M):
            dec = np.exp(-s * tau[m])
            tab[m, 0] = dec
            tab[m, 1] = -np.expm1(-s * tau[m]) / s
            tab[m, 2] = w * dec
        self.soe_tab = torch.from_numpy(tab).to(self.dev)
        # blocked SOE schedule (tsf_march.soe_block; csrc/tsf_soe.cuh k_soe_block)
        self.soe_block = (soe_block if soe_block is not None
                          else _soe_block_default(self.B, self.n))
        if self.soe_block > 1:
            alpha, beta = soe_block_tables(tab, self.soe_block)
            self.soe_alpha = torch.from_numpy(alpha).to(self.dev)
            self.soe_beta = beta
        self.kappa, self.source = kappa, source
        n, nexp = self.n, soe.n_exp
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.u0 = u0
        self.ubuf = [torch.empty((B, n), **f64), torch.empty((B, n), **f64)]
        self.W = torch.empty((B, nexp, n), **f64)
        self.rhs = torch.empty((B, n), **f64)
        self.kwork = torch.empty((B, n), **f64)
        self.iters = torch.zeros((M, B), dtype=torch.int32, device=self.dev)
        self.relres = torch.zeros((M, B), **f64)
        self.status = torch.zeros((M, B), dtype=torch.int32, device=self.dev)
        self.soe_ring = (torch.empty((2, self.soe_block, B, n), **f64) if self.soe_block > 1
                         else None)
        self.hist_B = int(hist_B)
        self.hist = torch.empty((M + 1, hist_B, n), **f64) if hist_B > 0 else None
        _native.check(_native.load().tsf_plan_reserve(self.plan.handle, self.B))
        self.reset()

    def reset(self):
        self.ubuf[0].copy_(self.u0)
        self.W.zero_()
        self.status.zero_()
        if self.hist is not None:
            self.hist[0].copy_(self.u0[: self.hist_B])
        self.next_level = 1

    def _desc(self, m_begin: int, m_end: int) -> _native.March:
        d = _native.March()
        d.B, d.M, d.nexp = self.B, self.M, self.soe.n_exp
        d.method, d.precond, d.tol, d.max_iters = self.method, self.precond, self.tol, self.max_iters
        d.G = self.G
        self._keep = (np.ascontiguousarray(self.shift), np.ascontiguousarray(self.a_mm))
        d.shift = self._keep[0].ctypes.data
        d.a_mm = self._keep[1].ctypes.data
        d.tau = self.tau.ctypes.data
        d.soe_tab = self.soe_tab.data_ptr()
        d.kappa = self.kappa.as_c()
        d.source = self.source.as_c()
        d.u_buf0 = self.ubuf[0].data_ptr()
        d.u_buf1 = self.ubuf[1].data_ptr()
        d.W = self.W.data_ptr()
        d.rhs = self.rhs.data_ptr()
        d.kwork = self.kwork.data_ptr()
        d.iters = self.iters.data_ptr()
        d.relres = self.relres.data_ptr()
        d.status = self.status.data_ptr()
        d.hist = self.hist.data_ptr() if self.hist is not None else None
        d.hist_B = self.hist_B
        d.m_begin, d.m_end = m_begin, m_end
        d.soe_block = self.soe_block if self.soe_block > 1 else 0
        if self.soe_block > 1:
            d.soe_alpha = self.soe_alpha.data_ptr()
            d.soe_beta = self.soe_beta.ctypes.data
            d.soe_ring = self.soe_ring.data_ptr()
        return d

    def run(self, levels: Optional[int] = None, stream=None, events=None):
        """Launch the next `levels` levels (all remaining by default); async.

        `events`: optional list of 3 torch.cuda.Event per level run (before
        the SOE kernel, between SOE and solve, after the solve)."""
        m0 = self.next_level
        m1 = self.M + 1 if levels is None else min(self.M + 1, m0 + levels)
        if m1 <= m0:
            return
        d = self._desc(m0, m1)
        if events is not None:
            if len(events) < 3 * (m1 - m0):
                raise ValueError("need 3 events per level")
            torch = _native.torch_mod()
            for e in events:  # materialise the lazily created CUDA events
                if e.cuda_event == 0:
                    e.record()
            torch.cuda.synchronize(self.dev)
            self._ev = (C.c_void_p * len(events))(*[e.cuda_event for e in events])
            d.events = C.cast(self._ev, C.c_void_p)
        if stream is not None:
            # reset() and the constructor's uploads ran on torch's current
            # stream of this device: order them before the march
            torch = _native.torch_mod()
            stream.wait_stream(torch.cuda.current_stream(self.dev))
        _native.check(_native.load().tsf_fids_march(self.plan.handle, C.byref(d),
                                                    _native.stream_ptr(stream, self.dev)))
        self.next_level = m1

    def u_level(self, m: int):
        return self.ubuf[m & 1]

    def result(self) -> MarchResult:
        torch = _native.torch_mod()
        torch.cuda.synchronize(self.dev)
        return MarchResult(self.u_level(self.next_level - 1), self.hist,
                           self.iters.cpu().numpy(), self.relres.cpu().numpy(),
                           self.status.cpu().numpy(), self.W)


def _raise_status(status: np.ndarray, iters, relres, t: np.ndarray, use_cg: bool):
    bad = np.argwhere(status != 0)
    if bad.size == 0:
        return
    m0, b0 = (int(v) for v in bad[0])
    st = int(status[m0, b0])
    tm = float(t[m0 + 1])
    if st == _native.ST_KAPPA_NONPOS:
        raise ValueError(f"kappa must be positive on the grid at t={tm}")
    if st == _native.ST_PRECOND_NONPOS:
        raise PreconditionerError("preconditioner has a non-positive eigenvalue")
    from .krylov import KrylovReport
    rep = KrylovReport(int(iters[m0, b0]), float(relres[m0, b0]), False,
                       _native.BREAKDOWN.get(st))
    raise RuntimeError(f"{'CG' if use_cg else 'BiCGSTAB'} did not converge: {rep}")


def run_fids(spec: ProblemSpec, M: int, r: float, N: int, epsilon: float = 1e-10,
             mu: Optional[float] = None, options: SolverOptions = SolverOptions(),
             keep_history: bool = True, soe: Optional[SoeApproximation] = None,
             device: int = 0):
    """Fast implicit scheme (scheme.py:236-303) on the B200."""
    t0 = time.perf_counter()
    if epsilon <= 0.0:
        raise ValueError(f"epsilon must be > 0, got {epsilon}")
    mesh, disc, x = _setup(spec, M, r, N, mu)
    n = N - 1
    tag = select_solver(N, options)
    if soe is None:
        soe = build_soe(spec.gamma, epsilon, (1.0 / M) ** r * spec.T, spec.T)
    u0 = np.asarray(spec.initial(x), dtype=float)
    if tag == "direct":
        hist, its = _run_direct(spec, mesh, disc, x, soe, u0, M, device)
        return _finish(spec, mesh, disc, x, hist, its, None, soe, t0, tag, keep_history)
    if tag not in ("krylov", "pkrylov"):
        raise ValueError(f"unknown solver {tag!r}")
    if tag == "pkrylov" and not (n >= 16 and n & (n - 1) == 0):
        hist, its, rel = _run_levels(spec, mesh, disc, x, soe, u0, M, options, device,
                                     keep_history or spec.exact is not None)
        return _finish(spec, mesh, disc, x, hist, its, rel, soe, t0, tag, keep_history)
    torch = _native.torch_mod()
    dev = torch.device(f"cuda:{device}")
    kap = _device_field(spec.kappa, x, mesh.t, n, M, dev, positive=True, chunk=MARCH_CHUNK)
    src = _device_field(spec.source, x, mesh.t, n, M, dev, positive=False, chunk=MARCH_CHUNK)
    u0_t = torch.from_numpy(np.ascontiguousarray(u0)[None, :]).to(dev)
    want_hist = keep_history or spec.exact is not None
    chunked = [f for f in (kap, src) if isinstance(f, _ChunkField)]
    if chunked:
        for f in chunked:
            f.fill(1, min(M + 1, 1 + MARCH_CHUNK))
    march = FidsMarch(spec.gamma, spec.alpha, spec.l, spec.T, M, r, N, soe,
                      method=1 if spec.kappa_x_independent else 0,
                      precond=1 if tag == "pkrylov" else 0, tol=options.tol,
                      max_iters=options.max_iters, B=1, kappa=kap, source=src, u0=u0_t,
                      hist_B=1 if want_hist else 0, device=device, mu=mu)
    for m0 in range(1, M + 1, MARCH_CHUNK):
        m1 = min(M + 1, m0 + MARCH_CHUNK)
        if m0 > 1:
            for f in chunked:
                f.fill(m0, m1)   # after the previous chunk (stream order + status sync)
        march.run(m1 - m0)
        st = march.status[m0 - 1: m1 - 1].cpu().numpy()
        if np.any(st != 0):
            _raise_status(st, march.iters[m0 - 1: m1 - 1].cpu().numpy(),
                          march.relres[m0 - 1: m1 - 1].cpu().numpy(), mesh.t[m0 - 1:],
                          spec.kappa_x_independent)
    res = march.result()
    if want_hist:
        hist = res.hist[:, 0, :].cpu().numpy()
    else:
        hist = res.u_final[0].cpu().numpy()[None, :]
    return _finish(spec, mesh, disc, x, hist, res.iterations[:, 0], res.relres[:, 0], soe, t0,
                   tag, keep_history)


def _run_levels(spec, mesh, disc, x, soe, u0, M, options, device, want_hist):
    """The reference's level loop (scheme.py:276-294) driven from the host,
    for the Strang preconditioner at non-power-of-two n: per level the SOE
    history term / RHS and the push run in the SOE kernel, the operator and
    P^{-1} = circ(IFFT(1/total)) in the Toeplitz kernels (toeplitz.py
    _circulant_plan), the BiCGSTAB/CG loop over device vectors."""
    from .krylov import LevelOperator, solve_bicgstab, solve_cg
    from .soe import FastHistory, fast_caputo_rhs, history_push
    from .toeplitz import build_preconditioner
    torch = _native.torch_mod()
    dev = torch.device(f"cuda:{device}")
    n = disc.N - 1
    G = math.exp(gammaln(1.0 - spec.gamma))
    op = build_toeplitz(disc.first_col, device=device)
    h = FastHistory.fresh(soe, n, device)
    u_prev = torch.from_numpy(np.ascontiguousarray(u0, dtype=np.float64)).to(dev)
    hist = np.empty((M + 1, n)) if want_hist else None
    if want_hist:
        hist[0] = u0
    its = np.zeros(M, dtype=np.int64)
    rel = np.zeros(M)
    solver = solve_cg if spec.kappa_x_independent else solve_bicgstab
    for m in range(1, M + 1):
        tau_m = float(mesh.tau[m - 1])
        tm = float(mesh.t[m])
        a_mm = _last_weight(tau_m, spec.gamma)
        kappa = _kappa_at(spec, x, tm)
        f = torch.from_numpy(np.ascontiguousarray(spec.source(x, tm), dtype=np.float64)).to(dev)
        rhs = f + fast_caputo_rhs(h, a_mm, u_prev, spec.gamma, tau_m)
        shift = a_mm / G
        lev = LevelOperator(op, shift, torch.from_numpy(kappa).to(dev))
        pc = build_preconditioner(disc.first_col, shift, float(kappa.mean()), device=device)
        u, rep = solver(lev, pc, rhs, tol=options.tol, max_iters=options.max_iters)
        if not rep.converged:
            raise RuntimeError(
                f"{'CG' if spec.kappa_x_independent else 'BiCGSTAB'} did not converge: {rep}")
        its[m - 1] = rep.iterations
        rel[m - 1] = rep.final_relative_residual
        history_push(h, u - u_prev, tau_m)
        u_prev = u
        if want_hist:
            hist[m] = u.cpu().numpy()
    if not want_hist:
        hist = u_prev.cpu().numpy()[None, :]
    return hist, its, rel


class _ChunkField(_FieldDev):
    """An arbitrary callable field tabulated CHUNK levels at a time: the
    device holds [CHUNK, n] instead of [M+1, n] (2.15 GB per field at
    configs[3] for the whole march).  `fill(m0, m1)` evaluates levels
    m0..m1-1 on the host as the reference does per level (scheme.py:280,283);
    the march descriptor's base pointer is offset so level m reads row m - m0
    (the march only touches levels inside the range it runs)."""

    def __init__(self, fn, x, t, n, dev, positive, chunk):
        torch = _native.torch_mod()
        buf = torch.empty((chunk, 1, n), dtype=torch.float64, device=dev)
        super().__init__(1, buf, 0, n, n, np.ones((t.size, 1)))
        self.fn, self.x, self.t, self.positive, self.m0 = fn, x, t, positive, 0

    def fill(self, m0: int, m1: int):
        torch = _native.torch_mod()
        tab = np.empty((m1 - m0, 1, self.x.size))
        for m in range(m0, m1):
            if self.positive:
                tab[m - m0, 0] = _kappa_at_fn(self.fn, self.x, self.t[m])
            else:
                tab[m - m0, 0] = np.asarray(self.fn(self.x, self.t[m]), dtype=float)
        self.modes[: m1 - m0].copy_(torch.from_numpy(tab))
        self.m0 = m0

    def as_c(self) -> _native.Field:
        base = self.modes.data_ptr() - self.m0 * self.t_stride * 8
        return _native.Field(1, base, 0, self.b_stride, self.t_stride, self.coef.ctypes.data)


# levels per native-march launch in run_fids: the status of a chunk is read
# back before the next one runs, so a failing level raises (as the
# reference does at that level, scheme.py:139-142) without the whole march
# running first, and callable fields are tabulated per chunk
MARCH_CHUNK = 32


def _device_field(fn, x, t, n, M, dev, positive, chunk=None):
    if isinstance(fn, SeparableField):
        return _field_separable(fn, x, t, 1, None, dev)
    if chunk:
        return _ChunkField(fn, x, t, n, dev, positive, min(chunk, M))
    tab = np.empty((M + 1, 1, n))
    tab[0] = 0.0
    for m in range(1, M + 1):
        if positive:
            tab[m, 0] = _kappa_at_fn(fn, x, t[m])
        else:
            tab[m, 0] = np.asarray(fn(x, t[m]), dtype=float)
    return _field_tabulated(tab, 1, n, M, dev)


def _kappa_at_fn(fn, x, t):
    k = np.broadcast_to(np.asarray(fn(x, t), dtype=float), x.shape).copy()
    if np.any(k <= 0.0):
        raise ValueError(f"kappa must be positive on the grid at t={t}")
    return k


def _finish(spec, mesh, disc, x, hist, its, rel, soe, t0, tag, keep_history):
    M = mesh.M
    n = disc.N - 1
    err_inf = err_2 = None
    if spec.exact is not None and hist.shape[0] == M + 1:
        sh = math.sqrt(disc.h)
        e_inf, e_2 = 0.0, 0.0
        for m in range(M + 1):
            e = hist[m] - spec.exact(x, mesh.t[m])
            e_inf = max(e_inf, float(np.max(np.abs(e))))
            e_2 = max(e_2, sh * float(np.linalg.norm(e)))
        err_inf, err_2 = e_inf, e_2
    its = np.asarray(its, dtype=np.int64)
    rep = SolveReport(
        err_inf=err_inf, err_2=err_2, avg_iterations=float(its.sum()) / M,
        wall_time=time.perf_counter() - t0, scheme_tag="FIDS", solver_tag=tag,
        history_ops=np.full(M, soe.n_exp * n, dtype=np.int64),
        history_memory_values=soe.n_exp * n, iterations=its,
        relres=None if rel is None else np.asarray(rel))
    out = hist if keep_history else hist[-1]
    return out, rep


def _run_direct(spec, mesh, disc, x, soe, u0, M, device):
    """Dense direct level solves for n <= direct_threshold (scheme.py:115-123;
    out of the FIDS hot path).  History via the device SOE kernels."""
    torch = _native.torch_mod()
    from .soe import FastHistory, fast_caputo_rhs, history_push
    dev = torch.device(f"cuda:{device}")
    n = disc.N - 1
    A = torch.from_numpy(disc.dense()).to(dev)
    g1mg = math.exp(gammaln(1.0 - spec.gamma))
    fast = FastHistory.fresh(soe, n, device)
    u_prev = torch.from_numpy(u0.copy()).to(dev)
    hist = np.empty((M + 1, n))
    hist[0] = u0
    eye = torch.eye(n, dtype=torch.float64, device=dev)
    for m in range(1, M + 1):
        tau_m = float(mesh.tau[m - 1])
        tm = float(mesh.t[m])
        a_mm = _last_weight(tau_m, spec.gamma)
        kappa = torch.from_numpy(_kappa_at(spec, x, tm)).to(dev)
        f = torch.from_numpy(np.asarray(spec.source(x, tm), dtype=float).copy()).to(dev)
        rhs = f + fast_caputo_rhs(fast, a_mm, u_prev, spec.gamma, tau_m)
        mat = (a_mm / g1mg) * eye + kappa[:, None] * A
        u = torch.linalg.solve(mat, rhs)
        history_push(fast, u - u_prev, tau_m)
        u_prev = u
        hist[m] = u.cpu().numpy()
    return hist, np.zeros(M, dtype=np.int64)


# ---------------------------------------------------------------- DIDS
class _DeviceLevelSolver:
    """Per-run level solver of scheme.py:105-143 (_LevelSolver) over device
    vectors: dense LU for the 'direct' tag, else the fused device BiCGSTAB /
    PCG on the structured operator with the Strang preconditioner
    ('pkrylov') — the same solves run_fids uses."""

    def __init__(self, spec: ProblemSpec, disc: IflDiscretization, tag: str,
                 options: SolverOptions, device: int):
        torch = _native.torch_mod()
        self.tag = tag
        self.options = options
        self.disc = disc
        self.device = device
        self.dev = torch.device(f"cuda:{device}")
        self.n = disc.N - 1
        self.use_cg = spec.kappa_x_independent
        if tag == "direct":
            self.A = torch.from_numpy(disc.dense()).to(self.dev)
            self.eye = torch.eye(self.n, dtype=torch.float64, device=self.dev)
        else:
            self.op = build_toeplitz(disc.first_col, device=device)

    def solve(self, shift: float, kappa: np.ndarray, rhs):
        torch = _native.torch_mod()
        from .krylov import LevelOperator, solve_bicgstab, solve_cg
        from .toeplitz import build_preconditioner
        kap = torch.from_numpy(kappa).to(self.dev)
        if self.tag == "direct":
            mat = shift * self.eye + kap[:, None] * self.A
            return torch.linalg.solve(mat, rhs), 0, 0.0
        lev = LevelOperator(self.op, shift, kap)
        pc = None
        if self.tag == "pkrylov":
            pc = build_preconditioner(self.disc.first_col, shift, float(kappa.mean()),
                                      device=self.device)
        solver = solve_cg if self.use_cg else solve_bicgstab
        u, rep = solver(lev, pc, rhs, tol=self.options.tol, max_iters=self.options.max_iters)
        if not rep.converged:
            raise RuntimeError(f"{'CG' if self.use_cg else 'BiCGSTAB'} did not converge: {rep}")
        return u, rep.iterations, rep.final_relative_residual


def run_dids(spec: ProblemSpec, M: int, r: float, N: int, mu: Optional[float] = None,
             options: SolverOptions = SolverOptions(), device: int = 0):
    """Direct implicit scheme (scheme.py:184-233) on the B200; returns
    (history [M+1, n], SolveReport).

    The history lives on the device; at level m the L1 history term
    `(a[0]/G) u^0 + (diff(a) @ hist[1:m]) / G` streams levels 0..m-1 once
    through k_l1_history_rhs (tsf_l1_history_rhs, csrc/tsf_dids.cuh) with the
    weights a = l1_weights(mesh, gamma, m).a formed on the host exactly as
    the reference does (mesh.py:53-80); the level solve is the device solve
    run_fids uses.  O(m n) work and O((M+1) n) storage per run, like the
    reference.
    """
    t0 = time.perf_counter()
    mesh, disc, x = _setup(spec, M, r, N, mu)
    n = N - 1
    tag = select_solver(N, options)
    if tag not in ("direct", "krylov", "pkrylov"):
        raise ValueError(f"unknown solver {tag!r}")
    torch = _native.torch_mod()
    dev = torch.device(f"cuda:{device}")
    lib = _native.load()
    solver = _DeviceLevelSolver(spec, disc, tag, options, device)
    G = math.exp(gammaln(1.0 - spec.gamma))
    hist = torch.empty((M + 1, n), dtype=torch.float64, device=dev)
    hist[0] = torch.from_numpy(np.ascontiguousarray(spec.initial(x), dtype=np.float64)).to(dev)
    rhs = torch.empty(n, dtype=torch.float64, device=dev)
    its = np.zeros(M, dtype=np.int64)
    rel = np.zeros(M)
    ops = np.empty(M, dtype=np.int64)
    for m in range(1, M + 1):
        a = l1_weights(mesh, spec.gamma, m).a
        tm = float(mesh.t[m])
        kappa = _kappa_at(spec, x, tm)
        f = torch.from_numpy(np.ascontiguousarray(spec.source(x, tm), dtype=np.float64)).to(dev)
        w = torch.from_numpy(np.diff(a)).to(dev) if m > 1 else None
        with torch.cuda.device(dev):
            _native.check(lib.tsf_l1_history_rhs(1, n, m, hist.data_ptr(), m * n,
                                                 None if w is None else w.data_ptr(),
                                                 a[0] / G, G, f.data_ptr(), rhs.data_ptr(),
                                                 _native.stream_ptr(device=dev)))
        ops[m - 1] = m * n
        u, it, rr = solver.solve(a[-1] / G, kappa, rhs)
        its[m - 1] = it
        rel[m - 1] = rr
        hist[m] = u
    hist_np = hist.cpu().numpy()
    err_inf = err_2 = None
    if spec.exact is not None:
        sh = math.sqrt(disc.h)
        err_inf = err_2 = 0.0
        for m in range(M + 1):
            e = hist_np[m] - spec.exact(x, mesh.t[m])
            err_inf = max(err_inf, float(np.max(np.abs(e))))
            err_2 = max(err_2, sh * float(np.linalg.norm(e)))
    rep = SolveReport(
        err_inf=err_inf, err_2=err_2, avg_iterations=float(its.sum()) / M,
        wall_time=time.perf_counter() - t0, scheme_tag="DIDS", solver_tag=tag,
        history_ops=ops, history_memory_values=hist_np.size, iterations=its,
        relres=None if tag == "direct" else rel)
    return hist_np, rep


# ---------------------------------------------------------------- batched
def run_fids_batched(gamma: float, alpha: float, M: int, r: float, N: int,
                     kappa: SeparableField, source: SeparableField, initial,
                     kappa_modes: Optional[np.ndarray] = None,
                     source_modes: Optional[np.ndarray] = None, l: float = 1.0,
                     T: float = 1.0, epsilon: float = 1e-10, mu: Optional[float] = None,
                     options: SolverOptions = SolverOptions(solver="pkrylov"),
                     hist_B: int = 0, device: int = 0, use_cg: bool = False):
    """B independent FIDS instances in one device march.

    initial:      [B, n] u^0 per instance (numpy or torch)
    kappa_modes:  optional [Q, B, n] per-instance spatial modes (else the
                  field's shared modes); `kappa.coef(t)` gives the Q time
                  coefficients.  Same for `source_modes`.
    Returns (u^M [B, n] in the input's array type, report dict).
    """
    t0 = time.perf_counter()
    torch = _native.torch_mod()
    dev = torch.device(f"cuda:{device}")
    mesh = build_mesh(M, r, T)
    mu_ = 1.0 + alpha / 2.0 if mu is None else mu
    disc = build_ifl(alpha, mu_, l, N)
    x = disc.interior_points()
    u0, as_np = _arrays.to_device(initial, device)
    B = u0.shape[0]
    kap = _field_separable(kappa, x, mesh.t, B, kappa_modes, dev)
    src = _field_separable(source, x, mesh.t, B, source_modes, dev)
    soe = build_soe(gamma, epsilon, (1.0 / M) ** r * T, T)
    tag = options.solver if options.solver != "auto" else "pkrylov"
    march = FidsMarch(gamma, alpha, l, T, M, r, N, soe, method=1 if use_cg else 0,
                      precond=1 if tag == "pkrylov" else 0, tol=options.tol,
                      max_iters=options.max_iters, B=B, kappa=kap, source=src, u0=u0,
                      hist_B=hist_B, device=device, mu=mu)
    march.run()
    res = march.result()
    _raise_status(res.status, res.iterations, res.relres, mesh.t, use_cg)
    rep = dict(iterations=res.iterations, relres=res.relres, n_exp=soe.n_exp,
               wall_time=time.perf_counter() - t0,
               hist=None if res.hist is None else res.hist.cpu().numpy(),
               W=res.W, soe_block=march.soe_block)
    return _arrays.back(res.u_final, as_np), rep
