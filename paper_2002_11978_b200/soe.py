"""Sum-of-exponentials kernel compression and the device history state.

`build_soe` is host setup (as in the reference, soe.py:90-184): a uniform
log-lattice midpoint rule for t^{-gamma} = (1/Gamma(gamma)) int e^{-ts}
s^{gamma-1} ds with the left tail collapsed into one moment-matched node,
refined x0.85 until an a-posteriori check on a 4096-point log grid passes.
It is restated step for step so nodes/weights match the reference to
1e-13 (pinned by tests against tests/golden/setup.npz).

`FastHistory` keeps W (N_exp x n, row per exponential, soe.py:73-87) in HBM;
`history_push` and `fast_caputo_rhs` run on the device
(csrc/tsf_soe.cuh, fused in the time march).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
from scipy.special import gammaln

from . import _arrays, _native

DEFAULT_NODE_CAP = 256


class SoeConstructionError(RuntimeError):
    """Tolerance not reachable within the node cap (soe.py:48-49)."""


@dataclass(frozen=True)
class SoeApproximation:
    gamma: float
    epsilon: float
    delta: float
    T: float
    nodes: np.ndarray
    weights: np.ndarray

    @property
    def n_exp(self) -> int:
        return int(self.nodes.size)

    def evaluate(self, t) -> np.ndarray:
        tt = np.atleast_1d(np.asarray(t, dtype=float))
        return np.exp(-np.outer(tt, self.nodes)) @ self.weights


def _step_for(gamma: float, target: float) -> float:
    # aliasing error of the log-variable midpoint rule ~ 2|Gamma(gamma + 2 pi i/h)|/Gamma(gamma);
    # fixed point of y = (2/pi)(log(8 sqrt(2pi)) + (gamma-1/2) log y - lgamma(gamma) - log target)
    lg = gammaln(gamma)
    c0 = math.log(8.0 * math.sqrt(2.0 * math.pi)) - lg - math.log(target)
    y = 20.0
    for _ in range(60):
        y = (2.0 / math.pi) * (c0 + (gamma - 0.5) * math.log(max(y, 1.0)))
    return 2.0 * math.pi / y


def _lattice_nodes(gamma, eps, delta, T, h):
    lg = gammaln(gamma)
    inv_gamma_fn = math.exp(-lg)
    # tail below s = a collapses into one node; error budget eps/8
    a = (eps * gamma * math.exp(lg) / (4.0 * T * T)) ** (1.0 / (gamma + 2.0))
    j0 = math.floor(math.log(a) / h - 0.5)
    u0 = (j0 + 0.5) * h
    mass = h * inv_gamma_fn * math.exp(gamma * u0) / (1.0 - math.exp(-gamma * h))
    moment = (h * inv_gamma_fn * math.exp((gamma + 1.0) * u0)
              / (1.0 - math.exp(-(gamma + 1.0) * h)))
    s_out = [moment / mass]
    w_out = [mass]
    j = j0 + 1
    while True:
        u = (j + 0.5) * h
        sj = math.exp(u)
        wj = h * math.exp(gamma * u) * inv_gamma_fn
        s_out.append(sj)
        w_out.append(wj)
        if sj * delta > gamma + 1.0 and wj * math.exp(-min(sj * delta, 700.0)) < eps / 32.0:
            break
        j += 1
        if len(s_out) > 100_000:
            raise SoeConstructionError("right tail of the lattice does not terminate")
    return np.array(s_out), np.array(w_out)


def _passes_check(gamma, s, w, eps, delta, T) -> bool:
    grid = np.logspace(math.log10(delta), math.log10(T), 4096)
    exact = grid ** (-gamma)
    err = np.abs(exact - np.exp(-np.outer(grid, s)) @ w)
    return bool(np.all(err <= np.maximum(eps, 4.0 * np.finfo(float).eps * exact)))


def build_soe(gamma: float, epsilon: float, delta: float, T: float,
              node_cap: int = DEFAULT_NODE_CAP) -> SoeApproximation:
    """soe.py:145-184: |t^{-gamma} - sum w e^{-s t}| <= epsilon on [delta, T]."""
    if not 0.0 < gamma < 1.0:
        raise ValueError(f"gamma must lie in (0, 1), got {gamma}")
    if epsilon <= 0.0:
        raise ValueError(f"epsilon must be > 0, got {epsilon}")
    if not 0.0 < delta < T:
        raise SoeConstructionError(
            f"cutoff must satisfy 0 < delta < T, got delta={delta}, T={T}")
    h = _step_for(gamma, epsilon * delta ** gamma / 4.0)
    for _ in range(6):
        s, w = _lattice_nodes(gamma, epsilon, delta, T, h)
        if s.size > node_cap:
            raise SoeConstructionError(
                f"tolerance {epsilon:g} on [{delta:g}, {T:g}] needs {s.size} "
                f"exponentials, cap is {node_cap}")
        if _passes_check(gamma, s, w, epsilon, delta, T):
            return SoeApproximation(gamma=float(gamma), epsilon=float(epsilon),
                                    delta=float(delta), T=float(T), nodes=s, weights=w)
        h *= 0.85
    raise SoeConstructionError(f"validation failed to reach {epsilon:g} on [{delta:g}, {T:g}]")


def fast_coefficients(soe: SoeApproximation, mesh, m: int) -> np.ndarray:
    """Direct b_k (soe.py:187-206); host-side checker of the recurrence."""
    from .mesh import l1_weights
    if not 1 <= m <= mesh.M:
        raise ValueError(f"level m must lie in [1, {mesh.M}], got {m}")
    s, w = soe.nodes, soe.weights
    b = np.empty(m)
    for k in range(1, m):
        tk = mesh.tau[k - 1]
        ek = np.exp(-s * (mesh.t[m] - mesh.t[k])) * (-np.expm1(-s * tk))
        b[k - 1] = np.dot(w, ek / s) / tk
    b[m - 1] = l1_weights(mesh, soe.gamma, m).a[-1]
    return b


@dataclass
class FastHistory:
    """Accumulators W (N_exp, n); single owner (soe.py:73-87).

    `fresh(soe, n)` — the reference's call — gives W as a host numpy array, as
    the reference's does (callers index, copy and multiply it with numpy);
    `history_push` / `fast_caputo_rhs` still run on the device (the array is
    staged to the GPU and written back in place).  `fresh(soe, n, device=d)`
    keeps W resident on device d as a torch tensor (the package's own level
    loops); the batched march holds its W[B][N_exp][n] itself (scheme.py).
    """

    soe: SoeApproximation
    W: object = field(default=None)  # numpy (N_exp, n) or torch CUDA tensor (N_exp, n)
    level: int = 0

    @classmethod
    def fresh(cls, soe: SoeApproximation, n_spatial: int,
              device: Optional[int] = None) -> "FastHistory":
        if device is None:
            return cls(soe=soe, W=np.zeros((soe.n_exp, n_spatial)), level=0)
        torch = _native.torch_mod()
        return cls(soe=soe, W=torch.zeros((soe.n_exp, n_spatial), dtype=torch.float64,
                                          device=f"cuda:{device}"), level=0)


def _device_W(h: FastHistory):
    """(device tensor, write-back) for h.W: a host array is staged to cuda:0
    and copied back in place after the kernel."""
    if _arrays.is_torch(h.W):
        return h.W, None
    torch = _native.torch_mod()
    host = h.W
    if host.dtype != np.float64 or not host.flags.c_contiguous:
        raise ValueError("FastHistory.W must be a C-contiguous float64 array")
    dW = torch.from_numpy(host).to("cuda:0")
    return dW, lambda: np.copyto(host, dW.cpu().numpy())


def _coef_tables(soe: SoeApproximation, tau_push: Optional[float], tau_next: Optional[float],
                 device):
    torch = _native.torch_mod()
    s, w = soe.nodes, soe.weights
    dec = np.exp(-s * tau_push) if tau_push is not None else np.zeros_like(s)
    cof = -np.expm1(-s * tau_push) / s if tau_push is not None else np.zeros_like(s)
    hc = w * np.exp(-s * tau_next) if tau_next is not None else np.zeros_like(s)
    tab = torch.from_numpy(np.stack([dec, cof, hc])).to(device)
    return tab


def history_push(h: FastHistory, delta_u, tau_m: float) -> FastHistory:
    """W_j <- e^{-s_j tau} W_j + (delta_u/tau)(1-e^{-s_j tau})/s_j on the device.

    soe.py:209-225.  Bit-identical to numpy given identical inputs (the
    kernel disables FMA contraction and uses a true division).
    """
    if tau_m <= 0.0:
        raise ValueError(f"tau_m must be > 0, got {tau_m}")
    torch = _native.torch_mod()
    n = h.W.shape[1]
    if tuple(getattr(delta_u, 'shape', np.shape(delta_u))) != (n,):
        raise ValueError("delta_u length does not match the history width")
    W, write_back = _device_W(h)
    dev = W.device
    du, _ = _arrays.to_device(delta_u, dev.index or 0)
    tab = _coef_tables(h.soe, tau_m, None, dev)
    zero = torch.zeros(n, dtype=torch.float64, device=dev)
    # push with u = delta_u, uprev = 0 reproduces (u - 0)/tau == delta_u/tau exactly
    with torch.cuda.device(dev):
        _native.check(_native.load().tsf_soe_push_rhs(
            1, n, h.soe.n_exp, W.data_ptr(), du.data_ptr(), zero.data_ptr(),
            float(tau_m), tab[0].data_ptr(), tab[1].data_ptr(), tab[2].data_ptr(), 1, 0, 0,
            0.0, 1.0, None, None, _native.stream_ptr(device=dev)))
    if write_back:
        write_back()
    h.level += 1
    return h


def fast_caputo_rhs(h: FastHistory, a_mm: float, u_prev, gamma: float, tau_m: float):
    """(a_mm u^{m-1} - sum_j w_j e^{-s_j tau_m} W_j) / Gamma(1-gamma)  (soe.py:228-246)."""
    torch = _native.torch_mod()
    n = h.W.shape[1]
    if tuple(getattr(u_prev, 'shape', np.shape(u_prev))) != (n,):
        raise ValueError("u_prev length does not match the history width")
    W, _ = _device_W(h)
    dev = W.device
    up, as_np = _arrays.to_device(u_prev, dev.index or 0)
    tab = _coef_tables(h.soe, None, tau_m, dev)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    zero_f = torch.zeros(n, dtype=torch.float64, device=dev)
    G = math.exp(gammaln(1.0 - gamma))
    with torch.cuda.device(dev):
        _native.check(_native.load().tsf_soe_push_rhs(
            1, n, h.soe.n_exp, W.data_ptr(), up.data_ptr(), None, 0.0,
            None, None, tab[2].data_ptr(), 0, 0, 1, float(a_mm), G, zero_f.data_ptr(),
            out.data_ptr(), _native.stream_ptr(device=dev)))
    return _arrays.back(out, as_np)
