"""IFL Toeplitz first column — host setup (ifl.py:27-115 of the reference).

The diagonal's long positive series is summed with math.fsum (exactly
rounded), which agrees with the reference's Kahan loop (ifl.py:60-70) to
the last bit or one ulp while running in C instead of a Python loop (the
reference loop takes 7 s at N = 2^24).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
from scipy.special import gammaln


@dataclass(frozen=True)
class IflDiscretization:
    alpha: float
    mu: float
    nu: float
    kappa_mu: int
    l: float
    N: int
    h: float
    c_norm: float
    scale: float
    first_col: np.ndarray

    def dense(self) -> np.ndarray:
        from scipy.linalg import toeplitz
        return toeplitz(self.first_col)

    def interior_points(self) -> np.ndarray:
        """x_i = -l + i h, i = 1..N-1 (ifl.py:43-45)."""
        return -self.l + self.h * np.arange(1, self.N)


def normalization_constant(alpha: float) -> float:
    """c_{1,alpha} (ifl.py:48-57)."""
    if not 0.0 < alpha < 2.0:
        raise ValueError(f"alpha must lie in (0, 2), got {alpha}")
    return (2.0 ** (alpha - 1.0) * alpha
            * math.exp(gammaln((alpha + 1.0) / 2.0) - gammaln(1.0 - alpha / 2.0))
            / math.sqrt(math.pi))


def build_ifl(alpha: float, mu: float, l: float, N: int) -> IflDiscretization:
    """First column of the order-(N-1) symmetric Toeplitz IFL matrix (ifl.py:73-115)."""
    if not 0.0 < alpha < 2.0:
        raise ValueError(f"alpha must lie in (0, 2), got {alpha}")
    if not alpha < mu <= 2.0:
        raise ValueError(f"mu must lie in (alpha, 2], got mu={mu}, alpha={alpha}")
    if N < 3:
        raise ValueError(f"N must be >= 3, got {N}")
    if l <= 0.0:
        raise ValueError(f"half-width l must be > 0, got {l}")
    nu = mu - alpha
    kmu = 2 if mu == 2.0 else 1
    h = 2.0 * l / N
    cn = normalization_constant(alpha)
    scale = cn / (nu * h ** alpha)
    lv = np.arange(2.0, N)
    terms = ((lv + 1.0) ** nu - (lv - 1.0) ** nu) / lv ** mu
    diag = (math.fsum(terms.tolist())
            + (N ** nu - (N - 1.0) ** nu) / N ** mu
            + (2.0 ** nu + kmu - 1.0)
            + 2.0 * nu / (alpha * N ** alpha))
    col = np.empty(N - 1)
    col[0] = scale * diag
    col[1] = -scale * (2.0 ** nu + kmu - 1.0) / 2.0
    kv = np.arange(2.0, N - 1)
    col[2:] = -scale * ((kv + 1.0) ** nu - (kv - 1.0) ** nu) / (2.0 * kv ** mu)
    return IflDiscretization(alpha=float(alpha), mu=float(mu), nu=float(nu), kappa_mu=kmu,
                             l=float(l), N=int(N), h=h, c_norm=cn, scale=scale,
                             first_col=col)
