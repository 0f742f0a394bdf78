"""Shared helpers for the test suite (golden fixture loading, tolerances)."""

from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"

_cache = {}


def golden(name: str):
    if name not in _cache:
        path = GOLDEN / f"{name}.npz"
        if not path.exists():
            pytest.skip(f"golden fixture {path.name} not generated")
        _cache[name] = dict(np.load(path))
    return _cache[name]


def rel_err(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def cfg0_fields():
    """BASELINE.json configs[0] coefficient fields (numpy callables)."""
    kappa = lambda x, t: 1.0 + 0.5 * np.sin(np.pi * x) * np.exp(-t)  # noqa: E731
    source = lambda x, t: (1.0 + t) * np.sin(np.pi * x)  # noqa: E731
    initial = lambda x: (1.0 - x * x) ** 2  # noqa: E731
    return kappa, source, initial
