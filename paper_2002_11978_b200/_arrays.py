"""numpy <-> torch CUDA conversion for the drop-in entry points.

Entry points accept numpy arrays (copied to the device, result copied back
as numpy, matching the reference's return types) or torch CUDA tensors
(zero-copy, result returned as a torch tensor on the same device).
"""

from __future__ import annotations

import numpy as np

from . import _native


def is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def to_device(x, device: int = 0):
    """Return (contiguous fp64 CUDA tensor, came_from_numpy)."""
    torch = _native.torch_mod()
    if is_torch(x):
        t = x
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        if not t.is_cuda:
            t = t.to(f"cuda:{device}")
        return t.contiguous(), False
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(a).to(f"cuda:{device}", non_blocking=False), True


def back(t, as_numpy: bool):
    if as_numpy:
        return t.detach().cpu().numpy()
    return t
