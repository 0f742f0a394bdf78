"""ctypes binding of libtsfrac_b200.so (the C ABI in include/tsfrac_b200.h).

The product path has no CPU fallback: if the shared library is missing or
CUDA is unavailable, every device entry point raises.  Only host-side setup
(mesh, IFL column, SOE nodes — as in the reference) runs without a GPU.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Optional

import numpy as np

LIB_NAME = "libtsfrac_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

# per-instance status codes (include/tsfrac_b200.h)
ST_OK = 0
ST_NOT_CONVERGED = 1
ST_RHO_VANISHED = 2
ST_R0V_VANISHED = 3
ST_OMEGA_DEN_VANISHED = 4
ST_OMEGA_VANISHED = 5
ST_NONPOS_CURVATURE = 6
ST_KAPPA_NONPOS = 7
ST_PRECOND_NONPOS = 8

BREAKDOWN = {
    ST_RHO_VANISHED: "rho vanished",
    ST_R0V_VANISHED: "r0.v vanished",
    ST_OMEGA_DEN_VANISHED: "omega denominator vanished",
    ST_OMEGA_VANISHED: "omega vanished",
    ST_NONPOS_CURVATURE: "non-positive curvature",
}

# every symbol include/tsfrac_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "tsf_abi_version", "tsf_last_error", "tsf_plan_create", "tsf_plan_destroy",
    "tsf_plan_info", "tsf_plan_reserve", "tsf_toeplitz_matvec", "tsf_precond_solve",
    "tsf_krylov_solve", "tsf_krylov_solve_circ", "tsf_soe_push_rhs", "tsf_fids_march",
    "tsf_fft_debug", "tsf_l1_history_rhs", "tsf_half_debug",
)

P = C.c_void_p
D = C.c_double
I = C.c_int
I64 = C.c_int64


class Field(C.Structure):
    _fields_ = [("nmodes", I), ("modes", P), ("q_stride", I64), ("b_stride", I64),
                ("t_stride", I64), ("coef", P)]


class March(C.Structure):
    _fields_ = [
        ("B", I), ("M", I), ("nexp", I), ("method", I), ("precond", I), ("tol", D),
        ("max_iters", I), ("G", D), ("shift", P), ("a_mm", P), ("tau", P),
        ("soe_tab", P), ("kappa", Field), ("source", Field), ("u_buf0", P),
        ("u_buf1", P), ("W", P), ("rhs", P), ("kwork", P), ("iters", P),
        ("relres", P), ("status", P), ("hist", P), ("hist_B", I), ("m_begin", I),
        ("m_end", I), ("events", P), ("soe_block", I), ("soe_alpha", P), ("soe_beta", P),
        ("soe_ring", P),
    ]


class NativeError(RuntimeError):
    pass


_lib = None


def load(path: Optional[os.PathLike] = None):
    """Load (once) and return the CDLL; raises NativeError when absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # TSF_LIB: an alternative build of the same ABI (kernel-variant experiments)
    p = Path(path) if path else Path(os.environ.get("TSF_LIB", LIB_PATH))
    if not p.exists():
        raise NativeError(
            f"{p.name} is not built ({p}); run `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -j` — there is no CPU fallback for the device path")
    lib = C.CDLL(str(p))
    sig = {
        "tsf_abi_version": (I, []),
        "tsf_last_error": (C.c_char_p, []),
        "tsf_plan_create": (I, [C.POINTER(P), I, I, P, P, I]),
        "tsf_plan_destroy": (I, [P]),
        "tsf_plan_info": (I, [P, P]),
        "tsf_plan_reserve": (I, [P, I]),
        "tsf_toeplitz_matvec": (I, [P, I, P, P, P, D, P]),
        "tsf_precond_solve": (I, [P, I, P, P, D, D, P, P]),
        "tsf_krylov_solve": (I, [P, I, I, I, P, P, P, D, D, D, I, P, P, P, P]),
        "tsf_krylov_solve_circ": (I, [P, I, I, P, P, P, D, P, I64, D, I, P, P, P, P]),
        "tsf_soe_push_rhs": (I, [I, I, I, P, P, P, D, P, P, P, I, I, I, D, D, P, P, P]),
        "tsf_fids_march": (I, [P, C.POINTER(March), P]),
        "tsf_fft_debug": (I, [I, I, I, P, P, P]),
        "tsf_l1_history_rhs": (I, [I, I, I, P, C.c_int64, P, D, D, P, P, P]),
        "tsf_half_debug": (I, [P, I, I, P, P, D, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int):
    if rc != 0:
        msg = load().tsf_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        if rc == -3:
            raise NotImplementedError(msg)
        raise NativeError(f"tsfrac_b200 error {rc}: {msg}")


def torch_mod():
    import torch
    if not torch.cuda.is_available():
        raise NativeError("CUDA is not available: the tsfrac_b200 device path has no CPU fallback")
    return torch


def stream_ptr(stream=None, device=None) -> int:
    """The launch stream: `stream`, else torch's current stream OF `device`
    (the tensors' device — not whichever device happens to be current)."""
    torch = torch_mod()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


def ptr(t) -> Optional[int]:
    if t is None:
        return None
    return int(t.data_ptr())


class Plan:
    """Owns one native plan (tables + Krylov workspaces) on one device."""

    def __init__(self, n: int, L: int, symbol_re: np.ndarray, lam: Optional[np.ndarray],
                 device: int = 0):
        torch_mod()
        lib = load()
        self.n, self.L, self.device = int(n), int(L), int(device)
        sym = np.ascontiguousarray(symbol_re, dtype=np.float64)
        if sym.size != L:
            raise ValueError("symbol length must equal L")
        lam_c = None if lam is None else np.ascontiguousarray(lam, dtype=np.float64)
        h = P()
        check(lib.tsf_plan_create(C.byref(h), self.n, self.L, sym.ctypes.data,
                                  None if lam_c is None else lam_c.ctypes.data, self.device))
        self._h = h
        self.has_precond = lam is not None

    @property
    def handle(self):
        return self._h

    def info(self):
        out = (I64 * 5)()
        check(load().tsf_plan_info(self._h, C.addressof(out)))
        return list(out)

    def close(self):
        if getattr(self, "_h", None):
            load().tsf_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def src_sha256() -> str:
    """sha256 over the kernel sources the library is built from (csrc/, the C
    header, the Makefile): ties a profile to the CODE it measured.  nvcc's
    output is not bit-reproducible (a fresh build of the same sources has a
    different file hash), so the library file's own hash cannot do that."""
    import hashlib
    root = Path(__file__).resolve().parent
    files = sorted(p for p in (root / "csrc").rglob("*") if p.is_file())
    files += [root.parent / "include" / "tsfrac_b200.h", root.parent / "Makefile"]
    h = hashlib.sha256()
    for p in files:
        h.update(str(p.relative_to(root.parent)).encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def lib_sha256(path: Optional[os.PathLike] = None) -> str:
    """sha256 of the loaded library file (ties profiles to the build they measured)."""
    import hashlib
    p = Path(path) if path else Path(os.environ.get("TSF_LIB", LIB_PATH))
    h = hashlib.sha256()
    with open(p, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 20), b""):
            h.update(chunk)
    return h.hexdigest()
