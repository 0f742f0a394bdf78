"""Noise floor of the reference itself on BASELINE configs[1] (test infrastructure).

Runs the UNMODIFIED reference march (n = 16384, M = 1024, tol 1e-12) with
only its FFT engine swapped (tsfrac.fourier.fft/ifft: numpy pocketfft ->
scipy.fft, both correctly-rounded-quality FFTs) and compares per-step
BiCGSTAB iterations and u^64 / u^M with tests/golden/cfg1.npz (the stock
run).  The resulting spread is what any second FFT implementation (ours
included) must be allowed; tests/test_gpu_large.py gates on it.

    python oracle/engine_swap_floor.py   # writes tests/golden/cfg1_floor.json
"""
from __future__ import annotations

import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))

COMBOS = [(g, a) for g in (0.3, 0.5, 0.8) for a in (0.5, 1.0, 1.5, 1.9)]


def _one(ga):
    import scipy.fft as sf
    from gen_golden import _import_reference, _march
    from tsf_testlib import cfg0_fields
    g, a = ga
    tsfrac = _import_reference()
    import tsfrac.fourier as fourier
    import tsfrac.toeplitz as tz
    fourier.fft = lambda x: sf.fft(x)
    fourier.ifft = lambda x: sf.ifft(x)
    tz.fourier = fourier
    from tsfrac.scheme import ProblemSpec
    kappa, source, initial = cfg0_fields()
    spec = ProblemSpec(gamma=g, alpha=a, l=1.0, T=1.0, kappa=kappa, source=source,
                       initial=initial)
    hist, rep, its, rel = _march(tsfrac, spec, 1024, (2.0 - g) / g, 16385, 1e-12, 1e-12)
    return its, hist[64], hist[-1]


def main():
    gold = np.load(ROOT / "tests" / "golden" / "cfg1.npz")
    out = {}
    with ProcessPoolExecutor(max_workers=min(len(COMBOS), os.cpu_count() or 1)) as ex:
        for (g, a), (its, u64, uM) in zip(COMBOS, ex.map(_one, COMBOS)):
            tag = f"cfg1_g{int(g * 10)}_a{int(a * 10)}"
            d = its - gold[f"{tag}_its"]
            rl2 = lambda x, y: float(np.linalg.norm(x - y) / np.linalg.norm(y))  # noqa: E731
            out[tag] = {"within1": float(np.mean(np.abs(d) <= 1)),
                        "within2": float(np.mean(np.abs(d) <= 2)),
                        "mean_d": float(d.mean()), "max_abs_d": int(np.abs(d).max()),
                        "rel_l2_u64": rl2(u64, gold[f"{tag}_u64"]),
                        "rel_l2_uM": rl2(uM, gold[f"{tag}_uM"])}
            print(tag, out[tag], flush=True)
    (ROOT / "tests" / "golden" / "cfg1_floor.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
