"""Setup-path timing: host stages of one large-n run and
the native plan creation (tables permuted / uploaded by tsf_plan_create).

    python tools/setup_timing.py [log2 n ...]   (default 20 24)
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2002_11978_b200 as P  # noqa: E402
from paper_2002_11978_b200 import toeplitz as TZ  # noqa: E402


def main():
    import torch
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    for lg in [int(a) for a in sys.argv[1:]] or [20, 24]:
        n = 1 << lg
        r = {"n": n}
        t = time.perf_counter()
        d = P.build_ifl(1.2, 1.6, 1.0, n + 1)
        r["build_ifl_s"] = time.perf_counter() - t
        t = time.perf_counter()
        op = P.build_toeplitz(d.first_col)
        r["build_toeplitz_symbol_fft_s"] = time.perf_counter() - t
        t = time.perf_counter()
        lam = np.fft.fft(TZ.strang_first_column(d.first_col)).real
        r["strang_eigs_fft_s"] = time.perf_counter() - t
        t = time.perf_counter()
        soe = P.build_soe(0.7, 1e-12, (1.0 / 256) ** ((2 - 0.7) / 0.7), 1.0)
        r["build_soe_s"] = time.perf_counter() - t
        t = time.perf_counter()
        pl = op.plan            # hashing, symbol/Strang tables, native plan (tsf_plan_create)
        torch.cuda.synchronize()
        r["plan_create_s"] = time.perf_counter() - t
        x = np.random.default_rng(0).standard_normal(n)
        t = time.perf_counter()
        y = P.toeplitz_matvec(op, x)
        r["first_matvec_s"] = time.perf_counter() - t
        t = time.perf_counter()
        y = P.toeplitz_matvec(op, x)
        r["second_matvec_s"] = time.perf_counter() - t
        print(json.dumps(r), flush=True)
        del pl, op
        TZ.clear_plans()


if __name__ == "__main__":
    main()
