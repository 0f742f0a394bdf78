"""Spread of the configs[1] iteration-count statistics under rounding-level
reformulations of the SOE history term alone (test infrastructure, CPU).

The oracle march (numpy restatement of tsfrac.run_fids, pinned to the
reference) is run with its history term H = (w e^{-s tau}) @ W replaced by
mathematically identical forms, and per-level iteration counts / u^M are
compared with the stock reference run (tests/golden/cfg1.npz):
  gemv-rev   : the same dot with the exponentials summed in reverse order
  blocked-K  : the device's blocked schedule (W at block bases + du terms,
               paper_2002_11978_b200.scheme.soe_block_tables)
The spread of mean(d) across these is the statistical floor the GPU march
test's bias gate must allow (tests/test_gpu_large.py).

    python tools/soe_perturb_floor.py  [writes tests/golden/cfg1_soe_floor.json]
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
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

COMBOS = [(0.3, 1.5), (0.5, 1.5), (0.8, 1.5), (0.3, 1.9)]
MODES = ["gemv-rev", "blocked-8", "blocked-4"]


def _run(job):
    (g, a), mode = job
    import oracle.tsfrac_oracle as O   # patch the module fids_step resolves names in
    from paper_2002_11978_b200.scheme import soe_block_tables
    from tsf_testlib import cfg0_fields
    M, N = 1024, 16385
    r = (2.0 - g) / g
    if mode == "gemv-rev":
        O.soe_history_term = lambda W, s, w, tau: (w * np.exp(-s * tau))[::-1] @ W[::-1]
    else:
        K = int(mode.split("-")[1])
        t, tau = O.graded_mesh(M, r, 1.0)
        s, w = O.soe_build(g, 1e-12, (1.0 / M) ** r, 1.0)
        tab = np.empty((M, 3, s.size))
        for m in range(M):
            dec = np.exp(-s * tau[m])
            tab[m] = dec, -np.expm1(-s * tau[m]) / s, w * dec
        alpha, beta = soe_block_tables(tab, K)
        st = {"m": 0, "Wb": None, "du": {}}
        push0 = O.soe_push

        def push(W, s_, du, tau_m):
            st["du"][st["m"]] = du / tau_m
            push0(W, s_, du, tau_m)

        def hist(W, s_, w_, tau_m):
            st["m"] += 1
            m = st["m"]
            mb = K * ((m - 1) // K)
            if m - 1 == mb:
                st["Wb"] = W.copy()
            H = alpha[m - 1] @ st["Wb"]
            for q in range(m - 1 - mb):
                H = H + beta[m - 1, q] * st["du"][mb + 1 + q]
            return H
        O.soe_push = push
        O.soe_history_term = hist
    k, f, phi = cfg0_fields()
    rec = O.fids_march(g, a, 1.0, 1.0, M, r, N, k, f, phi, epsilon=1e-12, tol=1e-12)
    return rec.iterations, rec.hist[-1]


def main():
    gold = np.load(ROOT / "tests" / "golden" / "cfg1.npz")
    jobs = [(c, m) for c in COMBOS for m in MODES]
    out = {}
    with ProcessPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
        for ((g, a), mode), (its, uM) in zip(jobs, ex.map(_run, jobs)):
            tag = f"cfg1_g{int(g * 10)}_a{int(a * 10)}"
            d = its - gold[f"{tag}_its"]
            rl2 = float(np.linalg.norm(uM - gold[f"{tag}_uM"]) / np.linalg.norm(gold[f"{tag}_uM"]))
            out.setdefault(tag, {})[mode] = {
                "within1": float(np.mean(np.abs(d) <= 1)), "mean_d": float(d.mean()),
                "std_d": float(d.std()), "rel_l2_uM": rl2}
            print(tag, mode, out[tag][mode], flush=True)
    (ROOT / "tests" / "golden" / "cfg1_soe_floor.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
