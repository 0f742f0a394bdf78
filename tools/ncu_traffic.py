"""DRAM traffic of the level-solve and SOE kernels of one bench workload,
from an ncu capture of THIS build (run on the GPU box):

    python tools/ncu_traffic.py --workload cfg2 [--batch 1024] [--steps 3]

runs `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,...` over
`bench.py --workload W` with TSF_SOLVE_GRAPH=0 (the same kernels launched one
by one, so every launch is captured), sums the bytes of the solve kernels and
of the SOE kernels over the timed levels, normalises by the instance-
iterations the bench line reports, and records the result with the
library's and the kernel sources' sha256 in profiles/ncu_traffic.json —
bench.py quotes roofline.traffic only when one of them matches what it runs.
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SOLVE = ("k_solve_begin", "k_bicg_v", "k_bicg_t", "k_bicg_h", "k_krylov_persist", "k_cg_iter", "k_lcol_fwd", "k_lcol_inv",
         "k_lrow", "k_lsc", "k_lel_", "k_lspec", "k_lloop_cond", "k_loop_cond", "k_set_int",
         "k_hcol_fwd", "k_hcol_inv", "k_hrow_strang", "k_hrow_mv", "k_hspec")
SOE = ("k_soe",)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "ncu_traffic.json"))
    args = ap.parse_args()
    from paper_2002_11978_b200 import _native
    env = dict(os.environ, TSF_SOLVE_GRAPH="0")   # (the persistent solve is one kernel anyway)
    bench = [sys.executable, str(ROOT / "bench.py"), "--workload", args.workload, "--steps",
             str(args.steps), "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-matvec"]
    if args.batch:
        bench += ["--batch", str(args.batch)]
    log = ROOT / "gpurun_out" / f"ncu_traffic_{args.workload}.csv"
    log.parent.mkdir(exist_ok=True)
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "--cache-control", "none", "--csv", "--log-file",
           str(log)] + bench
    out = subprocess.run(cmd, env=env, capture_output=True, text=True)
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    if out.returncode != 0 or not line:
        raise SystemExit(f"ncu run failed: {out.returncode}\n{out.stderr[-2000:]}")
    bl = json.loads(line[-1])
    txt = log.read_text().splitlines()
    start_row = next(i for i, ln in enumerate(txt) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[start_row:]))))
    # kernels of the timed region: the last `steps` levels' launches (the
    # bench's warm-up levels run first); take every launch after the
    # (warmup)th SOE launch, i.e. group the list by level via the SOE kernels
    per = {}
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        per.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        per[key]["unit_" + r["Metric Name"]] = r["Metric Unit"]
    launches = [(int(k[0]), k[1], v) for k, v in per.items()]
    launches.sort()
    soe_idx = [i for i, (_, nm, _) in enumerate(launches) if any(s in nm for s in SOE)]
    warm = 3
    start = soe_idx[warm] if len(soe_idx) > warm else 0

    def nbytes(v):
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            u = v.get("unit_" + m, "byte").lower()
            mul = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
            tot += v.get(m, 0.0) * mul
        return tot
    solve = sum(nbytes(v) for _, nm, v in launches[start:] if any(s in nm for s in SOLVE))
    soe = sum(nbytes(v) for _, nm, v in launches[start:] if any(s in nm for s in SOE))
    K = bl["steps"]
    its = bl["kernels"]["level_solve"]["iterations_per_launch"] * K
    rec = {"lib_sha256": _native.lib_sha256(), "src_sha256": _native.src_sha256(),
           "B": bl["config"]["instances_per_gpu"],
           "dram_bytes_per_instance_iteration": solve / its,
           "soe_dram_bytes_per_level": soe / K,
           "algorithmic_bytes_per_instance_iteration": 216 * bl["config"]["n"],
           "capture": f"ncu dram__bytes_read/write.sum --cache-control none, {K} levels of "
                      f"bench.py --workload {args.workload} (B = {bl['config']['instances_per_gpu']}), "
                      "TSF_SOLVE_GRAPH=0"}
    p = Path(args.out)
    allr = json.loads(p.read_text()) if p.exists() else {}
    allr[args.workload] = rec
    p.write_text(json.dumps(allr, indent=1) + "\n")
    print(json.dumps({args.workload: rec}))


if __name__ == "__main__":
    main()
