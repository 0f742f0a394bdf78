"""Key ncu metrics of one or more .ncu-rep files side by side (first kernel
in each): duration, pipes, shared/L1 wavefronts, DRAM bytes, stall split.
    python tools/ncu_summary.py A.ncu-rep [B.ncu-rep ...]"""
import csv
import subprocess
import sys

KEYS = [
    ("duration us", "gpu__time_duration.sum"),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("FP64 pipe %", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
    ("LSU data wavefronts % elapsed", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
    ("shared wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    ("shared bank conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("global ld requests", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
    ("global ld sectors", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
    ("instructions", "smsp__inst_executed.sum"),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("dram read", "dram__bytes_read.sum"),
    ("dram write", "dram__bytes_write.sum"),
    ("registers", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    h, units, vals = rows[0], rows[1], rows[2]
    return {k: (v, u) for k, u, v in zip(h, units, vals)}


def main():
    reps = [load(r) for r in sys.argv[1:]]
    print("| metric | " + " | ".join(sys.argv[1:]) + " |")
    print("|---" * (len(reps) + 1) + "|")
    for name, key in KEYS:
        cells = [f"{r[key][0]} {r[key][1]}".strip() if key in r else "-" for r in reps]
        print(f"| {name} | " + " | ".join(cells) + " |")
    stall = sorted({k for r in reps for k in r if k.startswith("smsp__average_warps_issue_stalled_")
                    and k.endswith("_per_issue_active.ratio")})
    for k in stall:
        vals = [float(r[k][0]) if k in r else 0.0 for r in reps]
        if max(vals) >= 0.3:
            nm = k.replace("smsp__average_warps_issue_stalled_", "stall ").replace(
                "_per_issue_active.ratio", "")
            print(f"| {nm} | " + " | ".join(f"{v:.2f}" for v in vals) + " |")


if __name__ == "__main__":
    main()
