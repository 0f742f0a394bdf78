"""Like tools/ncu_lines.py for a report holding several kernels: map the
SASS stall samples of kernel #idx (0-based, report order) onto source lines.

    python tools/ncu_lines_multi.py REPORT DISASM MANGLED idx [top]
"""
import csv
import re
import subprocess
import sys
from collections import Counter

rep, dis, kname, idx = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
        continue
    if cur is not None:
        cur.append(r)
blk = blocks[idx]
h, data = blk[0], blk[1:]
ci = {k: i for i, k in enumerate(h)}
base = int(data[0][ci["Address"]], 16)
lines = open(dis).read().split("\n")
start = [i for i, l in enumerate(lines) if f".text.{kname}" in l][0]
cur, off2line = None, {}
for l in lines[start + 3:]:
    if l.startswith("//---------------------"):
        break
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
    m2 = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m2 and cur:
        off2line[int(m2.group(1), 16)] = cur
agg, agg_l = Counter(), Counter()
for r in data:
    off = int(r[ci["Address"]], 16) - base
    s = float(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    ls = float(r[ci["stall_long_sb"]] or 0)
    key = off2line.get(off, ("?", 0))
    agg[key] += s
    agg_l[key] += ls
tot = sum(agg.values())
print(f"total samples {tot:.0f}, long-scoreboard {sum(agg_l.values()) / tot:.1%}")
for k, v in agg.most_common(top):
    print(f"{k[0]}:{k[1]:<5} {v / tot:6.1%}  long_sb {agg_l[k] / tot:6.1%}")
