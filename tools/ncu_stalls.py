"""Where the warps of one ncu --set full launch wait: stall samples per SASS
opcode and the top SASS lines (with their stall-reason columns).

    python tools/ncu_stalls.py REPORT.ncu-rep [top_n]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
iS, iA, iN, iE = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Warp Stall Sampling (Not-issued Samples)"), hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or h.startswith("Stall") or "smsp__pcsamp" in h]


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


by_op, total = Counter(), 0.0
lines = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    src = r[iS].strip()
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    a = num(r[iA])
    total += a
    by_op[op] += a
    lines.append((a, r[0][-5:], src[:70], num(r[iE])))
print(f"stall samples: {total:.0f}")
print("by opcode: " + ", ".join(f"{op} {v / total * 100:.1f}%" for op, v in by_op.most_common(15)))
for a, addr, src, ex in sorted(lines, reverse=True)[:top]:
    print(f"{a / total * 100:5.1f}%  {addr}  {src}")
