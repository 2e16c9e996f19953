"""Summarise an ncu --set full report of owq_gemv_kernel: pipe utilisation,
stall reasons, and instructions per warp-item by opcode and source line.
python tools/ncu_analyze.py report.ncu-rep [warp_items]"""
import csv, subprocess, sys
from collections import Counter, defaultdict
rep = sys.argv[1]
W = float(sys.argv[2]) if len(sys.argv) > 2 else 73728.0
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
import ncu_csv  # noqa: E402  (unit row applied: values in bytes / seconds)
for get_d in ncu_csv.launches(rep, "owq_")[:1]:
    def get(name, d=get_d):
        v = d.get(name, float("nan"))
        return v if isinstance(v, float) else float("nan")
    print("duration us", get("gpu__time_duration.sum") * 1e6, " dram GB/s", get("dram__bytes.sum.per_second") / 1e9)
    for n in ["alu", "fma", "fmaheavy", "lsu", "adu", "cbu", "uniform", "tc", "xu"]:
        v = get(f"sm__inst_executed_pipe_{n}.avg.pct_of_peak_sustained_active")
        if v == v: print(f"  pipe {n:9s} {v:6.1f}%")
    st = [(get(n), n) for n in get_d if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
    print("  stalls:", ", ".join(f"{n[34:]}={v:.0f}" for v, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[2]
iE = hdr.index("Instructions Executed")
def num(x):
    try: return int(x)
    except Exception: return 0
c = Counter(); byline = defaultdict(Counter); linetext = {}
cur = None
for r in rows[3:]:
    if not r: continue
    if r[0] != "":
        cur = r[0]; linetext[cur] = r[1].strip(); continue
    s = r[3].strip()
    op = s.split()[0] if s else ""
    if op.startswith("@"): op = s.split()[1]
    op = op.split(".")[0]
    c[op] += num(r[iE]); byline[cur][op] += num(r[iE])
tot = sum(c.values())
print(f"instructions {tot}  per warp-item {tot / W:.1f}")
print("  " + ", ".join(f"{op}:{n / W:.1f}" for op, n in c.most_common(24)))
ALU = {"LOP3", "SHF", "ISETP", "IADD3", "SEL", "LEA", "PLOP3", "VIADDMNMX", "FSETP", "ISCADD", "PRMT", "IABS", "LOP", "MOV", "P2R", "R2P", "FLO", "POPC", "BREV"}
print("all instructions per warp-item by source line:")
for v, l in sorted(((sum(ops.values()), l) for l, ops in byline.items()), reverse=True)[:30]:
    print(f"  L{l:>4s} {v / W:6.2f}  {linetext.get(l, '')[:90]}")
print("ALU-pipe ops per warp-item by source line:")
al = sorted(((sum(v for k, v in ops.items() if k in ALU), l) for l, ops in byline.items()), reverse=True)[:25]
for v, l in al:
    print(f"  L{l:>4s} {v / W:6.2f}  {linetext.get(l, '')[:90]}")
