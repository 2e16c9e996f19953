"""Summarise an ncu report: key throughput metrics, stall reasons, top stalled opcodes."""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
d = dict(zip(r[0], r[2] if len(r) > 2 else r[1]))
def f(v):
    try: return float(str(v).replace(',', ''))
    except Exception: return 0.0
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'smsp__warps_active.avg.per_cycle_active',
        'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg.per_second', 'launch__registers_per_thread', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
for k in keys:
    print(f"{k:70s} {d.get(k)}")
st = [(k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), f(v))
      for k, v in d.items() if 'average_warps_issue_stalled' in k and 'per_issue_active' in k]
print("stalls/issue:", ", ".join(f"{k}:{v:.2f}" for k, v in sorted(st, key=lambda kv: -kv[1])[:10]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; data = rows[2:]
isrc = hdr.index("Source"); iall = hdr.index("Warp Stall Sampling (All Samples)"); iex = hdr.index("Instructions Executed")
cols = {h: i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h}
tot = sum(f(x[iall]) for x in data) or 1
agg = collections.Counter(); aggs = collections.defaultdict(collections.Counter); exe = collections.Counter()
for x in data:
    t = x[isrc].split()
    if not t: continue
    op = (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
    agg[op] += f(x[iall]); exe[op] += f(x[iex])
    for h, i in cols.items(): aggs[op][h] += f(x[i])
print(f"samples {tot:.0f}; executed warp-instr {sum(exe.values()):.0f}")
for op, w in agg.most_common(12):
    print(f"  {op:9s} {100*w/tot:5.1f}% exec {exe[op]:>9.0f}  " + ", ".join(f"{h[6:]}:{v:.0f}" for h, v in aggs[op].most_common(3)))
