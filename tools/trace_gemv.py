"""Run one GEMV with OWQ_TRACE set and summarise per-CTA timelines (globaltimer ns)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 2 and sys.argv[1] == "--file":   # summarise an existing dump (tools/trace_graph.py)
    import numpy as np
    t = np.fromfile(sys.argv[2], dtype=np.uint64).reshape(-1, 256).astype(np.int64)
    M = K = bits = "?"
else:
    path = "gpurun_out/trace.bin"
    if os.path.exists(path): os.remove(path)
    os.environ["OWQ_TRACE"] = path
    import numpy as np, torch
    import paper_2306_02272_b200 as owq, synth
    a = [int(v) for v in sys.argv[1:]] + [12288, 12288, 3, 0, 15, 1][len(sys.argv) - 1:]
    M, K, bits, group, k, B = a[:6]
    d = synth.representation(M, K, bits, group, k, seed=1)
    L = owq.OwqLinear(d, device="cuda")
    x = torch.from_numpy(synth.activations(B, K, seed=2)).cuda()
    for _ in range(3):
        L(x)
    torch.cuda.synchronize()
    t = np.fromfile(path, dtype=np.uint64).reshape(3, -1, 256)[-1].astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
def rel(v): return (v - t0) / 1e3
print(f"{M}x{K} b{bits} CTAs={len(t)}  (us from first CTA start; median over CTAs)")
print(f" start med {np.median(rel(t[:,0])):.2f}  fin-in {np.median(rel(t[:,50])):.2f}  fin-out {np.median(rel(t[:,56])):.2f}  end {np.median(rel(t[:,62])):.2f} max {rel(t[:,62]).max():.2f}")
print(" stage  prod_issue  dec_full dec_aempty  dec_done mma_afull  mma_done  epi_done")
for kk in range(0, 16):
    cols = [64 + kk, 192 + kk, 18 + kk, 96 + kk, 224 + kk, 128 + kk, 160 + kk]
    vals = []
    for c in cols:
        v = t[:, c]; v = v[v > 0]
        vals.append(f"{np.median(rel(v)):9.2f}" if len(v) else "        -")
    print(f" {kk:5d} " + " ".join(vals))
print(" MMA warps (cycles, mean over CTAs): wait afull", [int(t[:, 1 + w].mean()) for w in range(4)],
      " issue", [int(t[:, 5 + w].mean()) for w in range(4)], " commit(wg3)", int(t[:, 9].mean()), " MMAs(wg3)", int(t[:, 52].mean()))
print(" MMA waits (cycles, mean): tready", [int(t[:, 42 + w].mean()) for w in range(4)], " dempty", [int(t[:, 46 + w].mean()) for w in range(4)])
print(" epilogue (grouped per-stage mode) cycles: ring", int(t[:, 53].mean()), " dfull", int(t[:, 54].mean()), " ld", int(t[:, 55].mean()), " combine", int(t[:, 57].mean()))
print(" kernel cycles ~", int((np.median(t[:, 62]) - np.median(t[:, 0])) * 1.9))
order = np.argsort(-t[:, 62])
print(" slowest CTAs: idx  start  fin-in  fin-out  end   (us)   last-stage epi_done")
for c in order[:6]:
    eds = [v for v in t[c, 160:192] if v > 0]
    print(f"   {c:4d} {rel(t[c,0]):6.2f} {rel(t[c,50]):7.2f} {rel(t[c,56]):8.2f} {rel(t[c,62]):6.2f}    stages {len(eds)}  epi_done " +
          " ".join(f"{rel(v):.2f}" for v in eds))
print(" group ends of the slowest CTAs: [stage-seen, S done, sz done, D+combine done] (us)")
for c in order[:4]:
    print("   ", c, [[round(rel(t[c, 18 + 6 * j + i]), 2) for i in range(4)] for j in range(2) if t[c, 18 + 6 * j] > 0])
med = [[float(np.median(rel(t[t[:, 18 + 6 * j] > 0, 18 + 6 * j + i]))) for i in range(4)] for j in range(2)]
print(" median group-end timeline:", [[round(v, 2) for v in m] for m in med])
st, en = rel(t[:, 0]), rel(t[:, 62])
du = en - st
q = [0, 10, 50, 90, 100]
print(" start  pct", [round(float(np.percentile(st, v)), 2) for v in q])
print(" end    pct", [round(float(np.percentile(en, v)), 2) for v in q])
print(" dur    pct", [round(float(np.percentile(du, v)), 2) for v in q], " corr(start, end) %.2f" % float(np.corrcoef(st, en)[0, 1]))
if t[:, 61].max() > 0:
    nrb = int(t[:, 61].max())
    spans = sorted((int(t[c, 58]), int(t[c, 59]), c) for c in range(len(t)))
    def role(c):
        i0, i1 = int(t[c, 58]), int(t[c, 59])
        r0, r1 = i0 // nrb, (i1 - 1) // nrb
        parts = []
        for r in range(r0, r1 + 1):
            a, b = max(i0, r * nrb), min(i1, (r + 1) * nrb)
            whole = a == r * nrb and b == (r + 1) * nrb
            summer = a == r * nrb and not whole
            parts.append("W" if whole else ("S" if summer else "p") + f"{b - a}")
        return " ".join(parts)
    order = np.argsort(du)
    print(" fastest / slowest CTAs: idx start end dur | parts (W whole rb, S summer piece, p other piece, items)")
    for c in list(order[:5]) + list(order[-6:]):
        print(f"   {c:4d} {st[c]:6.2f} {en[c]:6.2f} {du[c]:6.2f} | {role(c):24s} fin-in {rel(t[c,50]):6.2f} fin-out {rel(t[c,56]):6.2f}"
              f" fin1 {rel(t[c,51]):6.2f}-{rel(t[c,60]):6.2f} open2 {rel(t[c,17]) if t[c,17] else -1:6.2f} groups [seen, S, D, comb] " + str([round(rel(t[c, 18 + 6 * j + i]), 2) for j in range(4) for i in range(4) if t[c, 18 + 6 * j] > 0][-8:]))
