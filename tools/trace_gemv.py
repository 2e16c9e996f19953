"""Run one GEMV with OWQ_TRACE set and summarise per-CTA timelines (globaltimer ns)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
