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
t = np.fromfile(path, dtype=np.uint64).reshape(3, -1, 64)[-1].astype(np.int64)
live = t[:, 0] > 0
t = t[live]
t0 = t[:, 0].min()
def q(col, name):
    v = t[:, col]; v = v[v > 0]
    if len(v): print(f" {name:24s} min {(v.min()-t0)/1e3:7.2f} med {(np.median(v)-t0)/1e3:7.2f} max {(v.max()-t0)/1e3:7.2f}  (n={len(v)})")
print(f"{M}x{K} b{bits} CTAs={live.sum()} stages/CTA {t[:,63].min()}..{t[:,63].max()} (us from first CTA start)")
q(0, "start"); q(1, "init done"); q(2, "first full")
for kk in range(8): q(35 + kk, f"producer issue {kk}")
for kk in [0, 1, 2, 3, 4, 8, 12, 16, 24, 31]: q(3 + kk, f"stage {kk} done")
for c, n in zip(range(50, 57), ["fin in", "fin sync1", "fin partial st", "fin atomic", "fin sync2", "fin reads", "fin out"]): q(c, n)
q(62, "end")
iv = []
for c in range(len(t)):
    st = t[c, 3:3 + min(32, t[c, 63])]
    st = st[st > 0]
    iv += list(np.diff(st) / 1e3)
if iv: print(f" stage interval us: p10 {np.percentile(iv,10):.3f} med {np.median(iv):.3f} p90 {np.percentile(iv,90):.3f}")
