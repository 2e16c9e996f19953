"""Graph timing of mixed layer sequences (are shape transitions expensive?)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2306_02272_b200 as owq, synth
D = 12288
spec = {"q": (D, D, 15), "k": (D, D, 15), "v": (D, D, 15), "o": (D, D, 15), "f1": (4 * D, D, 3), "f2": (D, 4 * D, 15)}
L = {}
for i, (n, (M, K, k)) in enumerate(spec.items()):
    d = synth.representation(M, K, 3, 0, k, seed=10 + i)
    sh = owq.Shape(M, K, 3, 0, k)
    L[n] = dict(shape=sh, packed=owq.owq_pack(sh, d, device="cuda"),
                x=torch.from_numpy(synth.activations(1, K, seed=20 + i)).cuda(),
                y=torch.empty((1, M), dtype=torch.float16, device="cuda"), ws=owq.workspace(sh, 1), bytes=3 * M * K / 8)
    del d
s = torch.cuda.Stream()
def call(l):
    owq.owq_gemm_small_batch(l["shape"], l["packed"], l["x"], y=l["y"], ws=l["ws"])
def timed(seq, R=20):
    with torch.cuda.stream(s):
        for n in seq: call(L[n])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(R):
            for n in seq: call(L[n])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g.replay(); e0.record(); g.replay(); e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / R
for seq, R in [(["q", "k", "v", "o", "f1", "f2"], 20), (["q", "k", "v", "o", "f1", "f2"], 50), (["q", "k", "v", "o", "f1", "f2"], 5)]:
    t = timed(seq, R)
    print(f"{'+'.join(seq):22s} {t:8.2f} us per sequence  ({t / len(seq):6.2f} us per call)")
