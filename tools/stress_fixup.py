"""Stress the stream-K fixup: a CUDA graph of back-to-back calls of mixed shapes,
batches and grids sharing one workspace, replayed many times; every replay must
give bit-identical outputs (the fixup sums pieces in a fixed order)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2306_02272_b200 as owq, synth
dev = torch.device("cuda:0")
cases = [(12288, 12288, 3, 0, 15, 1, 0), (4096, 2048, 3, 0, 9, 2, 0), (3000, 4096, 4, 128, 7, 1, 0),
         (2048, 4096, 4, 0, 3, 8, 0), (768, 768, 3, 0, 8, 1, 300), (8192, 1024, 3, 0, 5, 3, 0), (12288, 12288, 3, 0, 15, 1, 49)]
layers, xs, ys, ws_bytes = [], [], [], 0
for i, (M, K, bits, g, k, B, grid) in enumerate(cases):
    d = synth.representation(M, K, bits, g, k, seed=500 + i)
    x = synth.activations(B, K, seed=600 + i)
    L = owq.OwqLinear(d, device=dev)
    layers.append((L, grid))
    xs.append(torch.from_numpy(x).to(dev))
    ys.append(torch.empty((B, M), dtype=torch.float32, device=dev))
    ws_bytes = max(ws_bytes, owq.workspace(L.shape, B, dev, grid=grid).numel())
ws = torch.zeros(ws_bytes, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()
def chain():
    for (L, grid), x, y in zip(layers, xs, ys):
        if grid:
            owq.owq_gemm_small_batch_grid(L.shape, L.packed, x, grid, y=y, y_f32=True, ws=ws)
        else:
            owq.owq_gemm_small_batch(L.shape, L.packed, x, y=y, y_f32=True, ws=ws)
with torch.cuda.stream(s):
    chain()
torch.cuda.synchronize()
ref = [y.clone() for y in ys]
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for _ in range(4):
        chain()
bad = 0
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
for r in range(n):
    for y in ys:
        y.fill_(float("nan"))
    g.replay()
    torch.cuda.synchronize()
    for i, (y, y0) in enumerate(zip(ys, ref)):
        if not torch.equal(y, y0):
            bad += 1
            print("mismatch replay", r, "layer", i, float((y - y0).abs().max()))
slots = 512 * 16 * 128 * 4
print(f"{n} replays x {4 * len(cases)} calls: {bad} mismatches; sync prefix nonzero words: "
      f"{int(torch.count_nonzero(ws[:slots]).item())}")
