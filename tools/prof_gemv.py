"""Device-timed single-layer GEMV: N launches captured in one CUDA graph,
rotating over enough packed copies that the working set exceeds L2.
python tools/prof_gemv.py [M K bits group k B iters layout]   (layout 3 = tcgen05, 4 = CUDA-core)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2306_02272_b200 as owq, synth
a = [int(v) for v in sys.argv[1:]] + [12288, 12288, 3, 0, 15, 1, 10, 3][len(sys.argv) - 1:]
M, K, bits, group, k, B, iters, layout = a[:8]
flags = owq.OWQ_PACK_LAYOUT_CC if layout == 4 else 0
d = synth.representation(M, K, bits, group, k, seed=1)
shape = owq.Shape(M, K, bits, group, k)
nbytes = owq.owq_packed_bytes_layout(shape, layout)
ncopies = max(1, min(8, -(-400_000_000 // nbytes)))        # > 3x L2
packed = [owq.owq_pack(shape, d, flags=flags, device="cuda") for _ in range(ncopies)]
x = torch.from_numpy(synth.activations(B, K, seed=2)).cuda()
y = torch.empty((B, M), dtype=torch.float16, device="cuda")
ws = owq.workspace(shape, B)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for i in range(2 * ncopies):
        owq.owq_gemm_small_batch(shape, packed[i % ncopies], x, y=y, ws=ws)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for i in range(iters):
        owq.owq_gemm_small_batch(shape, packed[i % ncopies], x, y=y, ws=ws)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(); g.replay(); e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / iters * 1e3
alg = bits * M * K / 8 + 4 * M * (1 if group == 0 else -(-K // group)) + 2 * M * k + 2 * k + 2 * K * B + 2 * M * B
print(f"L{layout} {M}x{K} b{bits} g{group} k{k} B{B}: {us:.2f} us/launch, {alg / us / 1e3:.0f} GB/s (graph, {ncopies} rotating copies)")
