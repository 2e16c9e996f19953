"""Device time of the prefill GEMM (NEXT-2): python tools/prof_prefill.py M K B [iters] [ws: 1 = with a workspace (K split)]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_02272_b200 as owq  # noqa: E402
import synth  # noqa: E402

a = [int(v) for v in sys.argv[1:]] + [12288, 12288, 2048, 10, 0][len(sys.argv) - 1:]
M, K, B, iters, use_ws = a[:5]
k = 15
d = synth.representation(M, K, 3, 0, k, seed=1)
shape = owq.Shape(M, K, 3, 0, k)
packed = owq.owq_pack(shape, d, device="cuda")
x = torch.from_numpy(synth.activations(B, K, seed=2)).cuda()
y = torch.empty((B, M), dtype=torch.float16, device="cuda")
ws = owq.prefill_workspace(shape, B) if use_ws else None
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    owq.owq_gemm_prefill(shape, packed, x, y=y, ws=ws)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for _ in range(iters):
        owq.owq_gemm_prefill(shape, packed, x, y=y, ws=ws)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(); g.replay(); e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / iters * 1e3
flops = 2.0 * M * K * B
print(f"prefill {M}x{K} B={B}{' ws' if ws is not None else ''}: {us:.1f} us, {flops / us / 1e6:.1f} TFLOP/s (dense-equivalent 2MKB)")
