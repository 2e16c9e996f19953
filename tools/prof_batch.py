"""Device time per call of the batched paths on one layer shape:
python tools/prof_batch.py M K bits group k B [iters]  (tcgen05 i8 kernel vs the f16 batch kernel)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_02272_b200 as owq  # noqa: E402
import synth  # noqa: E402

a = [int(v) for v in sys.argv[1:]] + [12288, 12288, 3, 0, 15, 8, 24][len(sys.argv) - 1:]
M, K, bits, group, k, B, iters = a[:7]
d = synth.representation(M, K, bits, group, k, seed=1)
shape = owq.Shape(M, K, bits, group, k)
nb = owq.owq_packed_bytes(shape)
ncop = max(1, min(8, -(-400_000_000 // nb)))
packs = [owq.owq_pack(shape, d, device="cuda") for _ in range(ncop)]
x = torch.from_numpy(synth.activations(B, K, seed=2)).cuda()
y = torch.empty((B, M), dtype=torch.float16, device="cuda")
ws = owq.workspace(shape, min(B, 16))
alg = bits * M * K / 8 + 4 * M * (1 if group == 0 else -(-K // group)) + 2 * M * k + 2 * k + 2 * K * B + 2 * M * B
for name, fn in (("i8", owq.owq_gemm_small_batch), ("f16", owq.owq_gemm_batch_f16)):
    if name == "i8" and B > 16:
        continue
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for P in packs:
            fn(shape, P, x, y=y, ws=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(iters):
            fn(shape, packs[i % ncop], x, y=y, ws=ws)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(); g.replay(); e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    print(f"{name:4s} {M}x{K} b{bits} g{group} k{k} B{B}: {us:.2f} us, {alg / us / 1e3:.0f} GB/s")
