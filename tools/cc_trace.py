"""Per-CTA timeline (globaltimer) of the last CUDA-core GEMV call of a graph of R
back-to-back calls (experiment build):
OWQ_LIB=paper_2306_02272_b200/_ab/exp.so python tools/cc_trace.py M K bits group k [R]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_02272_b200 as owq  # noqa: E402
import synth  # noqa: E402

a = [int(v) for v in sys.argv[1:]] + [4096, 4096, 3, 0, 5, 8][len(sys.argv) - 1:]
M, K, bits, group, k, R = a[:6]
d = synth.representation(M, K, bits, group, k, seed=1)
shape = owq.Shape(M, K, bits, group, k)
nb = owq.owq_packed_bytes_layout(shape, owq.OWQ_LAYOUT_CC)
ncop = max(2, min(8, -(-400_000_000 // nb)))
packs = [owq.owq_pack(shape, d, flags=owq.OWQ_PACK_LAYOUT_CC, device="cuda") for _ in range(ncop)]
x = torch.from_numpy(synth.activations(1, K, seed=2)).cuda()
y = torch.empty((1, M), dtype=torch.float16, device="cuda")
ws = owq.workspace(shape, 1)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for i in range(ncop):
        owq.owq_gemm_small_batch(shape, packs[i], x, y=y, ws=ws)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for i in range(R):
        owq.owq_gemm_small_batch(shape, packs[i % ncop], x, y=y, ws=ws)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record(); g.replay(); e1.record()
torch.cuda.synchronize()
print(f"{M}x{K} b{bits} g{group} k{k}: {e0.elapsed_time(e1) * 1e3 / R:.2f} us per call (graph of {R})")
c = np.zeros((4, 1024), dtype=np.uint64)
owq.lib().owq_exp_cc_cta(c.ctypes.data_as(ctypes.c_void_p))
n = int((c[0] > 0).sum())
c = c[:, :n].astype(np.int64)
t0 = c[0].min()
st, pw, ml, ex = [(c[i] - t0) / 1e3 for i in range(4)]
q = lambda v: " ".join(f"{np.percentile(v, p):7.2f}" for p in (0, 10, 50, 90, 100))
print(f"last call, {n} CTAs, us since the first CTA start (p0 p10 p50 p90 p100)")
print(f"  start      {q(st)}\n  x ready    {q(pw)}\n  loop done  {q(ml)}\n  exit       {q(ex)}\n  loop       {q(ml - pw)}\n  fixup      {q(ex - ml)}")
