"""Per-stage timeline of CTA (0, 0) of the batched f16 kernel (experiment build):
OWQ_LIB=paper_2306_02272_b200/_ab/exp.so python tools/sb_trace.py M K bits group k B"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_02272_b200 as owq  # noqa: E402
import synth  # noqa: E402

a = [int(v) for v in sys.argv[1:]] + [12288, 12288, 3, 0, 15, 8][len(sys.argv) - 1:]
M, K, bits, group, k, B = a[:6]
d = synth.representation(M, K, bits, group, k, seed=1)
shape = owq.Shape(M, K, bits, group, k)
P = owq.owq_pack(shape, d, device="cuda")
x = torch.from_numpy(synth.activations(B, K, seed=2)).cuda()
y = torch.empty((B, M), dtype=torch.float16, device="cuda")
ws = owq.workspace(shape, min(B, 16))
for _ in range(3):
    owq.owq_gemm_batch_f16(shape, P, x, y=y, ws=ws)
torch.cuda.synchronize()
t = np.zeros((8, 64), dtype=np.int64)
owq.lib().owq_exp_sb_trace(t.ctypes.data_as(ctypes.c_void_p))
names = ["prod.empty", "dec.full", "dec.afull", "mma.afull", "mma.bfull", "ld.empty", "ld.arrive", "epi.dfull"]
t0 = t[t > 0].min()
print("cycles since the first stamp; columns:", " ".join(names))
for l in range(64):
    if not t[:, l].any():
        break
    print(f"{l:3d} " + " ".join(f"{(v - t0) if v else -1:9d}" for v in t[:, l]))

# per-CTA start / after-pdl_wait / exit (globaltimer ns) of one call timed alone and of
# the last call of a CUDA graph of 8 back-to-back calls
def cta_times(tag):
    c = np.zeros((3, 1024), dtype=np.uint64)
    owq.lib().owq_exp_sb_cta(c.ctypes.data_as(ctypes.c_void_p))
    n = int((c[0] > 0).sum())
    c = c[:, :n].astype(np.int64)
    t0 = c[0].min()
    st, pw, ex = (c[0] - t0) / 1e3, (c[1] - t0) / 1e3, (c[2] - t0) / 1e3
    q = lambda v: " ".join(f"{np.percentile(v, p):7.1f}" for p in (0, 10, 50, 90, 100))
    print(f"[{tag}] {n} CTAs, us since the first CTA start (p0 p10 p50 p90 p100)")
    print(f"  start      {q(st)}\n  pdl done   {q(pw)}\n  exit       {q(ex)}\n  duration   {q(ex - st)}\n  work       {q(ex - pw)}")


torch.cuda.synchronize()
c = torch.zeros(1 << 26, dtype=torch.uint8, device="cuda")
c.fill_(1); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); owq.owq_gemm_batch_f16(shape, P, x, y=y, ws=ws); e1.record(); torch.cuda.synchronize()
print(f"single call: {e0.elapsed_time(e1) * 1e3:.1f} us")
cta_times("single")
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    owq.owq_gemm_batch_f16(shape, P, x, y=y, ws=ws)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    for _ in range(8):
        owq.owq_gemm_batch_f16(shape, P, x, y=y, ws=ws)
g.replay(); torch.cuda.synchronize()
with torch.cuda.stream(s):
    e0.record(); g.replay(); e1.record()
torch.cuda.synchronize()
print(f"graph: {e0.elapsed_time(e1) * 1e3 / 8:.1f} us per call")
cta_times("graph, last call")
