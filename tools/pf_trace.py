"""Per-stage timeline of CTA (0, 0) and per-CTA start / exit of the prefill kernel
(experiment build): OWQ_LIB=paper_2306_02272_b200/_ab/exp.so python tools/pf_trace.py M K tokens"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_02272_b200 as owq  # noqa: E402
import synth  # noqa: E402

a = [int(v) for v in sys.argv[1:]] + [12288, 12288, 2048, 15][len(sys.argv) - 1:]
M, K, B, k = a[:4]
d = synth.representation(M, K, 3, 0, k, seed=1)
shape = owq.Shape(M, K, 3, 0, k)
P = owq.owq_pack(shape, d, device="cuda")
x = torch.from_numpy(synth.activations(B, K, seed=2)).cuda()
y = torch.empty((B, M), dtype=torch.float16, device="cuda")
for _ in range(2):
    owq.owq_gemm_prefill(shape, P, x, y=y)
torch.cuda.synchronize()
c = torch.zeros(1 << 26, dtype=torch.uint8, device="cuda")
c.fill_(1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); owq.owq_gemm_prefill(shape, P, x, y=y); e1.record(); torch.cuda.synchronize()
print(f"single call {e0.elapsed_time(e1) * 1e3:.1f} us")
t = np.zeros((8, 256), dtype=np.int64)
owq.lib().owq_exp_pf_trace(t.ctypes.data_as(ctypes.c_void_p))
names = ["prod.empty", "dec.full", "dec.arrive", "mma.afull", "mma.bfull", "ld.empty", "ld.arrive"]
t0 = t[t > 0].min()
print("CTA (0,0) cycles since the first stamp:", " ".join(names))
for l in list(range(0, 12)) + list(range(180, 192)):
    if not t[:, l].any():
        continue
    print(f"{l:3d} " + " ".join(f"{(v - t0) if v else -1:9d}" for v in t[:7, l]))
e = t[7]
print("epilogue of CTA (0,0), cycles after dfull: staged", e[0] - e[15], " gathered", e[1] - e[15], " passes",
      [int(e[2 + i] - e[15]) for i in range(8)])
cc = np.zeros((4, 2048), dtype=np.uint64)
owq.lib().owq_exp_pf_cta(cc.ctypes.data_as(ctypes.c_void_p))
n = int((cc[0] > 0).sum())
cc = cc[:, :n].astype(np.int64)
t0 = cc[0].min()
q = lambda v: " ".join(f"{np.percentile(v, p):8.1f}" for p in (0, 10, 50, 90, 100))
st, pw, df, ex = [(cc[i] - t0) / 1e3 for i in range(4)]
print(f"{n} CTAs, us since the first CTA start (p0 p10 p50 p90 p100)")
print(f"  start      {q(st)}\n  pdl done   {q(pw)}\n  dfull      {q(df)}\n  exit       {q(ex)}\n  mainloop   {q(df - pw)}\n  epilogue   {q(ex - df)}")
