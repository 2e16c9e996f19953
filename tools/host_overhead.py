"""Host-side cost of one eager owq_gemm_small_batch call (binding + C-ABI +
launches), measured as the issue rate of a long loop of calls on a tiny layer."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2306_02272_b200 as owq, synth
d = synth.representation(512, 512, 3, 0, 3, seed=1)
L = owq.OwqLinear(d, device="cuda")
x = torch.from_numpy(synth.activations(1, 512, seed=2)).cuda()
y = torch.empty((1, 512), dtype=torch.float16, device="cuda")
ws = owq.workspace(L.shape, 1)
for _ in range(100):
    owq.owq_gemm_small_batch(L.shape, L.packed, x, y=y, ws=ws)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    owq.owq_gemm_small_batch(L.shape, L.packed, x, y=y, ws=ws)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e6 * (t1 - t0) / n:.1f} us/call, with drain {1e6 * (t2 - t0) / n:.1f} us/call")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(500):
    owq.owq_gemm_small_batch(L.shape, L.packed, x, y=y, ws=ws)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
