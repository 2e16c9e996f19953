"""Wall time of the GPU OWQ quantizer (NEXT-1) per layer shape, fp64, synthetic
W / calibration X (N = 2048 tokens).  python tools/quant_time.py M K [bits k group]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_02272_b200 as owq  # noqa: E402

a = [int(v) for v in sys.argv[1:]] + [768, 768, 3, 8, 0][len(sys.argv) - 1:]
M, K, bits, k, group = a[:5]
g = torch.Generator(device="cuda").manual_seed(1)
W = torch.randn((M, K), dtype=torch.float64, device="cuda", generator=g) * 0.02
X = torch.randn((K, 2048), dtype=torch.float64, device="cuda", generator=g)
X[:8] *= 50.0
owq.owq_quantize_gpu(W, X, bits, k, group=group)   # warm-up (kernel attributes, first launches)
torch.cuda.synchronize()
t0 = time.perf_counter()
owq.owq_quantize_gpu(W, X, bits, k, group=group)
torch.cuda.synchronize()
print(f"quantize {M}x{K} b{bits} k{k} g{group} N=2048: {time.perf_counter() - t0:.3f} s")
