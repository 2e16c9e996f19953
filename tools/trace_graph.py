"""Trace the LAST of R back-to-back GEMV launches replayed from a CUDA graph
(OWQ_TRACE + OWQ_TRACE_DEFER), i.e. the per-CTA timeline in the steady state
of the bench, then summarise it with tools/trace_gemv.py's printer.
python tools/trace_graph.py [M K bits group k B R]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = "gpurun_out/trace.bin"
os.environ["OWQ_TRACE"] = path
os.environ["OWQ_TRACE_DEFER"] = "1"
import numpy as np, torch
import paper_2306_02272_b200 as owq, synth
a = [int(v) for v in sys.argv[1:]] + [12288, 12288, 3, 0, 15, 1, 6][len(sys.argv) - 1:]
M, K, bits, group, k, B, R = a[:7]
d = synth.representation(M, K, bits, group, k, seed=1)
shape = owq.Shape(M, K, bits, group, k)
packed = [owq.owq_pack(shape, d, device="cuda") for _ in range(max(2, min(8, -(-400_000_000 // owq.owq_packed_bytes(shape)))))]
x = torch.from_numpy(synth.activations(B, K, seed=2)).cuda()
y = torch.empty((B, M), dtype=torch.float16, device="cuda")
ws = owq.workspace(shape, B)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for i in range(4):
        owq.owq_gemm_small_batch(shape, packed[i % len(packed)], x, y=y, ws=ws)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for i in range(R):
        owq.owq_gemm_small_batch(shape, packed[i % len(packed)], x, y=y, ws=ws)
g.replay(); g.replay()
torch.cuda.synchronize()
lib = ctypes.CDLL(owq.LIB_PATH)
lib.owq_debug_trace_dump.argtypes = [ctypes.c_char_p]
assert lib.owq_debug_trace_dump(path.encode()) == 0
sys.argv = [sys.argv[0], "--file", path]
import runpy
runpy.run_path(os.path.join(os.path.dirname(__file__), "trace_gemv.py"), run_name="__main__")
