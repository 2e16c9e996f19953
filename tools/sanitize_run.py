"""Small calls of every kernel of libowq, for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): each result is also checked against the
oracle so a run that "passes" the tool also computed the right thing.
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2306_02272_b200 as owq  # noqa: E402
import synth  # noqa: E402
from owq_testutil import TOL, dict_from_stored, rel_err, rep_from_synth, synthetic_stored  # noqa: E402

dev = torch.device("cuda:0")
fails = 0


def check(name, y, ref):
    global fails
    e = rel_err(y, ref)[0]
    ok = e <= TOL
    fails += not ok
    print(f"{name:40s} err {e:.2e} {'ok' if ok else 'FAIL'}", flush=True)


cases = [(300, 700, 3, 0, 11, 1), (300, 700, 3, 0, 11, 3), (260, 1100, 4, 128, 6, 1), (130, 640, 4, 128, 5, 2)]
for M, K, bits, group, k, B in cases:
    d = synth.representation(M, K, bits, group, k, seed=M + K + B)
    x = synth.activations(B, K, seed=B, outliers=d["weak_idx"])
    ref = O.matvec(rep_from_synth(d), x.astype(np.float64))
    xt = torch.from_numpy(x).to(dev)
    for lay in (owq.OWQ_LAYOUT_TC, owq.OWQ_LAYOUT_CC):
        L = owq.OwqLinear(d, device=dev, layout=lay)
        for grid in (0, 2):
            if grid:
                y = owq.owq_gemm_small_batch_grid(L.shape, L.packed, xt, grid, y_f32=True)
            else:
                y = L(xt, y_f32=True)
            check(f"gemv L{lay} {M}x{K} b{bits} g{group} B{B} grid{grid}", y.cpu().numpy(), ref)
        if lay == owq.OWQ_LAYOUT_TC and K % 8 == 0:
            y = owq.owq_gemm_batch_f16(L.shape, L.packed, xt, y_f32=True, ws=L.ws)
            check(f"batch_f16 {M}x{K} b{bits} g{group} B{B}", y.cpu().numpy(), ref)
            if group == 0:
                y = owq.owq_gemm_prefill(L.shape, L.packed, xt, y_f32=True)
                check(f"prefill {M}x{K} b{bits} B{B}", y.cpu().numpy(), ref)
rep = synthetic_stored(200, 900, 4, 128, 7, "storage", seed=1)
x = synth.activations(2, 900, seed=2, outliers=rep.weak_idx)
L = owq.OwqLinear(dict_from_stored(rep), device=dev)
check("colmap storage-favored g128 B2", L(torch.from_numpy(x).to(dev), y_f32=True).cpu().numpy(),
      O.matvec_stored(rep, x.astype(np.float64)))
W, X, ch = synth.weights_and_calib(64, 256, N=512, n_outliers=2, seed=3)
q = owq.owq_quantize_gpu(torch.from_numpy(W).to(dev), torch.from_numpy(X).to(dev), 3, 4)
r = O.owq_quantize(W, X, 3, 4)
ok = np.array_equal(q["codes"].cpu().numpy(), r.codes)
fails += not ok
print(f"{'quantizer 64x256 k4':40s} codes {'identical' if ok else 'DIFFER'}")
torch.cuda.synchronize()
print("sanitize_run:", "FAIL" if fails else "all results correct")
sys.exit(1 if fails else 0)
