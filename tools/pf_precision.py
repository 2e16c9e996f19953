"""Prefill (no K split) error against the fp64 oracle as K grows: the fp32 TMEM
accumulator over the whole K loop.  python tools/pf_precision.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2306_02272_b200 as owq  # noqa: E402
import synth  # noqa: E402
from owq_testutil import rel_err, rep_from_synth  # noqa: E402

M, B = 1024, 128
for bits, K in [(4, 2048), (4, 4096), (4, 6144), (4, 8192), (4, 11008), (4, 16384), (3, 12288), (3, 24576), (3, 49152)]:
    d = synth.representation(M, K, bits, 0, 4, seed=K + bits)
    x = synth.activations(B, K, seed=7, outliers=d["weak_idx"])
    L = owq.OwqLinear(d, device="cuda", layout=owq.OWQ_LAYOUT_TC)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float16)).cuda()
    rows = list(range(0, M, 4))
    ref = O.matvec_rows(rep_from_synth(d), x.astype(np.float64), rows)
    y = owq.owq_gemm_prefill(L.shape, L.packed, xt, y_f32=True).cpu().numpy().astype(np.float64)
    ws = owq.prefill_workspace(L.shape, B)
    line = f"bits {bits} K {K:6d}: no split {rel_err(y[:, rows], ref)[0]:.2e}"
    if ws is not None:
        ys = owq.owq_gemm_prefill(L.shape, L.packed, xt, y_f32=True, ws=ws).cpu().numpy().astype(np.float64)
        line += f"  split {rel_err(ys[:, rows], ref)[0]:.2e}"
    print(line, flush=True)
