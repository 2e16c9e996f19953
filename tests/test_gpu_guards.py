"""Out-of-bounds write guards (compute-sanitizer is refused on this pool --
profiles/r2_compute_sanitizer_refused.txt -- so every kernel entry point is run
with guard bands after its output and its workspace, filled with a sentinel,
and the guards must come back untouched).  Outputs are checked against the
oracle too, so a kernel cannot pass by writing nothing."""
import numpy as np
import pytest

import oracle as O
import synth
from owq_testutil import TOL, rel_err, rep_from_synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2306_02272_b200 as owq  # noqa: E402

SENT = 0x7FC0DEAD   # a NaN bit pattern no kernel writes
GUARD = 4096


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch.device("cuda:0")


def guarded(n, dev, dtype):
    buf = torch.full((n + GUARD,), 0, dtype=torch.int32, device=dev)
    buf[:] = SENT
    return buf


@pytest.mark.parametrize("path,B,group", [
    ("tc", 1, 0), ("tc", 3, 0), ("tc", 1, 128), ("cc", 1, 0), ("cc", 3, 128), ("cc", 6, 0),
    ("f16", 5, 0), ("f16", 9, 128), ("prefill", 40, 0),
])
def test_no_write_outside_outputs(dev, path, B, group):
    M, K, k = 200 if group == 0 else 257, 1024, 5
    bits = 3 if group == 0 else 4
    d = synth.representation(M, K, bits, group, k, seed=B + group)
    x = synth.activations(B, K, seed=B, outliers=d["weak_idx"])
    lay = owq.OWQ_LAYOUT_CC if path == "cc" else owq.OWQ_LAYOUT_TC
    L = owq.OwqLinear(d, device=dev, layout=lay)
    ybuf = guarded(B * M, dev, torch.float32)
    y = ybuf[:B * M].view(torch.float32).view(B, M)
    nws = L.ws.numel()
    wsbuf = torch.zeros(nws + GUARD * 4, dtype=torch.uint8, device=dev)
    wsbuf[nws:] = 0xA5
    ws = wsbuf[:nws]
    xt = torch.from_numpy(x).to(dev)
    if path in ("tc", "cc"):
        owq.owq_gemm_small_batch(L.shape, L.packed, xt, y=y, y_f32=True, ws=ws)
    elif path == "f16":
        owq.owq_gemm_batch_f16(L.shape, L.packed, xt, y=y, y_f32=True, ws=ws)
    else:
        owq.owq_gemm_prefill(L.shape, L.packed, xt, y=y, y_f32=True)
    torch.cuda.synchronize()
    assert bool((ybuf[B * M:] == SENT).all()), "write past y"
    assert bool((wsbuf[nws:] == 0xA5).all()), "write past the workspace"
    e, _ = rel_err(y.cpu().numpy().astype(np.float64), O.matvec(rep_from_synth(d), x.astype(np.float64)))
    assert e <= TOL
