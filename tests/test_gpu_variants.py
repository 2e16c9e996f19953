"""GPU parity of the NEXT-4 variants: act-order and
storage-favored representations -- a code matrix in stored column
order plus a column map, blob layout 4, the CUDA-core kernel -- against the
oracle's matvec_stored (oracle/owq_variants.py).  Same tolerance as every
GPU parity test (2e-3 per element with the reading-s16 floor)."""
import numpy as np
import pytest

import oracle as O
import synth
from owq_testutil import TOL, dict_from_stored, rel_err, synthetic_stored

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2306_02272_b200 as owq  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch.device("cuda:0")


def run(rep, x, dev, grid=0):
    d = dict_from_stored(rep)
    layer = owq.OwqLinear(d, device=dev)
    assert layer.layout == owq.OWQ_LAYOUT_CC
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float16)).to(dev)
    if grid:
        y = owq.owq_gemm_small_batch_grid(layer.shape, layer.packed, xt, grid, y_f32=True)
    else:
        y = layer(xt, y_f32=True)
    torch.cuda.synchronize()
    return y.cpu().numpy().astype(np.float64), layer


@pytest.mark.parametrize("act_order", [False, True])
@pytest.mark.parametrize("mode", ["latency", "storage"])
@pytest.mark.parametrize("group", [0, 128])
def test_oracle_quantized_variants(dev, act_order, mode, group):
    # the oracle's own OWQ quantizer in the variant, then the GPU hot path on its output
    W, X, ch = synth.weights_and_calib(256, 512, N=1024, n_outliers=6, seed=11 + group)
    rep = O.owq_quantize_variant(W, X, 4 if group else 3, 6, group=group, act_order=act_order, mode=mode)
    x = synth.activations(2, 512, seed=3, outliers=ch)
    y, _ = run(rep, x, dev)
    e, eu = rel_err(y, O.matvec_stored(rep, x.astype(np.float64)))
    assert e <= TOL, (e, eu)


@pytest.mark.parametrize("mode", ["latency", "storage"])
@pytest.mark.parametrize("M,K,bits,group,k,B", [
    (4096, 4096, 4, 128, 4, 1), (4096, 4096, 4, 128, 4, 3), (11008, 4096, 4, 128, 1, 2),
    (4096, 11008, 4, 128, 4, 1), (3000, 2000, 3, 0, 15, 1), (700, 5000, 3, 256, 7, 4),
])
def test_synthetic_variants_real_shapes(dev, mode, M, K, bits, group, k, B):
    rep = synthetic_stored(M, K, bits, group, k, mode, seed=M + K + B)
    x = synth.activations(B, K, seed=B, outliers=rep.weak_idx)
    y, _ = run(rep, x, dev)
    e, eu = rel_err(y, O.matvec_stored(rep, x.astype(np.float64)))
    assert e <= TOL, (e, eu)


@pytest.mark.parametrize("grid", [1, 2, 5])
def test_variants_small_grids(dev, grid):
    rep = synthetic_stored(300, 3000, 4, 128, 9, "storage", seed=grid)
    x = synth.activations(1, 3000, seed=grid, outliers=rep.weak_idx)
    y, _ = run(rep, x, dev, grid=grid)
    e, _ = rel_err(y, O.matvec_stored(rep, x.astype(np.float64)))
    assert e <= TOL


def test_variant_probes_bit_exact(dev):
    # x = e_j: weak j -> the fp16 weak column; mapped j at stored position p -> s (q - z) exactly
    rep = synthetic_stored(130, 600, 3, 128, 5, "storage", seed=9)
    js = [int(j) for j in rep.weak_idx] + [int(rep.colmap[p]) for p in (0, 1, 31, 32, 127, 128, 500, rep.Ks - 1)]
    X = np.zeros((len(js), 600), np.float16)
    for n, j in enumerate(js):
        X[n, j] = 1.0
    for a in range(0, len(js), 4):
        y, _ = run(rep, X[a:a + 4], dev)
        assert np.array_equal(y, O.matvec_stored(rep, X[a:a + 4].astype(np.float64)))


def test_latency_and_storage_agree(dev):
    # the same quantization stored both ways: identical products (zero-filled columns add 0)
    lat = synthetic_stored(512, 2048, 4, 128, 8, "latency", seed=4)
    sto = O.stored_from_rep(lat)
    x = synth.activations(1, 2048, seed=4, outliers=lat.weak_idx)
    y1, _ = run(lat, x, dev)
    y2, _ = run(sto, x, dev)
    ref = O.matvec_stored(sto, x.astype(np.float64))
    assert rel_err(y1, ref)[0] <= TOL and rel_err(y2, ref)[0] <= TOL
