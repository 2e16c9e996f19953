"""Batched GEMV on tensor cores with the exact fp16 (q - z) A operand
(owq_gemm_batch_f16) against the fp64 oracle: BASELINE
config 3 (LLaMA-7B 4-bit g128, B = 4 / 8 / 16), OPT-175B 12288^2 at B = 8 / 16
(sampled rows), ragged batches, split-K over several CTAs per row-block."""
import numpy as np
import pytest

import oracle as O
import synth
from owq_testutil import TOL, rel_err, rep_from_synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2306_02272_b200 as owq  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch.device("cuda:0")


def run(d, x, dev, y_f32=True):
    L = owq.OwqLinear(d, device=dev, layout=owq.OWQ_LAYOUT_TC)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float16)).to(dev)
    y = owq.owq_gemm_batch_f16(L.shape, L.packed, xt, y_f32=y_f32, ws=L.ws)
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("B", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("M,K,k", [(4096, 4096, 4), (11008, 4096, 1), (4096, 11008, 4)])
def test_llama7b_g128(dev, M, K, k, B):
    d = synth.representation(M, K, 4, 128, k, seed=M + K + B)
    x = synth.activations(B, K, seed=B, outliers=d["weak_idx"])
    y = run(d, x, dev)
    rep = rep_from_synth(d)
    if M * K <= 4096 * 4096:
        ref = O.matvec(rep, x.astype(np.float64))
        e, eu = rel_err(y, ref)
    else:
        rows = sorted(set([0, 127, 128, M - 1] + list(np.random.default_rng(0).choice(M, 200, replace=False))))
        e, eu = rel_err(y[:, rows], O.matvec_rows(rep, x.astype(np.float64), rows))
    assert e <= TOL, (e, eu)


@pytest.mark.parametrize("B", [3, 8, 16, 24, 32])
def test_opt175b_per_row(dev, B):
    M = K = 12288
    d = synth.representation(M, K, 3, 0, 15, seed=B)
    x = synth.activations(B, K, seed=B, outliers=d["weak_idx"][:8])
    y = run(d, x, dev)
    rows = sorted(set([0, 127, 128, M - 1] + list(np.random.default_rng(1).choice(M, 200, replace=False))))
    e, eu = rel_err(y[:, rows], O.matvec_rows(rep_from_synth(d), x.astype(np.float64), rows))
    assert e <= TOL, (e, eu)


@pytest.mark.parametrize("M,K,bits,group,k,B", [
    (300, 4000, 3, 0, 11, 5), (130, 640, 4, 128, 3, 7), (257, 1024, 3, 256, 5, 2), (64, 64, 3, 0, 0, 16),
    (512, 1024, 4, 128, 3, 5), (384, 2048, 3, 128, 4, 32),   # groups of two super-steps, ragged rows, B = 32
])
def test_small_and_ragged(dev, M, K, bits, group, k, B):
    d = synth.representation(M, K, bits, group, k, seed=M + B)
    x = synth.activations(B, K, seed=B, outliers=d["weak_idx"])
    y = run(d, x, dev)
    e, eu = rel_err(y, O.matvec(rep_from_synth(d), x.astype(np.float64)))
    assert e <= TOL, (e, eu)


@pytest.mark.parametrize("B", [4, 9, 16])
def test_small_batch_routes_grouped(dev, B):
    """owq_gemm_small_batch with grouped scales at B >= 4 runs this kernel (DESIGN.md
    §6.5): its result equals owq_gemm_batch_f16's bit for bit and the oracle's within
    the bound."""
    M, K, k = 1100, 2048, 3
    d = synth.representation(M, K, 4, 128, k, seed=40 + B)
    x = synth.activations(B, K, seed=50 + B, outliers=d["weak_idx"])
    L = owq.OwqLinear(d, device=dev, layout=owq.OWQ_LAYOUT_TC)
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float16)).to(dev)
    a = owq.owq_gemm_small_batch(L.shape, L.packed, xt, y_f32=True, ws=L.ws).cpu().numpy()
    b = owq.owq_gemm_batch_f16(L.shape, L.packed, xt, y_f32=True, ws=L.ws).cpu().numpy()
    assert np.array_equal(a, b)
    e, eu = rel_err(a.astype(np.float64), O.matvec(rep_from_synth(d), x.astype(np.float64)))
    assert e <= TOL, (e, eu)


def test_probes_and_repeat_deterministic(dev):
    M, K, k = 256, 1024, 4
    d = synth.representation(M, K, 4, 128, k, seed=3)
    js = list(d["weak_idx"]) + [0, 1, 127, 128, 1023]
    X = np.zeros((len(js), K), np.float16)
    for n, j in enumerate(js):
        X[n, j] = 1.0
    y1 = run(d, X, dev)
    assert np.array_equal(y1, O.matvec(rep_from_synth(d), X.astype(np.float64)))
    x = synth.activations(8, K, seed=4, outliers=d["weak_idx"])
    a, b = run(d, x, dev), run(d, x, dev)
    assert np.array_equal(a, b)
