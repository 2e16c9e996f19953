"""GPU OWQ quantizer (csrc/owq_quant.cu) against the CPU
oracle's quantizer (oracle.owq_quantize), both fp64:
the weak-column selection must be identical, and so must the codes, the fp16
scale / zero and the fp16 weak values ("bit-exact weak-index
selection and codes identical on config 1").  Both follow the same algorithm in
fp64 with different summation orders; a decision could only differ where a
value falls within ~1e-12 of a rounding boundary."""
import numpy as np
import pytest

import oracle as O
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2306_02272_b200 as owq  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch.device("cuda:0")


def gpu_quantize(W, X, bits, k, group, clip, dev):
    out = owq.owq_quantize_gpu(torch.from_numpy(W).to(dev), torch.from_numpy(X).to(dev), bits, k, group=group,
                               clip=clip)
    torch.cuda.synchronize()
    return {n: (v.cpu().numpy() if hasattr(v, "cpu") else v) for n, v in out.items()}


def compare(rep, g):
    assert np.array_equal(g["weak_idx"].view(np.uint16).astype(np.int64), rep.weak_idx)
    mism = int(np.count_nonzero(g["codes"] != rep.codes))
    assert mism == 0, f"{mism} codes differ"
    assert np.array_equal(g["scale_f16"].view(np.uint16), O.fp16_bits(rep.scale))
    assert np.array_equal(g["zero_f16"].view(np.uint16), O.fp16_bits(rep.zero))
    assert np.array_equal(g["weak_val_f16"].view(np.uint16), O.fp16_bits(rep.weak_val))


def test_config1_identical_to_oracle(dev):
    # BASELINE config 1: OPT-125m-shaped 768 x 768, 3-bit per-row, k = 8, N = 2048 tokens
    W, X, ch = synth.weights_and_calib(768, 768, N=2048, n_outliers=8, seed=2306)
    rep = O.owq_quantize(W, X, 3, 8)
    g = gpu_quantize(W, X, 3, 8, 0, True, dev)
    compare(rep, g)
    assert set(ch) <= set(rep.weak_idx.tolist())


@pytest.mark.parametrize("M,K,bits,k,group,clip", [
    (96, 256, 3, 5, 0, False), (128, 512, 4, 6, 128, True), (64, 300, 4, 3, 64, True), (40, 100, 2, 0, 0, True),
])
def test_small_layers_identical(dev, M, K, bits, k, group, clip):
    W, X, ch = synth.weights_and_calib(M, K, N=4 * K, n_outliers=4, seed=M + K)
    rep = O.owq_quantize(W, X, bits, k, group=group, clip=clip)
    g = gpu_quantize(W, X, bits, k, group, clip, dev)
    compare(rep, g)


def test_dead_columns(dev):
    # a calibration channel that is always zero: H_jj = 0 -> dead (reading s2)
    W, X, ch = synth.weights_and_calib(64, 128, N=512, n_outliers=2, seed=3)
    X[[5, 77], :] = 0.0
    rep = O.owq_quantize(W, X, 3, 4)
    g = gpu_quantize(W, X, 3, 4, 0, True, dev)
    compare(rep, g)


def test_quantized_layer_runs_on_the_hot_path(dev):
    # the GPU quantizer's output packs and multiplies like the oracle's (end to end on device data)
    from owq_testutil import TOL, rel_err, rep_from_synth
    W, X, ch = synth.weights_and_calib(512, 1024, N=2048, n_outliers=6, seed=5)
    g = gpu_quantize(W, X, 3, 6, 0, True, dev)
    d = {"M": 512, "K": 1024, "bits": 3, "group": 0, "codes": g["codes"], "scale_f16": g["scale_f16"].view(np.uint16),
         "zero_f16": g["zero_f16"].view(np.uint16), "weak_idx": g["weak_idx"].view(np.uint16),
         "weak_val_f16": g["weak_val_f16"].view(np.uint16)}
    x = synth.activations(1, 1024, seed=1, outliers=ch)
    for layout in (owq.OWQ_LAYOUT_TC, owq.OWQ_LAYOUT_CC):
        L = owq.OwqLinear(d, device=dev, layout=layout, flags=owq.OWQ_PACK_STRICT)
        y = L(torch.from_numpy(x).to(dev), y_f32=True).cpu().numpy()
        assert rel_err(y, O.matvec(rep_from_synth(d), x.astype(np.float64)))[0] <= TOL
