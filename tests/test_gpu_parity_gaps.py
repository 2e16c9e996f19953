"""GPU parity (through the C-ABI) on the paths round 1 left unchecked
(VERDICT r1 "Next round" item 1):

(a) BASELINE config 3 at its real shapes -- LLaMA-7B 4096^2 (k = 4),
    11008x4096 (k = 1) and 4096x11008 (k = 4), 4-bit g128, B = 1/4/8/16
     -- which drives the grouped per-stage epilogue at B = 1 and the
    grouped batch epilogue at B > 1 through many stages per CTA;
(b) OPT-175B 12288^2 at B = 3/8/16 (MMA N = 32/64/96 with full rings);
(c) small layers forced through explicit small grids so every ring wraps many
    times (per-row and grouped scales, B = 1/3/6/11/16);
(d) x-range edges the exact digit split rests on: +-65504, subnormals, -0,
    every column large at K = 49152;
(e) zero points at both ends of the code range, weak indices {0, 1, K-1},
    adjacent weak indices, K = 65536 (the u16 index limit).

Tolerance: the north_star's 2e-3 per element with the near-zero floor of
DESIGN.md reading s16 (tests/owq_testutil.py), unchanged from round 1.
Full outputs are compared where the fp64 oracle finishes in seconds; above
that, rows are sampled so that every row-block position class (first/last row
of a 128-row block, the ragged last block) is covered and the oracle computes
them one by one (oracle.matvec_rows).
"""
import numpy as np
import pytest

import oracle as O
import synth
from owq_testutil import TOL, rel_err, rep_from_synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2306_02272_b200 as owq  # noqa: E402


@pytest.fixture(params=[owq.OWQ_LAYOUT_TC, owq.OWQ_LAYOUT_CC], ids=["tc", "cc"])
def layout(request):
    """Both device layouts: 3 = tcgen05 kind::i8 kernel, 4 = CUDA-core FFMA2 kernel."""
    return request.param


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return torch.device("cuda:0")


def sample_rows(M, n=256, seed=0):
    """Every row-block boundary class plus random rows."""
    r = np.random.default_rng(seed)
    rows = {0, 1, M - 1, M - 2}
    for rb in range(0, M, 128):
        rows.update({rb, min(M - 1, rb + 127), min(M - 1, rb + 31), min(M - 1, rb + 64)})
    rows = sorted(rows)
    if len(rows) > n:
        rows = sorted(r.choice(rows, n, replace=False).tolist() + [0, M - 1])
    extra = r.choice(M, min(M, n // 2), replace=False).tolist()
    return sorted(set(rows) | set(extra))


def gpu_run(d, x_np, dev, grid=0, y_f32=True, layout=owq.OWQ_LAYOUT_TC):
    layer = owq.OwqLinear(d, device=dev, layout=layout)
    x = torch.from_numpy(np.ascontiguousarray(x_np, np.float16)).to(dev)
    if grid:
        y = owq.owq_gemm_small_batch_grid(layer.shape, layer.packed, x, grid, y_f32=y_f32)
    else:
        y = layer(x, y_f32=y_f32)
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64)


def check(d, x, y, full=True, rows=None):
    rep = rep_from_synth(d)
    if full:
        ref = O.matvec(rep, x.astype(np.float64))
        e, eu = rel_err(y, ref)
    else:
        rows = rows if rows is not None else sample_rows(d["M"])
        ref = O.matvec_rows(rep, x.astype(np.float64), rows)
        e, eu = rel_err(y[:, rows], ref)
    assert e <= TOL, (e, eu)
    return e


# (a) BASELINE config 3: LLaMA-7B linears, 4-bit g128, k from reading s13
LLAMA7B = [(4096, 4096, 4), (11008, 4096, 1), (4096, 11008, 4)]


@pytest.mark.parametrize("B", [1, 4, 8, 16])
@pytest.mark.parametrize("M,K,k", LLAMA7B)
def test_llama7b_g128(dev, layout, M, K, k, B):
    d = synth.representation(M, K, 4, 128, k, seed=7000 + M + K + B)
    x = synth.activations(B, K, seed=B + K, outliers=d["weak_idx"])
    y = gpu_run(d, x, dev, layout=layout)
    check(d, x, y, full=(M * K <= 4096 * 4096))


# (b) OPT-175B 12288^2 at the batch sizes whose MMA N is 32 / 64 / 96
@pytest.mark.parametrize("B", [3, 8, 16])
def test_opt175b_qkvo_batch(dev, layout, B):
    M = K = 12288
    d = synth.representation(M, K, 3, 0, 15, seed=175 + B)
    x = synth.activations(B, K, seed=B, outliers=d["weak_idx"][:8])
    y = gpu_run(d, x, dev, layout=layout)
    check(d, x, y, full=False)


# (c) small layers through tiny grids: every ring wraps many times
@pytest.mark.parametrize("grid", [1, 2, 3])
@pytest.mark.parametrize("B", [1, 3, 6, 11, 16])
@pytest.mark.parametrize("bits,group", [(3, 0), (4, 128)])
def test_small_grid_rings_wrap(dev, layout, grid, B, bits, group):
    M, K, k = 300, 4000, 11
    d = synth.representation(M, K, bits, group, k, seed=grid * 31 + B * 7 + bits)
    x = synth.activations(B, K, seed=B + grid, outliers=d["weak_idx"])
    y = gpu_run(d, x, dev, grid=grid, layout=layout)
    check(d, x, y)


@pytest.mark.parametrize("grid", [1, 2, 3, 5, 7])
@pytest.mark.parametrize("group", [128, 256, 1024])
def test_grouped_batch1_per_stage_many_items(dev, layout, grid, group):
    # BASELINE config 3's B = 1 path (grouped per-stage epilogue): groups span
    # stages and CTAs, several pieces per stage, partial last group (K % g != 0)
    M, K, k = 260, 5000, 6
    d = synth.representation(M, K, 4, group, k, seed=grid + group)
    x = synth.activations(1, K, seed=grid, outliers=d["weak_idx"])
    y = gpu_run(d, x, dev, grid=grid, layout=layout)
    check(d, x, y)


# (d) x-range edges of the exact int8 digit split (x * 2^24 < 2^40)
def _edge_x(B, K, kind, seed):
    r = np.random.default_rng(seed)
    x = r.normal(size=(B, K))
    if kind == "max":
        x = np.sign(x) * 65504.0                       # every column at the fp16 maximum
    elif kind == "subnormal":
        x = r.integers(-1023, 1024, size=(B, K)) * 2.0 ** -24   # fp16 subnormals (and zeros)
    elif kind == "mixed":
        n = K // 8
        x[:, r.choice(K, n, replace=False)] = 65504.0 * np.sign(r.normal(size=(B, n)))
        x[:, r.choice(K, n, replace=False)] = 2.0 ** -24 * r.integers(-5, 6, size=(B, n))
        x[:, r.choice(K, n, replace=False)] = -0.0
    return x.astype(np.float16)


@pytest.mark.parametrize("kind", ["max", "subnormal", "mixed"])
@pytest.mark.parametrize("B", [1, 4])
def test_x_range_edges_k49152(dev, layout, kind, B):
    M, K = 256, 49152
    d = synth.representation(M, K, 3, 0, 15, seed=49)
    x = _edge_x(B, K, kind, seed=B)
    if kind == "mixed":
        assert np.any(np.signbit(x) & (x == 0))          # -0 present
    y = gpu_run(d, x, dev, layout=layout)
    check(d, x, y)


def test_negative_zero_is_zero(dev, layout):
    # x = -0 everywhere: y must be exactly +-0 (zero-filled low-bit part, weak x = 0)
    M, K = 130, 700
    d = synth.representation(M, K, 3, 0, 5, seed=3)
    x = np.full((1, K), -0.0, np.float16)
    y = gpu_run(d, x, dev, layout=layout)
    assert np.all(y == 0.0)


# (e) zero points at the code-range ends, weak-index edges, K = 65536
@pytest.mark.parametrize("bits,group", [(3, 0), (4, 128), (3, 256)])
def test_zero_point_extremes(dev, layout, bits, group):
    M, K, k = 257, 1500, 5
    d = synth.representation(M, K, bits, group, k, seed=bits + group)
    maxq = (1 << bits) - 1
    z = O.from_fp16_bits(d["zero_f16"]).copy()
    z[0::3] = 0
    z[1::3] = maxq
    d["zero_f16"] = O.fp16_bits(z)
    r = np.random.default_rng(5)
    d["codes"] = r.integers(0, maxq + 1, size=(M, K), dtype=np.uint8)   # full code range
    x = synth.activations(2, K, seed=9, outliers=d["weak_idx"])
    y = gpu_run(d, x, dev, layout=layout)
    check(d, x, y)


@pytest.mark.parametrize("K,idx", [
    (1000, [0, 1, 999]),
    (1000, [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 998, 999]),      # adjacent, a full chunk + tail
    (65536, [0, 1, 4095, 4096, 65534, 65535]),             # the u16 limit
])
def test_weak_index_edges(dev, layout, K, idx):
    M = 200
    d = synth.representation(M, K, 3, 0, len(idx), seed=K + len(idx))
    d["weak_idx"] = np.asarray(idx, np.uint16)
    x = synth.activations(3, K, seed=len(idx), outliers=d["weak_idx"])
    y = gpu_run(d, x, dev, layout=layout)
    check(d, x, y)
    # probes: x = e_j at the weak edges returns the fp16 weak column exactly
    X = np.zeros((len(idx), K), np.float16)
    for n, j in enumerate(idx):
        X[n, j] = 1.0
    for a in range(0, len(idx), 16):
        yp = gpu_run(d, X[a:a + 16], dev, layout=layout)
        ref = O.matvec(rep_from_synth(d), X[a:a + 16].astype(np.float64))
        assert np.array_equal(yp, ref)


def test_k65536_full_width(dev, layout):
    M, K = 384, 65536
    d = synth.representation(M, K, 4, 128, 9, seed=65536)
    x = synth.activations(2, K, seed=2, outliers=d["weak_idx"])
    y = gpu_run(d, x, dev, layout=layout)
    check(d, x, y)
