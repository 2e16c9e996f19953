"""GPU parity of the CUDA path (through the C-ABI) against the CPU oracle.

Tolerance (BASELINE.json north_star): relative error <= 2e-3 per output element
(fp32 accumulation vs the fp64 oracle), with the near-zero floor of DESIGN.md
reading s16.  Packing, unpacking and index work are bit-exact; probes with a
closed-form answer are bit-exact too.
"""
import numpy as np
import pytest

import oracle as O
import synth
from owq_testutil import TOL, rel_err, rep_from_synth, synth_from_rep

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


def run(d, x_np, dev, y_f32=True, grid=0, layout=owq.OWQ_LAYOUT_TC):
    layer = owq.OwqLinear(d, device=dev, layout=layout)
    x = torch.from_numpy(np.ascontiguousarray(x_np, np.float16)).to(dev)
    if grid:
        y = owq.owq_gemm_small_batch_grid(layer.shape, layer.packed, x, grid, y_f32=y_f32)
    else:
        y = layer(x, y_f32=y_f32)
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64), layer


SHAPES = [
    # (M, K, bits, group, k)             what it covers
    (768, 768, 3, 0, 8),                 # BASELINE config 1
    (100, 200, 3, 0, 5),                 # ragged rows / columns / k tail
    (64, 64, 3, 0, 0),                   # one super-step, no weak columns
    (1, 1, 3, 0, 1),                     # degenerate: one weight, weak
    (130, 1100, 4, 128, 9),              # 4-bit g128, partial last group
    (4096, 4096, 3, 0, 5),               # OPT-6.7B qkvo
    (512, 2048, 4, 1024, 3),             # g1024
    (192, 3000, 3, 0, 153),              # many weak columns (3.1-bit style), 10 full chunks + tail
    (64, 5000, 3, 0, 136),               # two weak units
]


@pytest.mark.parametrize("M,K,bits,group,k", SHAPES)
def test_gemv_parity_vs_oracle(dev, layout, M, K, bits, group, k):
    d = synth.representation(M, K, bits, group, k, seed=M * 7 + K)
    rep = rep_from_synth(d)
    x = synth.activations(1, K, seed=K, outliers=d["weak_idx"][:8])
    y, _ = run(d, x, dev, layout=layout)
    y_ref = O.matvec(rep, x.astype(np.float64))
    e, eu = rel_err(y, y_ref)
    assert e <= TOL, (e, eu)


@pytest.mark.parametrize("B", [2, 3, 8, 9, 16])
@pytest.mark.parametrize("M,K,bits,group,k", [(256, 1024, 4, 128, 4), (300, 700, 3, 0, 11)])
def test_small_batch_parity(dev, layout, B, M, K, bits, group, k):
    d = synth.representation(M, K, bits, group, k, seed=B + M)
    rep = rep_from_synth(d)
    x = synth.activations(B, K, seed=B * 3, outliers=d["weak_idx"])
    y, _ = run(d, x, dev, layout=layout)
    y_ref = O.matvec(rep, x.astype(np.float64))
    assert y.shape == (B, M)
    e, _ = rel_err(y, y_ref)
    assert e <= TOL


def test_fp16_output(dev, layout):
    d = synth.representation(333, 1500, 3, 0, 7, seed=5)
    x = synth.activations(4, 1500, seed=6, outliers=d["weak_idx"])
    y16, _ = run(d, x, dev, y_f32=False, layout=layout)
    y_ref = O.matvec(rep_from_synth(d), x.astype(np.float64))
    e, _ = rel_err(y16, y_ref)
    assert e <= TOL


def test_oracle_quantizer_output_config1(dev, layout):
    # BASELINE config 1 end to end: OWQ quantization by the oracle (768x768, k=8),
    # then the GPU hot path on the oracle's representation.
    W, X, ch = synth.weights_and_calib(768, 768, N=2048, n_outliers=8, seed=2306)
    rep = O.owq_quantize(W, X, 3, 8)
    d = synth_from_rep(rep)
    x = synth.activations(1, 768, seed=2307, outliers=ch)
    y, layer = run(d, x, dev, layout=layout)
    e, _ = rel_err(y, O.matvec(rep, x.astype(np.float64)))
    assert e <= TOL
    # strict packing accepts it (codes of weak columns already equal z)
    owq.owq_pack(layer.shape, d, flags=owq.OWQ_PACK_STRICT, device=dev)


@pytest.mark.parametrize("bits,group", [(3, 0), (4, 128)])
def test_device_unpack_bit_exact(dev, layout, bits, group):
    M, K, k = 200, 1500, 6
    d = synth.representation(M, K, bits, group, k, seed=9)
    shape = owq.Shape(M, K, bits, group, k)
    packed = owq.owq_pack(shape, d, device=dev, flags=owq.OWQ_PACK_LAYOUT_CC if layout == owq.OWQ_LAYOUT_CC else 0)
    codes = owq.owq_unpack_codes(shape, packed).cpu().numpy()
    expect = d["codes"].copy()
    z = O.from_fp16_bits(d["zero_f16"]).astype(np.uint8)
    for j in d["weak_idx"]:
        expect[:, j] = z[:, j // group if group else 0]
    assert np.array_equal(codes, expect)


@pytest.mark.parametrize("bits,group", [(3, 0), (4, 128)])
def test_probes_bit_exact(dev, layout, bits, group):
    # x = e_j: weak j -> y = v[:, t] exactly; non-weak j -> y_i = s_i (q_ij - z_i) exactly
    # (fp16 s times an integer <= 15 is exact in fp32).  Covers index, layout, zero fill.
    M, K, k = 130, 600, 5
    d = synth.representation(M, K, bits, group, k, seed=11)
    rep = rep_from_synth(d)
    layer = owq.OwqLinear(d, device=dev, layout=layout)
    js = list(d["weak_idx"]) + [0, 1, 63, 64, 127, 128, 300, 599]
    X = np.zeros((len(js), K), np.float16)
    for n, j in enumerate(js):
        X[n, j] = 1.0
    for a in range(0, len(js), 16):
        xb = torch.from_numpy(X[a:a + 16]).to(dev)
        y = layer(xb, y_f32=True).cpu().numpy().astype(np.float64)
        y_ref = O.matvec(rep, X[a:a + 16].astype(np.float64))
        assert np.array_equal(y, y_ref)


@pytest.mark.parametrize("grid", [1, 2, 3, 7, 13, 64, 500])
def test_stream_k_any_grid_and_deterministic(dev, layout, grid):
    M, K, bits, group, k = 700, 5000, 3, 0, 20
    d = synth.representation(M, K, bits, group, k, seed=grid)
    rep = rep_from_synth(d)
    x = synth.activations(2, K, seed=3, outliers=d["weak_idx"])
    y1, layer = run(d, x, dev, grid=grid, layout=layout)
    e, _ = rel_err(y1, O.matvec(rep, x.astype(np.float64)))
    assert e <= TOL
    xt = torch.from_numpy(x).to(dev)
    for _ in range(3):     # counters reset to 0 after every call; results bit-identical
        y2 = owq.owq_gemm_small_batch_grid(layer.shape, layer.packed, xt, grid, y_f32=True)
        assert np.array_equal(y2.cpu().numpy().astype(np.float64), y1)


@pytest.mark.parametrize("M,K,k", [(12288, 12288, 15), (49152, 12288, 3), (12288, 49152, 15)])
def test_full_size_opt175b_sampled(dev, layout, M, K, k):
    # BASELINE config 5 at full size in the bench launch configuration; the oracle
    # computes a sample of rows one by one (every row-block boundary class covered).
    d = synth.representation(M, K, 3, 0, k, seed=M + K)
    rep = rep_from_synth(d)
    x = synth.activations(1, K, seed=1, outliers=d["weak_idx"][:8])
    y, _ = run(d, x, dev, layout=layout)
    r = np.random.default_rng(0)
    rows = sorted(set([0, 1, 63, 64, M - 1, M - 64] + list(r.choice(M, 120, replace=False))))
    y_ref = O.matvec_rows(rep, x.astype(np.float64), rows)
    e, _ = rel_err(y[:, rows], y_ref)
    assert e <= TOL
    # a property that holds at any size: sum_i y_i = sum_j x_j * colsum_j(W_hat) -- skipped;
    # row-sample parity above is exact per element.


def test_tp_world1_nccl(dev):
    # NCCL communicator of one rank: both TP modes reproduce the single-GPU result.
    M, K, bits, group, k = 512, 2048, 4, 128, 6
    d = synth.representation(M, K, bits, group, k, seed=21)
    shape = owq.Shape(M, K, bits, group, k)
    x = synth.activations(2, K, seed=22, outliers=d["weak_idx"])
    xt = torch.from_numpy(x).to(dev)
    y_ref = O.matvec(rep_from_synth(d), x.astype(np.float64))
    tp = owq.owq_tp_init(owq.owq_tp_get_unique_id(), 1, 0)
    try:
        for mode in (owq.OWQ_TP_ROWS, owq.OWQ_TP_COLS):
            ss, packed = owq.owq_tp_shard(shape, d, mode, 1, 0, device=dev)
            ws = torch.zeros(owq.owq_tp_workspace_bytes(shape, mode, 1, 2), dtype=torch.uint8, device=dev)
            y = torch.empty((2, M), dtype=torch.float32, device=dev)
            owq.owq_tp_gemv(tp, mode, shape, ss, packed, xt, y, y_f32=True, ws=ws)
            torch.cuda.synchronize()
            e, _ = rel_err(y.cpu().numpy(), y_ref)
            assert e <= TOL
    finally:
        owq.owq_tp_destroy(tp)


def test_errors_are_loud(dev, layout):
    d = synth.representation(64, 128, 3, 0, 2, seed=1)
    layer = owq.OwqLinear(d, device=dev, layout=layout)
    x = torch.zeros((17, 128), dtype=torch.float16, device=dev)
    with pytest.raises(owq.OwqError, match="UNSUPPORTED"):
        owq.owq_gemm_small_batch(layer.shape, layer.packed, x)
    wrong = owq.Shape(64, 128, 3, 0, 3)
    with pytest.raises(owq.OwqError, match="BAD_BLOB"):
        owq.owq_gemv(wrong, layer.packed, x[0])


def test_back_to_back_graph_shared_workspace(dev):
    """Chained calls with no host synchronisation in between, captured in one CUDA
    graph, all sharing ONE workspace (the launches overlap through programmatic
    dependent launch): every output must still match the oracle, and replays are
    bit-identical.  Mixed shapes, bits, groups and batch sizes in one chain."""
    cases = [(768, 768, 3, 0, 8, 1), (4096, 1024, 3, 0, 5, 1), (300, 2000, 4, 128, 7, 2), (1000, 700, 3, 0, 11, 1),
             (512, 4096, 4, 0, 3, 3), (2048, 2048, 3, 0, 9, 1)]
    layers, xs, ys, refs = [], [], [], []
    ws_bytes = 0
    for i, (M, K, bits, g, k, B) in enumerate(cases):
        d = synth.representation(M, K, bits, g, k, seed=100 + i)
        x = synth.activations(B, K, seed=200 + i, outliers=d["weak_idx"][:4])
        L = owq.OwqLinear(d, device=dev, layout=owq.OWQ_LAYOUT_CC if i % 2 else owq.OWQ_LAYOUT_TC)   # both layouts in one chain
        layers.append(L)
        xs.append(torch.from_numpy(x).to(dev))
        ys.append(torch.empty((B, M), dtype=torch.float32, device=dev))
        refs.append(O.matvec(rep_from_synth(d), x.astype(np.float64)))
        ws_bytes = max(ws_bytes, owq.owq_workspace_bytes(L.shape, B))
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for L, x, y in zip(layers, xs, ys):   # eager warm-up
            owq.owq_gemm_small_batch(L.shape, L.packed, x, y=y, y_f32=True, ws=ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(3):
            for L, x, y in zip(layers, xs, ys):
                owq.owq_gemm_small_batch(L.shape, L.packed, x, y=y, y_f32=True, ws=ws)
    outs = []
    for _ in range(2):
        for y in ys:
            y.zero_()
        g.replay()
        torch.cuda.synchronize()
        outs.append([y.cpu().numpy().astype(np.float64) for y in ys])
    for y, ref in zip(outs[0], refs):
        e, _ = rel_err(y, ref)
        assert e <= TOL
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


def test_concurrent_streams_partial_grids(dev):
    """The bench's q/k/v schedule: three independent layers on three streams, each
    on a third of the SMs (explicit grid, own workspace), captured in one graph."""
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    cases = [(2048, 3072, 3, 0, 9), (2048, 3072, 3, 0, 11), (1536, 3072, 4, 0, 5)]
    main = torch.cuda.Stream()
    side = [torch.cuda.Stream() for _ in cases]
    runs = []
    for i, (M, K, bits, g, k) in enumerate(cases):
        d = synth.representation(M, K, bits, g, k, seed=300 + i)
        x = synth.activations(1, K, seed=400 + i, outliers=d["weak_idx"][:4])
        L = owq.OwqLinear(d, device=dev)
        grid = sms // 3
        runs.append(dict(L=L, grid=grid, x=torch.from_numpy(x).to(dev),
                         y=torch.empty((1, M), dtype=torch.float32, device=dev),
                         ws=owq.workspace(L.shape, 1, dev, grid=grid),
                         ref=O.matvec(rep_from_synth(d), x.astype(np.float64))))

    def step():
        cur = torch.cuda.current_stream()
        for sd, r in zip(side, runs):
            sd.wait_stream(cur)
            with torch.cuda.stream(sd):
                owq.owq_gemm_small_batch_grid(r["L"].shape, r["L"].packed, r["x"], r["grid"], y=r["y"], y_f32=True,
                                              ws=r["ws"], stream=sd)
        for sd in side:
            cur.wait_stream(sd)

    with torch.cuda.stream(main):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=main):
        for _ in range(3):
            step()
    for r in runs:
        r["y"].zero_()
    g.replay()
    torch.cuda.synchronize()
    for r in runs:
        e, _ = rel_err(r["y"].cpu().numpy().astype(np.float64), r["ref"])
        assert e <= TOL


@pytest.mark.timeout(300)
@pytest.mark.parametrize("layout", [owq.OWQ_LAYOUT_TC, owq.OWQ_LAYOUT_CC])
def test_concurrent_full_grids(dev, layout):
    """Two full-grid (one CTA per SM) calls running concurrently on two streams, so
    neither grid is wholly resident.  The stream-K fixups'
    summer is each row-block's highest-index piece, which waits only on
    lower-index CTAs: both calls must complete and match the oracle, repeatedly."""
    cases = [(12288, 4096, 3, 0, 15), (8192, 6144, 3, 0, 9)]
    streams = [torch.cuda.Stream() for _ in cases]
    runs = []
    for i, (M, K, bits, g, k) in enumerate(cases):
        d = synth.representation(M, K, bits, g, k, seed=500 + i)
        x = synth.activations(1, K, seed=600 + i, outliers=d["weak_idx"][:4])
        L = owq.OwqLinear(d, device=dev, layout=layout)
        rows = sorted(set([0, 127, 128, M - 1] + list(np.random.default_rng(i).choice(M, 100, replace=False))))
        runs.append(dict(L=L, x=torch.from_numpy(x).to(dev), y=torch.empty((1, M), dtype=torch.float32, device=dev),
                         rows=rows, ref=O.matvec_rows(rep_from_synth(d), x.astype(np.float64), rows)))
    torch.cuda.synchronize()
    for it in range(20):
        for sd, r in zip(streams, runs):
            with torch.cuda.stream(sd):
                r["L"](r["x"], y=r["y"], y_f32=True)
    torch.cuda.synchronize()
    for r in runs:
        e, _ = rel_err(r["y"].cpu().numpy().astype(np.float64)[:, r["rows"]], r["ref"])
        assert e <= TOL


@pytest.mark.timeout(300)
def test_concurrent_full_grids_batched(dev):
    """As above at B = 8 on the tcgen05 kernel (MMA N = 48, eight batch rows per
    fixup slot): two full grids compete for the SMs; every call completes and
    matches the oracle."""
    cases = [(12288, 4096, 3, 0, 15), (8192, 6144, 3, 0, 9)]
    B = 8
    streams = [torch.cuda.Stream() for _ in cases]
    runs = []
    for i, (M, K, bits, g, k) in enumerate(cases):
        d = synth.representation(M, K, bits, g, k, seed=700 + i)
        x = synth.activations(B, K, seed=800 + i, outliers=d["weak_idx"][:4])
        L = owq.OwqLinear(d, device=dev, layout=owq.OWQ_LAYOUT_TC)
        rows = sorted(set([0, 127, 128, M - 1] + list(np.random.default_rng(i).choice(M, 60, replace=False))))
        runs.append(dict(L=L, x=torch.from_numpy(x).to(dev), y=torch.empty((B, M), dtype=torch.float32, device=dev),
                         rows=rows, ref=O.matvec_rows(rep_from_synth(d), x.astype(np.float64), rows)))
    torch.cuda.synchronize()
    for it in range(20):
        for sd, r in zip(streams, runs):
            with torch.cuda.stream(sd):
                r["L"](r["x"], y=r["y"], y_f32=True)
    torch.cuda.synchronize()
    for r in runs:
        e, _ = rel_err(r["y"].cpu().numpy().astype(np.float64)[:, r["rows"]], r["ref"])
        assert e <= TOL


def test_workspace_sync_words_left_zero(dev):
    """One workspace shared by calls of different shapes, batches and grids --
    co-resident (zero-word slot protocol) and larger than the SM count (counter
    protocol) -- in one stream with no synchronisation in between: every output
    matches the oracle and the fixed synchronisation prefix of the workspace
    (partial-row slots, 0 = not written) is all zero afterwards."""
    cases = [(1000, 700, 3, 0, 11, 1, 0), (4096, 2048, 3, 0, 9, 2, 500), (300, 2000, 4, 128, 7, 1, 0),
             (2048, 4096, 4, 0, 3, 8, 0), (768, 768, 3, 0, 8, 1, 300), (4096, 1024, 3, 0, 5, 3, 0),
             (1000, 700, 3, 0, 11, 1, -1), (4096, 2048, 4, 128, 9, 2, -700), (768, 768, 3, 0, 8, 4, -3)]
    layers, xs, refs, ws_bytes = [], [], [], 0
    for i, (M, K, bits, g, k, B, grid) in enumerate(cases):
        d = synth.representation(M, K, bits, g, k, seed=300 + i)
        x = synth.activations(B, K, seed=400 + i, outliers=d["weak_idx"][:4])
        cc = grid < 0                      # negative grid: the CUDA-core layout at grid |grid| (-1: default)
        grid = 0 if grid == -1 else abs(grid)
        L = owq.OwqLinear(d, device=dev, layout=owq.OWQ_LAYOUT_CC if cc else owq.OWQ_LAYOUT_TC)
        layers.append((L, grid))
        xs.append(torch.from_numpy(x).to(dev))
        refs.append(O.matvec(rep_from_synth(d), x.astype(np.float64)))
        ws_bytes = max(ws_bytes, owq.workspace(L.shape, B, dev, grid=grid).numel())
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device=dev)
    for _ in range(2):
        ys = []
        for (L, grid), x in zip(layers, xs):
            y = torch.empty((x.shape[0], L.shape.c_out), dtype=torch.float32, device=dev)
            if grid:
                owq.owq_gemm_small_batch_grid(L.shape, L.packed, x, grid, y=y, y_f32=True, ws=ws)
            else:
                owq.owq_gemm_small_batch(L.shape, L.packed, x, y=y, y_f32=True, ws=ws)
            ys.append(y)
        torch.cuda.synchronize()
        for y, ref in zip(ys, refs):
            e, _ = rel_err(y.cpu().numpy().astype(np.float64), ref)
            assert e <= TOL
        slots = 512 * 16 * 128 * 4   # kMaxGrid x OWQ_MAX_BATCH x 128 rows x 4 B (owq_gemv.cu ws_sync)
        assert int(torch.count_nonzero(ws[:slots]).item()) == 0   # both layouts' slot prefixes
