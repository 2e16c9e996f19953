"""C-ABI boundary on the CPU: the library loads, exports every symbol declared
in include/owq.h, and the host packer / shard logic are bit-exact.  No compute
call needs a GPU here."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2306_02272_b200 as owq
import synth
from owq_testutil import rep_from_synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_and_exports_header_symbols():
    L = owq.lib()
    hdr = open(os.path.join(ROOT, "include", "owq.h")).read()
    declared = set(re.findall(r"^\s*(?:owq_status|size_t|const char \*)\s*(owq_\w+)\(", hdr, re.M))
    assert declared == set(owq.EXPORTED_SYMBOLS)
    for name in declared:
        assert getattr(L, name) is not None
    assert owq.lib().owq_status_string(0) == b"OWQ_OK"


def test_canonical_pack_matches_oracle_stream():
    # product-side numpy packbits vs the oracle's bit loop, and the SPEC S:403 bytes
    r = np.random.default_rng(1)
    for bits in (3, 4):
        c = r.integers(0, 2 ** bits, size=(5, 37)).astype(np.uint8)
        assert np.array_equal(owq.canonical_pack(c, bits), O.pack_canonical(c, bits))
    assert [format(b, "08b") for b in owq.canonical_pack(np.arange(8, dtype=np.uint8)[None], 3)[0]] == \
        ["10001000", "11000110", "11111010"]


@pytest.mark.parametrize("M,K,bits,group,k", [
    (64, 64, 3, 0, 0), (100, 200, 3, 0, 5), (768, 768, 3, 0, 8), (130, 1100, 4, 128, 9),
    (16, 4096, 4, 1024, 1), (65, 129, 3, 128, 17), (1, 1, 3, 0, 1), (200, 1500, 3, 0, 153)])
def test_host_pack_roundtrip_bit_exact(M, K, bits, group, k):
    d = synth.representation(M, K, bits, group, k, seed=M + K)
    shape = owq.Shape(M, K, bits, group, k)
    blob = owq.owq_pack_host(shape, d)
    assert blob.size == owq.owq_packed_bytes(shape)
    back = owq.owq_blob_decode_host(blob)
    assert back["shape"].tup() == shape.tup()
    # zero fill: weak-column codes become the row/group zero point (reading s10)
    expect = d["codes"].copy()
    z = O.from_fp16_bits(d["zero_f16"]).astype(np.uint8)
    for j in d["weak_idx"]:
        expect[:, j] = z[:, (j // group) if group else 0]
    assert np.array_equal(back["codes"], expect)
    for key in ("scale_f16", "zero_f16", "weak_idx", "weak_val_f16"):
        assert np.array_equal(back[key], d[key]), key
    # canonical input gives the same blob
    dc = dict(d, codes=owq.canonical_pack(d["codes"], bits), canonical=True)
    assert np.array_equal(owq.owq_pack_host(shape, dc), blob)


def test_blob_bytes_close_to_algorithmic():
    # code units + weak units + scale/zero + idx: padding overhead small at real sizes
    for (M, K, bits, g, k) in [(12288, 12288, 3, 0, 15), (49152, 12288, 3, 0, 3), (4096, 4096, 4, 128, 4)]:
        n = owq.owq_packed_bytes(owq.Shape(M, K, bits, g, k))
        G = 1 if g == 0 else K // g
        alg = bits * M * K / 8 + 4 * M * G + 2 * M * k + 2 * k
        # padding: k -> multiple of 8 weak columns (mma k8), rows -> 64, header 256 B
        kpad = -(-k // 8) * 8
        assert alg <= n <= alg + 2 * M * (kpad - k) + 256 + 2 * kpad + 16
        assert n <= alg * 1.003


def test_pack_validation_errors():
    d = synth.representation(64, 128, 3, 0, 3, seed=3)
    shape = owq.Shape(64, 128, 3, 0, 3)
    with pytest.raises(owq.OwqError, match="ZERO_FILL"):
        owq.owq_pack_host(shape, d, flags=owq.OWQ_PACK_STRICT)      # synthetic weak codes != z
    bad = dict(d, weak_idx=d["weak_idx"][::-1].copy())
    with pytest.raises(owq.OwqError, match="WEAK_INDEX"):
        owq.owq_pack_host(shape, bad)
    bad = dict(d, zero_f16=np.full_like(d["zero_f16"], np.float16(2.5).view(np.uint16)))
    with pytest.raises(owq.OwqError, match="ZERO_POINT"):
        owq.owq_pack_host(shape, bad)
    bad = dict(d, codes=np.full_like(d["codes"], 9))
    with pytest.raises(owq.OwqError, match="CODE_RANGE"):
        owq.owq_pack_host(shape, bad)
    with pytest.raises(owq.OwqError, match="UNSUPPORTED"):
        owq.owq_pack_host(owq.Shape(64, 128, 5, 0, 3), d)
    with pytest.raises(owq.OwqError, match="UNSUPPORTED"):
        owq.owq_pack_host(owq.Shape(64, 128, 3, 64, 3), d)
    assert owq.owq_packed_bytes(owq.Shape(64, 70000, 3, 0, 0)) == 0
    # strict mode accepts a properly zero-filled representation (oracle quantizer output)
    W, X, _ = synth.weights_and_calib(32, 64, N=128, n_outliers=2, seed=4)
    rep = O.owq_quantize(W, X, 3, 2)
    from owq_testutil import synth_from_rep
    owq.owq_pack_host(owq.Shape(32, 64, 3, 0, 2), synth_from_rep(rep), flags=owq.OWQ_PACK_STRICT)


@pytest.mark.parametrize("mode", [owq.OWQ_TP_ROWS, owq.OWQ_TP_COLS])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_tp_shards_partition_the_layer(mode, world):
    M, K, bits, g, k = 1376 * 2, 11008 // 4, 4, 128, 9
    d = synth.representation(M, K, bits, g, k, seed=7)
    shape = owq.Shape(M, K, bits, g, k)
    full = rep_from_synth(d)
    x = synth.activations(2, K, seed=8).astype(np.float64)
    y_ref = O.matvec(full, x)
    acc = np.zeros_like(y_ref)
    covered = 0
    for r in range(world):
        a, b = owq.owq_tp_bounds(shape, mode, world, r)
        ss, blob = owq.owq_tp_shard_host(shape, d, mode, world, r)
        dec = owq.owq_blob_decode_host(blob)
        sr = O.Rep(M=ss.c_out, K=ss.c_in, bits=bits, group=g, codes=dec["codes"],
                   scale=O.from_fp16_bits(dec["scale_f16"]), zero=O.from_fp16_bits(dec["zero_f16"]),
                   weak_idx=dec["weak_idx"].astype(np.int64), weak_val=O.from_fp16_bits(dec["weak_val_f16"]))
        if mode == owq.OWQ_TP_ROWS:
            assert a % 16 == 0 and ss.c_out == b - a
            acc[:, a:b] = O.matvec(sr, x)
        else:
            assert a % 128 == 0 and ss.c_in == b - a
            acc += O.matvec(sr, x[:, a:b])
        covered += b - a
    assert covered == (M if mode == owq.OWQ_TP_ROWS else K)
    assert np.allclose(acc, y_ref, rtol=1e-12, atol=1e-12)


def test_prefill_workspace_sizing():
    """owq_prefill_workspace_bytes (host logic, no GPU needed): K pieces of at most
    64 super-steps (4096 columns) are needed whenever c_in > 4096 -- B x c_out(padded
    to 128) fp32 partial rows per piece -- and none for c_in <= 4096 on a wide layer."""
    s = owq.Shape(12288, 12288, 3, 0, 15)
    n = owq.owq_prefill_workspace_bytes(s, 2048)
    assert n >= 3 * 2048 * 12288 * 4 and n % (2048 * 12288 * 4) == 0
    assert owq.owq_prefill_workspace_bytes(owq.Shape(12288, 4096, 3, 0, 15), 2048) == 0
    assert owq.owq_prefill_workspace_bytes(owq.Shape(130, 49152, 4, 0, 3), 17) >= 12 * 17 * 256 * 4
    assert owq.owq_prefill_workspace_bytes(owq.Shape(0, 4096, 3, 0, 0), 8) == 0   # invalid shape
