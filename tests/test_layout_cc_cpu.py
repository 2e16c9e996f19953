"""Device layout version 4 (the CUDA-core GEMV's blob, csrc/owq_layout_cc.h),
checked on the host without a GPU.

The kernel isolates the code of column j of a 32-column step with ONE LOP3,
m = reg & ((2^b - 1) << p(j)), where reg is one of the stored words or a word
assembled from their top bytes with PRMT, and reads m as the fp32 subnormal
q 2^(p(j) - 149).  That is only correct if the packer put every code in the
field the kernel masks and if p(j) + b <= 24.  These tests emulate the
kernel's register arithmetic in numpy on blobs the C packer wrote (so a
packer / extraction mismatch fails here, before any GPU run), and check the
host round trip and the metadata regions bit-exactly.
"""
import numpy as np
import pytest

import paper_2306_02272_b200 as owq
import synth

ROWBLOCK, STEP = 128, 32


def cdiv(a, b):
    return -(-a // b)


def geo(M, K, bits, group, k):
    """Region offsets restated from the owq_layout_cc.h comment (not imported)."""
    nrb, nsteps, kpad = cdiv(M, ROWBLOCK), cdiv(K, STEP), cdiv(k, 8) * 8
    G = cdiv(K, group) if group else 1
    W = 3 if bits == 3 else 4
    item = W * 32 * 16
    units = 256
    sz = units + nrb * nsteps * item
    weak = sz + nrb * G * 512
    widx = weak + nrb * (kpad // 8) * 2048
    wmask = widx + cdiv(kpad * 2 + 2, 16) * 16
    total = wmask + cdiv(nsteps * 4, 16) * 16
    return dict(nrb=nrb, nsteps=nsteps, kpad=kpad, G=G, W=W, item=item, units=units, sz=sz, weak=weak,
                widx=widx, wmask=wmask, total=total)


def prmt(a, b, sel):
    """PTX prmt.b32 (default mode): byte i of the result = byte sel[4i:4i+4] & 7 of {b, a}."""
    src = (np.uint64(b) << np.uint64(32)) | np.uint64(a)
    out = 0
    for i in range(4):
        n = (sel >> (4 * i)) & 7
        out |= int((src >> np.uint64(8 * n)) & np.uint64(0xFF)) << (8 * i)
    return out


def kernel_registers(words, bits):
    """The registers owq_gemv_cc.cu extract<BITS>() masks: stored words, then t (t1), then t2."""
    w = [int(v) for v in words]
    t = prmt(prmt(w[0], w[1], 0x0073), w[2], 0x0710)
    if bits == 3:
        return w + [t]
    return w + [t, prmt(w[3], w[3], 0x0003)]


def kernel_fields(bits):
    """(register, bit offset p) of columns 0..31 as extract<BITS>() reads them."""
    out = []
    for j in range(32):
        if bits == 3:
            out.append((j // 8 if j < 24 else 3, 3 * (j % 8)))
        else:
            if j < 24:
                out.append((j // 6, 4 * (j % 6)))
            elif j < 30:
                out.append((4, 4 * (j - 24)))
            else:
                out.append((5, 4 * (j - 30)))
    return out


@pytest.mark.parametrize("M,K,bits,group,k", [
    (130, 100, 3, 0, 5), (256, 96, 4, 0, 3), (77, 300, 4, 128, 9), (128, 64, 3, 0, 0), (1, 1, 3, 0, 1),
])
def test_kernel_extraction_recovers_every_code(M, K, bits, group, k):
    d = synth.representation(M, K, bits, group, k, seed=M + K + bits)
    shape = owq.Shape(M, K, bits, group, k)
    blob = owq.owq_pack_host(shape, d, flags=owq.OWQ_PACK_LAYOUT_CC)
    g = geo(M, K, bits, group, k)
    assert blob.size == g["total"] == owq.owq_packed_bytes_layout(shape, owq.OWQ_LAYOUT_CC)
    hdr = blob[:8].view(np.uint32)
    assert hdr[1] == 4
    # expected codes: weak columns zero-filled to the row/group zero point (reading s10)
    codes = d["codes"].copy()
    z = d["zero_f16"].view(np.float16).astype(np.int64)
    for j in d["weak_idx"]:
        codes[:, j] = z[:, (j // group) if group else 0]
    fields = kernel_fields(bits)
    mask = (1 << bits) - 1
    for _, p in fields:
        assert p + bits <= 24          # the masked pattern is an exact fp32 subnormal/low normal
    u32 = blob.view(np.uint32)
    for rb in range(g["nrb"]):
        for st in range(g["nsteps"]):
            base = (g["units"] + (rb * g["nsteps"] + st) * g["item"]) // 4
            for rr in range(ROWBLOCK):
                row = rb * ROWBLOCK + rr
                lane, r = rr >> 2, rr & 3
                words = [u32[base + (c * 32 + lane) * 4 + r] for c in range(g["W"])]
                regs = kernel_registers(words, bits)
                for j in range(32):
                    col = st * STEP + j
                    reg, p = fields[j]
                    m = regs[reg] & (mask << p)
                    want = (int(codes[row, col]) if (row < M and col < K) else 0) << p
                    assert m == want, (rb, st, rr, j, m, want)


@pytest.mark.parametrize("M,K,bits,group,k", [(300, 1000, 3, 0, 11), (200, 700, 4, 128, 6), (64, 33, 3, 0, 33)])
def test_cc_host_round_trip_and_regions(M, K, bits, group, k):
    d = synth.representation(M, K, bits, group, k, seed=3 * M + K)
    shape = owq.Shape(M, K, bits, group, k)
    blob = owq.owq_pack_host(shape, d, flags=owq.OWQ_PACK_LAYOUT_CC)
    out = owq.owq_blob_decode_host(blob)
    codes = d["codes"].copy()
    z = d["zero_f16"].view(np.float16).astype(np.int64)
    for j in d["weak_idx"]:
        codes[:, j] = z[:, (j // group) if group else 0]
    assert np.array_equal(out["codes"], codes)
    assert np.array_equal(out["scale_f16"], d["scale_f16"])
    assert np.array_equal(out["zero_f16"], d["zero_f16"])
    assert np.array_equal(out["weak_idx"], d["weak_idx"])
    assert np.array_equal(out["weak_val_f16"], d["weak_val_f16"])
    g = geo(M, K, bits, group, k)
    # scale/zero: [nrb][G][128] (s, z) pairs
    sz = blob[g["sz"]:g["weak"]].view(np.uint16).reshape(g["nrb"], g["G"], 128, 2)
    for row in (0, M // 2, M - 1):
        assert np.array_equal(sz[row // 128, :, row % 128, 0], d["scale_f16"][row])
        assert np.array_equal(sz[row // 128, :, row % 128, 1], d["zero_f16"][row])
    # weak values: [nrb][kpad/8][128][8], zero-padded
    wv = blob[g["weak"]:g["widx"]].view(np.uint16).reshape(g["nrb"], g["kpad"] // 8, 128, 8)
    for row in (0, M - 1):
        flat = wv[row // 128, :, row % 128, :].reshape(-1)
        assert np.array_equal(flat[:k], d["weak_val_f16"][row]) and not flat[k:].any()
    # weak-column bitmask
    wm = blob[g["wmask"]:g["total"]].view(np.uint32)[:g["nsteps"]]
    bitsset = [j for j in range(K) if (wm[j >> 5] >> (j & 31)) & 1]
    assert bitsset == sorted(int(j) for j in d["weak_idx"])


def test_cc_strict_and_errors():
    d = synth.representation(64, 128, 3, 0, 2, seed=1)
    shape = owq.Shape(64, 128, 3, 0, 2)
    with pytest.raises(owq.OwqError, match="ZERO_FILL"):
        owq.owq_pack_host(shape, d, flags=owq.OWQ_PACK_LAYOUT_CC | owq.OWQ_PACK_STRICT)
    assert owq.owq_packed_bytes_layout(shape, 5) == 0
    assert owq.owq_packed_bytes_layout(owq.Shape(64, 128, 5, 0, 2), owq.OWQ_LAYOUT_CC) == 0


# ---------------------------------------------------------------- NEXT-4: column-mapped blobs
@pytest.mark.parametrize("mode,group", [("latency", 0), ("storage", 0), ("latency", 128), ("storage", 128)])
def test_colmap_round_trip(mode, group):
    from owq_testutil import dict_from_stored, synthetic_stored
    rep = synthetic_stored(200, 700, 4 if group else 3, group, 9, mode, seed=5)
    d = dict_from_stored(rep)
    shape = owq.Shape(200, 700, rep.bits, group, 9)
    blob = owq.owq_pack_host_colmap(shape, d, d["colmap"], flags=owq.OWQ_PACK_U8_CODES)
    assert blob.size == owq.owq_packed_bytes_colmap(shape, d["colmap"])
    assert np.array_equal(owq.owq_blob_colmap_host(blob), d["colmap"])
    out = owq.owq_blob_decode_host(blob)
    assert out["codes"].shape == (200, rep.Ks)
    assert np.array_equal(out["codes"], d["codes"])
    assert np.array_equal(out["scale_f16"], d["scale_f16"]) and np.array_equal(out["zero_f16"], d["zero_f16"])
    assert np.array_equal(out["weak_val_f16"], d["weak_val_f16"])
    # weak mask over stored positions
    g = geo(200, rep.Ks, rep.bits, group, 9)
    hdr = blob[:256]
    wmask_off = g["wmask"]
    wm = blob[wmask_off:wmask_off + 4 * g["nsteps"]].view(np.uint32)
    ws = set(int(j) for j in rep.weak_idx)
    for p in range(rep.Ks):
        assert bool((wm[p >> 5] >> (p & 31)) & 1) == (int(rep.colmap[p]) in ws)


def test_colmap_validation():
    from owq_testutil import dict_from_stored, synthetic_stored
    rep = synthetic_stored(64, 100, 3, 0, 4, "storage", seed=1)
    d = dict_from_stored(rep)
    shape = owq.Shape(64, 100, 3, 0, 4)
    bad = d["colmap"].copy()
    bad[1] = bad[0]                                     # repeated column
    with pytest.raises(owq.OwqError, match="INVALID_ARG"):
        owq.owq_pack_host_colmap(shape, d, bad, flags=owq.OWQ_PACK_U8_CODES)
    bad = d["colmap"].copy()
    bad[0] = 100                                        # out of range
    with pytest.raises(owq.OwqError, match="INVALID_ARG"):
        owq.owq_pack_host_colmap(shape, d, bad, flags=owq.OWQ_PACK_U8_CODES)
    # latency-favored with a weak stored position not zero-filled: strict rejects
    lat = synthetic_stored(64, 100, 3, 0, 4, "latency", seed=2)
    dl = dict_from_stored(lat)
    dl["codes"] = dl["codes"].copy()
    dl["codes"][:, -1] = (dl["codes"][:, -1] + 1) % 8
    with pytest.raises(owq.OwqError, match="ZERO_FILL"):
        owq.owq_pack_host_colmap(owq.Shape(64, 100, 3, 0, 4), dl, dl["colmap"],
                                 flags=owq.OWQ_PACK_U8_CODES | owq.OWQ_PACK_STRICT)
