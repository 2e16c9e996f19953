"""Seeded synthetic inputs shared by the oracle-side tests, the GPU tests and
bench.py.  This module holds NONE of OWQ's arithmetic: it only draws random
numbers (numpy PCG64) with the shapes, value distributions and structure of the
paper's workloads.  Recipe:

* W ~ N(0, 0.02^2) (M x K), calibration X (K x N, N = 2048 tokens)
  ~ N(0, 1) with a few outlier input channels scaled by U(20, 100) -- "a few
  outliers ... concentrated in specific feature dimensions".
* activations x [B][K] fp16 ~ N(0, 1) with the same kind of outlier channels.
* a synthetic *quantized representation* (for layer sizes where running the
  oracle's quantizer is too slow): codes ~ clip(z + round(N(0, 1.6)), 0, 2^b-1),
  integer zero points z ~ U{2^(b-1)-1, 2^(b-1)} per row/group, fp16 scales
  ~ 0.02 * U(5, 7) / (2^b - 1), weak indices = k distinct sorted channels,
  weak values fp16 ~ N(0, 0.02^2).  Weak-column codes are drawn like every
  other code: zero-filling them is the method's job (packer / oracle), not
  the generator's.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 2306


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def outlier_channels(K: int, n: int, seed: int) -> np.ndarray:
    r = rng(seed * 7919 + 17)
    n = min(n, K)
    return np.sort(r.choice(K, size=n, replace=False)).astype(np.int64)


def weights_and_calib(M: int, K: int, N: int = 2048, n_outliers: int = 8,
                      seed: int = SEED_BASE, outlier_lo: float = 20.0,
                      outlier_hi: float = 100.0):
    """W (M x K) and calibration X (K x N) in fp64, plus the outlier channels."""
    r = rng(seed)
    W = r.normal(0.0, 0.02, size=(M, K))
    X = r.normal(0.0, 1.0, size=(K, N))
    ch = outlier_channels(K, n_outliers, seed)
    X[ch, :] *= r.uniform(outlier_lo, outlier_hi, size=(ch.size, 1))
    return W, X, ch


def activations(B: int, K: int, seed: int = SEED_BASE, outliers=None,
                outlier_lo: float = 20.0, outlier_hi: float = 100.0) -> np.ndarray:
    """x [B][K] as fp16 (numpy float16)."""
    r = rng(seed + 1_000_003)
    x = r.normal(0.0, 1.0, size=(B, K))
    if outliers is not None and len(outliers):
        oc = np.asarray(outliers, dtype=np.int64)
        x[:, oc] *= r.uniform(outlier_lo, outlier_hi, size=(1, oc.size))
    return x.astype(np.float16)


def representation(M: int, K: int, bits: int, group: int, k: int,
                   seed: int = SEED_BASE):
    """A synthetic quantized layer in the paper's representation.

    Returns a dict of numpy arrays:
      codes u8 [M][K], scale_f16 u16-bits [M][G], zero_f16 u16-bits [M][G],
      weak_idx u16 [k] (strictly ascending), weak_val_f16 u16-bits [M][k].
    """
    r = rng(seed + 31337)
    maxq = (1 << bits) - 1
    G = 1 if group == 0 else (K + group - 1) // group
    zero = r.integers((maxq + 1) // 2 - 1, (maxq + 1) // 2 + 1, size=(M, G))
    scale = (0.02 * r.uniform(5.0, 7.0, size=(M, G)) / maxq).astype(np.float16)
    gi = (np.arange(K) // group) if group else np.zeros(K, dtype=np.int64)
    # codes ~ clip(z + round(N(0, 1.6)), 0, 2^b - 1), drawn through a 256-entry
    # quantile table of N(0, 1.6) so that 600M-weight layers generate in seconds
    from statistics import NormalDist
    nd = NormalDist(0.0, 1.6)
    table = np.array([round(nd.inv_cdf((u + 0.5) / 256.0)) for u in range(256)], dtype=np.int16)
    codes = np.empty((M, K), dtype=np.uint8)
    rc = rng(seed + 4242)
    for a in range(0, M, 2048):              # chunked: bounded temporaries
        b = min(M, a + 2048)
        u = rc.integers(0, 256, size=(b - a, K), dtype=np.uint8)
        zb = zero[a:b].astype(np.int16)
        zb = zb[:, :1] if group == 0 else np.repeat(zb, group, axis=1)[:, :K]
        blk = table[u]
        blk += zb
        np.clip(blk, 0, maxq, out=blk)
        codes[a:b] = blk
    weak_idx = np.sort(r.choice(K, size=k, replace=False)).astype(np.uint16) if k else np.zeros(0, np.uint16)
    weak_val = r.normal(0.0, 0.02, size=(M, k)).astype(np.float16)
    return {
        "M": M, "K": K, "bits": bits, "group": group,
        "codes": codes,
        "scale_f16": scale.view(np.uint16),
        "zero_f16": zero.astype(np.float16).view(np.uint16),
        "weak_idx": weak_idx,
        "weak_val_f16": weak_val.view(np.uint16),
    }
