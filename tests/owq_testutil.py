"""Shared test helpers: representation conversion and the per-element error
metric of DESIGN.md §3 reading s16."""
import numpy as np

import oracle as O


def rep_from_synth(d) -> "O.Rep":
    return O.Rep(M=d["M"], K=d["K"], bits=d["bits"], group=d["group"], codes=d["codes"],
                 scale=O.from_fp16_bits(d["scale_f16"]), zero=O.from_fp16_bits(d["zero_f16"]),
                 weak_idx=np.asarray(d["weak_idx"]).astype(np.int64),
                 weak_val=O.from_fp16_bits(d["weak_val_f16"]))


def synth_from_rep(rep: "O.Rep") -> dict:
    """Oracle quantizer output -> the dict the binding packs (fp16 bit patterns)."""
    return {"M": rep.M, "K": rep.K, "bits": rep.bits, "group": rep.group,
            "codes": np.ascontiguousarray(rep.codes, np.uint8),
            "scale_f16": O.fp16_bits(rep.scale), "zero_f16": O.fp16_bits(rep.zero),
            "weak_idx": np.asarray(rep.weak_idx, np.uint16),
            "weak_val_f16": O.fp16_bits(rep.weak_val)}


def rel_err(y, y_ref):
    """err_i = |y_i - ref_i| / max(|ref_i|, 1e-3 * rms(ref)) (reading s16); also the unfloored max."""
    y = np.asarray(y, np.float64)
    y_ref = np.asarray(y_ref, np.float64)
    rms = np.sqrt(np.mean(y_ref ** 2)) if y_ref.size else 1.0
    d = np.abs(y - y_ref)
    floored = d / np.maximum(np.abs(y_ref), 1e-3 * rms)
    unfloored = d / np.maximum(np.abs(y_ref), 1e-300)
    return float(floored.max()) if d.size else 0.0, float(unfloored.max()) if d.size else 0.0


TOL = 2e-3   # BASELINE.json north_star: relative error <= 2e-3 per output element


def dict_from_stored(rep) -> dict:
    """oracle.RepStored (NEXT-4 variants) -> the dict the binding packs with a column map."""
    return {"M": rep.M, "K": rep.K, "bits": rep.bits, "group": rep.group,
            "codes": np.ascontiguousarray(rep.codes, np.uint8),
            "scale_f16": O.fp16_bits(rep.scale), "zero_f16": O.fp16_bits(rep.zero),
            "weak_idx": np.asarray(rep.weak_idx, np.uint16), "weak_val_f16": O.fp16_bits(rep.weak_val),
            "colmap": np.asarray(rep.colmap, np.uint16)}


def synthetic_stored(M, K, bits, group, k, mode, seed):
    """A synthetic NEXT-4 representation at sizes the oracle quantizer cannot reach:
    a random quantization order (act-order-like permutation of the non-weak
    columns, weak columns last), codes/grids drawn like synth.representation."""
    import synth
    r = np.random.default_rng(seed)
    weak = np.sort(r.choice(K, size=k, replace=False)).astype(np.int64) if k else np.zeros(0, np.int64)
    ws = set(weak.tolist())
    rest = np.array([j for j in range(K) if j not in ws], dtype=np.int64)
    r.shuffle(rest)
    order = np.concatenate([rest, weak])
    Ks = K if mode == "latency" else K - k
    d = synth.representation(M, Ks, bits, group, 0, seed=seed)
    rep = O.RepStored(M=M, K=K, bits=bits, group=group, codes=d["codes"], colmap=order[:Ks],
                      scale=O.from_fp16_bits(d["scale_f16"]), zero=O.from_fp16_bits(d["zero_f16"]),
                      weak_idx=weak, weak_val=O.fp16(r.normal(0, 0.02, size=(M, k))), mode=mode)
    if mode == "latency":   # zero fill of the weak stored positions (the packer would do it too)
        for p in range(K - k, K):
            gi = p // group if group else 0
            rep.codes[:, p] = rep.zero[:, gi]
    return rep
