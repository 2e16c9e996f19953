"""OWQ representation variants -- TEST INFRASTRUCTURE ONLY.

Same status as owq_oracle.py: plain fp64 numpy, only tests/, smoke() and
bench.py's CPU legs may import it; nothing on the product path does.

Two variants the paper describes besides the default latency-favored format:

* act-order (App. "act-order" P:845-846): OPTQ quantizes the
  columns "based on activation magnitude" instead of sequentially -- in the
  OPTQ code the paper cites, in descending order of diag(H); with grouped
  grids the groups are consecutive runs of g columns IN THAT ORDER (each
  group's grid is fitted when the sweep reaches it).  OWQ keeps its weak
  columns out of the sweep (reading s6: they go last).
* storage-favored: "storing the reduced size low-precision matrix
  and fp16 weak columns ... to avoid storing unnecessary zeros corresponding
  to weak columns"; the latency-favored format keeps the zero-filled columns.

Both are expressed by one representation, RepStored: the code matrix in
STORED column order plus a column map colmap[p] = the original column of
stored position p.  Grids are per (row, group of g consecutive stored
positions) (reading s20: the paper does not say how groups are
laid out in a reduced / reordered matrix; quantization order = stored order
makes them contiguous).  Latency-favored stores all K columns (weak columns
last, codes zero-filled to their group's zero point, reading s10);
storage-favored stores the K - k non-weak columns only.

Parity status: act_order_perm (closed form), optq_quantize_ordered (diagonal-H
== RTN special case, per-step least-squares optimality solved independently,
brute force on tiny layers), matvec_stored (probes x = e_j, latency ==
storage on the same quantization, fp64 re-association against dequant +
matmul in the original order) -- tests/test_oracle_variants.py.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .owq_oracle import (PERCDAMP, chol_inv_upper, dampen, dequantize, fp16, hessian, minmax_grid, quantize,
                         rtn_delta, search_clip, select_weak, sensitivity)

__all__ = ["RepStored", "act_order_perm", "optq_quantize_ordered", "owq_quantize_variant", "matvec_stored",
           "dequant_matrix_stored", "stored_from_rep"]


@dataclass
class RepStored:
    M: int
    K: int                        # original input width (x has K columns)
    bits: int
    group: int                    # g over STORED positions; 0 = per output row
    codes: np.ndarray             # uint8 [M][Ks], stored order
    colmap: np.ndarray            # int64 [Ks]: stored position -> original column
    scale: np.ndarray             # fp64 values of fp16 [M][G]
    zero: np.ndarray              # fp64 integers [M][G]
    weak_idx: np.ndarray          # int64 [k], ascending, original columns
    weak_val: np.ndarray          # fp64 values of fp16 [M][k]
    mode: str = "latency"         # "latency" (Ks = K) or "storage" (Ks = K - k)
    extra: dict = field(default_factory=dict)

    @property
    def Ks(self) -> int:
        return int(self.colmap.size)

    @property
    def k(self) -> int:
        return int(self.weak_idx.size)

    @property
    def G(self) -> int:
        return 1 if self.group == 0 else (self.Ks + self.group - 1) // self.group


def act_order_perm(H: np.ndarray, weak=()) -> np.ndarray:
    """Quantization order of act-order OWQ: non-weak columns by descending
    H_jj ("based on activation magnitude"; diag(H) = 2 sum_n x_jn^2),
    ties to the smaller index, then the weak columns ascending (reading s6)."""
    d = np.diag(np.asarray(H, dtype=np.float64))
    weak = sorted(int(j) for j in weak)
    ws = set(weak)
    rest = sorted((j for j in range(d.size) if j not in ws), key=lambda j: (-d[j], j))
    return np.array(rest + weak, dtype=np.int64)


def optq_quantize_ordered(W, H_damped, bits, order, nq, group=0, clip=True, on_step=None):
    """OPTQ column sweep (Eq. 1, Cholesky-row form) over the columns
    in `order`: positions 0..nq-1 are quantized, the rest (the weak columns)
    absorb every compensation and are never quantized.  Grids: one per row
    (group = 0) fitted on the nq quantized columns, or one per run of `group`
    consecutive positions fitted when the sweep reaches the run's first
    position, on the run's current values.

    Returns (codes_p [M][K] in order positions (weak positions hold 0),
             scale [M][G], zero [M][G] with G over the K positions,
             Wp (the final working matrix, order positions))."""
    W = np.array(W, dtype=np.float64, copy=True)
    M, K = W.shape
    order = np.asarray(order, dtype=np.int64)
    Wp = W[:, order]
    Hp = np.asarray(H_damped, dtype=np.float64)[np.ix_(order, order)]
    U = chol_inv_upper(Hp)
    G = 1 if group == 0 else (K + group - 1) // group
    scale = np.ones((M, G))
    zero = np.zeros((M, G))
    fit = search_clip if clip else minmax_grid
    codes_p = np.zeros((M, K))
    cur = -1
    for i in range(nq):
        gi = 0 if group == 0 else i // group
        if gi != cur:
            hi = nq if group == 0 else min(nq, (gi + 1) * group)
            for r in range(M):
                scale[r, gi], zero[r, gi] = fit(Wp[r, i:hi], bits)
            cur = gi
        s, z = scale[:, gi], zero[:, gi]
        w = Wp[:, i]
        q = quantize(w, s, z, bits)
        codes_p[:, i] = q
        e = (w - dequantize(q, s, z)) / U[i, i]
        Wp[:, i + 1:] -= np.outer(e, U[i, i + 1:])
        if on_step is not None:
            on_step(i, order, Wp.copy())
    return codes_p.astype(np.uint8), scale, zero, Wp


def owq_quantize_variant(W, X, bits, k, group=0, act_order=False, mode="latency", clip=True, percdamp=PERCDAMP):
    """OWQ with the quantization order of act-order
     when `act_order`, stored latency- or storage-favored
    (P:486-490).  Weak-column selection is the default's (Eq. 5)."""
    if mode not in ("latency", "storage"):
        raise ValueError("mode")
    W = np.array(W, dtype=np.float64, copy=True)
    M, K = W.shape
    H = hessian(X)
    Hd, dead = dampen(H, percdamp)
    W[:, dead] = 0.0
    sens = sensitivity(H, rtn_delta(W, bits, group))
    sens[dead] = 0.0
    weak = select_weak(sens, k)
    if act_order:
        order = act_order_perm(H, weak)
    else:
        ws = set(weak.tolist())
        order = np.array([j for j in range(K) if j not in ws] + weak.tolist(), dtype=np.int64)
    nq = K - weak.size
    codes_p, scale, zero, Wp = optq_quantize_ordered(W, Hd, bits, order, nq, group, clip)
    # weak positions (nq..K-1): code := the zero point of their group (reading s10)
    for p in range(nq, K):
        gi = 0 if group == 0 else p // group
        codes_p[:, p] = zero[:, gi]
    # weak values: the compensated columns, in ascending original index
    wpos = {int(order[p]): p for p in range(nq, K)}
    weak_val = fp16(np.stack([Wp[:, wpos[int(j)]] for j in weak], axis=1)) if weak.size else np.zeros((M, 0))
    if mode == "storage":
        Gs = 1 if group == 0 else (nq + group - 1) // group
        rep = RepStored(M=M, K=K, bits=bits, group=group, codes=codes_p[:, :nq].copy(), colmap=order[:nq].copy(),
                        scale=fp16(scale[:, :Gs]), zero=zero[:, :Gs].copy(), weak_idx=weak, weak_val=weak_val,
                        mode="storage")
    else:
        rep = RepStored(M=M, K=K, bits=bits, group=group, codes=codes_p, colmap=order.copy(), scale=fp16(scale),
                        zero=zero, weak_idx=weak, weak_val=weak_val, mode="latency")
    rep.extra = {"H": H, "sens": sens, "order": order}
    return rep


def _stored_groups(rep: RepStored) -> np.ndarray:
    return np.array([p // rep.group if rep.group else 0 for p in range(rep.Ks)], dtype=np.int64)


def matvec_stored(rep: RepStored, x: np.ndarray) -> np.ndarray:
    """y[b, i] = sum_p s_{i,g(p)} (q_ip - z_{i,g(p)}) x[b, colmap[p]]   (stored positions
    p whose column is not weak) + sum_t v_{i,t} x[b, idx_t]  (P:114 with the
    column remap of P:486-490), fp64."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    gp = _stored_groups(rep)
    low = rep.scale[:, gp] * (rep.codes.astype(np.float64) - rep.zero[:, gp])
    weak = set(int(j) for j in rep.weak_idx)
    keep = np.array([int(c) not in weak for c in rep.colmap], dtype=bool)
    y = x[:, rep.colmap[keep]] @ low[:, keep].T
    if rep.k:
        y += x[:, rep.weak_idx] @ rep.weak_val.T
    return y


def dequant_matrix_stored(rep: RepStored) -> np.ndarray:
    """W_hat in ORIGINAL column order (M x K): scatter of the stored columns,
    zero on weak and unmapped columns, plus the fp16 weak columns."""
    gp = _stored_groups(rep)
    low = rep.scale[:, gp] * (rep.codes.astype(np.float64) - rep.zero[:, gp])
    What = np.zeros((rep.M, rep.K))
    What[:, rep.colmap] = low
    What[:, rep.weak_idx] = 0.0
    What[:, rep.weak_idx] += rep.weak_val
    return What


def stored_from_rep(rep_latency: RepStored) -> RepStored:
    """The storage-favored form of a latency-favored act-order/ordered rep: drop
    the stored positions of the weak columns (they are the last k positions)."""
    weak = set(int(j) for j in rep_latency.weak_idx)
    keep = np.array([int(c) not in weak for c in rep_latency.colmap], dtype=bool)
    nq = int(keep.sum())
    assert np.all(keep[:nq]) and not np.any(keep[nq:])
    g = rep_latency.group
    Gs = 1 if g == 0 else (nq + g - 1) // g
    return RepStored(M=rep_latency.M, K=rep_latency.K, bits=rep_latency.bits, group=g,
                     codes=rep_latency.codes[:, :nq].copy(), colmap=rep_latency.colmap[:nq].copy(),
                     scale=rep_latency.scale[:, :Gs].copy(), zero=rep_latency.zero[:, :Gs].copy(),
                     weak_idx=rep_latency.weak_idx.copy(), weak_val=rep_latency.weak_val.copy(), mode="storage")
