"""OWQ CPU oracle — TEST INFRASTRUCTURE ONLY.

This module is the plain, slow, obviously-correct CPU statement of what the
OWQ (arXiv 2306.02272) inference hot path computes, plus the quantizer steps
that produce its inputs.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product path (``paper_2306_02272_b200``) never imports, links or calls
anything under ``oracle/``, and this module shares no code with it.

Precision: float64 throughout (numpy).  fp16 appears only where the paper fixes
it as a *storage* format ("we store the weak columns as fp16"; scale and
zero stored as fp16 per the OPTQ lineage the paper builds on).

Citation keys: ``P:n`` = /root/reference/PAPER.md line n (LaTeX source of the
paper), ``S:n`` = SPEC.md line n, ``reading sN`` = the reading listed in
DESIGN.md §3 (copied from SURVEY.md §8(c)) where the paper is silent/ambiguous.

Parity status per function (DESIGN.md §3 repeats this):
  hessian, dampen, chol_inv_upper, minmax_grid, quantize, dequantize,
  search_clip, rtn_delta, sensitivity, select_weak, budget_to_k,
  effective_bits, pack_canonical, unpack_canonical, dequant_matrix, matvec
      -- pinned by tests/test_oracle_*.py (closed forms, brute force,
         paper-printed numbers under tests/golden/).
  optq_quantize / owq_quantize
      -- pinned by special cases (diagonal H == RTN, one-step least-squares
         optimality, brute force on tiny layers, statistical error ordering).
         The exact codes OPTQ emits on large random layers have no external
         pin: "parity unpinned" for that part (the GPU path never consumes
         them except as opaque inputs, so GPU parity does not depend on it).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Rep", "hessian", "dampen", "chol_inv_upper", "fp16", "minmax_grid",
    "quantize", "dequantize", "search_clip", "rtn_delta", "sensitivity",
    "select_weak", "optq_quantize", "owq_quantize", "budget_to_k",
    "effective_bits", "pack_canonical", "unpack_canonical", "dequant_matrix",
    "matvec", "matvec_rows", "layer_error", "fp16_bits", "from_fp16_bits",
]

PERCDAMP = 0.01        # reading s2: OPTQ lineage
CLIP_POINTS = 80       # reading s8: p in {1 - i/100 : i = 0..79} (maxshrink 0.8)


# --------------------------------------------------------------------------
# fp16 storage helpers (IEEE binary16, round-half-to-even; reading s9)
# --------------------------------------------------------------------------
def fp16(a):
    """Round to IEEE fp16 (RNE) and widen back to fp64 exactly."""
    return np.asarray(a, dtype=np.float64).astype(np.float16).astype(np.float64)


def fp16_bits(a) -> np.ndarray:
    """fp64 values -> uint16 fp16 bit patterns (RNE)."""
    return np.asarray(a, dtype=np.float64).astype(np.float16).view(np.uint16)


def from_fp16_bits(b) -> np.ndarray:
    return np.asarray(b, dtype=np.uint16).view(np.float16).astype(np.float64)


# --------------------------------------------------------------------------
# L0: Hessian  (Eq. 3: H_i = d2E/dW_i^2 = 2 X X^T, same for all rows)
# --------------------------------------------------------------------------
def hessian(X: np.ndarray) -> np.ndarray:
    """H = 2 X X^T for calibration features X in R^{C_in x N}.

    Summed over the N samples, not averaged (reading s1)."""
    X = np.asarray(X, dtype=np.float64)
    return 2.0 * (X @ X.T)


def dampen(H: np.ndarray, percdamp: float = PERCDAMP):
    """OPTQ-lineage conditioning ("based on OPTQ"; reading s2).

    Dead columns (H_jj == 0) get H_jj := 1; then H += percdamp*mean(diag H)*I.
    Returns (H_damped, dead_mask)."""
    if percdamp <= 0:
        raise ValueError("percdamp must be positive")
    H = np.array(H, dtype=np.float64, copy=True)
    d = np.diag(H).copy()
    if not np.any(d > 0):
        raise ValueError("all-zero Hessian (no calibration signal)")
    dead = d == 0
    H[dead, dead] = 1.0
    damp = percdamp * np.mean(np.diag(H))
    H[np.diag_indices_from(H)] += damp
    return H, dead


def chol_inv_upper(H: np.ndarray) -> np.ndarray:
    """Upper-triangular U with U^T U = H^{-1} (the Cholesky-row form of Eq. 1's
    [H_F^{-1}]).  H^{-1} is formed from H's own Cholesky factor."""
    L = np.linalg.cholesky(H)                 # H = L L^T
    Linv = np.linalg.inv(L)
    Hinv = Linv.T @ Linv                      # H^{-1}
    Hinv = 0.5 * (Hinv + Hinv.T)
    return np.linalg.cholesky(Hinv).T         # upper: U^T U = H^{-1}


# --------------------------------------------------------------------------
# L2: linear grid, RTN, truncation search  (P:118-123, P:160 RTN baseline)
# --------------------------------------------------------------------------
def _grid_from_range(xmin, xmax, bits):
    """Asymmetric integer-zero-point grid (reading s7): 0 always on the grid.
    Scale rounded to fp16 before computing z (reading s12)."""
    maxq = (1 << bits) - 1
    xmin = np.minimum(np.asarray(xmin, dtype=np.float64), 0.0)
    xmax = np.maximum(np.asarray(xmax, dtype=np.float64), 0.0)
    both0 = (xmin == 0) & (xmax == 0)
    xmin = np.where(both0, -1.0, xmin)
    xmax = np.where(both0, 1.0, xmax)
    s = fp16((xmax - xmin) / maxq)
    # an fp16 underflow to 0 would make the grid degenerate: smallest subnormal
    s = np.where(s == 0, 2.0 ** -24, s)
    z = np.clip(np.rint(-xmin / s), 0, maxq)
    return s, z


def minmax_grid(w: np.ndarray, bits: int):
    """Min-max grid of one vector (the OPTQ baseline grid)."""
    w = np.asarray(w, dtype=np.float64)
    s, z = _grid_from_range(w.min(), w.max(), bits)
    return float(s), float(z)


def quantize(w, s, z, bits):
    """q = clamp(rne(w/s) + z, 0, 2^b - 1)  (round-to-nearest with truncation)."""
    maxq = (1 << bits) - 1
    return np.clip(np.rint(np.asarray(w, dtype=np.float64) / s) + z, 0, maxq)


def dequantize(q, s, z):
    """w_hat = s * (q - z)."""
    return s * (np.asarray(q, dtype=np.float64) - z)


def search_clip(w: np.ndarray, bits: int, points: int = CLIP_POINTS):
    """Greedy truncation search: shrink (xmin, xmax) by
    p in {1 - i/100}, keep the first p minimising sum |w - dequant(quant(w))|^2
    (reading s8).  p = 1 is the min-max grid, so the result never loses to it."""
    w = np.asarray(w, dtype=np.float64)
    xmin0 = min(w.min(), 0.0)
    xmax0 = max(w.max(), 0.0)
    best = None
    for i in range(points):
        p = 1.0 - i / 100.0
        s, z = _grid_from_range(p * xmin0, p * xmax0, bits)
        s, z = float(s), float(z)
        err = float(np.sum((w - dequantize(quantize(w, s, z, bits), s, z)) ** 2))
        if best is None or err < best[0]:
            best = (err, s, z)
    return best[1], best[2]


def _groups(K: int, g: int):
    if g == 0:
        return [(0, K)]
    return [(a, min(a + g, K)) for a in range(0, K, g)]


def rtn_delta(W: np.ndarray, bits: int, group: int = 0) -> np.ndarray:
    """Delta W = W - RTN_b(W) with per-row (per-group) min-max grids fitted on
    all columns (reading s4), used by Eq. 5."""
    W = np.asarray(W, dtype=np.float64)
    D = np.empty_like(W)
    for a, b in _groups(W.shape[1], group):
        for i in range(W.shape[0]):
            s, z = minmax_grid(W[i, a:b], bits)
            D[i, a:b] = W[i, a:b] - dequantize(quantize(W[i, a:b], s, z, bits), s, z)
    return D


# --------------------------------------------------------------------------
# L1: sensitivity and weak-column selection  (Eq. 5)
# --------------------------------------------------------------------------
def sensitivity(H: np.ndarray, dW: np.ndarray) -> np.ndarray:
    """sensitivity_j = lambda_j * ||dW_{:,j}||_2^2, lambda_j = H_jj (undamped,
    reading s3) -- Eq. 5."""
    lam = np.diag(np.asarray(H, dtype=np.float64))
    return lam * np.sum(np.asarray(dW, dtype=np.float64) ** 2, axis=0)


def select_weak(sens: np.ndarray, k: int) -> np.ndarray:
    """Top-k columns by sensitivity; ties -> smaller index (reading s5);
    returned ascending."""
    sens = np.asarray(sens, dtype=np.float64)
    if not 0 <= k <= sens.size:
        raise ValueError("k out of range")
    order = sorted(range(sens.size), key=lambda j: (-sens[j], j))
    return np.array(sorted(order[:k]), dtype=np.int64)


# --------------------------------------------------------------------------
# The paper's quantized representation
# --------------------------------------------------------------------------
@dataclass
class Rep:
    """Zero-filled b-bit codes + fp16 scale/zero per row (or per group) +
    fp16 weak columns + u16 weak-column indices."""
    M: int
    K: int
    bits: int
    group: int                    # 0 = per output row
    codes: np.ndarray             # uint8 [M][K]
    scale: np.ndarray             # fp64 values of fp16 [M][G]
    zero: np.ndarray              # fp64 integer values [M][G]
    weak_idx: np.ndarray          # int64 [k], strictly ascending, < K
    weak_val: np.ndarray          # fp64 values of fp16 [M][k]
    extra: dict = field(default_factory=dict)

    @property
    def k(self) -> int:
        return int(self.weak_idx.size)

    @property
    def G(self) -> int:
        return 1 if self.group == 0 else (self.K + self.group - 1) // self.group


# --------------------------------------------------------------------------
# L2: OPTQ with weak columns excluded  (Eq. 1)
# --------------------------------------------------------------------------
def optq_quantize(W, H_damped, bits, group=0, weak=(), clip=True, on_step=None):
    """OPTQ column sweep in the Cholesky-row form of Eq. 1.

    Weak columns are moved to the end of the order (reading s6): they are never
    quantized, absorb every compensation update, and their final values are
    returned.  Grids: per row on the non-weak columns ("after removing the
    weak columns"), truncation-searched when ``clip`` else min-max;
    with ``group`` > 0 a group's grid is fitted when the sweep reaches its first
    non-weak column, on the group's current (compensated) non-weak values.

    ``on_step(i, perm, Wp, dequantized_col)`` (tests only) is called after
    every column step with the current permuted working matrix.

    Returns (codes [M][K] with weak columns = the row/group zero point,
             scale [M][G], zero [M][G], weak_values [M][k] (fp64, compensated)).
    """
    W = np.array(W, dtype=np.float64, copy=True)
    M, K = W.shape
    weak = np.array(sorted(int(j) for j in weak), dtype=np.int64)
    k = weak.size
    is_weak = np.zeros(K, dtype=bool)
    is_weak[weak] = True
    perm = np.concatenate([np.flatnonzero(~is_weak), weak])
    Wp = W[:, perm]
    Hp = np.asarray(H_damped, dtype=np.float64)[np.ix_(perm, perm)]
    U = chol_inv_upper(Hp)
    groups = _groups(K, group)
    G = len(groups)
    scale = np.zeros((M, G))
    zero = np.zeros((M, G))
    fit = search_clip if clip else minmax_grid
    nq = K - k                                   # quantized (non-weak) columns
    codes_p = np.zeros((M, K))
    grp_of = np.array([j // group if group else 0 for j in range(K)])
    cur = -1
    for i in range(nq):
        j = perm[i]
        gidx = grp_of[j]
        if gidx != cur:
            # fit this group's grid on its non-weak columns' current values
            cols = [ii for ii in range(i, nq) if grp_of[perm[ii]] == gidx]
            for r in range(M):
                scale[r, gidx], zero[r, gidx] = fit(Wp[r, cols], bits)
            cur = gidx
        s, z = scale[:, gidx], zero[:, gidx]
        w = Wp[:, i]
        q = quantize(w, s, z, bits)
        d = dequantize(q, s, z)
        codes_p[:, i] = q
        e = (w - d) / U[i, i]
        Wp[:, i + 1:] -= np.outer(e, U[i, i + 1:])
        if on_step is not None:
            on_step(i, perm, Wp.copy(), d.copy())
    # groups containing only weak columns keep a valid grid (min-max of values)
    for gidx in range(G):
        if not np.any(scale[:, gidx]):
            scale[:, gidx], zero[:, gidx] = 1.0, 0.0
    codes = np.zeros((M, K))
    codes[:, perm] = codes_p
    # zero fill (reading s10): weak-column code := that row/group's zero point
    for j in weak:
        codes[:, j] = zero[:, grp_of[j]]
    weak_values = Wp[:, nq:]
    return codes.astype(np.uint8), scale, zero, weak_values


def owq_quantize(W, X, bits, k, group=0, clip=True, percdamp=PERCDAMP):
    """OWQ as the paper states it, step by step:
    H = 2XX^T (Eq. 3) -> RTN Delta W -> Eq. 5 sensitivity -> top-k ->
    OPTQ with weak columns excluded + truncation-tuned grid ->
    zero-filled codes + fp16 weak columns + u16 indices."""
    W = np.array(W, dtype=np.float64, copy=True)
    H = hessian(X)
    Hd, dead = dampen(H, percdamp)
    W[:, dead] = 0.0
    sens = sensitivity(H, rtn_delta(W, bits, group))
    sens[dead] = 0.0
    weak = select_weak(sens, k)
    codes, scale, zero, wv = optq_quantize(W, Hd, bits, group, weak, clip)
    return Rep(M=W.shape[0], K=W.shape[1], bits=bits, group=group,
               codes=codes, scale=fp16(scale), zero=zero,
               weak_idx=weak, weak_val=fp16(wv),
               extra={"sens": sens, "H": H})


# --------------------------------------------------------------------------
# Budget and effective bit-width
# --------------------------------------------------------------------------
def budget_to_k(extra_bits, layer_dims, bits, mode="latency"):
    """Extra bits spread evenly over the L linear layers (reading s13):
    B_layer = extra * sum(M*K) / L;  k = floor(B_layer / cost_per_column),
    cost = 16*M + 16 (latency-favored, zero-filled column kept) or
    (16 - b)*M + 16 (storage-favored)."""
    if extra_bits < 0:
        raise ValueError("negative budget")
    total = extra_bits * sum(m * kk for m, kk in layer_dims)
    per = total / len(layer_dims)
    out = []
    for m, kk in layer_dims:
        cost = 16 * m + 16 if mode == "latency" else (16 - bits) * m + 16
        out.append(min(kk, int(math.floor(per / cost + 1e-12))))
    return out


def effective_bits(M, K, bits, k, mode="latency"):
    """Appendix B.3.  storage: (b*M*(K-k) + 16*M*k + 16*k)/(M*K);
    latency additionally keeps the b*M*k zero-filled codes."""
    num = bits * M * (K - k) + 16 * M * k + 16 * k
    if mode == "latency":
        num += bits * M * k
    return num / (M * K)


# --------------------------------------------------------------------------
# Canonical bit packing (reading s11)
# --------------------------------------------------------------------------
def pack_canonical(codes: np.ndarray, bits: int) -> np.ndarray:
    """Row-major, LSB-first bit stream, each row padded to a whole byte.
    Bit t of code (i, j) is bit (j*b + t) of row i's stream."""
    codes = np.asarray(codes)
    M, K = codes.shape
    if np.any(codes >= (1 << bits)) or np.any(codes < 0):
        raise ValueError("code out of range")
    rb = (K * bits + 7) // 8
    out = np.zeros((M, rb), dtype=np.uint8)
    for j in range(K):
        for t in range(bits):
            pos = j * bits + t
            bit = ((codes[:, j].astype(np.int64) >> t) & 1).astype(np.uint8)
            out[:, pos // 8] |= (bit << (pos % 8)).astype(np.uint8)
    return out


def unpack_canonical(blob: np.ndarray, M: int, K: int, bits: int) -> np.ndarray:
    blob = np.asarray(blob, dtype=np.uint8).reshape(M, -1)
    if blob.shape[1] != (K * bits + 7) // 8:
        raise ValueError("length mismatch")
    codes = np.zeros((M, K), dtype=np.int64)
    for j in range(K):
        for t in range(bits):
            pos = j * bits + t
            codes[:, j] |= ((blob[:, pos // 8] >> (pos % 8)) & 1).astype(np.int64) << t
    return codes.astype(np.uint8)


# --------------------------------------------------------------------------
# L4: the hot path's definition  (SPEC mixed_forward S:468-476)
# --------------------------------------------------------------------------
def dequant_matrix(rep: Rep) -> np.ndarray:
    """W_hat = (zero-filled low-bit matrix) + weak columns, fp64.  The low-bit
    part is s_{i,g(j)} (q_ij - z_{i,g(j)}) and is zero on weak columns
    ("zero-filled weak columns"; "set weak columns ... to zero")."""
    M, K = rep.M, rep.K
    gi = np.array([j // rep.group if rep.group else 0 for j in range(K)])
    low = rep.scale[:, gi] * (rep.codes.astype(np.float64) - rep.zero[:, gi])
    low[:, rep.weak_idx] = 0.0
    What = low
    What[:, rep.weak_idx] += rep.weak_val
    return What


def matvec(rep: Rep, x: np.ndarray) -> np.ndarray:
    """y[b, i] = sum_j s(q_ij - z) x[b, j] (non-weak j) + sum_t v_{i,t} x[b, idx_t]
    -- the sum of (zero-filled quantized matrix x fp16 activation) and
    (fp16 weak columns x the matching activation channels).  x is
    [B][K] (torch layout; the paper's X is C_in x N, reading s18); every
    operand is widened exactly to fp64 and summed in fp64."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    M, K = rep.M, rep.K
    gi = np.array([j // rep.group if rep.group else 0 for j in range(K)])
    low = rep.scale[:, gi] * (rep.codes.astype(np.float64) - rep.zero[:, gi])
    low[:, rep.weak_idx] = 0.0
    y = x @ low.T
    if rep.k:
        y += x[:, rep.weak_idx] @ rep.weak_val.T
    return y


def matvec_rows(rep: Rep, x: np.ndarray, rows) -> np.ndarray:
    """The same definition as ``matvec`` evaluated for selected output rows only
    (for sampled parity at sizes where the full fp64 matrix does not fit):
    y[b, r] for r in rows, one row at a time."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    K = rep.K
    gi = np.array([j // rep.group if rep.group else 0 for j in range(K)])
    weak = np.asarray(rep.weak_idx, dtype=np.int64)
    out = np.zeros((x.shape[0], len(rows)))
    for n, i in enumerate(rows):
        low = rep.scale[i, gi] * (rep.codes[i].astype(np.float64) - rep.zero[i, gi])
        low[weak] = 0.0
        out[:, n] = x @ low
        if weak.size:
            out[:, n] += x[:, weak] @ rep.weak_val[i]
    return out


def layer_error(W, What, X) -> float:
    """Eq. 2 objective ||W X - W_hat X||_2^2."""
    D = (np.asarray(W, dtype=np.float64) - np.asarray(What, dtype=np.float64))
    return float(np.sum((D @ np.asarray(X, dtype=np.float64)) ** 2))
