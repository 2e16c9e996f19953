"""Pins for the oracle's OPTQ / OWQ quantizer (Eq. 1).
Its exact codes on large random layers have no external pin ("parity unpinned",
DESIGN.md §3); these special cases and properties pin its arithmetic."""
import itertools

import numpy as np
import pytest

import oracle as O
import synth


def test_diagonal_hessian_reduces_to_rtn():
    # diagonal H -> no compensation -> codes == per-row RTN on the same grid
    r = np.random.default_rng(20)
    for clip in (False, True):
        W = r.normal(0, 0.02, size=(12, 24))
        H = np.diag(r.uniform(0.5, 3.0, size=24))
        codes, s, z, wv = O.optq_quantize(W, H, 3, 0, (), clip)
        for i in range(12):
            assert np.array_equal(codes[i], O.quantize(W[i], s[i, 0], z[i, 0], 3).astype(np.uint8))
    # with weak columns: the weak ones keep their original values (nothing to absorb)
    codes, s, z, wv = O.optq_quantize(W, H, 3, 0, (3, 17), True)
    assert np.array_equal(wv, W[:, [3, 17]])


def test_every_step_is_the_constrained_least_squares_optimum():
    # S:254 / acceptance 3: after each OPTQ step the not-yet-quantized coordinates equal
    # argmin dW H dW^T with the quantized coordinates fixed -- solved here independently
    # with np.linalg.solve on H's blocks (no Cholesky, no sequential updates).
    r = np.random.default_rng(21)
    worst = 0.0
    for trial in range(200):
        K = int(r.integers(2, 9)); M = int(r.integers(1, 4))
        W = r.normal(size=(M, K))
        X = r.normal(size=(K, 3 * K)) * r.uniform(0.2, 3, size=(K, 1))
        X += 0.7 * r.normal(size=(1, 3 * K))            # correlated channels
        Hd, _ = O.dampen(O.hessian(X))
        nweak = int(r.integers(0, min(2, K - 1) + 1))
        weak = tuple(sorted(r.choice(K, size=nweak, replace=False))) if nweak else ()
        fixed = {}

        def on_step(i, perm, Wp, dcol):
            fixed[i] = dcol
            Q = list(range(i + 1)); F = list(range(i + 1, K))
            if not F:
                return
            Hp = Hd[np.ix_(perm, perm)]
            W0 = W[:, perm]
            dQ = W0[:, Q] - np.stack([fixed[q] for q in Q], axis=1)
            dF = -np.linalg.solve(Hp[np.ix_(F, F)], Hp[np.ix_(F, Q)] @ dQ.T).T
            expect = W0[:, F] - dF
            nonlocal worst
            err = np.abs(Wp[:, F] - expect).max() / max(np.abs(expect).max(), 1e-12)
            worst = max(worst, err)

        O.optq_quantize(W, Hd, 2, 0, weak, False, on_step=on_step)
    assert worst < 1e-8


def test_optq_1x2_example():
    # 1x2 layer w = [0.6, 0.4], H = [[4,2],[2,3]], 1-bit grid {0, 1}
    W = np.array([[0.6, 0.4]]); H = np.array([[4.0, 2.0], [2.0, 3.0]])
    seen = {}
    O.optq_quantize(W, H, 1, 0, (), False, on_step=lambda i, p, Wp, d: seen.setdefault(i, Wp))
    # grid: xmin=0, xmax=0.6 -> s = fp16(0.6); column 0 -> code 1 -> value s
    s = float(np.float16(0.6))
    d0 = 0.6 - s
    # unconstrained optimum for the free coordinate: w1' = 0.4 + (H01/H11) * d0
    assert seen[0][0, 1] == pytest.approx(0.4 + (2.0 / 3.0) * d0, rel=1e-12)


def test_brute_force_tiny_layers():
    # M=1, K<=6, b=2: enumerate every code vector on OPTQ's grid; the global optimum of
    # ||(W - What) X||^2 <= OPTQ's, and OPTQ <= RTN (same grid) in >= 95% of seeds.
    r = np.random.default_rng(22)
    better_than_rtn = 0
    n = 100
    for seed in range(n):
        K = int(r.integers(3, 7))
        W = r.normal(size=(1, K))
        X = r.normal(size=(K, 40)) + 0.8 * r.normal(size=(1, 40))
        H = O.hessian(X)
        Hd, _ = O.dampen(H)
        codes, s, z, _ = O.optq_quantize(W, Hd, 2, 0, (), False)
        s0, z0 = s[0, 0], z[0, 0]
        e_optq = O.layer_error(W, O.dequantize(codes, s0, z0), X)
        e_rtn = O.layer_error(W, O.dequantize(O.quantize(W, s0, z0, 2), s0, z0), X)
        best = min(O.layer_error(W, O.dequantize(np.array([c]), s0, z0), X)
                   for c in itertools.product(range(4), repeat=K))
        assert best <= e_optq + 1e-12
        better_than_rtn += int(e_optq <= e_rtn + 1e-12)
    assert better_than_rtn >= 95


def _outlier_fixture(seed, c_out=16, c_in=64, n=2048):
    r = np.random.default_rng(1000 + seed)
    W = r.normal(size=(c_out, c_in))
    X = r.normal(size=(c_in, n))
    ch = int(r.integers(c_in))
    X[ch] *= 100.0
    return W, X, ch


def test_error_ordering_owq_optq_rtn():
    # SPEC acceptance 5: E(OWQ, k=1) < E(OPTQ) and E(OPTQ) < E(RTN) in >= 95/100 seeds
    a = b = sel = 0
    for seed in range(100):
        W, X, ch = _outlier_fixture(seed)
        rep = O.owq_quantize(W, X, 3, 1, clip=True)
        e_owq = O.layer_error(W, O.dequant_matrix(rep), X)
        Hd, _ = O.dampen(O.hessian(X))
        codes, s, z, _ = O.optq_quantize(W, Hd, 3, 0, (), False)
        e_optq = O.layer_error(W, s[:, [0]] * (codes - z[:, [0]]), X)
        e_rtn = O.layer_error(W, W - O.rtn_delta(W, 3), X)
        a += int(e_owq < e_optq); b += int(e_optq < e_rtn)
        sel += int(list(rep.weak_idx) == [ch])              # acceptance 6
    assert a >= 95 and b >= 95 and sel >= 95


def test_owq_representation_invariants():
    # BASELINE north_star invariants: codes in [0, 2^b-1]; weak columns reproduced exactly
    # in fp16; dequant of weak columns' low-bit part is exactly 0 (zero-filled).
    W, X, ch = synth.weights_and_calib(48, 96, N=256, n_outliers=3, seed=5)
    for group in (0, 32):
        rep = O.owq_quantize(W, X, 3, 4, group=group)
        assert rep.codes.max() <= 7 and rep.codes.dtype == np.uint8
        assert set(ch) <= set(rep.weak_idx.tolist())         # outlier channels are picked
        gi = np.array([j // group if group else 0 for j in range(96)])
        for j in rep.weak_idx:
            assert np.array_equal(rep.codes[:, j], rep.zero[:, gi[j]])
        Wh = O.dequant_matrix(rep)
        assert np.array_equal(Wh[:, rep.weak_idx], rep.weak_val)
        assert np.array_equal(rep.weak_val, O.fp16(rep.weak_val))
        assert np.array_equal(rep.scale, O.fp16(rep.scale))
        # k = 0 (extra_bits = 0) is bit-identical to plain OPTQ with the tuned grid (acceptance 9)
    rep0 = O.owq_quantize(W, X, 3, 0)
    Hd, dead = O.dampen(O.hessian(X))
    codes, s, z, _ = O.optq_quantize(W, Hd, 3, 0, (), True)
    assert np.array_equal(rep0.codes, codes)


def test_grouped_grid_fits_per_group():
    r = np.random.default_rng(23)
    W = r.normal(size=(4, 16)); W[:, 8:] *= 10
    X = r.normal(size=(16, 64))
    rep = O.owq_quantize(W, X, 3, 0, group=8, clip=False)
    assert rep.scale.shape == (4, 2)
    assert np.all(rep.scale[:, 1] > 3 * rep.scale[:, 0])


def test_grouped_grid_refit_on_compensated_values():
    # SURVEY §8(c) step 7 (the grid is fitted "after removing the weak columns";
    # every not-yet-quantized column carries the compensation): with g > 0 a
    # group's grid is fitted when the sweep reaches the group, on the group's CURRENT
    # non-weak values.  Those values are solved here independently: the constrained
    # least-squares optimum with the earlier group's dequantized values fixed,
    # W_F + (W_A - D_A) H_AF H_FF^-1 (np.linalg.solve, no Cholesky, no sequential
    # updates); the min-max grid is s = fp16((max(v,0) - min(v,0)) / (2^b - 1)),
    # z = rne(-min(v,0)/s) (pinned by the S:174-176 examples).  The alternatives a
    # plausible bug would use -- the original W, or every non-weak column at once --
    # must give a different grid in most seeds, so the test has teeth.
    r = np.random.default_rng(77)
    bits, g, K, M = 2, 4, 8, 3
    weak = (5,)
    A, F = [0, 1, 2, 3], [4, 5, 6, 7]
    grp1 = [4, 6, 7]                              # group 1 without its weak column
    n_orig_differs = n_all_differs = 0
    trials = 60
    for _ in range(trials):
        W = r.normal(size=(M, K))
        X = r.normal(size=(K, 4 * K)) + 0.9 * r.normal(size=(1, 4 * K))   # correlated channels
        Hd, _ = O.dampen(O.hessian(X))
        codes, s, z, wv = O.optq_quantize(W, Hd, bits, g, weak, clip=False)
        D_A = s[:, [0]] * (codes[:, A].astype(np.float64) - z[:, [0]])
        HAF, HFF = Hd[np.ix_(A, F)], Hd[np.ix_(F, F)]
        cur = W[:, F] + np.linalg.solve(HFF.T, ((W[:, A] - D_A) @ HAF).T).T
        v = cur[:, [F.index(j) for j in grp1]]

        def minmax(vals):
            lo, hi = min(vals.min(), 0.0), max(vals.max(), 0.0)
            sc = float(np.float16((hi - lo) / (2 ** bits - 1)))
            return sc, float(np.clip(np.rint(-lo / sc), 0, 2 ** bits - 1))

        for i in range(M):
            se, ze = minmax(v[i])
            assert s[i, 1] == se and z[i, 1] == ze, (i, s[i, 1], se, z[i, 1], ze)
            if minmax(W[i, grp1]) != (se, ze):
                n_orig_differs += 1
            if minmax(W[i, [0, 1, 2, 3, 4, 6, 7]]) != (se, ze):
                n_all_differs += 1
    assert n_orig_differs > trials * M // 2 and n_all_differs > trials * M // 2
