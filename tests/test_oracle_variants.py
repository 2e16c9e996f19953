"""Pins for oracle/owq_variants.py (NEXT-4: act-order P:411-412, storage-favored
P:486-490).  Nothing here re-types the functions under test: the permutation
is checked against hand-made Hessians, OPTQ steps against an independent
least-squares solve, the grids against the RTN special case, and the matvec
against probes and a different association order."""
import itertools

import numpy as np
import pytest

import oracle as O
import synth


def test_act_order_perm_hand_made():
    H = np.diag([1.0, 5.0, 3.0, 5.0, 0.5, 9.0])
    # descending diag, ties -> smaller index; weak columns last, ascending
    assert O.act_order_perm(H).tolist() == [5, 1, 3, 2, 0, 4]
    assert O.act_order_perm(H, weak=[5, 0]).tolist() == [1, 3, 2, 4, 0, 5]


@pytest.mark.parametrize("group", [0, 4])
def test_ordered_sweep_diagonal_h_is_rtn_on_order_groups(group):
    # diagonal H: no compensation, so each column's code is RTN on its group's
    # grid, and the grid of group c is the min-max grid of order positions
    # c*g .. c*g+g-1 (consecutive in the QUANTIZATION order, not by index)
    r = np.random.default_rng(3)
    M, K = 5, 12
    W = r.normal(size=(M, K))
    d = r.uniform(0.5, 4.0, size=K)
    H = np.diag(d)
    order = O.act_order_perm(H)
    codes, s, z, Wp = O.optq_quantize_ordered(W, H, 3, order, K, group, clip=False)
    for i in range(K):
        gi = i // group if group else 0
        lo, hi = (gi * group, min(K, gi * group + group)) if group else (0, K)
        for row in range(M):
            vals = W[row, order[lo:hi]]
            a, b = min(vals.min(), 0.0), max(vals.max(), 0.0)
            sc = float(np.float16((b - a) / 7))
            zz = float(np.clip(np.rint(-a / sc), 0, 7))
            assert s[row, gi] == sc and z[row, gi] == zz
            assert codes[row, i] == np.clip(np.rint(W[row, order[i]] / sc) + zz, 0, 7)
    assert np.array_equal(Wp, W[:, order])   # nothing moved


def test_ordered_sweep_steps_are_least_squares_optimal():
    # after each step the not-yet-quantized coordinates equal the constrained
    # least-squares optimum given the quantized ones (independent np.linalg.solve)
    r = np.random.default_rng(4)
    worst = 0.0
    for trial in range(60):
        K = int(r.integers(3, 9)); M = 2
        W = r.normal(size=(M, K))
        X = r.normal(size=(K, 3 * K)) + 0.8 * r.normal(size=(1, 3 * K))
        Hd, _ = O.dampen(O.hessian(X))
        order = O.act_order_perm(Hd, weak=[int(r.integers(0, K))])
        nq = K - 1
        deq = {}

        def on_step(i, order_, Wp):
            deq[i] = Wp.copy()

        codes, s, z, _ = O.optq_quantize_ordered(W, Hd, 2, order, nq, 0, clip=False, on_step=on_step)
        Wo, Ho = W[:, order], Hd[np.ix_(order, order)]
        for i in range(nq):
            A, F = list(range(i + 1)), list(range(i + 1, K))
            D_A = s[:, [0]] * (codes[:, A].astype(np.float64) - z[:, [0]])
            want = Wo[:, F] + np.linalg.solve(Ho[np.ix_(F, F)].T, ((Wo[:, A] - D_A) @ Ho[np.ix_(A, F)]).T).T
            worst = max(worst, float(np.max(np.abs(deq[i][:, F] - want))))
    assert worst < 1e-9


def test_act_order_brute_force_tiny():
    # M = 1, K <= 5, b = 2: the global optimum over all 4^K code vectors on the
    # fixed grid <= ordered OPTQ <= RTN, in >= 95 % of seeds
    r = np.random.default_rng(5)
    ok = 0
    n = 60
    for _ in range(n):
        K = int(r.integers(2, 6))
        W = r.normal(size=(1, K))
        X = r.normal(size=(K, 4 * K)) * r.uniform(0.3, 3.0, size=(K, 1))
        H = O.hessian(X)
        Hd, _ = O.dampen(H)
        order = O.act_order_perm(H)
        codes, s, z, _ = O.optq_quantize_ordered(W, Hd, 2, order, K, 0, clip=False)
        sc, zz = s[0, 0], z[0, 0]
        q_opt = np.zeros(K)
        q_opt[order] = codes[0]

        def err(q):
            dlt = W[0] - sc * (q - zz)
            return float(dlt @ H @ dlt)

        best = min(err(np.array(c, dtype=np.float64)) for c in itertools.product(range(4), repeat=K))
        rtn = err(np.clip(np.rint(W[0] / sc) + zz, 0, 3))
        ok += best <= err(q_opt) + 1e-12 and err(q_opt) <= rtn + 1e-12
    assert ok >= 0.95 * n


@pytest.mark.parametrize("act_order", [False, True])
@pytest.mark.parametrize("group", [0, 16])
def test_variant_representation_invariants(act_order, group):
    W, X, ch = synth.weights_and_calib(24, 64, N=256, n_outliers=3, seed=7)
    lat = O.owq_quantize_variant(W, X, 3, 4, group=group, act_order=act_order, mode="latency")
    sto = O.owq_quantize_variant(W, X, 3, 4, group=group, act_order=act_order, mode="storage")
    assert set(ch) <= set(lat.weak_idx.tolist())
    assert lat.Ks == 64 and sto.Ks == 60
    assert sorted(lat.colmap.tolist()) == list(range(64))
    assert set(sto.colmap.tolist()) == set(range(64)) - set(lat.weak_idx.tolist())
    assert lat.codes.max() <= 7 and np.array_equal(lat.weak_val, O.fp16(lat.weak_val))
    # zero fill (reading s10): weak stored positions hold their group's zero point
    for p in range(60, 64):
        gi = p // group if group else 0
        assert np.array_equal(lat.codes[:, p], lat.zero[:, gi])
    # the same quantization stored both ways gives the same W_hat and the same y
    assert np.array_equal(O.dequant_matrix_stored(lat), O.dequant_matrix_stored(sto))
    x = synth.activations(3, 64, seed=1, outliers=lat.weak_idx)
    assert np.allclose(O.matvec_stored(lat, x), O.matvec_stored(sto, x), rtol=0, atol=1e-12)
    # re-association: matvec == x @ W_hat^T (original order), fp64
    y = O.matvec_stored(sto, x)
    assert np.max(np.abs(y - x.astype(np.float64) @ O.dequant_matrix_stored(sto).T)) <= 1e-12 * np.max(np.abs(y))
    assert np.array_equal(O.stored_from_rep(lat).codes, sto.codes)


def test_matvec_stored_probes():
    # x = e_j: weak j -> v[:, t] exactly; mapped j at stored position p -> s(q - z)
    W, X, ch = synth.weights_and_calib(8, 40, N=128, n_outliers=2, seed=9)
    rep = O.owq_quantize_variant(W, X, 4, 3, group=8, act_order=True, mode="storage")
    pos = {int(c): p for p, c in enumerate(rep.colmap)}
    for j in range(40):
        x = np.zeros((1, 40)); x[0, j] = 1.0
        y = O.matvec_stored(rep, x)[0]
        if j in set(rep.weak_idx.tolist()):
            t = rep.weak_idx.tolist().index(j)
            assert np.array_equal(y, rep.weak_val[:, t])
        else:
            p = pos[j]
            assert np.array_equal(y, rep.scale[:, p // 8] * (rep.codes[:, p] - rep.zero[:, p // 8]))


def test_act_order_helps_on_outlier_fixture():
    # the paper's observation: act-order improves OPTQ, OWQ improves both;
    # statistical: layer error of OWQ(k) with act-order < OPTQ act-order (k = 0) in most seeds
    wins = 0
    for seed in range(12):
        W, X, ch = synth.weights_and_calib(16, 48, N=192, n_outliers=2, seed=100 + seed)
        a0 = O.owq_quantize_variant(W, X, 3, 0, act_order=True)
        a2 = O.owq_quantize_variant(W, X, 3, 2, act_order=True)
        e0 = O.layer_error(W, O.dequant_matrix_stored(a0), X)
        e2 = O.layer_error(W, O.dequant_matrix_stored(a2), X)
        wins += e2 < e0
    assert wins >= 11
