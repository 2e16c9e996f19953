"""Pins for the oracle's statement of the hot path, y = W_hat x:
brute-force loops, probes with closed-form answers, linearity."""
import numpy as np
import pytest

import oracle as O
import synth


def _rep_from_synth(d):
    return O.Rep(M=d["M"], K=d["K"], bits=d["bits"], group=d["group"],
                 codes=d["codes"], scale=O.from_fp16_bits(d["scale_f16"]),
                 zero=O.from_fp16_bits(d["zero_f16"]), weak_idx=d["weak_idx"].astype(np.int64),
                 weak_val=O.from_fp16_bits(d["weak_val_f16"]))


@pytest.mark.parametrize("bits,group,k", [(3, 0, 4), (4, 8, 3), (3, 8, 0), (4, 0, 9)])
def test_matvec_brute_force_loops(bits, group, k):
    rep = _rep_from_synth(synth.representation(7, 24, bits, group, k, seed=3))
    x = synth.activations(2, 24, seed=4).astype(np.float64)
    y = O.matvec(rep, x)
    weak = {int(j): t for t, j in enumerate(rep.weak_idx)}
    for b in range(2):
        for i in range(7):
            acc = 0.0
            for j in range(24):
                g = j // group if group else 0
                if j in weak:
                    acc += rep.weak_val[i, weak[j]] * x[b, j]          # fp16 weak column
                else:
                    acc += rep.scale[i, g] * (int(rep.codes[i, j]) - rep.zero[i, g]) * x[b, j]
            assert y[b, i] == pytest.approx(acc, rel=1e-13, abs=1e-15)


def test_probes_are_exact():
    # x = e_j, weak j -> y = weak_val[:, t] exactly (low-bit part zero-filled);
    # x = e_j, non-weak j -> y_i = s_i (q_ij - z_i) exactly.
    d = synth.representation(16, 40, 3, 0, 5, seed=9)
    rep = _rep_from_synth(d)
    for t, j in enumerate(rep.weak_idx):
        e = np.zeros((1, 40)); e[0, j] = 1.0
        assert np.array_equal(O.matvec(rep, e)[0], rep.weak_val[:, t])
    for j in range(40):
        if j in set(rep.weak_idx.tolist()):
            continue
        e = np.zeros((1, 40)); e[0, j] = 1.0
        assert np.array_equal(O.matvec(rep, e)[0], rep.scale[:, 0] * (rep.codes[:, j] - rep.zero[:, 0]))


def test_matvec_linear_and_matches_materialized_matrix():
    rep = _rep_from_synth(synth.representation(33, 70, 4, 16, 6, seed=11))
    r = np.random.default_rng(12)
    x1, x2 = r.normal(size=(3, 70)), r.normal(size=(3, 70))
    a, b = 1.7, -0.3
    lhs = O.matvec(rep, a * x1 + b * x2)
    assert np.allclose(lhs, a * O.matvec(rep, x1) + b * O.matvec(rep, x2), rtol=1e-12, atol=1e-14)
    Wh = O.dequant_matrix(rep)
    assert np.allclose(O.matvec(rep, x1), x1 @ Wh.T, rtol=1e-12, atol=1e-14)


def test_zero_fill_ignores_stored_weak_codes():
    # the low-precision matrix is zero on weak columns whatever code is stored
    d = synth.representation(8, 20, 3, 0, 3, seed=13)
    rep = _rep_from_synth(d)
    y0 = O.matvec(rep, np.ones((1, 20)))
    rep.codes = rep.codes.copy(); rep.codes[:, rep.weak_idx] = 7
    assert np.array_equal(O.matvec(rep, np.ones((1, 20))), y0)


def test_quantizer_output_feeds_matvec():
    W, X, ch = synth.weights_and_calib(24, 64, N=256, n_outliers=2, seed=14)
    rep = O.owq_quantize(W, X, 3, 2)
    x = synth.activations(1, 64, seed=15, outliers=ch).astype(np.float64)
    assert np.allclose(O.matvec(rep, x), x @ O.dequant_matrix(rep).T, rtol=1e-12)
    # the mixed representation approximates W x far better than zero
    err = np.abs(O.matvec(rep, x) - x @ W.T).max()
    assert err < 0.25 * np.abs(x @ W.T).max()


def test_matvec_rows_brute_force():
    rep = _rep_from_synth(synth.representation(9, 30, 3, 0, 4, seed=21))
    x = synth.activations(2, 30, seed=22).astype(np.float64)
    rows = [0, 4, 8]
    y = O.matvec_rows(rep, x, rows)
    weak = {int(j): t for t, j in enumerate(rep.weak_idx)}
    for b in range(2):
        for n, i in enumerate(rows):
            acc = 0.0
            for j in range(30):
                acc += (rep.weak_val[i, weak[j]] if j in weak else
                        rep.scale[i, 0] * (int(rep.codes[i, j]) - rep.zero[i, 0])) * x[b, j]
            assert y[b, n] == pytest.approx(acc, rel=1e-13, abs=1e-15)
