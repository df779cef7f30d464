"""The Kalman/RTS oracle and the three-way agreement of the
sparse-precision oracle, the Kalman filter + RTS smoother and the dense GP
(acceptance criterion 1): MLL, posterior mean and variance at the
training points, and predictions at test times (the filter over the merged grid with
test times as missing observations)."""
import numpy as np
import pytest

import oracle_lib as O
from test_oracle_engine import data, dense_gp
from test_predict import dense_predict

KERNELS = [
    ([O.MATERN12], [0.8, 1.7]),
    ([O.MATERN32], [1.3, 0.9]),
    ([O.MATERN52], [2.1, 1.2]),
    ([(O.EQ, 6)], [1.1, 1.4]),
    ([O.MATERN32, O.MATERN12], [1.0, 0.7, 0.5, 2.0]),
]


def tols(leaves):
    # EQ order 6: the modal Pinf is ill-conditioned and Q cancels below the jitter; the
    # fp64 floor of the SPEC formulation is ~1e-5 (tests/test_oracle_engine.py)
    return (3e-5, 2e-4) if leaves[0] == (O.EQ, 6) else (1e-7, 1e-6)


@pytest.mark.parametrize("leaves,theta", KERNELS)
@pytest.mark.parametrize("n", [1, 2, 50, 300])
def test_three_way_training_points(leaves, theta, n):
    rng = np.random.default_rng(100 + n)
    t, y = data(rng, n)
    sp = O.evaluate(leaves, theta, t, y, 0.3)
    kf = O.kf_rts(leaves, theta, t, y, 0.3)
    ll_d, mean_d, var_d = dense_gp(leaves, theta, t, y, 0.3)
    tol, mtol = tols(leaves)
    assert kf["loglik"] == pytest.approx(sp["loglik"], rel=tol)
    assert kf["loglik"] == pytest.approx(ll_d, rel=tol)
    for a, b in ((kf["mean"], sp["mean"]), (kf["mean"], mean_d), (kf["var"], sp["var"]), (kf["var"], var_d)):
        assert np.abs(a - b).max() < mtol


@pytest.mark.parametrize("leaves,theta", KERNELS)
def test_kf_rts_predict_matches_dense_gp(leaves, theta):  # SPEC.md:396 (N=30, M=10)
    rng = np.random.default_rng(7)
    t = np.cumsum(rng.uniform(0.1, 0.4, 30))
    y = np.sin(t) + 0.3 * rng.standard_normal(30)
    ts = rng.uniform(t[0] - 1.0, t[-1] + 1.0, 10)
    ll, mean, var = O.kf_rts_predict(leaves, theta, t, y, ts, 0.3)
    ll_d, mean_d, var_d = dense_predict(leaves, theta, t, y, ts, 0.3)
    tol, mtol = tols(leaves)
    assert ll == pytest.approx(ll_d, rel=tol)
    assert np.abs(mean - mean_d).max() < mtol and np.abs(var - var_d).max() < mtol


@pytest.mark.parametrize("leaves,theta", KERNELS[:3] + KERNELS[4:])
def test_smoothed_variance_never_exceeds_filtered(leaves, theta):
    rng = np.random.default_rng(11)
    t, y = data(rng, 200)
    kf = O.kf_rts(leaves, theta, t, y, 0.3)
    assert np.all(kf["var"] <= kf["fvar"] + 1e-10)
    assert kf["var"][-1] == kf["fvar"][-1]  # no future data after the last point


def test_single_point_smoother_equals_filter():
    kf = O.kf_rts([O.MATERN32], [1.0, 2.0], [0.5], [0.3], 0.3)
    assert kf["var"][0] == kf["fvar"][0]
    # N=1 closed form: posterior variance of f given y = k - k^2 / (k + s^2)
    assert kf["var"][0] == pytest.approx(1.0 - 1.0 / (1.0 + 0.09), rel=1e-9)


def test_kf_mll_time_translation_invariant():
    rng = np.random.default_rng(3)
    t, y = data(rng, 100)
    a = O.kf_rts([O.MATERN52], [2.0, 1.5], t, y, 0.2)["loglik"]
    b = O.kf_rts([O.MATERN52], [2.0, 1.5], t + 1234.5, y, 0.2)["loglik"]
    assert a == pytest.approx(b, rel=1e-10)
