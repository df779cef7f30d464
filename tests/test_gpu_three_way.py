"""The GPU path (sm_100a kernels through the C ABI) in the oracle triangle of
SPEC.md:399,507 (acceptance criterion 1): GPU vs the Kalman filter + RTS smoother vs the
dense GP, on the MLL, the posterior mean/variance at the training points and the
predictions at test times (spingp_predict vs kf_rts_predict over the merged grid)."""
import numpy as np
import pytest

import oracle_lib as O
import paper_1610_08035_b200 as P
from test_oracle_engine import data, dense_gp
from test_oracle_kf_rts import KERNELS, tols
from test_predict import dense_predict

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("leaves,theta", KERNELS)
@pytest.mark.parametrize("n", [1, 2, 50, 300])
def test_gpu_kf_dense_training_points(ctx, leaves, theta, n):
    rng = np.random.default_rng(100 + n)
    t, y = data(rng, n)
    g = ctx.eval(leaves, theta, t, y, 0.3, grad=False, mean=True, var=True)
    kf = O.kf_rts(leaves, theta, t, y, 0.3)
    ll_d, mean_d, var_d = dense_gp(leaves, theta, t, y, 0.3)
    tol, mtol = tols(leaves)
    assert g["loglik"] == pytest.approx(kf["loglik"], rel=tol)
    assert g["loglik"] == pytest.approx(ll_d, rel=tol)
    for ref in (kf["mean"], mean_d):
        assert np.abs(g["mean"] - ref).max() < mtol
    for ref in (kf["var"], var_d):
        assert np.abs(g["var"] - ref).max() < mtol


@pytest.mark.parametrize("leaves,theta", KERNELS)
def test_gpu_predict_kf_rts_dense(ctx, leaves, theta):  # SPEC.md:396, 303 (N=30, M=10)
    rng = np.random.default_rng(7)
    t = np.cumsum(rng.uniform(0.1, 0.4, 30))
    y = np.sin(t) + 0.3 * rng.standard_normal(30)
    ts = rng.uniform(t[0] - 1.0, t[-1] + 1.0, 10)
    p = ctx.predict(leaves, theta, t, y, ts, 0.3, grad=False)
    ll_k, mean_k, var_k = O.kf_rts_predict(leaves, theta, t, y, ts, 0.3)
    ll_d, mean_d, var_d = dense_predict(leaves, theta, t, y, ts, 0.3)
    tol, mtol = tols(leaves)
    assert p["loglik"] == pytest.approx(ll_k, rel=tol) and p["loglik"] == pytest.approx(ll_d, rel=tol)
    for m_, v_ in ((mean_k, var_k), (mean_d, var_d)):
        assert np.abs(p["mean"] - m_).max() < mtol and np.abs(p["var"] - v_).max() < mtol


def test_gpu_matches_kf_rts_on_a_long_series(ctx):
    """20,000 points through the multi-level GPU path vs the sequential KF/RTS."""
    rng = np.random.default_rng(5)
    t = np.cumsum(rng.uniform(0.05, 0.15, 20_000))
    y = np.sin(0.5 * t) + 0.3 * rng.standard_normal(len(t))
    g = ctx.eval([P.MATERN32], [1.0, 2.0], t, y, 0.3, grad=False, mean=True, var=True)
    kf = O.kf_rts([O.MATERN32], [1.0, 2.0], t, y, 0.3)
    assert g["loglik"] == pytest.approx(kf["loglik"], rel=1e-9)
    assert np.abs(g["mean"] - kf["mean"]).max() < 1e-9
    assert np.abs(g["var"] - kf["var"]).max() < 1e-9
