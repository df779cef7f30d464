"""predict at arbitrary test times.

The test points join the training grid without an observation term (SPEC.md:251-254,
"infinity in the limit sense"), so the same partitioned elimination and selected inverse
give their posterior mean and latent variance.  Checked against:
* a dense GP on the state-space implied covariance (1e-6 absolute);
* the training-only evaluation (mask invariance);
* the prior variance far from the data.
The CPU half runs the exact kernel code through the host emulation; the GPU half runs
the sm_100a kernels through the C ABI (spingp_predict)."""
import math

import numpy as np
import pytest

import emu_lib as E
import oracle_lib as O
from conftest import rel

KERNELS = [
    ([O.MATERN12], [0.8, 1.7]),
    ([O.MATERN32], [1.3, 0.9]),
    ([O.MATERN52], [2.1, 1.2]),
    ([O.MATERN32, O.MATERN12], [1.0, 0.7, 0.5, 2.0]),
    ([(O.QP, 3)], [1.0, 0.8, 1.3, 5.0]),
]


def dense_predict(leaves, theta, t, y, ts, s):
    k = lambda a, b: np.array([[O.implied_covariance(leaves, theta, u - v) for v in b] for u in a])  # noqa: E731
    C = k(t, t) + s * s * np.eye(len(t))
    Ks = k(ts, t)
    mean = Ks @ np.linalg.solve(C, y)
    var = O.implied_covariance(leaves, theta, 0.0) - np.einsum("ij,ji->i", Ks, np.linalg.solve(C, Ks.T))
    ll = -0.5 * y @ np.linalg.solve(C, y) - 0.5 * np.linalg.slogdet(C)[1] - 0.5 * len(t) * math.log(2 * math.pi)
    return ll, mean, var


def case(seed, n=30, m=10):
    rng = np.random.default_rng(seed)
    t = np.cumsum(rng.uniform(0.1, 0.4, n))
    y = np.sin(t) + 0.3 * rng.standard_normal(n)
    ts = rng.uniform(t[0] - 1.0, t[-1] + 1.0, m)  # interleaved and beyond both ends, unsorted
    return t, y, ts


@pytest.mark.parametrize("leaves,theta", KERNELS)
def test_emu_predict_matches_dense_gp(leaves, theta):
    t, y, ts = case(3)
    p = E.predict(leaves, theta, t, y, ts, 0.3)
    ll, mean, var = dense_predict(leaves, theta, t, y, ts, 0.3)
    assert np.abs(p["mean"] - mean).max() < 1e-6
    assert np.abs(p["var"] - var).max() < 1e-6
    assert abs(p["loglik"] - ll) <= 1e-7 * abs(ll)  # SPEC.md:307 oracle triangle bound


@pytest.mark.parametrize("leaves,theta", KERNELS[:3])
def test_emu_predict_training_posterior_is_mask_invariant(leaves, theta):
    """Adding test points changes nothing about the training data's loglik and gradient
    (SPEC.md:311), up to the jitter of the extra process-noise blocks."""
    t, y, ts = case(5, n=60, m=25)
    p = E.predict(leaves, theta, t, y, ts, 0.3)
    e = E.evaluate(leaves, theta, t, y, 0.3)
    assert rel(p["loglik"], e["loglik"]) < 1e-9
    assert rel(p["grad"], e["grad"]) < 1e-6


def test_emu_predict_at_training_times_is_nudged():
    """A test time equal to a training time is nudged by 1e-9 x span: its
    prediction equals the training posterior there, up to the jitter-sized process noise
    (1e-10 tr(Pinf)/b) of the nudged step (SPEC.md:302 example allows 1e-4)."""
    leaves, theta = [O.MATERN32], [1.0, 2.0]
    t, y, _ = case(7, n=40)
    ts = t[[0, 7, 39]].copy()
    p = E.predict(leaves, theta, t, y, ts, 0.3, include_noise=True)
    e = E.evaluate(leaves, theta, t, y, 0.3, include_noise=True)
    assert np.abs(p["mean"] - e["mean"][[0, 7, 39]]).max() < 1e-6
    assert np.abs(p["var"] - e["var"][[0, 7, 39]]).max() < 1e-6


def test_emu_predict_far_from_data_reverts_to_prior():
    leaves, theta = [O.MATERN52], [1.5, 0.7]
    t, y, _ = case(9)
    ts = np.array([t[-1] + 50.0, t[0] - 40.0])
    p = E.predict(leaves, theta, t, y, ts, 0.2)
    k0 = O.implied_covariance(leaves, theta, 0.0)
    assert np.abs(p["mean"]).max() < 1e-6
    assert np.abs(p["var"] - k0).max() < 1e-6


def test_emu_predict_tiny_and_duplicate_tests():
    leaves, theta = [O.MATERN32], [1.0, 2.0]
    t, y = np.array([0.5]), np.array([0.3])
    ts = np.array([0.5, 0.5, 1.0, -2.0])
    p = E.predict(leaves, theta, t, y, ts, 0.3)
    ll, mean, var = dense_predict(leaves, theta, t, y, ts, 0.3)
    assert np.abs(p["mean"] - mean).max() < 1e-6 and np.abs(p["var"] - var).max() < 1e-6


# ------------------------------------------------------------------------- GPU ----

@pytest.mark.gpu
@pytest.mark.parametrize("leaves,theta", KERNELS)
def test_gpu_predict_matches_dense_gp_and_emulation(ctx, leaves, theta):
    t, y, ts = case(11)
    g = ctx.predict(leaves, theta, t, y, ts, 0.3)
    e = E.predict(leaves, theta, t, y, ts, 0.3)
    ll, mean, var = dense_predict(leaves, theta, t, y, ts, 0.3)
    assert np.abs(g["mean"] - mean).max() < 1e-6 and np.abs(g["var"] - var).max() < 1e-6
    assert abs(g["loglik"] - ll) <= 1e-7 * abs(ll)
    # device vs host emulation of the same kernels: different FMA contraction, so the
    # (conditioning-amplified, e.g. Matérn-5/2) rounding differs; both sit on the dense GP
    assert rel(g["mean"], e["mean"]) < 1e-6 and rel(g["var"], e["var"]) < 1e-6
    assert rel(g["grad"], e["grad"]) < 1e-6


@pytest.mark.gpu
def test_gpu_predict_large_grid_mask_invariance(ctx):
    """200k training points + 50k test points through the full tree path."""
    rng = np.random.default_rng(13)
    n, m = 200_000, 50_000
    t = np.cumsum(rng.exponential(0.01, n))
    y = np.sin(3 * t) + 0.2 * rng.standard_normal(n)
    ts = rng.uniform(t[0], t[-1], m)
    leaves, theta = [O.MATERN52], [2.0, 1.5]
    import paper_1610_08035_b200 as P
    g = ctx.predict([P.MATERN52], theta, t, y, ts, 0.2)
    e = ctx.eval([P.MATERN52], theta, t, y, 0.2, grad=True, mean=True, var=True)
    assert rel(g["loglik"], e["loglik"]) < 1e-8
    # a test point's mean lies within the range of its neighbours' posterior means +- 4 sd
    idx = np.searchsorted(t, ts)
    idx = np.clip(idx, 1, n - 1)
    lo = np.minimum(e["mean"][idx - 1], e["mean"][idx]) - 4 * np.sqrt(np.maximum(e["var"][idx - 1], e["var"][idx]))
    hi = np.maximum(e["mean"][idx - 1], e["mean"][idx]) + 4 * np.sqrt(np.maximum(e["var"][idx - 1], e["var"][idx]))
    assert np.all((g["mean"] >= lo) & (g["mean"] <= hi))
    assert np.all(g["var"] >= 0)
