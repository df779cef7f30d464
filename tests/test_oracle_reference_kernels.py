"""The reference's own kernel_ss test suite (proj/tests/test_kernels.cpp:40-288),
ported case by case and run against the CPU oracle's restatement.

These are the executable pins the reference holds for the path:
printed forms, Taylor-expm oracle, group property, PSD Q, magnitude shortcut,
finite differences, EQ convergence, closed-form Matérn covariances, names.
"""
import math

import numpy as np
import pytest

import oracle_lib as O

ALL_KERNELS = [  # test_kernels.cpp:15-21
    ([O.MATERN12], [0.8, 1.7]),
    ([O.MATERN32], [1.3, 0.9]),
    ([O.MATERN52], [2.1, 1.2]),
    ([(O.EQ, 10)], [1.1, 1.4]),
    ([O.MATERN32, O.MATERN12], [1.0, 0.7, 0.5, 2.0]),
]


def taylor_expm(a):  # test_support.hpp:15-32
    norm = np.abs(a).sum(axis=0).max()
    sq = 0
    while norm > 0.25 and sq < 60:
        norm *= 0.5
        sq += 1
    s = a / 2.0 ** sq
    term = np.eye(len(a))
    tot = term.copy()
    for k in range(1, 31):
        term = term @ s / k
        tot = tot + term
    for _ in range(sq):
        tot = tot @ tot
    return tot


def closed_form(typ, var, ln, tau):  # test_kernels.cpp:23-36
    if typ == O.MATERN12:
        return var * math.exp(-tau / ln)
    if typ == O.MATERN32:
        a = math.sqrt(3) * tau / ln
        return var * (1 + a) * math.exp(-a)
    a = math.sqrt(5) * tau / ln
    return var * (1 + a + a * a / 3) * math.exp(-a)


def test_state_space_of_matern32_matches_printed_form():  # :40-53
    ss = O.state_space([O.MATERN32], [1.0, 0.5])
    l = 0.5
    assert ss["b"] == 2
    F, H, P = ss["F"], ss["H"], ss["Pinf"]
    assert F[0, 0] == 0.0 and F[0, 1] == 1.0
    assert abs(F[1, 0] + 3.0 / (l * l)) < 1e-14
    assert abs(F[1, 1] + 2.0 * math.sqrt(3) / l) < 1e-14
    assert H[0] == 1.0 and H[1] == 0.0
    assert abs(P[0, 0] - 1.0) < 1e-15
    assert abs(P[1, 1] - 3.0 / (l * l)) < 1e-12
    assert P[0, 1] == 0.0


def test_sum_of_matern32_and_eq10_has_block_size_12():  # :55-59
    assert O.state_space([O.MATERN32, (O.EQ, 10)], [1.0, 1.0, 1.0, 1.0])["b"] == 12


def test_matern12_is_ornstein_uhlenbeck():  # :61-69
    ss = O.state_space([O.MATERN12], [1.0, 2.0])
    assert ss["b"] == 1
    assert abs(ss["F"][0, 0] + 0.5) < 1e-15
    assert ss["H"][0] == 1.0 and ss["Pinf"][0, 0] == 1.0
    for tau in (0.0, 0.3, 1.5, 4.0):
        assert abs(O.implied_covariance([O.MATERN12], [1.0, 2.0], tau) - math.exp(-tau / 2.0)) < 1e-12


@pytest.mark.parametrize("leaves,theta", ALL_KERNELS)
def test_stability_and_stationarity(leaves, theta):  # :71-82
    ss = O.state_space(leaves, theta)
    assert np.linalg.eigvals(ss["F"]).real.max() < 0.0
    lyap = ss["F"] @ ss["Pinf"] + ss["Pinf"] @ ss["F"].T
    lyap = 0.5 * (lyap + lyap.T)
    assert np.linalg.eigvalsh(lyap).max() <= 1e-9 * np.linalg.norm(ss["Pinf"])


def test_rejects_bad_input():  # :84-92
    for leaves, theta in [([O.MATERN32], [1.0]), ([O.MATERN32], [-1.0, 1.0]), ([O.MATERN32], [1.0, 0.0]),
                          ([(O.EQ, 3)], [1.0, 1.0]), ([(O.EQ, 0)], [1.0, 1.0]), ([(O.EQ, 18)], [1.0, 1.0])]:
        with pytest.raises(O.OracleError) as e:
            O.state_space(leaves, theta)
        assert e.value.status == 3  # std::invalid_argument


@pytest.mark.parametrize("leaves,theta", ALL_KERNELS)
def test_discretize_zero_gap_is_identity(leaves, theta):  # :94-101
    Phi, Q = O.discretize(leaves, theta, 0.0)
    assert np.array_equal(Phi, np.eye(len(Phi)))
    assert not Q.any()


def test_discretize_transition_matches_taylor_reference():  # :103-108
    ss = O.state_space([O.MATERN32], [1.0, 1.0])
    Phi, _ = O.discretize([O.MATERN32], [1.0, 1.0], 0.5)
    assert np.abs(Phi - taylor_expm(ss["F"] * 0.5)).max() < 1e-10


@pytest.mark.parametrize("leaves,theta", ALL_KERNELS)
def test_discretize_group_property(leaves, theta):  # :110-123
    rng = np.random.default_rng(11)
    for _ in range(10):
        a, b = rng.uniform(0.01, 2.0, 2)
        lhs = O.discretize(leaves, theta, a)[0] @ O.discretize(leaves, theta, b)[0]
        assert np.abs(lhs - O.discretize(leaves, theta, a + b)[0]).max() < 1e-9


@pytest.mark.parametrize("leaves,theta", ALL_KERNELS)
def test_process_noise_is_positive_semidefinite(leaves, theta):  # :125-136
    rng = np.random.default_rng(12)
    for _ in range(20):
        _, Q = O.discretize(leaves, theta, rng.uniform(1e-3, 5.0))
        assert np.linalg.eigvalsh(Q).min() >= -1e-10 * np.trace(Q)


def test_discretize_with_grad_magnitude_shortcut():  # :138-143
    Phi, Q, dPhi, dQ = O.discretize([O.MATERN32], [2.5, 1.3], 0.7, grad=True)
    assert not dPhi[0].any()
    assert np.abs(dQ[0] - Q / 2.5).max() < 1e-12


@pytest.mark.parametrize("leaves,theta", ALL_KERNELS)
def test_discretize_with_grad_zero_gap(leaves, theta):  # :145-152
    _, _, dPhi, dQ = O.discretize(leaves, theta, 0.0, grad=True)
    assert not dPhi.any() and not dQ.any()


@pytest.mark.parametrize("leaves,theta", ALL_KERNELS)
def test_discretize_with_grad_matches_finite_differences(leaves, theta):  # :159-183
    dt = 0.3
    _, _, dPhi, dQ = O.discretize(leaves, theta, dt, grad=True)
    for p in range(len(theta)):
        h = 1e-6 * theta[p]
        tp, tm = list(theta), list(theta)
        tp[p] += h
        tm[p] -= h
        Pp, Qp = O.discretize(leaves, tp, dt)
        Pm, Qm = O.discretize(leaves, tm, dt)
        fd_phi, fd_q = (Pp - Pm) / (2 * h), (Qp - Qm) / (2 * h)
        assert np.abs(dPhi[p] - fd_phi).max() / max(np.abs(fd_phi).max(), 1e-8) < 1e-4
        assert np.abs(dQ[p] - fd_q).max() / max(np.abs(fd_q).max(), 1e-8) < 1e-4


def test_matern32_lengthscale_against_tight_fd():  # :185-197
    th = [1.0, 1.1]
    _, _, dPhi, _ = O.discretize([O.MATERN32], th, 0.3, grad=True)
    h = 1e-6 * th[1]
    fd = (O.discretize([O.MATERN32], [1.0, 1.1 + h], 0.3)[0] - O.discretize([O.MATERN32], [1.0, 1.1 - h], 0.3)[0]) / (2 * h)
    assert np.abs(dPhi[1] - fd).max() / np.abs(fd).max() < 1e-5


def test_eq_order_ten_has_state_dimension_ten():  # :199-202
    assert O.state_space([(O.EQ, 10)], [1.0, 1.0])["b"] == 10


def test_eq_implied_variance_equals_magnitude():  # :204-207
    assert abs(O.implied_covariance([(O.EQ, 10)], [1.7, 0.8], 0.0) / 1.7 - 1.0) < 1e-6


def test_eq_converges_monotonically_to_exact_eq():  # :209-223
    var, ln = 1.3, 0.9
    prev = math.inf
    for order in (4, 6, 8, 10):
        dev = max(abs(O.implied_covariance([(O.EQ, order)], [var, ln], tau) - var * math.exp(-0.5 * (tau / ln) ** 2))
                  for tau in (5.0 * ln * i / 200 for i in range(201)))
        assert dev <= prev * (1 + 1e-12)
        prev = dev
    assert prev <= 0.02 * var


def test_kernel_eval_zero_gap_gives_magnitude():  # :225-227
    assert O.implied_covariance([O.MATERN32], [2.2, 1.0], 0.0) == pytest.approx(2.2, abs=1e-15)


def test_kernel_eval_matern32_printed_value():  # :229-233
    v = O.implied_covariance([O.MATERN32], [1.0, 1.0], 1.0)
    assert abs(v - (1 + math.sqrt(3)) * math.exp(-math.sqrt(3))) < 1e-12
    assert abs(v - 0.48335) < 1e-4


@pytest.mark.parametrize("leaves,theta", ALL_KERNELS)
def test_kernel_eval_symmetric_in_arguments(leaves, theta):  # :235-245
    rng = np.random.default_rng(5)
    for _ in range(5):
        t1, t2 = rng.uniform(-3, 3, 2)
        assert O.implied_covariance(leaves, theta, t1 - t2) == O.implied_covariance(leaves, theta, t2 - t1)


@pytest.mark.parametrize("typ,var,ln", [(O.MATERN12, 0.8, 1.7), (O.MATERN32, 1.3, 0.9), (O.MATERN52, 2.1, 1.2)])
def test_state_space_implied_matches_closed_form_materns(typ, var, ln):  # :247-261
    rng = np.random.default_rng(21)
    for _ in range(100):
        tau = rng.uniform(0.0, 10.0 * ln)
        exact = closed_form(typ, var, ln, tau)
        assert abs(O.implied_covariance([typ], [var, ln], tau) - exact) < 1e-8 * abs(exact) + 1e-14


def test_kernel_eval_sum_equals_sum_of_children():  # :263-276
    rng = np.random.default_rng(31)
    for _ in range(25):
        tau = rng.uniform(0, 5)
        s = O.implied_covariance([O.MATERN32, (O.EQ, 6)], [1.0, 0.7, 0.6, 1.5], tau)
        c = O.implied_covariance([O.MATERN32], [1.0, 0.7], tau) + O.implied_covariance([(O.EQ, 6)], [0.6, 1.5], tau)
        assert abs(s - c) < 1e-10


def test_expm_pade_matches_taylor_across_degree_branches():
    """matexp.hpp:11-13 (Eigen's Padé degree selection): every branch against the Taylor oracle."""
    rng = np.random.default_rng(3)
    for norm in (0.01, 0.2, 0.9, 2.0, 5.0, 20.0):
        A = rng.standard_normal((4, 4))
        A *= norm / np.abs(A).sum(axis=0).max()
        assert np.abs(O.expm(A) - taylor_expm(A)).max() < 1e-12 * max(1.0, np.abs(taylor_expm(A)).max())
