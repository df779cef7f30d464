"""btd_core known answers and dense-oracle checks,
against the CPU oracle (block Thomas + Takahashi).  These pin the oracle that the
GPU parity tests then use."""
import math

import numpy as np
import pytest

import oracle_lib as O


def dense(diag, upper):
    n, b, _ = diag.shape
    M = np.zeros((n * b, n * b))
    for i in range(n):
        M[i * b:(i + 1) * b, i * b:(i + 1) * b] = diag[i]
    for i in range(n - 1):
        M[i * b:(i + 1) * b, (i + 1) * b:(i + 2) * b] = upper[i]
        M[(i + 1) * b:(i + 2) * b, i * b:(i + 1) * b] = upper[i].T
    return M


def random_spd_btd(rng, n, b):
    A = rng.standard_normal((n, b, b))
    diag = np.einsum("nij,nkj->nik", A, A) + 4.0 * b * np.eye(b)
    upper = rng.standard_normal((max(n - 1, 0), b, b))
    return diag, upper


def test_factorize_scalar():
    _, ld = O.btd_solve(np.array([[[4.0]]]), np.zeros((0, 1, 1)))
    assert ld == pytest.approx(math.log(4.0), abs=1e-15)


def test_factorize_two_by_two():
    _, ld = O.btd_solve(np.array([[[2.0]], [[2.0]]]), np.array([[[-1.0]]]))
    assert ld == pytest.approx(math.log(3.0), abs=1e-15)


def test_solve_two_by_two():
    x, _ = O.btd_solve(np.array([[[2.0]], [[2.0]]]), np.array([[[-1.0]]]), np.array([1.0, 1.0]))
    assert np.allclose(x.ravel(), [1.0, 1.0], atol=1e-15)


def test_solve_identity_returns_rhs():
    rng = np.random.default_rng(0)
    diag = np.tile(np.eye(3), (5, 1, 1))
    rhs = rng.standard_normal((15, 2))
    x, _ = O.btd_solve(diag, np.zeros((4, 3, 3)), rhs)
    assert np.array_equal(x, rhs)


def test_selective_inverse_two_by_two():
    cd, cu, _ = O.btd_selinv(np.array([[[2.0]], [[2.0]]]), np.array([[[-1.0]]]))
    assert np.allclose(cd.ravel(), [2 / 3, 2 / 3], atol=1e-15)
    assert np.allclose(cu.ravel(), [1 / 3], atol=1e-15)


def test_logdet_diagonal():
    _, ld = O.btd_solve(np.tile(2.0 * np.eye(5), (1, 1, 1)), np.zeros((0, 5, 5)))
    assert ld == pytest.approx(5 * math.log(2.0), abs=1e-14)


def test_logdet_identity_is_zero():
    _, ld = O.btd_solve(np.tile(np.eye(2), (7, 1, 1)), np.zeros((6, 2, 2)))
    assert ld == 0.0


def test_trace_identity():  # trace_btd_product(I, I) with n*b = 7 -> 7
    cd, cu, _ = O.btd_selinv(np.tile(np.eye(1), (7, 1, 1)), np.zeros((6, 1, 1)))
    assert float(np.einsum("nii->", cd)) + 2 * float(np.einsum("nij,nij->", cu, np.zeros_like(cu))) == 7.0


def test_indefinite_input_raises_not_positive_definite():  # SPEC.md:515, errors.hpp:12-20
    with pytest.raises(O.OracleError) as e:
        O.btd_solve(np.array([[[-1.0]]]), np.zeros((0, 1, 1)))
    assert e.value.status == 1 and e.value.block == 0


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 8, 9, 15, 16, 17, 31, 33, 50])
@pytest.mark.parametrize("b", [1, 2, 3, 4])
def test_btd_suite_against_dense(n, b):  # SPEC.md:509 (criterion 3)
    rng = np.random.default_rng(100 * n + b)
    diag, upper = random_spd_btd(rng, n, b)
    M = dense(diag, upper)
    rhs = rng.standard_normal((n * b, 3))
    x, ld = O.btd_solve(diag, upper, rhs)
    assert np.abs(x - np.linalg.solve(M, rhs)).max() <= 1e-8 * np.abs(np.linalg.solve(M, rhs)).max()
    assert ld == pytest.approx(np.linalg.slogdet(M)[1], rel=1e-9, abs=1e-12)
    cd, cu, _ = O.btd_selinv(diag, upper)
    Minv = np.linalg.inv(M)
    for i in range(n):
        assert np.abs(cd[i] - Minv[i * b:(i + 1) * b, i * b:(i + 1) * b]).max() <= 1e-8 * np.abs(Minv).max()
    for i in range(n - 1):
        assert np.abs(cu[i] - Minv[i * b:(i + 1) * b, (i + 1) * b:(i + 2) * b]).max() <= 1e-8 * np.abs(Minv).max()
    # trace_btd_product(selinv(M), S) = Tr(M^-1 S) for a random symmetric BTD S
    sd, su = random_spd_btd(rng, n, b)
    tr = float(np.einsum("nij,nji->", cd, sd)) + 2.0 * float(np.einsum("nij,nij->", cu, su))
    assert tr == pytest.approx(float(np.trace(Minv @ dense(sd, su))), rel=1e-8)
