"""The product's device algorithm, executed on the CPU through the host emulation
of the exact kernel code (tests/emu/: engine.cuh compiled as host C++), against
the oracle.  Covers the partitioned elimination for every chunking (including the
cyclic-reduction limit m = 2), ragged and tiny series, batched series, the
closed-form discretisation and its θ-derivatives, and the btd_core operators."""
import numpy as np
import pytest

import emu_lib as E
import oracle_lib as O
from conftest import rel

KERNELS = [
    ([O.MATERN12], [0.8, 1.7]),
    ([O.MATERN32], [1.3, 0.9]),
    ([O.MATERN52], [2.1, 1.2]),
    ([(O.EQ, 6)], [1.1, 1.4]),
    ([O.MATERN32, O.MATERN12], [1.0, 0.7, 0.5, 2.0]),
    ([(O.QP, 3)], [1.0, 0.8, 1.3, 5.0]),
    ([O.MATERN32, (O.QP, 6)], [1.0, 10.0, 1.0, 1.0, 1.0, 20.0]),
]


def series(seed, n, lo=0.05, hi=0.15):
    rng = np.random.default_rng(seed)
    t = np.cumsum(rng.uniform(lo, hi, n))
    return t, np.sin(0.5 * t) + 0.3 * rng.standard_normal(n)


@pytest.mark.parametrize("leaves,theta", KERNELS)
@pytest.mark.parametrize("dt", [-1.0, 0.3, 0.01])
def test_closed_form_discretisation_matches_pade(leaves, theta, dt):
    """model_dev.cuh closed forms vs the oracle's Padé expm / Van Loan (kernels.hpp:392-443)."""
    Pe, Qe, dPe, dQe, jit = E.discretize(leaves, theta, dt)
    ss = O.state_space(leaves, theta)
    b = ss["b"]
    if dt < 0:  # anchor step: Φ := 0, Q = Pinf, dQ = dPinf
        Po, Qo = np.zeros((b, b)), ss["Pinf"]
        dPo, dQo = np.zeros((len(theta), b, b)), ss["dPinf"].copy()
    else:
        Po, Qo, dPo, dQo = O.discretize(leaves, theta, dt, grad=True)
    for p in range(len(theta)):  # + d jitter / dθ
        dQo[p] += 1e-10 * np.trace(ss["dPinf"][p]) / b * np.eye(b)
    assert np.abs(Pe - Po).max() < 1e-14
    assert np.abs(Qe - Qo).max() <= 1e-12 * max(1.0, np.abs(ss["Pinf"]).max())
    assert np.abs(dPe - dPo).max() <= 1e-12 * max(1.0, np.abs(dPo).max())
    assert np.abs(dQe - dQo).max() <= 1e-11 * max(1.0, np.abs(dQo).max())


@pytest.mark.parametrize("leaves,theta", [k for k in KERNELS if k[0][0] != (O.EQ, 6)])
@pytest.mark.parametrize("n", [1, 2, 3, 7, 8, 9, 31, 33, 100])
@pytest.mark.parametrize("m0", [0, 2, 3, 5])
def test_partitioned_elimination_matches_oracle(leaves, theta, n, m0):
    t, y = series(n * 7 + m0, n)
    e = E.evaluate(leaves, theta, t, y, 0.3, m0=m0)
    o = O.evaluate(leaves, theta, t, y, 0.3)
    for k, tol in (("loglik", 1e-10), ("grad", 1e-9), ("mean", 1e-9), ("var", 1e-9)):
        if rel(e[k], o[k]) >= tol:  # arbitrate with the long-double evaluation
            ld = O.evaluate(leaves, theta, t, y, 0.3, precision=1)
            assert rel(e[k], ld[k]) <= max(tol, 4 * rel(o[k], ld[k])), k


@pytest.mark.parametrize("m0", [0, 2, 4])
def test_eq_against_long_double_arbiter(m0):
    """EQ is ill-conditioned in fp64: the device algorithm must be at
    least as close to the long-double evaluation of the reference formulas as the fp64
    oracle itself (x4), or within 1e-9."""
    t, y = series(5, 120)
    lv, th = [(O.EQ, 6)], [1.1, 1.4]
    e = E.evaluate(lv, th, t, y, 0.3, m0=m0)
    o = O.evaluate(lv, th, t, y, 0.3)
    ld = O.evaluate(lv, th, t, y, 0.3, precision=1)
    for k in ("loglik", "grad", "mean", "var"):
        assert rel(e[k], ld[k]) <= max(1e-9, 4 * rel(o[k], ld[k])), k


def test_batched_series_match_individual_oracle_runs():
    rng = np.random.default_rng(3)
    S, n = 6, 50
    t = np.cumsum(rng.uniform(0.5, 1.5, (S, n)) * 0.01, axis=1)
    y = rng.standard_normal((S, n))
    theta = np.stack([np.exp(rng.uniform(np.log(0.5), np.log(2), S)), np.exp(rng.uniform(np.log(0.5), np.log(5), S))], 1)
    sig = np.full(S, 0.1)
    e = E.evaluate([O.MATERN52], theta, t, y, sig, var=False, mean=False)
    for s in range(S):
        o = O.evaluate([O.MATERN52], theta[s], t[s], y[s], 0.1, mean=False, var=False)
        assert rel(e["loglik"][s], o["loglik"]) < 1e-10
        assert rel(e["grad"][s], o["grad"]) < 1e-9


def test_duplicate_time_reported_with_index():
    with pytest.raises(E.EmuError) as ex:
        E.evaluate([O.MATERN32], [1.0, 1.0], [0.0, 0.5, 0.5, 1.0], [0.0] * 4, 0.3)
    assert ex.value.status == 6 and ex.value.block == 2


@pytest.mark.parametrize("n,b", [(1, 1), (2, 1), (3, 2), (17, 2), (100, 3), (33, 4), (50, 6), (20, 16), (129, 5)])
@pytest.mark.parametrize("m0", [0, 2, 3])
def test_btd_operators_match_thomas(n, b, m0):
    rng = np.random.default_rng(n * b + m0)
    A = rng.standard_normal((n, b, b))
    diag = np.einsum("nij,nkj->nik", A, A) + 4 * b * np.eye(b)
    upper = rng.standard_normal((max(n - 1, 0), b, b))
    rhs = rng.standard_normal((n * b, 2))
    xo, ldo = O.btd_solve(diag, upper, rhs)
    cdo, cuo, _ = O.btd_selinv(diag, upper)
    r = E.btd(diag, upper, rhs, selinv=True, m0=m0)
    assert rel(r["x"], xo) < 1e-12
    assert abs(r["logdet"] - ldo) <= 1e-12 * max(1.0, abs(ldo))
    assert rel(r["cdiag"], cdo) < 1e-12
    if n > 1:
        assert rel(r["cupper"], cuo) < 1e-12


def _segment_run(leaves, theta, t, y, sigma, P, m0=0):
    from paper_1610_08035_b200.partition import split, halos
    bounds = split(len(t), P)
    nrec, npart = E.seg_sizes(leaves)
    recs = []
    for r in range(P):
        tl, tr = halos(t, bounds, r)
        recs.append(E.seg_forward(leaves, theta, t[bounds[r]:bounds[r + 1]], y[bounds[r]:bounds[r + 1]], tl, tr, r, P,
                                  sigma, flags=7, m0=m0))
    recs = np.concatenate(recs)
    tot = np.zeros(npart)
    mean = np.zeros(len(t))
    var = np.zeros(len(t))
    for r in range(P):
        a, b = bounds[r], bounds[r + 1]
        tl, tr = halos(t, bounds, r)
        E.seg_forward(leaves, theta, t[a:b], y[a:b], tl, tr, r, P, sigma, flags=7, m0=m0)
        part, mu, v = E.seg_reverse(recs, b - a, npart, mean=True, var=True)
        tot += part
        mean[a:b], var[a:b] = mu, v
    ll, g = E.seg_finalize(tot, len(theta), len(t), sigma)
    return ll, g, mean, var


@pytest.mark.parametrize("leaves,theta", [k for k in KERNELS if k[0][0] != (O.EQ, 6)])
@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("m0", [0, 3])
def test_segment_partition_matches_oracle(leaves, theta, P, m0):
    """Multi-GPU partition with the ranks emulated in turn: segments,
    halos, the all-gathered 2-separator records, the redundant P-block solve and the
    summed partials reproduce the single-series oracle."""
    t, y = series(77 + P, 400)
    ll, g, mean, var = _segment_run(leaves, theta, t, y, 0.3, P, m0)
    o = O.evaluate(leaves, theta, t, y, 0.3)
    assert rel(ll, o["loglik"]) < 1e-10
    assert rel(g, o["grad"]) < 1e-9
    assert rel(mean, o["mean"]) < 1e-9
    assert rel(var, o["var"]) < 1e-9


@pytest.fixture
def tree_group():
    yield E.set_tree_group
    E.set_tree_group(0)


@pytest.mark.parametrize("leaves,theta", [KERNELS[1], KERNELS[2], KERNELS[4]])
@pytest.mark.parametrize("G", [2, 3, 4, 7, 16])
@pytest.mark.parametrize("n,m0", [(300, 2), (257, 3), (64, 1)])
def test_multilevel_tree_groups_match_oracle(leaves, theta, G, n, m0, tree_group):
    """Levels >= 1 as shared-memory tree groups (tree.cuh) with a forced small group size:
    several k_tree_fwd / k_tree_rev levels below the k_tree_one top, ragged last groups,
    non-power-of-two groups."""
    tree_group(G)
    t, y = series(n + G, n)
    e = E.evaluate(leaves, theta, t, y, 0.3, m0=m0)
    o = O.evaluate(leaves, theta, t, y, 0.3)
    for k, tol in (("loglik", 1e-10), ("grad", 1e-9), ("mean", 1e-9), ("var", 1e-9)):
        if rel(e[k], o[k]) >= tol:
            ld = O.evaluate(leaves, theta, t, y, 0.3, precision=1)
            assert rel(e[k], ld[k]) <= max(tol, 4 * rel(o[k], ld[k])), k


@pytest.mark.parametrize("G", [2, 5])
def test_multilevel_tree_groups_batched(G, tree_group):
    tree_group(G)
    rng = np.random.default_rng(11)
    S, n = 5, 90
    t = np.cumsum(rng.uniform(0.5, 1.5, (S, n)) * 0.01, axis=1)
    y = rng.standard_normal((S, n))
    theta = np.stack([np.exp(rng.uniform(np.log(0.5), np.log(2), S)), np.exp(rng.uniform(np.log(0.5), np.log(5), S))], 1)
    e = E.evaluate([O.MATERN52], theta, t, y, np.full(S, 0.1), var=True, mean=True, m0=2)
    for s in range(S):
        o = O.evaluate([O.MATERN52], theta[s], t[s], y[s], 0.1)
        for k, tol in (("loglik", 1e-10), ("grad", 1e-9), ("mean", 1e-9), ("var", 1e-9)):
            if rel(e[k][s], o[k]) >= tol:  # arbitrate with the long-double evaluation
                ld = O.evaluate([O.MATERN52], theta[s], t[s], y[s], 0.1, precision=1)
                assert rel(e[k][s], ld[k]) <= max(tol, 4 * rel(o[k], ld[k])), k


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("G", [2, 3])
def test_segment_partition_with_tree_levels(P, G, tree_group):
    tree_group(G)
    leaves, theta = KERNELS[2]
    t, y = series(91 + P, 300)
    ll, g, mean, var = _segment_run(leaves, theta, t, y, 0.3, P, 2)
    o = O.evaluate(leaves, theta, t, y, 0.3)
    assert rel(ll, o["loglik"]) < 1e-10
    assert rel(g, o["grad"]) < 1e-9
    assert rel(mean, o["mean"]) < 1e-9
    assert rel(var, o["var"]) < 1e-9


def test_plan_level_structure():
    """make_plan (host_model.cpp): the level-0 chunk count targets 75,776 chunks; tree
    levels of G(b) = 512 records at b = 3 end in one group per series; b >= 6 keeps the
    per-thread 4-record levels."""
    p = E.plan(1_000_000, 1, 3)  # cfg2
    assert p["tree"] and p["levels"][0] == (1_000_000, 14, 71429)
    assert p["levels"][1] == (71429, 512, 140) and p["levels"][2] == (140, 140, 1) and p["nlev"] == 3
    q = E.plan(2048, 4096, 3)  # cfg3: chunks lengthened so k_rev0's last wave is full
    assert q["levels"][0] == (2048, 114, 18) and 18 * 4096 <= 2 * 296 * 128
    r = E.plan(16_000_000, 1, 6)  # cfg4: b = 6, per-thread levels
    assert not r["tree"] and all(m == 4 for _, m, _ in r["levels"][1:-1])
    one = E.plan(1, 1, 3)  # a single point still gets a tree level (its top inverse)
    assert one["nlev"] == 2 and one["levels"][1] == (1, 1, 1)
