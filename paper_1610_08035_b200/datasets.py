"""Seeded synthetic inputs for the five BASELINE configurations (BASELINE.json
`configs`).  The paper's experiments ("two sinusoids", CO2) are
not reproducible here (no dataset ships with the reference), so these seeded
series with the stated shapes, gap laws and signal/noise mixes stand in for them.

RNG: numpy PCG64 (`np.random.default_rng(seed)`), one fixed seed per config.
Every config returns plain float64 arrays; times are strictly increasing.
"""
import math
from dataclasses import dataclass, field

import numpy as np

MATERN12, MATERN32, MATERN52, EQ, QP = 0, 1, 2, 3, 4

SEEDS = {"cfg1": 1001, "cfg2": 1002, "cfg3": 1003, "cfg4": 1004, "cfg5": 1005}


@dataclass
class Workload:
    name: str
    leaves: list
    theta: np.ndarray          # [n_theta] or [S, n_theta]
    sigma: object              # float or [S]
    t: np.ndarray              # [n] or [S, n]
    y: np.ndarray
    outputs: tuple             # subset of ("grad", "mean", "var")
    description: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def batched(self):
        return self.t.ndim == 2

    @property
    def points(self):
        return int(self.t.size)


def cfg1(n=10_000, seed=SEEDS["cfg1"]):
    """Matérn-3/2 (var 1, len 2), N=10,000, gaps U(0.05,0.15), y = sin(0.5t) + 0.3 N(0,1), σ=0.3."""
    rng = np.random.default_rng(seed)
    t = np.cumsum(rng.uniform(0.05, 0.15, n))
    y = np.sin(0.5 * t) + 0.3 * rng.standard_normal(n)
    return Workload("cfg1", [MATERN32], np.array([1.0, 2.0]), 0.3, t, y, ("grad", "mean", "var"),
                    "Matérn-3/2 b=2 single series N=%d" % n)


def cfg2(n=1_000_000, seed=SEEDS["cfg2"]):
    """Matérn-5/2 (var 2, len 1.5), N=1e6, gaps Exp(mean 0.01),
    y = sin(3t) + 0.5 cos(0.7t) + 0.2 N(0,1), σ=0.2."""
    rng = np.random.default_rng(seed)
    gaps = rng.exponential(0.01, n)
    gaps[gaps <= 0.0] = np.finfo(float).tiny  # exact zero gaps are impossible in practice; guard anyway
    t = np.cumsum(gaps)
    y = np.sin(3.0 * t) + 0.5 * np.cos(0.7 * t) + 0.2 * rng.standard_normal(n)
    return Workload("cfg2", [MATERN52], np.array([2.0, 1.5]), 0.2, t, y, ("grad", "mean"),
                    "Matérn-5/2 b=3 single series N=%d" % n)


def _matern52_prior_sample(rng, lens, vars_, t):
    """z_n = Φ_n z_{n-1} + chol(Q̃_n) ξ with the jittered Q̃, vectorised over series."""
    S, n = t.shape
    lam = math.sqrt(5.0) / lens
    kap = lam * lam / 3.0
    P = np.zeros((S, 3, 3))
    P[:, 0, 0] = vars_
    P[:, 1, 1] = vars_ * kap
    P[:, 2, 2] = vars_ * lam ** 4
    P[:, 0, 2] = P[:, 2, 0] = -vars_ * kap
    jit = 1e-10 * np.trace(P, axis1=1, axis2=2) / 3.0
    eye = np.eye(3)
    L0 = np.linalg.cholesky(P + jit[:, None, None] * eye)
    z = np.einsum("sij,sj->si", L0, rng.standard_normal((S, 3)))
    f = np.empty((S, n))
    f[:, 0] = z[:, 0]
    N = np.zeros((S, 3, 3))
    N[:, 0, 0] = lam; N[:, 0, 1] = 1.0
    N[:, 1, 1] = lam; N[:, 1, 2] = 1.0
    N[:, 2, 0] = -lam ** 3; N[:, 2, 1] = -3 * lam ** 2; N[:, 2, 2] = -2 * lam
    N2 = N @ N
    for k in range(1, n):
        dt = (t[:, k] - t[:, k - 1])[:, None, None]
        Phi = np.exp(-lam[:, None, None] * dt) * (eye + N * dt + 0.5 * N2 * dt * dt)
        Q = P - Phi @ P @ np.transpose(Phi, (0, 2, 1))
        Q = 0.5 * (Q + np.transpose(Q, (0, 2, 1))) + jit[:, None, None] * eye
        L = np.linalg.cholesky(Q)
        z = np.einsum("sij,sj->si", Phi, z) + np.einsum("sij,sj->si", L, rng.standard_normal((S, 3)))
        f[:, k] = z[:, 0]
    return f


def cfg3(S=4096, n=2048, seed=SEEDS["cfg3"]):
    """4096 x 2048 Matérn-5/2, per-series len ~ LogU(0.5,5), var ~ LogU(0.5,2), gaps U(0.5,1.5)*0.01,
    y = prior sample (state-space recursion, jittered Q̃) + 0.1 N(0,1), σ=0.1."""
    rng = np.random.default_rng(seed)
    lens = np.exp(rng.uniform(math.log(0.5), math.log(5.0), S))
    vars_ = np.exp(rng.uniform(math.log(0.5), math.log(2.0), S))
    t = np.cumsum(rng.uniform(0.5, 1.5, (S, n)) * 0.01, axis=1)
    y = _matern52_prior_sample(rng, lens, vars_, t) + 0.1 * rng.standard_normal((S, n))
    theta = np.stack([vars_, lens], axis=1)
    return Workload("cfg3", [MATERN52], theta, np.full(S, 0.1), t, y, ("grad",),
                    "Matérn-5/2 b=3 batched %d series x N=%d" % (S, n))


def cfg4(n=16_000_000, seed=SEEDS["cfg4"]):
    """EQ order 6 (var 1, len 1), N retained points of a dt=1e-3 grid with a seeded 5% drop
    (t = k*1e-3 computed directly), y = tanh(sin 2t) + 0.1 N(0,1), σ=0.1."""
    rng = np.random.default_rng(seed)
    grid = int(math.ceil(n / 0.95 * 1.02)) + 16
    keep = np.flatnonzero(rng.random(grid) >= 0.05)[:n]
    if len(keep) < n:
        raise ValueError("grid too short")
    t = keep.astype(np.float64) * 1e-3
    y = np.tanh(np.sin(2.0 * t)) + 0.1 * rng.standard_normal(n)
    return Workload("cfg4", [(EQ, 6)], np.array([1.0, 1.0]), 0.1, t, y, ("grad",),
                    "EQ order-6 b=6 single series N=%d" % n)


def cfg5(n=32_000_000, seed=SEEDS["cfg5"]):
    """Matérn-3/2 (var 1, len 10) + quasi-periodic (var 1, len_p 1, period 1, env 20, 6 harmonics,
    b=14); gaps U(0.5,1.5)*1e-3; y = sin(2πt) + 0.3 sin(0.05t) + 0.1 N(0,1), σ=0.1.
    var = 1 for both leaves and len_p = 1 are not fixed by BASELINE."""
    rng = np.random.default_rng(seed)
    t = np.cumsum(rng.uniform(0.5, 1.5, n) * 1e-3)
    y = np.sin(2.0 * math.pi * t) + 0.3 * np.sin(0.05 * t) + 0.1 * rng.standard_normal(n)
    theta = np.array([1.0, 10.0, 1.0, 1.0, 1.0, 20.0])
    return Workload("cfg5", [MATERN32, (QP, 6)], theta, 0.1, t, y, ("grad", "var"),
                    "Matérn-3/2 + quasi-periodic(6) b=16 single series N=%d" % n)


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}


def make(name, **kw):
    return CONFIGS[name](**kw)
