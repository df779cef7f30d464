"""Generates tests/golden/golden.json: an INDEPENDENT restatement of the reference's
kernel_ss formulas (proj/include/spingp/kernels.hpp) with scipy/numpy —
scipy.linalg.expm (Al-Mohy–Higham Padé), scipy.linalg.expm_frechet, scipy's
Lyapunov solver, numpy.roots for the EQ spectral factor — plus dense-GP
log-likelihoods.  The reference itself cannot be built or run here (Eigen/GTest
absent), so these vectors pin the C++ oracle against a second, unrelated
implementation of the same published formulas.

Run: python tests/golden/make_golden.py   (needs scipy; not needed at test time)
"""
import json
import math
import os

import numpy as np
from scipy import linalg


def matern(nu, var, ln):
    if nu == 1:
        lam = 1.0 / ln
        F = np.array([[-lam]]); P = np.array([[var]])
        dF = [np.zeros((1, 1)), np.array([[1.0 / ln ** 2]])]
        dP = [np.array([[1.0]]), np.zeros((1, 1))]
    elif nu == 3:
        lam = math.sqrt(3) / ln
        F = np.array([[0, 1], [-lam ** 2, -2 * lam]]); P = np.diag([var, var * lam ** 2])
        dF = [np.zeros((2, 2)), np.array([[0, 0], [2 * lam ** 2 / ln, 2 * lam / ln]])]
        dP = [P / var, np.diag([0, -2 * var * lam ** 2 / ln])]
    else:
        lam = math.sqrt(5) / ln
        kap = lam ** 2 / 3
        F = np.array([[0, 1, 0], [0, 0, 1], [-lam ** 3, -3 * lam ** 2, -3 * lam]])
        P = np.array([[var, 0, -var * kap], [0, var * kap, 0], [-var * kap, 0, var * lam ** 4]])
        dFl = np.zeros((3, 3)); dFl[2] = [-(3 - k) / ln * F[2, k] for k in range(3)]
        dPl = np.array([[-(i + j) / ln * P[i, j] for j in range(3)] for i in range(3)])
        dF = [np.zeros((3, 3)), dFl]; dP = [P / var, dPl]
    H = np.zeros(len(F)); H[0] = 1
    return F, H, P, dF, dP, [True, False]


def eq(var, ln, J):
    # roots of T_J(y) = sum_{k<=J} y^k/k!, then r = -sqrt(-2y) in the stable half plane
    coef = [1.0 / math.factorial(k) for k in range(J, -1, -1)]
    ys = np.roots(coef)
    r = -np.sqrt(-2 * ys + 0j)
    r = np.where(r.real > 0, -r, r)
    up = sorted([z for z in r if z.imag > 0], key=lambda z: (z.real, z.imag))
    F = np.zeros((J, J)); H = np.zeros(J); g = np.zeros(J)
    for p, z in enumerate(up):
        den = np.prod([z - o for o in r if abs(o - z) > 1e-12])
        res = 1 / den
        k = 2 * p
        F[k, k] = F[k + 1, k + 1] = z.real / ln
        F[k, k + 1] = z.imag / ln
        F[k + 1, k] = -z.imag / ln
        H[k], H[k + 1] = 2 * res.real, 2 * res.imag
        g[k] = 1
    p1 = linalg.solve_continuous_lyapunov(F * ln, -np.outer(g, g))
    p1 = 0.5 * (p1 + p1.T)
    P = var / (H @ p1 @ H) * p1
    return F, H, P, [np.zeros((J, J)), -F / ln], [P / var, np.zeros((J, J))], [True, False]


def step(F, P, dF, dP, fc, dt):
    Phi = linalg.expm(F * dt)
    Q = P - Phi @ P @ Phi.T
    Q = 0.5 * (Q + Q.T)
    dPhi, dQ = [], []
    for a, b_, c in zip(dF, dP, fc):
        dp = np.zeros_like(F) if c else linalg.expm_frechet(F * dt, a * dt, compute_expm=False)
        dq = b_ - dp @ P @ Phi.T - Phi @ b_ @ Phi.T - Phi @ P @ dp.T
        dPhi.append(dp); dQ.append(0.5 * (dq + dq.T))
    return Phi, Q, dPhi, dQ


def main():
    cases = []
    specs = [("matern12", [0], [0.8, 1.7], lambda th: matern(1, *th)),
             ("matern32", [1], [1.3, 0.9], lambda th: matern(3, *th)),
             ("matern52", [2], [2.1, 1.2], lambda th: matern(5, *th)),
             ("eq6", [[3, 6]], [1.1, 1.4], lambda th: eq(th[0], th[1], 6)),
             ("eq10", [[3, 10]], [1.1, 1.4], lambda th: eq(th[0], th[1], 10))]
    for name, leaves, th, fn in specs:
        F, H, P, dF, dP, fc = fn(th)
        steps = []
        for dt in (0.003, 0.3, 2.5):
            Phi, Q, dPhi, dQ = step(F, P, dF, dP, fc, dt)
            steps.append({"dt": dt, "Phi": Phi.tolist(), "Q": Q.tolist(), "dPhi": [x.tolist() for x in dPhi],
                          "dQ": [x.tolist() for x in dQ]})
        # dense GP loglik (no jitter) on a small seeded series
        rng = np.random.default_rng(42)
        t = np.sort(rng.uniform(0, 8, 25))
        y = np.sin(t) + 0.3 * rng.standard_normal(25)
        K = np.array([[H @ (linalg.expm(F * abs(a - b)) @ P) @ H for b in t] for a in t])
        C = K + 0.09 * np.eye(25)
        ll = -0.5 * y @ np.linalg.solve(C, y) - 0.5 * np.linalg.slogdet(C)[1] - 12.5 * math.log(2 * math.pi)
        cases.append({"name": name, "leaves": leaves, "theta": th, "F": F.tolist(), "H": H.tolist(), "Pinf": P.tolist(),
                      "steps": steps, "gp": {"t": t.tolist(), "y": y.tolist(), "sigma": 0.3, "loglik": ll}})
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(out, "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (scipy %s, numpy %s)" % (
            __import__("scipy").__version__, np.__version__), "cases": cases}, f)
    print("wrote", out)


if __name__ == "__main__":
    main()
