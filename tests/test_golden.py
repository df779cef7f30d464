"""The oracle against golden vectors from an independent scipy/numpy restatement of
the reference formulas (tests/golden/make_golden.py; the reference cannot run here)."""
import json
import os

import numpy as np
import pytest

import oracle_lib as O

G = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")))


def leaves_of(c):
    return [tuple(x) if isinstance(x, list) else x for x in c["leaves"]]


@pytest.mark.parametrize("case", G["cases"], ids=[c["name"] for c in G["cases"]])
def test_state_space_matches_golden(case):
    ss = O.state_space(leaves_of(case), case["theta"])
    tol = 1e-9 if case["name"].startswith("eq") else 1e-14
    for k in ("F", "H", "Pinf"):
        ref = np.array(case[k])
        assert np.abs(ss[k] - ref).max() <= tol * max(1.0, np.abs(ref).max()), k


@pytest.mark.parametrize("case", G["cases"], ids=[c["name"] for c in G["cases"]])
def test_discretisation_matches_golden(case):
    eqc = case["name"].startswith("eq")
    for s in case["steps"]:
        Phi, Q, dPhi, dQ = O.discretize(leaves_of(case), case["theta"], s["dt"], grad=True)
        P = np.abs(np.array(case["Pinf"])).max()
        assert np.abs(Phi - np.array(s["Phi"])).max() <= 1e-12
        # Q = Pinf - Phi Pinf Phi^T cancels; compare at the scale of Pinf (EQ: Lyapunov-solver dependent)
        assert np.abs(Q - np.array(s["Q"])).max() <= (1e-9 if eqc else 1e-13) * max(1.0, P)
        for a, b in zip(dPhi, s["dPhi"]):
            assert np.abs(a - np.array(b)).max() <= 1e-10 * max(1.0, np.abs(np.array(b)).max())
        for a, b in zip(dQ, s["dQ"]):
            assert np.abs(a - np.array(b)).max() <= (1e-8 if eqc else 1e-11) * max(1.0, P)


@pytest.mark.parametrize("case", [c for c in G["cases"] if not c["name"].startswith("eq1")],
                         ids=[c["name"] for c in G["cases"] if not c["name"].startswith("eq1")])
def test_loglik_matches_golden_dense_gp(case):
    gp = case["gp"]
    r = O.evaluate(leaves_of(case), case["theta"], gp["t"], gp["y"], gp["sigma"], grad=False, mean=False, var=False)
    tol = 2e-5 if case["name"].startswith("eq") else 1e-8  # the SPEC jitter shifts the EQ model (see test_oracle_engine)
    assert r["loglik"] == pytest.approx(gp["loglik"], rel=tol)
