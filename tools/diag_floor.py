"""Diagnostics for the parity floors: cfg3 per-series GPU / floor ratios with the
forward and time-reversed fp64 oracle, and cfg5 small-n team vs thread errors.
Usage: python tools/diag_floor.py  (GPU box; SPINGP_TEAM honoured)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle_lib as O  # noqa: E402
import paper_1610_08035_b200 as P  # noqa: E402
from paper_1610_08035_b200 import datasets  # noqa: E402
from conftest import rel  # noqa: E402

out = {}
with P.Context(0) as ctx:
    w = datasets.cfg3()
    g = ctx.eval_batched(w.leaves, w.theta, w.t, w.y, w.sigma, grad=True)
    ll, gr = O.evaluate_batched(w.leaves, w.theta, w.t, w.y, w.sigma, grad=True, threads=16)
    llr, grr = O.evaluate_batched(w.leaves, w.theta, -w.t[:, ::-1].copy(), w.y[:, ::-1].copy(), w.sigma, grad=True,
                                  threads=16)
    lld, grd = O.evaluate_batched(w.leaves, w.theta, w.t, w.y, w.sigma, grad=True, precision=1, threads=16)
    for name, got, o, orv, ld in (("loglik", g["loglik"][:, None], ll[:, None], llr[:, None], lld[:, None]),
                                  ("grad", g["grad"], gr, grr, grd)):
        den = np.abs(ld).max(axis=1)
        err = np.abs(got - ld).max(axis=1) / den
        f1 = np.abs(o - ld).max(axis=1) / den
        f2 = np.abs(orv - ld).max(axis=1) / den
        fl = np.maximum(f1, f2)
        ratio = err / np.maximum(fl, 1e-16)
        bad = err > np.maximum(1e-9, 4 * fl)
        out["cfg3_" + name] = {"max_err": float(err.max()), "max_floor": float(fl.max()),
                               "agg_ratio": float(err.max() / fl.max()), "n_bad_4x": int(bad.sum()),
                               "ratio_p99": float(np.quantile(ratio, 0.99)), "ratio_max": float(ratio.max()),
                               "worst": [int(i) for i in np.argsort(-ratio)[:5]],
                               "worst_err": [float(err[i]) for i in np.argsort(-ratio)[:5]],
                               "worst_floor": [float(fl[i]) for i in np.argsort(-ratio)[:5]]}
    for n, m0 in ((4000, 0), (4000, 423), (20000, 0), (100000, 423)):
        w = datasets.cfg5(n=n)
        ctx.set_chunk(m0)
        g = ctx.eval(w.leaves, w.theta, w.t, w.y, w.sigma, grad=True, var=True)
        ctx.set_chunk(0)
        o = O.evaluate(w.leaves, w.theta, w.t, w.y, w.sigma, grad=True, mean=False, var=True, threads=16)
        orv = O.evaluate(w.leaves, w.theta, -w.t[::-1].copy(), w.y[::-1].copy(), w.sigma, grad=True, mean=False,
                         var=True, threads=16)
        orv["var"] = orv["var"][::-1]
        ld = O.evaluate(w.leaves, w.theta, w.t, w.y, w.sigma, grad=True, mean=False, var=True, precision=1, threads=16)
        out[f"cfg5_{n}_{m0}"] = {k: {"gpu_ld": rel(g[k], ld[k]), "o_ld": rel(o[k], ld[k]), "orev_ld": rel(orv[k], ld[k]),
                                     "loglik_ld": ld["loglik"] if k == "loglik" else None}
                                 for k in ("loglik", "grad", "var")}
print(json.dumps(out, indent=1))
