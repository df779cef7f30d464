"""A/B check of the b >= 6 level-0 kernels: team (default) vs thread-per-chunk
(SPINGP_TEAM=0, run in a subprocess), both against the fp64 / long-double oracle, plus
timings of cfg4 / cfg5 prefixes.  Usage: python tools/team_check.py [n4] [n5]"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402


def run(n4, n5):
    import paper_1610_08035_b200 as P
    from paper_1610_08035_b200 import datasets
    out = {}
    with P.Context(0) as ctx:
        cases = [("eq6", [(P.EQ, 6)], [1.1, 1.4], 0), ("m32qp6", [P.MATERN32, (P.QP, 6)], [1.0, 10.0, 1.0, 1.0, 1.0, 20.0], 0),
                 ("g6_m32_m12_m12", [P.MATERN32, P.MATERN12, P.MATERN12], [1.0, 0.7, 0.5, 2.0, 0.3, 1.0], 0),
                 ("eq6_m5", [(P.EQ, 6)], [1.1, 1.4], 5), ("m32qp6_m7", [P.MATERN32, (P.QP, 6)], [1.0, 10.0, 1.0, 1.0, 1.0, 20.0], 7)]
        rng = np.random.default_rng(1)
        t = np.cumsum(rng.uniform(0.05, 0.15, 2000))
        y = np.sin(0.5 * t) + 0.3 * rng.standard_normal(len(t))
        for name, lv, th, m0 in cases:
            ctx.set_chunk(m0)
            g = ctx.eval(lv, th, t, y, 0.3, grad=True, mean=True, var=True)
            ctx.set_chunk(0)
            out[name] = {k: (np.asarray(g[k]).tolist() if k != "loglik" else g[k]) for k in ("loglik", "grad", "mean", "var")}
        for name, n in (("cfg4", n4), ("cfg5", n5)):
            w = datasets.make(name, n=n)
            ctx.eval(w.leaves, w.theta, w.t, w.y, w.sigma, grad=True, var="var" in w.outputs)
            t0 = time.time()
            g = ctx.eval(w.leaves, w.theta, w.t, w.y, w.sigma, grad=True, var="var" in w.outputs)
            out[name] = {"seconds": time.time() - t0, "loglik": g["loglik"], "grad": np.asarray(g["grad"]).tolist()}
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        print(json.dumps(run(int(sys.argv[2]), int(sys.argv[3]))))
        sys.exit(0)
    n4 = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    n5 = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
    res = {}
    for team in ("1", "0"):
        r = subprocess.run([sys.executable, __file__, "--child", str(n4), str(n5)], capture_output=True, text=True,
                           env=dict(os.environ, SPINGP_TEAM=team))
        if r.returncode:
            print("team", team, "FAILED", r.stderr[-3000:])
            continue
        res[team] = json.loads(r.stdout.strip().splitlines()[-1])
    import oracle_lib as O
    from conftest import rel
    import paper_1610_08035_b200 as P
    rng = np.random.default_rng(1)
    t = np.cumsum(rng.uniform(0.05, 0.15, 2000))
    y = np.sin(0.5 * t) + 0.3 * rng.standard_normal(len(t))
    cases = {"eq6": ([(P.EQ, 6)], [1.1, 1.4]), "m32qp6": ([P.MATERN32, (P.QP, 6)], [1.0, 10.0, 1.0, 1.0, 1.0, 20.0]),
             "g6_m32_m12_m12": ([P.MATERN32, P.MATERN12, P.MATERN12], [1.0, 0.7, 0.5, 2.0, 0.3, 1.0])}
    cases["eq6_m5"] = cases["eq6"]
    cases["m32qp6_m7"] = cases["m32qp6"]
    for name, (lv, th) in cases.items():
        o = O.evaluate(lv, th, t, y, 0.3)
        ld = O.evaluate(lv, th, t, y, 0.3, precision=1)
        for team, r in res.items():
            errs = {k: (rel(r[name][k], o[k]), rel(r[name][k], ld[k]), rel(o[k], ld[k])) for k in ("loglik", "grad", "mean", "var")}
            print(name, "team" if team == "1" else "thread", " ".join(f"{k}:{a:.1e}/{b:.1e}/floor {c:.1e}" for k, (a, b, c) in errs.items()))
    for cfg in ("cfg4", "cfg5"):
        for team, r in res.items():
            print(cfg, "team" if team == "1" else "thread", f"{r[cfg]['seconds'] * 1e3:.2f} ms", r[cfg]["loglik"], r[cfg]["grad"])
