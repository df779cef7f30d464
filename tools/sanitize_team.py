"""Small evaluations through every b >= 6 path (team kernels, fully inlined build) for
compute-sanitizer: memcheck / initcheck / racecheck / synccheck (run under the tool by
tools/run_sanitizer.sh).  Also the thread-per-chunk b >= 6 kernels (SPINGP_TEAM=0)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1610_08035_b200 as P  # noqa: E402

rng = np.random.default_rng(3)
t = np.cumsum(rng.uniform(0.05, 0.15, 600))
y = np.sin(0.5 * t) + 0.3 * rng.standard_normal(len(t))
cases = [([(P.EQ, 6)], [1.1, 1.4]), ([P.MATERN32, (P.QP, 6)], [1.0, 10.0, 1.0, 1.0, 1.0, 20.0]),
         ([P.MATERN32, P.MATERN12, P.MATERN12], [1.0, 0.7, 0.5, 2.0, 0.3, 1.0]), ([(P.QP, 3)], [1.0, 0.8, 1.3, 5.0]),
         ([P.MATERN32, (P.EQ, 10)], [1.0, 5.0, 1.0, 20.0])]
with P.Context(0) as ctx:
    for lv, th in cases:
        for m0 in (0, 5):
            ctx.set_chunk(m0)
            g = ctx.eval(lv, th, t, y, 0.3, grad=True, mean=True, var=True)
            assert np.isfinite(g["loglik"]) and np.all(np.isfinite(g["grad"]))
    ctx.set_chunk(0)
print("sanitize_team ok", os.environ.get("SPINGP_TEAM", "1"))
