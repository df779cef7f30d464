"""Device (library) vs host emulation of the same kernels, per output, small n (debug tool)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import emu_lib as E, paper_1610_08035_b200 as P
np.set_printoptions(precision=8, linewidth=200)
CASES = [([(P.EQ, 6)], [1.1, 1.4]), ([(P.QP, 3)], [1.0, 0.8, 1.3, 5.0]),
         ([P.MATERN32, (P.QP, 6)], [1.0, 10.0, 1.0, 1.0, 1.0, 20.0])]
ctx = P.Context(0)
for lv, th in CASES:
    for n in [1, 2, 5]:
        rng = np.random.default_rng(n); t = np.cumsum(rng.uniform(0.05, 0.15, n)); y = np.sin(0.5 * t) + 0.3 * rng.standard_normal(n)
        try:
            g = ctx.eval(lv, th, t, y, 0.3, grad=True, mean=True, var=True)
        except Exception as e:
            print(lv, n, "GPU ERR", e); continue
        e = E.evaluate(lv, th, t, y, 0.3, grad=True, mean=True, var=True)
        for k in ["loglik", "grad", "mean", "var"]:
            a, b = np.atleast_1d(g[k]), np.atleast_1d(e[k])
            d = np.abs(a - b).max() / max(1e-300, np.abs(b).max())
            if d > 1e-10:
                print(lv, n, k, "rel", d, "\n  gpu", a[:8], "\n  emu", b[:8])
print("done")
