import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import oracle_lib as O, emu_lib as E
import paper_1610_08035_b200 as P
np.set_printoptions(precision=12, linewidth=200)
rng = np.random.default_rng(0)
ctx = P.Context(0)
for lv, th in [([2], [2.0, 1.5]), ([1, 0], [1.0, 0.7, 0.5, 2.0]), ([(3, 6)], [1.0, 1.0])]:
    for n in [1, 2]:
        t = np.cumsum(rng.uniform(0.05, 0.15, n)); y = np.sin(0.5 * t) + 0.3 * rng.standard_normal(n); s = 0.3
        ro = O.evaluate(lv, th, t, y, s)
        re = E.evaluate(lv, th, t, y, s)
        try:
            rg = ctx.eval(lv, th, t, y, s, grad=True, mean=True, var=True)
        except Exception as e:
            rg = dict(loglik=str(e), grad=None, var=None)
        print(lv, n, "oracle", ro['loglik'], ro['grad'], ro['var'])
        print(lv, n, "emu   ", re['loglik'], re['grad'], re['var'])
        print(lv, n, "gpu   ", rg['loglik'], rg['grad'], rg['var'])
