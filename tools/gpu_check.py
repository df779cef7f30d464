"""Quick GPU-vs-oracle comparison (development tool; the real parity suite is tests/)."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import oracle_lib as O
import paper_1610_08035_b200 as P

rng = np.random.default_rng(0)
ctx = P.Context(0)

def rel(a, b):
    a = np.asarray(a, dtype=float); b = np.asarray(b, dtype=float)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))

cases = [([P.MATERN12], [0.8, 1.7]), ([P.MATERN32], [1.0, 2.0]), ([P.MATERN52], [2.0, 1.5]),
         ([(P.EQ, 6)], [1.0, 1.0]), ([P.MATERN32, P.MATERN12], [1.0, 0.7, 0.5, 2.0]),
         ([(P.QP, 3)], [1.0, 0.8, 1.3, 5.0]), ([P.MATERN32, (P.QP, 6)], [1.0, 10.0, 1.0, 1.0, 1.0, 20.0])]
for n in [1, 2, 3, 17, 100, 1000]:
    for lv, th in cases:
        t = np.cumsum(rng.uniform(0.05, 0.15, n)); y = np.sin(0.5 * t) + 0.3 * rng.standard_normal(n); s = 0.3
        ro = O.evaluate(lv, th, t, y, s, threads=4)
        for m0 in [0, 2, 3, 5]:
            ctx.set_chunk(m0)
            try:
                rg = ctx.eval(lv, th, t, y, s, grad=True, mean=True, var=True)
            except Exception as e:
                print("FAIL", n, lv, m0, e); continue
            print(f"n={n:5d} {str(lv):24s} m0={m0} ll {rel(rg['loglik'], ro['loglik']):.1e} grad {rel(rg['grad'], ro['grad']):.1e} "
                  f"mean {rel(rg['mean'], ro['mean']):.1e} var {rel(rg['var'], ro['var']):.1e}")
ctx.set_chunk(0)
# BTD ops
for n, b in [(1, 1), (2, 1), (17, 2), (100, 3), (33, 4), (50, 6), (20, 16)]:
    A = rng.standard_normal((n, b, b)); diag = np.einsum('nij,nkj->nik', A, A) + 4 * b * np.eye(b)
    upper = rng.standard_normal((max(n - 1, 0), b, b))
    rhs = rng.standard_normal((n * b, 2))
    xo, ldo = O.btd_solve(diag, upper, rhs)
    xg, ldg = ctx.btd_cr_solve(diag, upper, rhs)
    cdo, cuo, _ = O.btd_selinv(diag, upper)
    cdg, cug, _ = ctx.btd_selinv(diag, upper)
    print(f"btd n={n} b={b}: x {rel(xg, xo):.1e} logdet {rel(ldg, ldo):.1e} cd {rel(cdg, cdo):.1e} cu {rel(cug, cuo) if n > 1 else 0:.1e}")
# timing cfg2-like
n = 1_000_000
t = np.cumsum(rng.exponential(0.01, n)); y = np.sin(3 * t) + 0.5 * np.cos(0.7 * t) + 0.2 * rng.standard_normal(n)
for it in range(3):
    t0 = time.perf_counter(); rg = ctx.eval([P.MATERN52], [2.0, 1.5], t, y, 0.2, grad=True, mean=True); t1 = time.perf_counter()
    print(f"cfg2 host-api wall {1e3*(t1-t0):.2f} ms loglik {rg['loglik']:.10f}")
t0 = time.perf_counter(); ro = O.evaluate([O.MATERN52], [2.0, 1.5], t, y, 0.2, mean=True, var=False, threads=16); t1 = time.perf_counter()
print(f"cfg2 oracle 16 threads {t1-t0:.2f} s: ll {rel(rg['loglik'], ro['loglik']):.2e} grad {rel(rg['grad'], ro['grad']):.2e} mean {rel(rg['mean'], ro['mean']):.2e}")
print("launches", ctx.launch_count())
