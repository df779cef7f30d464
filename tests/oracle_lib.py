"""ctypes binding of the CPU oracle (oracle/build/libspingp_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline leg.  The product package never imports this module.
"""
import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.path.join(ROOT, "oracle", "build", "libspingp_oracle.so")

MATERN12, MATERN32, MATERN52, EQ, QP = 0, 1, 2, 3, 4
LEAF_NPARAMS = {MATERN12: 2, MATERN32: 2, MATERN52: 2, EQ: 2, QP: 4}

_P = ctypes.POINTER
_d = _P(ctypes.c_double)
_i32 = _P(ctypes.c_int32)
_i64 = _P(ctypes.c_int64)
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_last_error.restype = ctypes.c_char_p
        L.oracle_state_space.argtypes = [_i32, ctypes.c_int32, _d, ctypes.c_int32, _d, _d, _d, _d, _d, _i32, _i32, ctypes.c_int]
        L.oracle_discretize.argtypes = [_i32, ctypes.c_int32, _d, ctypes.c_int32, ctypes.c_double, ctypes.c_int, _d, _d, _d, _d, ctypes.c_int]
        L.oracle_implied_covariance.argtypes = [_i32, ctypes.c_int32, _d, ctypes.c_int32, ctypes.c_double]
        L.oracle_implied_covariance.restype = ctypes.c_double
        L.oracle_eval.argtypes = [_i32, ctypes.c_int32, _d, ctypes.c_int32, _d, _d, ctypes.c_int64, ctypes.c_double, ctypes.c_uint32,
                                  _d, _d, _d, _d, _d, _i64, ctypes.c_int, ctypes.c_int]
        L.oracle_eval_batched.argtypes = [_i32, ctypes.c_int32, _d, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, _d, _d, _d,
                                          ctypes.c_uint32, _d, _d, _i64, ctypes.c_int, ctypes.c_int]
        L.oracle_assemble.argtypes = [_i32, ctypes.c_int32, _d, ctypes.c_int32, _d, _d, ctypes.c_int64, ctypes.c_double, _d, _d, _d, _i64,
                                      ctypes.c_int, ctypes.c_int]
        L.oracle_btd_solve.argtypes = [ctypes.c_int64, ctypes.c_int32, _d, _d, _d, ctypes.c_int32, _d, _d, _i64, ctypes.c_int]
        L.oracle_btd_selinv.argtypes = [ctypes.c_int64, ctypes.c_int32, _d, _d, _d, _d, _d, _i64, ctypes.c_int]
        L.oracle_kf_rts.argtypes = [_i32, ctypes.c_int32, _d, ctypes.c_int32, _d, _d, ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_double, _d, _d, _d, _d, _i64, ctypes.c_int]
        L.oracle_expm.argtypes = [ctypes.c_int32, _d, _d, ctypes.c_int]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status, block, msg):
        super().__init__(f"oracle status {status} block {block}: {msg}")
        self.status, self.block = status, block


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(_d)


def _leaves(leaves):
    arr = np.zeros(2 * len(leaves), dtype=np.int32)
    for i, lf in enumerate(leaves):
        typ, order = (lf, 0) if isinstance(lf, int) else lf
        arr[2 * i], arr[2 * i + 1] = typ, order
    return arr


def n_theta(leaves):
    return sum(LEAF_NPARAMS[(lf if isinstance(lf, int) else lf[0])] for lf in leaves)


def _check(st, fb=None):
    if st != 0:
        raise OracleError(st, None if fb is None else fb.value, lib().oracle_last_error().decode())


def state_space(leaves, theta, precision=0):
    L = lib()
    lv = _leaves(leaves)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    b = ctypes.c_int32()
    _check(L.oracle_state_space(lv.ctypes.data_as(_i32), len(leaves), _p(th), len(th), None, None, None, None, None, None,
                                ctypes.byref(b), precision))
    b = b.value
    nt = len(th)
    F = np.zeros((b, b)); H = np.zeros(b); P = np.zeros((b, b))
    dF = np.zeros((nt, b, b)); dP = np.zeros((nt, b, b)); fc = np.zeros(nt, dtype=np.int32)
    _check(L.oracle_state_space(lv.ctypes.data_as(_i32), len(leaves), _p(th), nt, _p(F), _p(H), _p(P), _p(dF), _p(dP),
                                fc.ctypes.data_as(_i32), ctypes.byref(ctypes.c_int32()), precision))
    return dict(F=F, H=H, Pinf=P, dF=dF, dPinf=dP, f_constant=fc, b=b)


def discretize(leaves, theta, dt, grad=False, precision=0):
    ss = state_space(leaves, theta, precision)
    b, nt = ss["b"], len(theta)
    Phi = np.zeros((b, b)); Q = np.zeros((b, b)); dPhi = np.zeros((nt, b, b)); dQ = np.zeros((nt, b, b))
    lv = _leaves(leaves)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    _check(lib().oracle_discretize(lv.ctypes.data_as(_i32), len(leaves), _p(th), nt, float(dt), int(grad), _p(Phi), _p(Q),
                                   _p(dPhi), _p(dQ), precision))
    return (Phi, Q, dPhi, dQ) if grad else (Phi, Q)


def implied_covariance(leaves, theta, tau):
    lv = _leaves(leaves)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    return lib().oracle_implied_covariance(lv.ctypes.data_as(_i32), len(leaves), _p(th), len(th), float(tau))


def expm(A, precision=0):
    A = np.ascontiguousarray(A, dtype=np.float64)
    out = np.zeros_like(A)
    _check(lib().oracle_expm(A.shape[0], _p(A), _p(out), precision))
    return out


def evaluate(leaves, theta, t, y, sigma, grad=True, mean=True, var=True, include_noise=False, precision=0, threads=1,
             diagnostics=False):
    lv = _leaves(leaves)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n = len(t)
    flags = (1 if grad else 0) | (2 if mean else 0) | (4 if var else 0) | (8 if include_noise else 0)
    ll = ctypes.c_double()
    g = np.zeros(len(th) + 1)
    mu = np.zeros(n) if mean else None
    v = np.zeros(n) if var else None
    d4 = np.zeros(4)
    fb = ctypes.c_int64()
    st = lib().oracle_eval(lv.ctypes.data_as(_i32), len(leaves), _p(th), len(th), _p(t), _p(y), n, float(sigma), flags,
                           ctypes.byref(ll), _p(g), _p(mu), _p(v), _p(d4), ctypes.byref(fb), precision, threads)
    _check(st, fb)
    out = dict(loglik=ll.value, grad=g if grad else None, mean=mu, var=v)
    if diagnostics:
        out.update(logdetP=d4[0], logdetQ=d4[1], fit_y=d4[2], fit_e=d4[3])
    return out


def evaluate_batched(leaves, theta, t, y, sigma, grad=True, precision=0, threads=1):
    lv = _leaves(leaves)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    S, n = t.shape
    t = np.ascontiguousarray(t, dtype=np.float64); y = np.ascontiguousarray(y, dtype=np.float64)
    sg = np.ascontiguousarray(sigma, dtype=np.float64)
    nt = th.shape[1]
    ll = np.zeros(S); g = np.zeros((S, nt + 1)); fs = ctypes.c_int64()
    st = lib().oracle_eval_batched(lv.ctypes.data_as(_i32), len(leaves), _p(th), nt, S, n, _p(t), _p(y), _p(sg),
                                   1 if grad else 0, _p(ll), _p(g), ctypes.byref(fs), precision, threads)
    _check(st, fs)
    return ll, g


def assemble(leaves, theta, t, y, sigma, precision=0, threads=1):
    lv = _leaves(leaves)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64); y = np.ascontiguousarray(y, dtype=np.float64)
    n = len(t)
    b = state_space(leaves, theta)["b"]
    diag = np.zeros((n, b, b)); upper = np.zeros((max(n - 1, 0), b, b)); rhs = np.zeros((n, b))
    fb = ctypes.c_int64()
    _check(lib().oracle_assemble(lv.ctypes.data_as(_i32), len(leaves), _p(th), len(th), _p(t), _p(y), n, float(sigma),
                                 _p(diag), _p(upper), _p(rhs), ctypes.byref(fb), precision, threads), fb)
    return diag, upper, rhs


def btd_solve(diag, upper, rhs=None, precision=0):
    diag = np.ascontiguousarray(diag, dtype=np.float64)
    n, b, _ = diag.shape
    upper = np.ascontiguousarray(upper if len(upper) else np.zeros((0, b, b)), dtype=np.float64)
    ld = ctypes.c_double(); fb = ctypes.c_int64()
    if rhs is None:
        _check(lib().oracle_btd_solve(n, b, _p(diag), _p(upper), None, 0, None, ctypes.byref(ld), ctypes.byref(fb), precision), fb)
        return None, ld.value
    rhs = np.ascontiguousarray(rhs, dtype=np.float64).reshape(n * b, -1)
    k = rhs.shape[1]
    x = np.zeros_like(rhs)
    _check(lib().oracle_btd_solve(n, b, _p(diag), _p(upper), _p(rhs), k, _p(x), ctypes.byref(ld), ctypes.byref(fb), precision), fb)
    return x, ld.value


def btd_selinv(diag, upper, precision=0):
    diag = np.ascontiguousarray(diag, dtype=np.float64)
    n, b, _ = diag.shape
    upper = np.ascontiguousarray(upper if len(upper) else np.zeros((0, b, b)), dtype=np.float64)
    cd = np.zeros_like(diag); cu = np.zeros((max(n - 1, 0), b, b)); ld = ctypes.c_double(); fb = ctypes.c_int64()
    _check(lib().oracle_btd_selinv(n, b, _p(diag), _p(upper), _p(cd), _p(cu), ctypes.byref(ld), ctypes.byref(fb), precision), fb)
    return cd, cu, ld.value


def kf_rts(leaves, theta, t, y, sigma, observed=None, precision=0):
    """Kalman filter + RTS smoother over the grid t; observed: optional
    bool mask (False = a test time, processed as a missing observation).  Returns loglik
    (prediction-error decomposition over the observed points), the smoothed mean H m^s
    and variance H P^s H^T, and the filtered variance H P H^T, per grid point."""
    lv = _leaves(leaves)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n = len(t)
    obs = None if observed is None else np.ascontiguousarray(observed, dtype=np.uint8)
    ll = ctypes.c_double()
    mu, v, fv = np.zeros(n), np.zeros(n), np.zeros(n)
    fb = ctypes.c_int64()
    st = lib().oracle_kf_rts(lv.ctypes.data_as(_i32), len(leaves), _p(th), len(th), _p(t), _p(y),
                             None if obs is None else obs.ctypes.data, n, float(sigma), ctypes.byref(ll), _p(mu), _p(v),
                             _p(fv), ctypes.byref(fb), precision)
    _check(st, fb)
    return dict(loglik=ll.value, mean=mu, var=v, fvar=fv)


def kf_rts_predict(leaves, theta, t, y, test_t, sigma, precision=0):
    """kf_rts_predict: the filter over the merged train+test grid with the
    test times as missing observations; returns (loglik, mean, var) at test_t (input order)."""
    t = np.asarray(t, float)
    ts = np.asarray(test_t, float)
    grid = np.concatenate([t, ts])
    obs = np.concatenate([np.ones(len(t), bool), np.zeros(len(ts), bool)])
    yy = np.concatenate([np.asarray(y, float), np.zeros(len(ts))])
    order = np.argsort(grid, kind="stable")
    r = kf_rts(leaves, theta, grid[order], yy[order], sigma, observed=obs[order], precision=precision)
    pos = np.empty(len(grid), dtype=np.int64)
    pos[order] = np.arange(len(grid))
    at = pos[len(t):]
    return r["loglik"], r["mean"][at], r["var"][at]
