"""ctypes binding of the host emulation of the product kernels (tests/emu/).

TEST INFRASTRUCTURE ONLY.  Runs the exact kernel code of
paper_1610_08035_b200/csrc/engine.cuh on the CPU so the CPU suite can check the
partitioned-elimination algorithm against the oracle without a GPU.
"""
import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.environ.get("SPINGP_EMU_LIB") or os.path.join(ROOT, "tests", "emu", "build", "libspingp_emu.so")
_d = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "emu")], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.environ.get("SPINGP_EMU_LIB"):  # a sanitizer build passed in explicitly is used as is
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.emu_last_error.restype = ctypes.c_char_p
        L.emu_eval_batched.argtypes = [ctypes.c_void_p, ctypes.c_int32, _d, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                       _d, _d, _d, ctypes.c_uint32, _d, _d, _d, _d, _i64p, ctypes.c_int64, ctypes.c_int]
        L.emu_set_tree_group.argtypes = [ctypes.c_int64]
        L.emu_plan.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, _i64p, ctypes.c_int32]
        L.emu_predict.argtypes = [ctypes.c_void_p, ctypes.c_int32, _d, ctypes.c_int32, ctypes.c_int64, _d, _d, _d,
                                  ctypes.c_int64, ctypes.c_double, ctypes.c_uint32, _d, _d, _d, _d, _i64p,
                                  ctypes.c_int64]
        L.emu_btd.argtypes = [ctypes.c_int64, ctypes.c_int32, _d, _d, _d, ctypes.c_int32, _d, _d, _d, _d, _i64p,
                              ctypes.c_int64]
        _lib = L
    return _lib


def plan(n, S, Bsz, m0=0):
    """make_plan's level structure: dict(nlev, tree, levels=[(n, m, K), ...])."""
    out = np.zeros(2 + 3 * 24, dtype=np.int64)
    st = lib().emu_plan(int(n), int(S), int(Bsz), int(m0), out.ctypes.data_as(_i64p), len(out))
    if st:
        raise EmuError(st, -1, lib().emu_last_error().decode())
    L = int(out[0])
    return dict(nlev=L, tree=bool(out[1]), levels=[tuple(int(v) for v in out[2 + 3 * l:5 + 3 * l]) for l in range(L)])


def set_tree_group(g):
    """Cap the records per shared-memory tree group (0 = automatic): more tree levels."""
    lib().emu_set_tree_group(int(g))


class EmuError(RuntimeError):
    def __init__(self, status, block, msg):
        super().__init__(f"emu status {status} block {block}: {msg}")
        self.status, self.block = status, block


def _p(a):
    return None if a is None else a.ctypes.data_as(_d)


def _leaves(leaves):
    arr = np.zeros(2 * len(leaves), dtype=np.int32)
    for i, lf in enumerate(leaves):
        typ, order = (lf, 0) if isinstance(lf, (int, np.integer)) else lf
        arr[2 * i], arr[2 * i + 1] = typ, order
    return arr


def evaluate(leaves, theta, t, y, sigma, grad=True, mean=True, var=True, include_noise=False, m0=0, force_generic=False):
    t = np.ascontiguousarray(np.atleast_2d(t), dtype=np.float64)
    y = np.ascontiguousarray(np.atleast_2d(y), dtype=np.float64)
    S, n = t.shape
    th = np.ascontiguousarray(np.atleast_2d(theta), dtype=np.float64)
    th = np.ascontiguousarray(np.broadcast_to(th, (S, th.shape[1])))
    sg = np.ascontiguousarray(np.broadcast_to(np.asarray(sigma, dtype=np.float64), (S,)))
    flags = (1 if grad else 0) | (2 if mean else 0) | (4 if var else 0) | (8 if include_noise else 0)
    ll = np.zeros(S); g = np.zeros((S, th.shape[1] + 1)); mu = np.zeros((S, n)); v = np.zeros((S, n))
    fb = ctypes.c_int64()
    lv = _leaves(leaves)
    st = lib().emu_eval_batched(lv.ctypes.data, len(leaves), _p(th), th.shape[1], S, n, _p(t), _p(y), _p(sg), flags,
                                _p(ll), _p(g), _p(mu), _p(v), ctypes.byref(fb), int(m0), int(force_generic))
    if st:
        raise EmuError(st, fb.value, lib().emu_last_error().decode())
    if S == 1:
        return dict(loglik=ll[0], grad=g[0] if grad else None, mean=mu[0] if mean else None, var=v[0] if var else None)
    return dict(loglik=ll, grad=g if grad else None, mean=mu if mean else None, var=v if var else None)


def predict(leaves, theta, t, y, test_t, sigma, grad=True, include_noise=False, m0=0):
    """spingp_predict on the host emulation (merged grid, test points unobserved)."""
    t = np.ascontiguousarray(t, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    ts = np.ascontiguousarray(test_t, dtype=np.float64)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    m = len(ts)
    ll = np.zeros(1); g = np.zeros(len(th) + 1); mu = np.zeros(max(m, 1)); v = np.zeros(max(m, 1))
    fb = ctypes.c_int64()
    lv = _leaves(leaves)
    flags = (1 if grad else 0) | (8 if include_noise else 0)
    st = lib().emu_predict(lv.ctypes.data, len(leaves), _p(th), len(th), len(t), _p(t), _p(y), _p(ts), m,
                           float(sigma), flags, _p(ll), _p(g), _p(mu), _p(v), ctypes.byref(fb), int(m0))
    if st:
        raise EmuError(st, fb.value, lib().emu_last_error().decode())
    return dict(loglik=ll[0], grad=g if grad else None, mean=mu[:m], var=v[:m])


def btd(diag, upper, rhs=None, selinv=False, m0=0):
    diag = np.ascontiguousarray(diag, dtype=np.float64)
    n, b, _ = diag.shape
    upper = np.ascontiguousarray(upper if n > 1 else np.zeros((1, b, b)), dtype=np.float64)
    k = 0
    x = None
    if rhs is not None:
        rhs = np.ascontiguousarray(rhs, dtype=np.float64).reshape(n * b, -1)
        k = rhs.shape[1]
        x = np.zeros_like(rhs)
    cd = np.zeros_like(diag) if selinv else None
    cu = np.zeros((max(n - 1, 1), b, b)) if selinv else None
    ld = ctypes.c_double(); fb = ctypes.c_int64()
    st = lib().emu_btd(n, b, _p(diag), _p(upper), _p(rhs), k, _p(x), _p(cd), _p(cu), ctypes.byref(ld), ctypes.byref(fb),
                       int(m0))
    if st:
        raise EmuError(st, fb.value, "btd failure")
    return dict(x=x, cdiag=cd, cupper=None if cu is None else cu[:n - 1], logdet=ld.value)


def discretize(leaves, theta, dt, sigma=0.3):
    """Device closed-form step (T::step / T::grad) run on the host: Phi, Q, dPhi, dQt, jitter."""
    import oracle_lib
    b = oracle_lib.state_space(leaves, theta)["b"]
    nt = len(theta)
    L = lib()
    L.emu_discretize.argtypes = [ctypes.c_void_p, ctypes.c_int32, _d, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                 _d, _d, _d, _d, _d]
    th = np.ascontiguousarray(theta, dtype=np.float64)
    Phi = np.zeros((b, b)); Q = np.zeros((b, b)); dPhi = np.zeros((nt, b, b)); dQ = np.zeros((nt, b, b))
    jit = ctypes.c_double()
    lv = _leaves(leaves)
    st = L.emu_discretize(lv.ctypes.data, len(leaves), _p(th), nt, float(sigma), float(dt), _p(Phi), _p(Q), _p(dPhi),
                          _p(dQ), ctypes.byref(jit))
    if st:
        raise EmuError(st, -1, L.emu_last_error().decode())
    return Phi, Q, dPhi, dQ, jit.value


def seg_sizes(leaves):
    """(record, partials) lengths of the segment protocol (same rule as spingp_seg_sizes)."""
    nrec, npart = ctypes.c_int32(), ctypes.c_int32()
    lv = _leaves(leaves)
    nt = sum(4 if (not isinstance(lf, int) and lf[0] == 4) else 2 for lf in leaves)
    lib().emu_seg_sizes.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                    ctypes.POINTER(ctypes.c_int32)]
    st = lib().emu_seg_sizes(lv.ctypes.data, len(leaves), nt, ctypes.byref(nrec), ctypes.byref(npart))
    assert st == 0
    return nrec.value, npart.value


def seg_forward(leaves, theta, t, y, t_left, t_right, rank, nranks, sigma, flags=1, m0=0):
    L = lib()
    L.emu_seg_forward.argtypes = [ctypes.c_void_p, ctypes.c_int32, _d, ctypes.c_int32, _d, _d, ctypes.c_int64,
                                  ctypes.c_double, ctypes.c_double, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                  ctypes.c_uint32, ctypes.c_int64, _d]
    nrec, _ = seg_sizes(leaves)
    lv = _leaves(leaves)
    th = np.ascontiguousarray(theta, dtype=np.float64)
    global _seg_keep
    _seg_keep = (np.ascontiguousarray(t, dtype=np.float64), np.ascontiguousarray(y, dtype=np.float64))
    rec = np.zeros(nrec)
    st = L.emu_seg_forward(lv.ctypes.data, len(leaves), _p(th), len(th), _p(_seg_keep[0]), _p(_seg_keep[1]),
                           len(t), float(t_left), float(t_right), rank, nranks, float(sigma), flags, int(m0), _p(rec))
    if st:
        raise EmuError(st, -1, L.emu_last_error().decode())
    return rec


def seg_reverse(records, n_local, n_partials, mean=False, var=False):
    L = lib()
    L.emu_seg_reverse.argtypes = [_d, _d, _d, _d]
    records = np.ascontiguousarray(records, dtype=np.float64)
    part = np.zeros(n_partials)
    mu = np.zeros(n_local) if mean else None
    v = np.zeros(n_local) if var else None
    st = L.emu_seg_reverse(_p(records), _p(part), _p(mu), _p(v))
    if st:
        raise EmuError(st, -1, "seg reverse failure")
    return part, mu, v


def seg_finalize(partials, n_theta, n_total, sigma):
    import math
    s2 = sigma * sigma
    ll = -0.5 * (partials[1] + partials[2]) - 0.5 * (partials[0] + partials[3] + n_total * math.log(s2)) \
        - 0.5 * n_total * math.log(2 * math.pi)
    g = np.zeros(n_theta + 1)
    g[:n_theta] = partials[5:5 + n_theta]
    g[n_theta] = 2 * sigma * (-0.5 * n_total / s2 + partials[4] / (2 * s2 * s2))
    return ll, g
