"""ctypes binding of libspingp_b200.so (include/spingp_c.h).

Every symbol declared in include/spingp_c.h is bound here with its exact
signature; status codes are mapped onto the reference's exception hierarchy
(proj/include/spingp/errors.hpp:12-47).
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.environ.get("SPINGP_LIB") or os.path.join(_HERE, "libspingp_b200.so")  # override: experiments only

MATERN12, MATERN32, MATERN52, EQ, QP = 0, 1, 2, 3, 4
LEAF_NPARAMS = {MATERN12: 2, MATERN32: 2, MATERN52: 2, EQ: 2, QP: 4}
WANT_GRAD, WANT_MEAN, WANT_VAR, INCLUDE_NOISE = 1, 2, 4, 8

OK, NOT_PD, SINGULAR_Q, BAD_ARG, CUDA_ERR, NCCL_ERR, DUPLICATE_TIME, UNSUPPORTED, NEG_VARIANCE = range(9)


class SpingpError(RuntimeError):
    def __init__(self, status, msg, block=None):
        super().__init__(msg if block is None or block < 0 else f"{msg} (block {block})")
        self.status = status
        self.block = block

    def block_index(self):
        return self.block


class NotPositiveDefinite(SpingpError):
    """errors.hpp:12-20."""


class SingularProcessNoise(NotPositiveDefinite):
    """errors.hpp:23-27."""


class DuplicateTimestamp(SpingpError, ValueError):
    """errors.hpp:29-32."""


class DeviceError(SpingpError):
    """CUDA failure (no CPU fallback exists)."""


class NegativeVariance(SpingpError):
    """a posterior variance below -1e-10."""


class Unsupported(SpingpError):
    pass


class BadArgument(SpingpError, ValueError):
    """std::invalid_argument in the reference."""


_EXC = {NOT_PD: NotPositiveDefinite, SINGULAR_Q: SingularProcessNoise, BAD_ARG: BadArgument,
        CUDA_ERR: DeviceError, NCCL_ERR: DeviceError, DUPLICATE_TIME: DuplicateTimestamp,
        UNSUPPORTED: Unsupported, NEG_VARIANCE: NegativeVariance}

_P = ctypes.POINTER
_d = _P(ctypes.c_double)
_i32p = _P(ctypes.c_int32)
_i64p = _P(ctypes.c_int64)
_vp = ctypes.c_void_p
_i32, _i64, _u32, _dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_double

# name -> (restype, argtypes): exactly the declarations of include/spingp_c.h
SIGNATURES = {
    "spingp_abi_version": (ctypes.c_int, []),
    "spingp_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "spingp_last_error": (ctypes.c_char_p, []),
    "spingp_kernel_dims": (ctypes.c_int, [_vp, _i32, _i32p, _i32p]),
    "spingp_state_space": (ctypes.c_int, [_vp, _i32, _d, _i32, _d, _d, _d, _d, _d, _i32p]),
    "spingp_ctx_create": (ctypes.c_int, [_i32, _P(_vp)]),
    "spingp_ctx_destroy": (ctypes.c_int, [_vp]),
    "spingp_ctx_set_stream": (ctypes.c_int, [_vp, _vp]),
    "spingp_ctx_use_own_stream": (ctypes.c_int, [_vp]),
    "spingp_ctx_set_phase_stamps": (ctypes.c_int, [_vp, _vp]),
    "spingp_ctx_get_stream": (_vp, [_vp]),
    "spingp_ctx_status": (ctypes.c_int, [_vp, _i64p]),
    "spingp_ctx_launch_count": (_i64, [_vp]),
    "spingp_ctx_set_chunk": (ctypes.c_int, [_vp, _i64]),
    "spingp_ctx_set_tree_group": (ctypes.c_int, [_vp, _i64]),
    "spingp_ctx_set_profiling": (ctypes.c_int, [_vp, ctypes.c_int]),
    "spingp_ctx_kernel_times": (ctypes.c_int, [_vp, _P(ctypes.c_char_p), _d, _i32, _i32p]),
    "spingp_eval": (ctypes.c_int, [_vp, _vp, _i32, _d, _i32, _d, _d, _i64, _dbl, _u32, _d, _d, _d, _d, _i64p]),
    "spingp_predict": (ctypes.c_int, [_vp, _vp, _i32, _d, _i32, _d, _d, _i64, _d, _i64, _dbl, _u32, _d, _d, _d, _d,
                                      _i64p]),
    "spingp_eval_device": (ctypes.c_int, [_vp, _vp, _i32, _d, _i32, _vp, _vp, _i64, _dbl, _u32, _vp, _vp, _vp, _vp]),
    "spingp_eval_batched": (ctypes.c_int, [_vp, _vp, _i32, _d, _i32, _i64, _i64, _d, _d, _d, _u32, _d, _d, _d, _d,
                                           _i64p]),
    "spingp_eval_batched_device": (ctypes.c_int, [_vp, _vp, _i32, _d, _i32, _i64, _i64, _vp, _vp, _d, _u32, _vp, _vp,
                                                  _vp, _vp]),
    "spingp_assemble": (ctypes.c_int, [_vp, _vp, _i32, _d, _i32, _d, _d, _i64, _dbl, _d, _d, _d, _i64p]),
    "spingp_seg_sizes": (ctypes.c_int, [_vp, _i32, _i32p, _i32p]),
    "spingp_seg_forward_device": (ctypes.c_int, [_vp, _vp, _i32, _d, _i32, _vp, _vp, _i64, _dbl, _dbl, _i32, _i32, _dbl,
                                                 _u32, _vp]),
    "spingp_seg_reverse_device": (ctypes.c_int, [_vp, _vp, _i32, _d, _i32, _vp, _vp, _i64, _dbl, _dbl, _i32, _i32, _dbl,
                                                 _u32, _vp, _vp, _vp, _vp]),
    "spingp_seg_finalize_device": (ctypes.c_int, [_vp, _i32, _i64, _dbl, _u32, _vp, _vp, _vp]),
    "spingp_btd_cr_solve": (ctypes.c_int, [_vp, _i64, _i32, _d, _d, _d, _i32, _d, _d, _i64p]),
    "spingp_btd_cr_solve_device": (ctypes.c_int, [_vp, _i64, _i32, _vp, _vp, _vp, _i32, _vp, _vp]),
    "spingp_btd_selinv": (ctypes.c_int, [_vp, _i64, _i32, _d, _d, _d, _d, _d, _i64p]),
    "spingp_btd_selinv_device": (ctypes.c_int, [_vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "spingp_btd_matvec": (ctypes.c_int, [_vp, _i64, _i32, _d, _d, _d, _d]),
    "spingp_eval_multi_theta": (ctypes.c_int, [_vp, _vp, _i32, _d, _i32, _i64, _d, _d, _i64, _d, _u32, _d, _d,
                                               _i64p]),
    "spingp_mctx_create": (ctypes.c_int, [_i32, _i32p, _P(_vp)]),
    "spingp_mctx_destroy": (ctypes.c_int, [_vp]),
    "spingp_mctx_size": (_i32, [_vp]),
    "spingp_mctx_rank_ctx": (_vp, [_vp, _i32]),
    "spingp_eval_partitioned": (ctypes.c_int, [_vp, _vp, _i32, _d, _i32, _d, _d, _i64, _dbl, _u32, _d, _d, _d, _d,
                                               _i64p]),
    "spingp_btd_factorize": (ctypes.c_int, [_vp, _i64, _i32, _d, _d, _P(_vp), _d, _i64p]),
    "spingp_btd_factor_destroy": (ctypes.c_int, [_vp]),
    "spingp_btd_factor_info": (ctypes.c_int, [_vp, _i64p, _i32p, _d]),
    "spingp_btd_factor_blocks": (ctypes.c_int, [_vp, _vp, _d, _d]),
    "spingp_btd_factor_solve": (ctypes.c_int, [_vp, _vp, _d, _i32, _d]),
    "spingp_btd_factor_selinv": (ctypes.c_int, [_vp, _vp, _d, _d]),
}

_lib = None


def lib():
    """Load libspingp_b200.so; raise loudly when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(lib_path):
            raise ImportError(f"{lib_path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(lib_path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _raise(st, fb=None):
    if st == OK:
        return
    msg = lib().spingp_last_error().decode() or lib().spingp_status_string(st).decode()
    blk = None if fb is None else int(fb.value if hasattr(fb, "value") else fb)
    raise _EXC.get(st, SpingpError)(st, msg, blk)


def _p(a):
    return None if a is None else a.ctypes.data_as(_d)


def _leaves(leaves):
    arr = np.zeros(2 * len(leaves), dtype=np.int32)
    for i, lf in enumerate(leaves):
        typ, order = (lf, 0) if isinstance(lf, (int, np.integer)) else lf
        arr[2 * i], arr[2 * i + 1] = int(typ), int(order)
    return arr


def n_theta(leaves):
    return sum(LEAF_NPARAMS[(lf if isinstance(lf, (int, np.integer)) else lf[0])] for lf in leaves)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def kernel_dims(leaves):
    lv = _leaves(leaves)
    b, nt = _i32(), _i32()
    _raise(lib().spingp_kernel_dims(lv.ctypes.data, len(leaves), ctypes.byref(b), ctypes.byref(nt)))
    return b.value, nt.value


def seg_sizes(leaves):
    """(record length, partials length) of the multi-GPU segment protocol."""
    nrec, npart = _i32(), _i32()
    lv = _leaves(leaves)
    _raise(lib().spingp_seg_sizes(lv.ctypes.data, len(leaves), ctypes.byref(nrec), ctypes.byref(npart)))
    return nrec.value, npart.value


def state_space(leaves, theta):
    """state_space_of (kernels.hpp:326-381) through the library's host code."""
    b, nt = kernel_dims(leaves)
    th = _f64(theta)
    lv = _leaves(leaves)
    F = np.zeros((b, b)); H = np.zeros(b); P = np.zeros((b, b))
    dF = np.zeros((nt, b, b)); dP = np.zeros((nt, b, b)); fc = np.zeros(nt, dtype=np.int32)
    _raise(lib().spingp_state_space(lv.ctypes.data, len(leaves), _p(th), len(th), _p(F), _p(H), _p(P), _p(dF), _p(dP),
                                    fc.ctypes.data_as(_i32p)))
    return dict(F=F, H=H, Pinf=P, dF=dF, dPinf=dP, f_constant=fc, b=b)


def _out(out, key, shape):
    """A caller-supplied output array (validated) or a fresh zeroed one."""
    if out is None or out.get(key) is None:
        return np.zeros(shape)
    a = out[key]
    if a.dtype != np.float64 or not a.flags.c_contiguous or a.shape != tuple(shape) or not a.flags.writeable:
        raise ValueError(f"out[{key!r}] must be a writeable C-contiguous float64 array of shape {tuple(shape)}")
    return a


class Context:
    """spingp_ctx: one CUDA device + stream + workspace."""

    def __init__(self, device=0):
        self._h = _vp()
        _raise(lib().spingp_ctx_create(int(device), ctypes.byref(self._h)))

    def close(self):
        if self._h:
            lib().spingp_ctx_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    @property
    def stream(self):
        return lib().spingp_ctx_get_stream(self._h)

    def set_stream(self, stream_ptr):
        """Enqueue on an external cudaStream_t (an int handle; 0 = the legacy default
        stream, e.g. torch's default current stream).  None = the context's own stream."""
        if stream_ptr is None:
            _raise(lib().spingp_ctx_use_own_stream(self._h))
        else:
            _raise(lib().spingp_ctx_set_stream(self._h, ctypes.c_void_p(int(stream_ptr))))

    def set_phase_stamps(self, d_ptr):
        """Diagnostics: device buffer (>= 64 uint64) for per-phase timer stamps (0 = off)."""
        _raise(lib().spingp_ctx_set_phase_stamps(self._h, ctypes.c_void_p(int(d_ptr)) if d_ptr else None))

    def set_chunk(self, m0):
        _raise(lib().spingp_ctx_set_chunk(self._h, int(m0)))

    def set_tree_group(self, g):
        _raise(lib().spingp_ctx_set_tree_group(self._h, int(g)))

    def set_profiling(self, on=True):
        _raise(lib().spingp_ctx_set_profiling(self._h, 1 if on else 0))

    def kernel_times(self, cap=4096):
        """[(kernel name, ms)] for every launch since the last call (synchronises)."""
        names = (ctypes.c_char_p * cap)()
        ms = np.zeros(cap)
        cnt = _i32()
        _raise(lib().spingp_ctx_kernel_times(self._h, names, _p(ms), cap, ctypes.byref(cnt)))
        k = min(cnt.value, cap)
        return [(names[i].decode(), float(ms[i])) for i in range(k)]

    def launch_count(self):
        return int(lib().spingp_ctx_launch_count(self._h))

    def status(self):
        fb = _i64()
        _raise(lib().spingp_ctx_status(self._h, ctypes.byref(fb)), fb)

    # ---- host-pointer entry points (synchronous) ----------------------------------
    def eval(self, leaves, theta, t, y, sigma, grad=True, mean=False, var=False, include_noise=False, out=None):
        """log_marginal_likelihood + mll_gradient + training-point posterior.
        out: optional dict of preallocated float64 C-contiguous arrays ('grad', 'mean', 'var'),
        e.g. views of pinned host memory, written in place (no per-call allocation)."""
        lv = _leaves(leaves)
        th = _f64(theta); t = _f64(t); y = _f64(y)
        n = len(t)
        if len(y) != n:
            raise ValueError("t and y lengths differ")
        flags = (WANT_GRAD if grad else 0) | (WANT_MEAN if mean else 0) | (WANT_VAR if var else 0) | \
            (INCLUDE_NOISE if include_noise else 0)
        ll = _dbl()
        g = _out(out, "grad", (len(th) + 1,)) if grad else None
        mu = _out(out, "mean", (n,)) if mean else None
        v = _out(out, "var", (n,)) if var else None
        fb = _i64()
        st = lib().spingp_eval(self._h, lv.ctypes.data, len(leaves), _p(th), len(th), _p(t), _p(y), n, float(sigma), flags,
                               ctypes.byref(ll), _p(g), _p(mu), _p(v), ctypes.byref(fb))
        _raise(st, fb)
        return dict(loglik=ll.value, grad=g, mean=mu, var=v)

    def predict(self, leaves, theta, t, y, test_t, sigma, grad=True, include_noise=False):
        """predict at arbitrary test times: posterior mean / variance at
        test_t (input order) with the training loglik (+ gradient)."""
        lv = _leaves(leaves)
        th = _f64(theta); t = _f64(t); y = _f64(y); ts = _f64(test_t)
        if len(y) != len(t):
            raise ValueError("t and y lengths differ")
        m = len(ts)
        ll = _dbl()
        g = np.empty(len(th) + 1) if grad else None
        mu = np.empty(m)
        v = np.empty(m)
        fb = _i64()
        flags = (WANT_GRAD if grad else 0) | (INCLUDE_NOISE if include_noise else 0)
        st = lib().spingp_predict(self._h, lv.ctypes.data, len(leaves), _p(th), len(th), _p(t), _p(y), len(t), _p(ts),
                                  m, float(sigma), flags, ctypes.byref(ll), _p(g), _p(mu), _p(v), ctypes.byref(fb))
        _raise(st, fb)
        return dict(loglik=ll.value, grad=g, mean=mu, var=v)

    def eval_batched(self, leaves, theta, t, y, sigma, grad=True, mean=False, var=False, include_noise=False,
                     out=None):
        lv = _leaves(leaves)
        t = _f64(t); y = _f64(y)
        S, n = t.shape
        th = _f64(theta).reshape(S, -1)
        sg = _f64(np.broadcast_to(np.asarray(sigma, dtype=np.float64), (S,)))
        flags = (WANT_GRAD if grad else 0) | (WANT_MEAN if mean else 0) | (WANT_VAR if var else 0) | \
            (INCLUDE_NOISE if include_noise else 0)
        ll = _out(out, "loglik", (S,))
        g = _out(out, "grad", (S, th.shape[1] + 1)) if grad else None
        mu = _out(out, "mean", (S, n)) if mean else None
        v = _out(out, "var", (S, n)) if var else None
        fb = _i64()
        st = lib().spingp_eval_batched(self._h, lv.ctypes.data, len(leaves), _p(th), th.shape[1], S, n, _p(t), _p(y),
                                       _p(sg), flags, _p(ll), _p(g), _p(mu), _p(v), ctypes.byref(fb))
        _raise(st, fb)
        return dict(loglik=ll, grad=g, mean=mu, var=v)

    def assemble(self, leaves, theta, t, y, sigma):
        """assemble_prior_precision + add_observation_term."""
        lv = _leaves(leaves)
        th = _f64(theta); t = _f64(t); y = _f64(y)
        n = len(t)
        b, _ = kernel_dims(leaves)
        diag = np.zeros((n, b, b)); upper = np.zeros((max(n - 1, 0), b, b)); rhs = np.zeros((n, b))
        fb = _i64()
        st = lib().spingp_assemble(self._h, lv.ctypes.data, len(leaves), _p(th), len(th), _p(t), _p(y), n, float(sigma),
                                   _p(diag), _p(upper) if n > 1 else None, _p(rhs), ctypes.byref(fb))
        _raise(st, fb)
        return diag, upper, rhs

    def btd_cr_solve(self, diag, upper, rhs=None):
        """cr_solve: (x, logdet)."""
        diag = _f64(diag)
        n, b, _ = diag.shape
        upper = _f64(upper if n > 1 else np.zeros((0, b, b)))
        ld = _dbl(); fb = _i64()
        if rhs is None:
            _raise(lib().spingp_btd_cr_solve(self._h, n, b, _p(diag), _p(upper) if n > 1 else None, None, 0, None,
                                             ctypes.byref(ld), ctypes.byref(fb)), fb)
            return None, ld.value
        rhs = _f64(rhs)
        shape = rhs.shape
        r2 = rhs.reshape(n * b, -1)
        k = r2.shape[1]
        x = np.zeros_like(r2)
        _raise(lib().spingp_btd_cr_solve(self._h, n, b, _p(diag), _p(upper) if n > 1 else None, _p(r2), k, _p(x),
                                         ctypes.byref(ld), ctypes.byref(fb)), fb)
        return x.reshape(shape), ld.value

    def btd_selinv(self, diag, upper):
        """selective_inverse: (cdiag, cupper, logdet)."""
        diag = _f64(diag)
        n, b, _ = diag.shape
        upper = _f64(upper if n > 1 else np.zeros((0, b, b)))
        cd = np.zeros_like(diag); cu = np.zeros((max(n - 1, 0), b, b)); ld = _dbl(); fb = _i64()
        _raise(lib().spingp_btd_selinv(self._h, n, b, _p(diag), _p(upper) if n > 1 else None, _p(cd),
                                       _p(cu) if n > 1 else None, ctypes.byref(ld), ctypes.byref(fb)), fb)
        return cd, cu, ld.value

    def btd_matvec(self, diag, upper, v):
        diag = _f64(diag)
        n, b, _ = diag.shape
        upper = _f64(upper if n > 1 else np.zeros((0, b, b)))
        v = _f64(v).reshape(n * b)
        out = np.zeros(n * b)
        _raise(lib().spingp_btd_matvec(self._h, n, b, _p(diag), _p(upper) if n > 1 else None, _p(v), _p(out)))
        return out

    # ---- device-pointer entry points (asynchronous, on self.stream) ----------------
    def eval_device(self, leaves, theta, d_t, d_y, n, sigma, flags, d_loglik, d_grad=0, d_mean=0, d_var=0):
        lv = _leaves(leaves)
        th = _f64(theta)
        _raise(lib().spingp_eval_device(self._h, lv.ctypes.data, len(leaves), _p(th), len(th), d_t, d_y, int(n),
                                        float(sigma), int(flags), d_loglik, d_grad or None, d_mean or None,
                                        d_var or None))

    def eval_batched_device(self, leaves, theta, S, n, d_t, d_y, sigma, flags, d_loglik, d_grad=0, d_mean=0, d_var=0):
        lv = _leaves(leaves)
        th = _f64(theta).reshape(S, -1)
        sg = _f64(np.broadcast_to(np.asarray(sigma, dtype=np.float64), (S,)))
        _raise(lib().spingp_eval_batched_device(self._h, lv.ctypes.data, len(leaves), _p(th), th.shape[1], int(S),
                                                int(n), d_t, d_y, _p(sg), int(flags), d_loglik, d_grad or None,
                                                d_mean or None, d_var or None))

    # ---- multi-GPU partition of one series (segment protocol, include/spingp_c.h) -----
    def seg_forward_device(self, leaves, theta, d_t, d_y, n_local, t_left, t_right, rank, nranks, sigma, flags,
                           d_record):
        lv = _leaves(leaves)
        th = _f64(theta)
        _raise(lib().spingp_seg_forward_device(self._h, lv.ctypes.data, len(leaves), _p(th), len(th), d_t, d_y,
                                               int(n_local), float(t_left), float(t_right), int(rank), int(nranks),
                                               float(sigma), int(flags), d_record))

    def seg_reverse_device(self, leaves, theta, d_t, d_y, n_local, t_left, t_right, rank, nranks, sigma, flags,
                           d_records, d_partials, d_mean=0, d_var=0):
        lv = _leaves(leaves)
        th = _f64(theta)
        _raise(lib().spingp_seg_reverse_device(self._h, lv.ctypes.data, len(leaves), _p(th), len(th), d_t, d_y,
                                               int(n_local), float(t_left), float(t_right), int(rank), int(nranks),
                                               float(sigma), int(flags), d_records, d_partials, d_mean or None,
                                               d_var or None))

    def seg_finalize_device(self, n_theta, n_total, sigma, flags, d_partials, d_loglik, d_grad=0):
        _raise(lib().spingp_seg_finalize_device(self._h, int(n_theta), int(n_total), float(sigma), int(flags),
                                                d_partials, d_loglik, d_grad or None))

    def btd_factorize(self, diag, upper):
        """factorize: a device-resident BTDFactor bound to this context."""
        return BTDFactor(self, diag, upper)

    def btd_cr_solve_device(self, n, b, d_diag, d_upper, d_rhs, k, d_x, d_logdet):
        _raise(lib().spingp_btd_cr_solve_device(self._h, int(n), int(b), d_diag, d_upper, d_rhs, int(k), d_x, d_logdet))


class BTDFactor:
    """BTDFactor on the device: L_i, M_i, log det and the selected
    inverse, kept for solve / selective_inverse (spingp_btd_factorize)."""

    def __init__(self, ctx, diag, upper):
        d = _f64(diag)
        n, b = d.shape[0], d.shape[1]
        u = _f64(upper) if n > 1 else None
        self._ctx, self.n, self.b = ctx, n, b
        self._h = _vp()
        ld = _dbl()
        fb = _i64()
        _raise(lib().spingp_btd_factorize(ctx._h, n, b, _p(d), _p(u), ctypes.byref(self._h), ctypes.byref(ld),
                                          ctypes.byref(fb)), fb)
        self.logdet = ld.value

    def blocks(self):
        L = np.empty((self.n, self.b, self.b))
        M = np.empty((max(self.n - 1, 0), self.b, self.b))
        _raise(lib().spingp_btd_factor_blocks(self._ctx._h, self._h, _p(L), _p(M) if self.n > 1 else None))
        return L, M

    def solve(self, rhs):
        r = _f64(rhs)
        k = 1 if r.ndim == 1 else r.shape[1]
        x = np.empty_like(r)
        _raise(lib().spingp_btd_factor_solve(self._ctx._h, self._h, _p(r), k, _p(x)))
        return x

    def selective_inverse(self):
        cd = np.empty((self.n, self.b, self.b))
        cu = np.empty((max(self.n - 1, 0), self.b, self.b))
        _raise(lib().spingp_btd_factor_selinv(self._ctx._h, self._h, _p(cd), _p(cu) if self.n > 1 else None))
        return cd, cu

    def close(self):
        if self._h:
            lib().spingp_btd_factor_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MultiContext:
    """spingp_mctx: P devices of one box joined by NCCL (spingp_mctx_create); eval()
    partitions one long series over them (spingp_eval_partitioned)."""

    def __init__(self, devices):
        devs = np.ascontiguousarray(devices, dtype=np.int32)
        self._h = _vp()
        _raise(lib().spingp_mctx_create(len(devs), devs.ctypes.data_as(_i32p), ctypes.byref(self._h)))
        self.size = len(devs)

    def eval(self, leaves, theta, t, y, sigma, grad=True, mean=False, var=False):
        lv = _leaves(leaves)
        th = _f64(theta); t = _f64(t); y = _f64(y)
        n = len(t)
        flags = (WANT_GRAD if grad else 0) | (WANT_MEAN if mean else 0) | (WANT_VAR if var else 0)
        ll = _dbl()
        g = np.zeros(len(th) + 1) if grad else None
        mu = np.zeros(n) if mean else None
        v = np.zeros(n) if var else None
        fb = _i64()
        _raise(lib().spingp_eval_partitioned(self._h, lv.ctypes.data, len(leaves), _p(th), len(th), _p(t), _p(y), n,
                                             float(sigma), flags, ctypes.byref(ll), _p(g), _p(mu), _p(v),
                                             ctypes.byref(fb)), fb)
        return dict(loglik=ll.value, grad=g, mean=mu, var=v)

    def close(self):
        if self._h:
            lib().spingp_mctx_destroy(self._h)
            self._h = _vp()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
