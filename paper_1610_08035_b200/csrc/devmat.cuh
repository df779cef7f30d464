// devmat.cuh — fixed-size dense fp64 block algebra for one thread (b x b blocks,
// row-major arrays).  For b <= 3 everything lives in registers; the templates
// are fully unrolled so the compiler can schedule the independent DFMAs.
//
// These are the per-block operations of the SPEC's btd_core:
// Cholesky pivots (factorize :146), triangular solves, explicit SPD inverses
// (selective_inverse :170-178) and the Schur-complement updates.
#pragma once

#ifndef SPINGP_HOST_EMU
#include <cuda_runtime.h>
#endif

namespace spingp_dev {

// SP_DEV_NOINLINE (experiment for the b >= 6 builds): every block
// routine becomes a real call with its own frame instead of being inlined.
#ifdef SP_DEV_NOINLINE
#define SP_DEV __device__ __noinline__ inline
#else
#define SP_DEV __device__ __forceinline__
#endif
// The fixed-size primitives of this file: always inlined, unless SP_DEVM_NOINLINE (the
// whole-call-tree variant of the b >= 6 build).
#if defined(SP_DEV_NOINLINE) && defined(SP_DEVM_NOINLINE)
#define SP_DEVM __device__ __noinline__ inline
#else
#define SP_DEVM __device__ __forceinline__
#endif
// Loop-unrolling hint for the b x b loops.  Deliberately empty: nvcc fully
// unrolls the constant-trip loops of the register-resident sizes (b <= 4) on
// its own, and an explicit `#pragma unroll (B <= 4 ? 64 : 1)` was measured to
// MISCOMPILE the triangular loops (inner trip count depending on the outer
// index) with nvcc 12.9 for sm_100a — wrong covariance blocks on the device
// while the same source was correct on the host (tools/dbg/dbg_pipe.cu).
#ifndef SP_UNROLL
#define SP_UNROLL
#endif
// Compiler-level memory barrier (no instruction emitted): the optimiser may not move
// local-array loads/stores across it (used around the dynamically offset leaf writes).
#ifndef SP_MEMFENCE
#define SP_MEMFENCE() asm volatile("" ::: "memory")
#endif

// L1 prefetch hint for a global address (no register, no wait; no-op on the host).
SP_DEVM void prefetch_l1(const void* p) {
#ifndef SPINGP_HOST_EMU
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#else
    (void)p;
#endif
}

template <int B>
SP_DEVM void mzero(double* a) {
SP_UNROLL
    for (int i = 0; i < B * B; ++i) a[i] = 0.0;
}
template <int B>
SP_DEVM void mcopy(double* d, const double* s) {
SP_UNROLL
    for (int i = 0; i < B * B; ++i) d[i] = s[i];
}
template <int B>
SP_DEVM void vzero(double* a) {
SP_UNROLL
    for (int i = 0; i < B; ++i) a[i] = 0.0;
}

// C = A * B
template <int B>
SP_DEVM void mm(double* C, const double* A, const double* Bm) {
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) {
            double s = 0.0;
SP_UNROLL
            for (int k = 0; k < B; ++k) s = fma(A[i * B + k], Bm[k * B + j], s);
            C[i * B + j] = s;
        }
}
// C = A^T * B
template <int B>
SP_DEVM void mtm(double* C, const double* A, const double* Bm) {
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) {
            double s = 0.0;
SP_UNROLL
            for (int k = 0; k < B; ++k) s = fma(A[k * B + i], Bm[k * B + j], s);
            C[i * B + j] = s;
        }
}
// C = A * B^T
template <int B>
SP_DEVM void mmt(double* C, const double* A, const double* Bm) {
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) {
            double s = 0.0;
SP_UNROLL
            for (int k = 0; k < B; ++k) s = fma(A[i * B + k], Bm[j * B + k], s);
            C[i * B + j] = s;
        }
}
// C = A^T * B, known to be symmetric: compute the lower triangle and mirror.
template <int B>
SP_DEVM void mtm_sym(double* C, const double* A, const double* Bm) {
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j <= i; ++j) {
            double s = 0.0;
SP_UNROLL
            for (int k = 0; k < B; ++k) s = fma(A[k * B + i], Bm[k * B + j], s);
            C[i * B + j] = s;
            C[j * B + i] = s;
        }
}
// y = A x
template <int B>
SP_DEVM void mv(double* y, const double* A, const double* x) {
SP_UNROLL
    for (int i = 0; i < B; ++i) {
        double s = 0.0;
SP_UNROLL
        for (int k = 0; k < B; ++k) s = fma(A[i * B + k], x[k], s);
        y[i] = s;
    }
}
// y = A^T x
template <int B>
SP_DEVM void mtv(double* y, const double* A, const double* x) {
SP_UNROLL
    for (int i = 0; i < B; ++i) {
        double s = 0.0;
SP_UNROLL
        for (int k = 0; k < B; ++k) s = fma(A[k * B + i], x[k], s);
        y[i] = s;
    }
}
template <int B>
SP_DEVM void msym(double* a) {
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < i; ++j) {
            const double v = 0.5 * (a[i * B + j] + a[j * B + i]);
            a[i * B + j] = v;
            a[j * B + i] = v;
        }
}
template <int B>
SP_DEVM double mtrace(const double* a) {
    double s = 0.0;
SP_UNROLL
    for (int i = 0; i < B; ++i) s += a[i * B + i];
    return s;
}
// Tr(A B)
template <int B>
SP_DEVM double mtrprod(const double* A, const double* Bm) {
    double s = 0.0;
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int k = 0; k < B; ++k) s = fma(A[i * B + k], Bm[k * B + i], s);
    return s;
}

// Cholesky A = L L^T with INVERTED pivots: the returned lower-triangular L holds
// 1/l_jj on its diagonal (all substitutions below multiply by it; one rsqrt per
// pivot and no divisions).  Returns false on a non-positive / non-finite pivot.
// logdet = log det A = -2 log prod_j (1/l_jj), taken in groups of 4 pivots.
template <int B>
SP_DEVM bool chol_nolog(double* L, const double* A) {
    bool ok = true;
SP_UNROLL
    for (int j = 0; j < B; ++j) {
        double d = A[j * B + j];
SP_UNROLL
        for (int k = 0; k < j; ++k) d = fma(-L[j * B + k], L[j * B + k], d);
        ok = ok && (d > 0.0) && isfinite(d);
        const double inv = rsqrt(d);
        L[j * B + j] = inv;
SP_UNROLL
        for (int i = j + 1; i < B; ++i) {
            double s = A[i * B + j];
SP_UNROLL
            for (int k = 0; k < j; ++k) s = fma(-L[i * B + k], L[j * B + k], s);
            L[i * B + j] = s * inv;
        }
SP_UNROLL
        for (int i = 0; i < j; ++i) L[i * B + j] = 0.0;
    }
    return ok;
}
template <int B>
SP_DEVM double chol_logdet(const double* L) {
    double ld = 0.0;
SP_UNROLL
    for (int j0 = 0; j0 < B; j0 += 4) {
        double p = 1.0;
SP_UNROLL
        for (int j = j0; j < j0 + 4 && j < B; ++j) p *= L[j * B + j];
        ld += log(p);
    }
    return -2.0 * ld;
}
template <int B>
SP_DEVM bool chol(double* L, const double* A, double& logdet) {
    const bool ok = chol_nolog<B>(L, A);
    logdet = ok ? chol_logdet<B>(L) : 0.0;
    return ok;
}

// Running log-determinant without a log per factorisation: the product of the
// inverted pivots is kept as mantissa in [0.5, 1) times 2^e (renormalised by
// exponent-field arithmetic after every group of <= 4 pivots, so it never leaves the
// normal range); one log at the end of a chunk.
struct LogDetAcc {
    double m;
    int e;
    SP_DEVM void init() {
        m = 1.0;
        e = 0;
    }
    SP_DEVM void mul(double p) {  // p > 0 finite
        double x = m * p;
#ifdef SPINGP_HOST_EMU
        int ex;
        x = std::frexp(x, &ex);
        e += ex;
#else
        const int hi = __double2hiint(x);
        e += ((hi >> 20) & 0x7ff) - 1022;
        x = __hiloint2double((hi & 0x800fffff) | 0x3fe00000, __double2loint(x));
#endif
        m = x;
    }
    // log det of the factored matrices = -2 log prod(1/l_jj)
    SP_DEVM double logdet() const { return -2.0 * (log(m) + static_cast<double>(e) * 0.69314718055994530942); }
};
template <int B>
SP_DEVM void chol_accum(const double* L, LogDetAcc& acc) {
SP_UNROLL
    for (int j0 = 0; j0 < B; j0 += 4) {
        double p = 1.0;
SP_UNROLL
        for (int j = j0; j < j0 + 4 && j < B; ++j) p *= L[j * B + j];
        acc.mul(p);
    }
}
template <int B>
SP_DEVM bool chol(double* L, const double* A, LogDetAcc& acc) {
    const bool ok = chol_nolog<B>(L, A);
    if (ok) chol_accum<B>(L, acc);
    return ok;
}

// Ainv = (L L^T)^{-1} = L^{-T} L^{-1}, symmetric.
template <int B>
SP_DEVM void chol_inverse(double* Ainv, const double* L) {
    double Li[B * B];  // L^{-1}, lower
SP_UNROLL
    for (int j = 0; j < B; ++j) {
        const double dj = L[j * B + j];  // inverted pivot
SP_UNROLL
        for (int i = 0; i < B; ++i) {
            if (i < j) { Li[i * B + j] = 0.0; continue; }
            if (i == j) { Li[i * B + j] = dj; continue; }
            double s = 0.0;
SP_UNROLL
            for (int k = j; k < i; ++k) s = fma(L[i * B + k], (k == j ? dj : Li[k * B + j]), s);
            Li[i * B + j] = -s * L[i * B + i];
        }
    }
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j <= i; ++j) {
            double s = 0.0;
SP_UNROLL
            for (int k = i; k < B; ++k) s = fma(Li[k * B + i], Li[k * B + j], s);
            Ainv[i * B + j] = s;
            Ainv[j * B + i] = s;
        }
}

// ---- triangular-factor forms (the numerically preferred route) -------------
// Li = L^{-1} for lower-triangular L (Li lower, zero upper).
template <int B>
SP_DEVM void tri_inverse(double* Li, const double* L) {
SP_UNROLL
    for (int j = 0; j < B; ++j) {
        const double dj = L[j * B + j];  // inverted pivot
SP_UNROLL
        for (int i = 0; i < B; ++i) {
            if (i < j) {
                Li[i * B + j] = 0.0;
            } else if (i == j) {
                Li[i * B + j] = dj;
            } else {
                double s = L[i * B + j] * dj;
SP_UNROLL
                for (int k = j + 1; k < i; ++k) s = fma(L[i * B + k], Li[k * B + j], s);
                Li[i * B + j] = -s * L[i * B + i];
            }
        }
    }
}
// C = Li A   (Li lower triangular)
template <int B>
SP_DEVM void lmul(double* C, const double* Li, const double* A) {
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) {
            double s = 0.0;
SP_UNROLL
            for (int k = 0; k <= i; ++k) s = fma(Li[i * B + k], A[k * B + j], s);
            C[i * B + j] = s;
        }
}
// C = Li^T A   (Li lower triangular)
template <int B>
SP_DEVM void ltmul(double* C, const double* Li, const double* A) {
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) {
            double s = 0.0;
SP_UNROLL
            for (int k = i; k < B; ++k) s = fma(Li[k * B + i], A[k * B + j], s);
            C[i * B + j] = s;
        }
}
// y = Li x ; y = Li^T x
template <int B>
SP_DEVM void lmv(double* y, const double* Li, const double* x) {
SP_UNROLL
    for (int i = 0; i < B; ++i) {
        double s = 0.0;
SP_UNROLL
        for (int k = 0; k <= i; ++k) s = fma(Li[i * B + k], x[k], s);
        y[i] = s;
    }
}
template <int B>
SP_DEVM void ltmv(double* y, const double* Li, const double* x) {
SP_UNROLL
    for (int i = 0; i < B; ++i) {
        double s = 0.0;
SP_UNROLL
        for (int k = i; k < B; ++k) s = fma(Li[k * B + i], x[k], s);
        y[i] = s;
    }
}
// C = Li^T X Li for symmetric X (result symmetric)
template <int B>
SP_DEVM void sandwich(double* C, const double* Li, const double* X) {
    double T[B * B];
    // T = X Li
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) {
            double s = 0.0;
SP_UNROLL
            for (int k = j; k < B; ++k) s = fma(X[i * B + k], Li[k * B + j], s);
            T[i * B + j] = s;
        }
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j <= i; ++j) {
            double s = 0.0;
SP_UNROLL
            for (int k = i; k < B; ++k) s = fma(Li[k * B + i], T[k * B + j], s);
            C[i * B + j] = s;
            C[j * B + i] = s;
        }
}
// C = Li^T Li = (L L^T)^{-1}
template <int B>
SP_DEVM void ltl(double* C, const double* Li) {
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j <= i; ++j) {
            double s = 0.0;
SP_UNROLL
            for (int k = i; k < B; ++k) s = fma(Li[k * B + i], Li[k * B + j], s);
            C[i * B + j] = s;
            C[j * B + i] = s;
        }
}

// Triangular solves with the inverted-pivot Cholesky factor L (lower):
// forward L X = A, backward L^T X = A.
template <int B>
SP_DEVM void lsolve(double* X, const double* L, const double* A, int ncol = B) {
SP_UNROLL
    for (int c = 0; c < B; ++c) {
        if (c >= ncol) break;
SP_UNROLL
        for (int i = 0; i < B; ++i) {
            double s = A[i * B + c];
SP_UNROLL
            for (int k = 0; k < i; ++k) s = fma(-L[i * B + k], X[k * B + c], s);
            X[i * B + c] = s * L[i * B + i];
        }
    }
}
template <int B>
SP_DEVM void lsolve_v(double* x, const double* L, const double* a) {
SP_UNROLL
    for (int i = 0; i < B; ++i) {
        double s = a[i];
SP_UNROLL
        for (int k = 0; k < i; ++k) s = fma(-L[i * B + k], x[k], s);
        x[i] = s * L[i * B + i];
    }
}
template <int B>
SP_DEVM void ltsolve(double* X, const double* L, const double* A) {
SP_UNROLL
    for (int c = 0; c < B; ++c)
SP_UNROLL
        for (int i = B - 1; i >= 0; --i) {
            double s = A[i * B + c];
SP_UNROLL
            for (int k = i + 1; k < B; ++k) s = fma(-L[k * B + i], X[k * B + c], s);
            X[i * B + c] = s * L[i * B + i];
        }
}
template <int B>
SP_DEVM void ltsolve_v(double* x, const double* L, const double* a) {
SP_UNROLL
    for (int i = B - 1; i >= 0; --i) {
        double s = a[i];
SP_UNROLL
        for (int k = i + 1; k < B; ++k) s = fma(-L[k * B + i], x[k], s);
        x[i] = s * L[i * B + i];
    }
}

}  // namespace spingp_dev
