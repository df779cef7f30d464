// engine.cuh — partitioned block-tridiagonal elimination on the B200.
//
// What it replaces.  SPEC.md btd_core factorize/solve/logdet/selective_inverse/
// cr_solve (:143-205) and spingp_engine assemble/add_observation_term/
// log_marginal_likelihood/mll_gradient/predict (:262-306).  The reference design
// is a sequential block Thomas recursion over all N blocks; here the N blocks are
// cut into chunks and reduced hierarchically (the SPEC's "cyclic reduction"
// contract, generalised from 2 to m blocks per chunk):
//
//   level 0   one thread per chunk of m0 consecutive time points.  It discretises
//             every step in closed form, assembles D_i, U_i, rhs_i on the fly
//             (never materialising the SymBTD), and eliminates the chunk's
//             interior blocks in forward order against its two separators: the
//             previous chunk's last block (L, carried as a "spike" W) and its own
//             last block (R).  Output: a 2-separator Schur record per chunk.
//   level l   the records form a BTD of one block per chunk; it is reduced the
//             same way (one thread per chunk of m_l blocks) until one block is left.
//   top       the single remaining block is inverted.
//   reverse   levels are walked back down: every chunk back-substitutes its
//             interior mean and runs the Takahashi recursion,
//             seeded by its separators' mean, variance and cross-covariance.  At
//             level 0 the same sweep recomputes each step's Φ, Q̃ and their
//             θ-derivatives and accumulates the stationary-form log-likelihood
//             terms, the per-step gradient and the per-point mean/variance.
//
// Elimination with a left spike (chunk interior j = s .. e-2, separators L, R):
//   S_j = D_j - T_j,  G_j = S_j^{-1} U_j,  V_j = S_j^{-1} W_j,  h_j = S_j^{-1} r_j
//   T_{j+1} = U_j^T G_j,  W_{j+1} = -U_j^T V_j,  r_{j+1} = rhs_{j+1} - U_j^T h_j
//   acc_LL -= W_j^T V_j,  acc_rL -= W_j^T h_j,   logdet += log det S_j
// Back substitution / selected inverse (x_j = h_j - V_j x_L - G_j x_{j+1} + ε_j,
// Cov ε_j = S_j^{-1}):
//   C_{jL} = -V_j C_LL - G_j C_{j+1,L}
//   C_{j,j+1} = -V_j C_{L,j+1} - G_j C_{j+1,j+1}
//   C_jj = S_j^{-1} - C_{jL} V_j^T - C_{j,j+1} G_j^T
#pragma once

#include <cstdint>

// Minimum resident CTAs (of 128 threads) per SM requested for the level-0 kernels:
// caps their registers at 65536 / (128 * minB).  Tuned on B200 (profiles/).
#ifndef SP_FWD0_MINB
#define SP_FWD0_MINB 3
#endif
#ifndef SP_REV0_MINB
#define SP_REV0_MINB 1
#endif

#include "devmat.cuh"
#include "model_dev.cuh"
#ifndef SPINGP_HOST_EMU
#include <cooperative_groups.h>
#endif

namespace spingp_dev {

// status word: min over every failure seen on the device of
//   (priority << 60) | (index << 4) | code,
// priority 0 for invalid input (bad value, duplicate time) so that it is reported
// ahead of the numerical failures it may cause, 1 for numerical failures.
enum DevStatus {
    ST_NOT_PD = 1, ST_SINGULAR_Q = 2, ST_BAD_ARG = 3, ST_DUPLICATE = 6, ST_NEG_VAR = 8
};

SP_DEV void report(unsigned long long* st, long long idx, int code) {
    const unsigned long long prio = (code == ST_BAD_ARG || code == ST_DUPLICATE) ? 0ULL : 1ULL;
    atomicMin(st, (prio << 60) | (static_cast<unsigned long long>(idx) << 4) |
                      static_cast<unsigned long long>(code));
}

// A failure that may only be the echo of an earlier one (a pivot that is NaN because its
// inputs already were): priority 2, reported only if nothing else was.
SP_DEV void report_echo(unsigned long long* st, long long idx, int code) {
    atomicMin(st, (2ULL << 60) | (static_cast<unsigned long long>(idx) << 4) | static_cast<unsigned long long>(code));
}

// level-l block k -> level-0 block index (the separator chain)
SP_DEV long long to_global(const Geom& g, int lev, long long k) {
    for (int l = lev; l > 0; --l) {
        const long long e = min(g.n[l - 1], (k + 1) * static_cast<long long>(g.m[l - 1]));
        k = e - 1;
    }
    return k;
}

// record layout, component-major: rec[comp * SK + chunk]
template <int B>
struct Rec {
    static constexpr int RDIAG = 0;
    static constexpr int LDIAG = B * B;
    static constexpr int LR = 2 * B * B;
    static constexpr int RRHS = 3 * B * B;
    static constexpr int LRHS = 3 * B * B + B;
    static constexpr int LOGDET = 3 * B * B + 2 * B;
    static constexpr int N = 3 * B * B + 2 * B + 1;
};
// per-step factor layout: fac[(jj * NF + comp) * SK + chunk]
//   LI: the Cholesky factor L_j of S_j, packed lower (row-major),
//   Y: L_j^{-1} W_j, Z: L_j^{-1} r_j  (triangular solves, never explicit inverses)
template <int B>
struct Fac {
    static constexpr int NLI = B * (B + 1) / 2;
    static constexpr int LI = 0;
    static constexpr int Y = NLI;
    static constexpr int Z = NLI + B * B;
    static constexpr int N = NLI + B * B + B;
};
// solution layout at level >= 1: sol[comp * Sn + block]
template <int B>
struct Sol {
    static constexpr int X = 0;
    static constexpr int CD = B;
    static constexpr int CU = B + B * B;
    static constexpr int N = B + 2 * B * B;
};
// level-0 per-chunk partial sums: part[comp * SK + chunk]
enum Part { P_LOGDET = 0, P_FITY = 1, P_FITE = 2, P_LDQ = 3, P_NOISE = 4, P_GRAD = 5 };

template <int B>
struct ElimState {
    double T[B * B];    // carried Schur update X^T X for the next block
    double rc[B];       // carried rhs update X^T z
    double W[B * B];    // coupling of the current block with the left separator
    double accLL[B * B];
    double accrL[B];
    double logdet;   // log-dets carried in from child records (upper levels)
    LogDetAcc piv;   // this chunk's own pivots
    SP_DEV double total_logdet() const { return logdet + piv.logdet(); }
};

template <int B>
SP_DEV void elim_init(ElimState<B>& es) {
    mzero<B>(es.T);
    vzero<B>(es.rc);
    mzero<B>(es.W);
    mzero<B>(es.accLL);
    vzero<B>(es.accrL);
    es.logdet = 0.0;
    es.piv.init();
}

// Eliminate one interior block j with diagonal D, coupling U (to j+1) and rhs.
// With S = D - T = L L^T:  X = L^{-1} U, Y = L^{-1} W, z = L^{-1} r (forward solves).
// Schur updates in Gram form (symmetric PSD by construction):
//   T' = X^T X,  rc' = X^T z,  W' = -X^T Y,  accLL -= Y^T Y,  accrL -= Y^T z.
// Stores L (packed), Y and z at fp[comp * SK] for the reverse sweep.
template <int B>
SP_DEV bool elim_block(ElimState<B>& es, const double* D, const double* U, const double* rhs,
                       bool hasL, double* fp, long long SK) {
    double S[B * B];
SP_UNROLL
    for (int i = 0; i < B * B; ++i) S[i] = D[i] - es.T[i];
    msym<B>(S);  // pivot symmetrisation
    double L[B * B];
    if (!chol<B>(L, S, es.piv)) return false;
    double r[B], z[B];
SP_UNROLL
    for (int i = 0; i < B; ++i) r[i] = rhs[i] - es.rc[i];
    lsolve_v<B>(z, L, r);
    double X[B * B];
    lsolve<B>(X, L, U);
    if (hasL) {
        double Y[B * B], G[B * B];
        lsolve<B>(Y, L, es.W);
        mtm_sym<B>(G, Y, Y);
SP_UNROLL
        for (int i = 0; i < B * B; ++i) es.accLL[i] -= G[i];
        double yz[B];
        mtv<B>(yz, Y, z);
SP_UNROLL
        for (int i = 0; i < B; ++i) es.accrL[i] -= yz[i];
        mtm<B>(G, X, Y);
SP_UNROLL
        for (int i = 0; i < B * B; ++i) es.W[i] = -G[i];
SP_UNROLL
        for (int i = 0; i < B * B; ++i) fp[(Fac<B>::Y + i) * SK] = Y[i];
    }
    mtm_sym<B>(es.T, X, X);
    mtv<B>(es.rc, X, z);
    int q = 0;
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j <= i; ++j) fp[(Fac<B>::LI + q++) * SK] = L[i * B + j];
SP_UNROLL
    for (int i = 0; i < B; ++i) fp[(Fac<B>::Z + i) * SK] = z[i];
    return true;
}

template <int B>
SP_DEV void write_rec(double* rec, long long SK, long long g, const ElimState<B>& es,
                      const double* Rdiag, const double* Rrhs, bool hasL) {
    double* r = rec + g;
SP_UNROLL
    for (int i = 0; i < B * B; ++i) r[(Rec<B>::RDIAG + i) * SK] = Rdiag[i];
SP_UNROLL
    for (int i = 0; i < B * B; ++i) r[(Rec<B>::LDIAG + i) * SK] = es.accLL[i];
    // coupling (L, R) of the reduced system = (P'_{R,L})^T = W^T
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) r[(Rec<B>::LR + i * B + j) * SK] = hasL ? es.W[j * B + i] : 0.0;
SP_UNROLL
    for (int i = 0; i < B; ++i) r[(Rec<B>::RRHS + i) * SK] = Rrhs[i];
SP_UNROLL
    for (int i = 0; i < B; ++i) r[(Rec<B>::LRHS + i) * SK] = es.accrL[i];
    r[Rec<B>::LOGDET * SK] = es.total_logdet();
}

// Q̃ = Q + jit I = L_Q L_Q^T  ->  L_Q (and log det Q̃).
template <int B>
SP_DEV bool qt_factor(const double* Q, double jit, int breal, double* L, LogDetAcc* ldq) {
    double Qt[B * B];
SP_UNROLL
    for (int i = 0; i < B * B; ++i) Qt[i] = Q[i];
SP_UNROLL
    for (int i = 0; i < B; ++i)
        if (i < breal) Qt[i * B + i] += jit;
    bool ok;
    if (ldq) ok = chol<B>(L, Qt, *ldq);
    else ok = chol_nolog<B>(L, Qt);
    return ok;
}

// Q̃^{-1} from its Cholesky factor by substitution (as the oracle's chol_solve(L, I)).
template <int B>
SP_DEV void chol_inv_solve(double* Qinv, const double* L) {
    double I[B * B], X[B * B];
SP_UNROLL
    for (int i = 0; i < B * B; ++i) I[i] = (i % (B + 1) == 0) ? 1.0 : 0.0;
    lsolve<B>(X, L, I);
    ltsolve<B>(Qinv, L, X);
    msym<B>(Qinv);
}

// Assembly pieces from one step: with Z = L_Q^{-1} Φ (forward solve),
//   Φ^T Q̃^{-1} Φ = Z^T Z  and  U = -Φ^T Q̃^{-1} = -(L_Q^{-T} Z)^T.
template <int B>
SP_DEV void step_assembly(const double* Phi, const double* LQ, double* PQP, double* U) {
    double Z[B * B], W[B * B];
    lsolve<B>(Z, LQ, Phi);
    mtm_sym<B>(PQP, Z, Z);
    ltsolve<B>(W, LQ, Z);
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) U[i * B + j] = -W[j * B + i];
}

// ======================================================= level 0 (fused) ======

template <class T>
__global__ void __launch_bounds__(128, SP_FWD0_MINB) k_fwd0(ModelDesc md, const double* __restrict__ params,
                                              const double* __restrict__ t,
                                              const double* __restrict__ y, Geom geo,
                                              double* __restrict__ fac, double* __restrict__ rec,
                                              double* __restrict__ part,
                                              unsigned long long* status,
                                              const double* __restrict__ halo, long long g0, long long g1,
                                              const unsigned char* __restrict__ obs) {
    // chunks [g0, g1) of the S * K level-0 chunks (host-input pipelining launches pieces)
    constexpr int B = T::B;
    const long long K = geo.K[0], SK = K * geo.S;
    const long long g = g0 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (g >= g1) return;
    const int s = static_cast<int>(g / K);
    const long long c = g - s * K;
    const long long n = geo.n[0];
    const int m = geo.m[0];
    const long long st = c * m, en = min(n, st + m);
    const double* ts = t + s * n;
    const double* ys = y + s * n;
    const double* rp = params + static_cast<long long>(s) * md.rec_stride;
    const double sig = rp[0], jit = rp[1], is2 = 1.0 / (sig * sig);
    const long long gbase = static_cast<long long>(s) * n;
    const bool hasL = c > 0 || geo.segL;

    double Phi[B * B], Q[B * B], Mq[B * B];
    double dt = -1.0;
    if (st > 0 || geo.segL) {
        dt = ts[st] - (st > 0 ? ts[st - 1] : halo[2 * s]);
        if (!(dt > 0.0) || !isfinite(dt)) {
            report(status, gbase + st, dt == 0.0 ? ST_DUPLICATE : ST_BAD_ARG);
            return;
        }
    }
    T::step(md, rp, dt, Phi, Q);
    if (!qt_factor<B>(Q, jit, md.b, Mq, nullptr)) {
        report(status, gbase + st, ST_SINGULAR_Q);
        return;
    }
    double Qinv[B * B];  // Q̃_j^{-1} of the current block
    chol_inv_solve<B>(Qinv, Mq);
    ElimState<B> es;
    elim_init<B>(es);
    if (hasL) {  // P_{s, s-1} = U_{s-1}^T
        double PQP[B * B], U[B * B];
        step_assembly<B>(Phi, Mq, PQP, U);
SP_UNROLL
        for (int i = 0; i < B; ++i)
SP_UNROLL
            for (int j = 0; j < B; ++j) es.W[i * B + j] = U[j * B + i];
    }
    double HH[B * B];
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) HH[i * B + j] = T::H(md, i) * T::H(md, j) * is2;

    for (long long j = st; j < en - 1; ++j) {
        if (m >= 32 && j + 2 < en) {  // long chunks: next step's inputs, while this one computes
            prefetch_l1(ts + j + 2);
            prefetch_l1(ys + j + 1);
        }
        const double dtn = ts[j + 1] - ts[j];
        if (!(dtn > 0.0) || !isfinite(dtn)) {
            report(status, gbase + j + 1, dtn == 0.0 ? ST_DUPLICATE : ST_BAD_ARG);
            return;
        }
        double Phn[B * B], Qn[B * B], Mqn[B * B];
        T::step(md, rp, dtn, Phn, Qn);
        if (!qt_factor<B>(Qn, jit, md.b, Mqn, nullptr)) {
            report(status, gbase + j + 1, ST_SINGULAR_Q);
            return;
        }
        double D[B * B], U[B * B], r[B];
        step_assembly<B>(Phn, Mqn, D, U);
        // observation mask (predict at test times): a test point
        // has no observation term (Σ'^{-1} = 0 there)
        const double wo = (!obs || obs[gbase + j]) ? 1.0 : 0.0;
SP_UNROLL
        for (int i = 0; i < B * B; ++i) D[i] += Qinv[i] + wo * HH[i];
        const double yj = wo != 0.0 ? ys[j] : 0.0;
        if (!isfinite(yj)) {
            report(status, gbase + j, ST_BAD_ARG);
            return;
        }
SP_UNROLL
        for (int i = 0; i < B; ++i) r[i] = T::H(md, i) * yj * is2;
        double* fp = fac + (j - st) * Fac<B>::N * SK + g;
        if (!elim_block<B>(es, D, U, r, hasL, fp, SK)) {
            report(status, gbase + j, ST_NOT_PD);
            return;
        }
        chol_inv_solve<B>(Qinv, Mqn);
    }
    // separator R = en - 1
    double D[B * B], Rr[B];
    const double woR = (!obs || obs[gbase + en - 1]) ? 1.0 : 0.0;
SP_UNROLL
    for (int i = 0; i < B * B; ++i) D[i] = Qinv[i] + woR * HH[i];
    if (en < n || geo.segR) {
        const double dte = (en < n ? ts[en] : halo[2 * s + 1]) - ts[en - 1];
        if (!(dte > 0.0) || !isfinite(dte)) {
            report(status, gbase + en, dte == 0.0 ? ST_DUPLICATE : ST_BAD_ARG);
            return;
        }
        double Phn[B * B], Qn[B * B], Mqn[B * B], PQP[B * B], U[B * B];
        T::step(md, rp, dte, Phn, Qn);
        if (!qt_factor<B>(Qn, jit, md.b, Mqn, nullptr)) {
            report(status, gbase + en, ST_SINGULAR_Q);
            return;
        }
        step_assembly<B>(Phn, Mqn, PQP, U);
SP_UNROLL
        for (int i = 0; i < B * B; ++i) D[i] += PQP[i];
    }
    const double yR = woR != 0.0 ? ys[en - 1] : 0.0;
    if (!isfinite(yR)) {
        report(status, gbase + en - 1, ST_BAD_ARG);
        return;
    }
SP_UNROLL
    for (int i = 0; i < B * B; ++i) D[i] -= es.T[i];
SP_UNROLL
    for (int i = 0; i < B; ++i) Rr[i] = T::H(md, i) * yR * is2 - es.rc[i];
    write_rec<B>(rec, SK, g, es, D, Rr, hasL);
    part[P_LOGDET * SK + g] = es.total_logdet();
}

// ============================================= materialised / upper levels ====
// Block source for level l >= 1: the records of level l-1 chunks.
template <int B>
struct RecSource {
    const double* rec;  // level l-1 records
    long long SKp;      // S * K[l-1]
    long long n;        // blocks per series at this level (= K[l-1])
    SP_DEV void block(int s, long long k, double* D, double* U, double* r, bool wantU) const {
        const long long i0 = static_cast<long long>(s) * n + k;
        const bool nx = k + 1 < n;
SP_UNROLL
        for (int q = 0; q < B * B; ++q)
            D[q] = rec[(Rec<B>::RDIAG + q) * SKp + i0] + (nx ? rec[(Rec<B>::LDIAG + q) * SKp + i0 + 1] : 0.0);
SP_UNROLL
        for (int q = 0; q < B; ++q)
            r[q] = rec[(Rec<B>::RRHS + q) * SKp + i0] + (nx ? rec[(Rec<B>::LRHS + q) * SKp + i0 + 1] : 0.0);
        if (wantU) upper(s, k, U);
    }
    // upper block (k, k+1)
    SP_DEV void upper(int s, long long k, double* U) const {
        const long long i1 = static_cast<long long>(s) * n + k + 1;
SP_UNROLL
        for (int q = 0; q < B * B; ++q) U[q] = rec[(Rec<B>::LR + q) * SKp + i1];
    }
    // cumulative log-determinant carried by child record k
    SP_DEV double child_logdet(int s, long long k) const {
        return rec[Rec<B>::LOGDET * SKp + static_cast<long long>(s) * n + k];
    }
    // segment mode: what block 0's record contributes to the segment's left separator
    SP_DEV void left_contrib(int s, double* D, double* r) const {
        const long long i0 = static_cast<long long>(s) * n;
SP_UNROLL
        for (int q = 0; q < B * B; ++q) D[q] = rec[(Rec<B>::LDIAG + q) * SKp + i0];
SP_UNROLL
        for (int q = 0; q < B; ++q) r[q] = rec[(Rec<B>::LRHS + q) * SKp + i0];
    }
};

// Block source for a user SymBTD (row-major diag[n][b][b], upper[n-1][b][b],
// rhs[n][b] column `col` of k), padded from b to B with identity blocks.
template <int B>
struct UserSource {
    const double* diag;
    const double* up;
    const double* rhs;
    long long n;
    int b, k, col;
    SP_DEV void block(int, long long i, double* D, double* U, double* r, bool wantU) const {
SP_UNROLL
        for (int p = 0; p < B; ++p)
SP_UNROLL
            for (int q = 0; q < B; ++q)
                D[p * B + q] = (p < b && q < b) ? diag[(i * b + p) * b + q] : (p == q ? 1.0 : 0.0);
SP_UNROLL
        for (int p = 0; p < B; ++p) r[p] = (p < b && rhs) ? rhs[(i * b + p) * k + col] : 0.0;
        if (wantU) upper(0, i, U);
    }
    SP_DEV void upper(int, long long i, double* U) const {
SP_UNROLL
        for (int p = 0; p < B; ++p)
SP_UNROLL
            for (int q = 0; q < B; ++q) U[p * B + q] = (p < b && q < b) ? up[(i * b + p) * b + q] : 0.0;
    }
    SP_DEV double child_logdet(int, long long) const { return 0.0; }
    SP_DEV void left_contrib(int, double* D, double* r) const {
        mzero<B>(D);
        vzero<B>(r);
    }
};

// One chunk of level `lev` (global chunk index g = series * K + chunk).  The record's
// LOGDET is cumulative: this chunk's own pivots plus the LOGDET of every child record
// it absorbs, so the last level carries the whole log-determinant (no level scans).
template <int B, class Src>
SP_DEV void fwdL_item(const Src& src, const Geom& geo, int lev, double* __restrict__ fac,
                      double* __restrict__ rec, unsigned long long* status, long long g) {
    const long long K = geo.K[lev], SK = K * geo.S;
    const int s = static_cast<int>(g / K);
    const long long c = g - s * K;
    const long long n = geo.n[lev];
    const int m = geo.m[lev];
    const long long st = c * m, en = min(n, st + m);
    const bool hasL = c > 0 || geo.segL;
    const long long gbase = static_cast<long long>(s) * geo.n[0];
    ElimState<B> es;
    elim_init<B>(es);
    if (c == 0 && geo.segL) src.left_contrib(s, es.accLL, es.accrL);  // carried to the segment's L
    if (hasL) {  // P_{st, st-1} = upper(st-1)^T
        double U[B * B];
        src.upper(s, st - 1, U);
SP_UNROLL
        for (int i = 0; i < B; ++i)
SP_UNROLL
            for (int j = 0; j < B; ++j) es.W[i * B + j] = U[j * B + i];
    }
    // software-pipelined: the next block's (L2-resident) record is loaded while the
    // current block is eliminated — the upper levels are latency-bound chains
    double D[B * B], U[B * B], r[B];
    if (st < en - 1) src.block(s, st, D, U, r, true);
    for (long long j = st; j < en - 1; ++j) {
        double Dn[B * B], Un[B * B], rn[B];
        if (j + 1 < en - 1) src.block(s, j + 1, Dn, Un, rn, true);
        double* fp = fac + (j - st) * Fac<B>::N * SK + g;
        if (!elim_block<B>(es, D, U, r, hasL, fp, SK)) {
            report(status, gbase + to_global(geo, lev, j), ST_NOT_PD);
            return;
        }
        mcopy<B>(D, Dn);
        mcopy<B>(U, Un);
SP_UNROLL
        for (int q = 0; q < B; ++q) r[q] = rn[q];
    }
    src.block(s, en - 1, D, U, r, false);
SP_UNROLL
    for (int i = 0; i < B * B; ++i) D[i] -= es.T[i];
SP_UNROLL
    for (int i = 0; i < B; ++i) r[i] -= es.rc[i];
    for (long long j = st; j < en; ++j) es.logdet += src.child_logdet(s, j);
    write_rec<B>(rec, SK, g, es, D, r, hasL);
}
template <int B, class Src>
__global__ void __launch_bounds__(128) k_fwdL(Src src, Geom geo, int lev, double* __restrict__ fac,
                                              double* __restrict__ rec, unsigned long long* status) {
    const long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (g >= geo.K[lev] * geo.S) return;
    fwdL_item<B, Src>(src, geo, lev, fac, rec, status, g);
}

// The single block left per series: invert it.  toplogdet = log det of the whole
// precision (this pivot + the cumulative LOGDET of the last record).
template <int B>
SP_DEV void top_item(const Geom& geo, const double* __restrict__ rec, double* __restrict__ sol,
                     double* __restrict__ toplogdet, unsigned long long* status, int s) {
    const int L = geo.nlev;
    const long long SK = geo.S;  // K = 1 at the last level
    double D[B * B], r[B], Lc[B * B], Li[B * B], C[B * B], x[B], z[B], ld;
SP_UNROLL
    for (int q = 0; q < B * B; ++q) D[q] = rec[(Rec<B>::RDIAG + q) * SK + s];
SP_UNROLL
    for (int q = 0; q < B; ++q) r[q] = rec[(Rec<B>::RRHS + q) * SK + s];
    msym<B>(D);
    if (!chol<B>(Lc, D, ld)) {
        report(status, static_cast<long long>(s) * geo.n[0] + to_global(geo, L, 0), ST_NOT_PD);
        return;
    }
    chol_inv_solve<B>(C, Lc);
    lsolve_v<B>(z, Lc, r);
    ltsolve_v<B>(x, Lc, z);
    (void)Li;
    const long long Sn = geo.S;
SP_UNROLL
    for (int q = 0; q < B; ++q) sol[(Sol<B>::X + q) * Sn + s] = x[q];
SP_UNROLL
    for (int q = 0; q < B * B; ++q) sol[(Sol<B>::CD + q) * Sn + s] = C[q];
    toplogdet[s] = ld + rec[Rec<B>::LOGDET * SK + s];
}
template <int B>
__global__ void k_top(Geom geo, const double* __restrict__ rec, double* __restrict__ sol,
                      double* __restrict__ toplogdet, unsigned long long* status) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= geo.S) return;
    top_item<B>(geo, rec, sol, toplogdet, status, s);
}

// Separator data of chunk c from the level above.
template <int B>
struct SepData {
    double xR[B], CRR[B * B], xL[B], CLL[B * B], CLR[B * B];
};
template <int B>
SP_DEV void load_sep(const double* solU, long long SnU, long long iR, bool hasL, bool needC,
                     SepData<B>& sd) {
SP_UNROLL
    for (int q = 0; q < B; ++q) sd.xR[q] = solU[(Sol<B>::X + q) * SnU + iR];
    if (needC) {
SP_UNROLL
        for (int q = 0; q < B * B; ++q) sd.CRR[q] = solU[(Sol<B>::CD + q) * SnU + iR];
    } else {
        mzero<B>(sd.CRR);
    }
    if (hasL) {
SP_UNROLL
        for (int q = 0; q < B; ++q) sd.xL[q] = solU[(Sol<B>::X + q) * SnU + iR - 1];
        if (needC) {
SP_UNROLL
            for (int q = 0; q < B * B; ++q) sd.CLL[q] = solU[(Sol<B>::CD + q) * SnU + iR - 1];
SP_UNROLL
            for (int q = 0; q < B * B; ++q) sd.CLR[q] = solU[(Sol<B>::CU + q) * SnU + iR - 1];
            return;
        }
    } else {
        vzero<B>(sd.xL);
    }
    mzero<B>(sd.CLL);
    mzero<B>(sd.CLR);
}

// One step of the reverse sweep (all L^{-1}, L^{-T} by substitution).  With
// x_j = L^{-T}(z - X x_n - Y x_L) + ε_j,  Cov ε_j = S_j^{-1} = L^{-T} L^{-1}:
//   P1 = X C_nL + Y C_LL,   C_jL = -L^{-T} P1
//   P2 = X C_nn + Y C_Ln,   C_jn = -L^{-T} P2
//   C_jj = L^{-T} (I + P2 X^T + P1 Y^T) L^{-1}
template <int B>
SP_DEV void back_step(const double* L, const double* Y, const double* z, const double* X,
                      bool hasL, bool needC, const SepData<B>& sd, const double* xn,
                      const double* Cnn, const double* CnL, double* xj, double* CjL, double* Cjn,
                      double* Cjj) {
    double a[B], tmp[B];
    mv<B>(tmp, X, xn);
SP_UNROLL
    for (int i = 0; i < B; ++i) a[i] = z[i] - tmp[i];
    if (hasL) {
        mv<B>(tmp, Y, sd.xL);
SP_UNROLL
        for (int i = 0; i < B; ++i) a[i] -= tmp[i];
    }
    ltsolve_v<B>(xj, L, a);
    if (!needC) return;
    double P1[B * B], P2[B * B], M[B * B], N[B * B];
    mm<B>(P1, X, CnL);
    mm<B>(P2, X, Cnn);
    if (hasL) {
        mm<B>(M, Y, sd.CLL);
SP_UNROLL
        for (int i = 0; i < B * B; ++i) P1[i] += M[i];
        mmt<B>(M, Y, CnL);  // Y C_{L,n} = Y C_{n,L}^T
SP_UNROLL
        for (int i = 0; i < B * B; ++i) P2[i] += M[i];
    }
    ltsolve<B>(CjL, L, P1);
    ltsolve<B>(Cjn, L, P2);
SP_UNROLL
    for (int i = 0; i < B * B; ++i) {
        CjL[i] = -CjL[i];
        Cjn[i] = -Cjn[i];
    }
    mmt<B>(M, P2, X);
    if (hasL) {
        mmt<B>(N, P1, Y);
SP_UNROLL
        for (int i = 0; i < B * B; ++i) M[i] += N[i];
    }
SP_UNROLL
    for (int i = 0; i < B; ++i) M[i * B + i] += 1.0;
    msym<B>(M);
    // Cjj = L^{-T} M L^{-1} = L^{-T} (L^{-T} M)^T
    ltsolve<B>(N, L, M);
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < i; ++j) {
            const double tmp2 = N[i * B + j];
            N[i * B + j] = N[j * B + i];
            N[j * B + i] = tmp2;
        }
    ltsolve<B>(Cjj, L, N);
    msym<B>(Cjj);
}

template <int B>
SP_DEV void load_fac(const double* fp, long long SK, bool hasL, double* Li, double* Y, double* z) {
    int q = 0;  // Li receives the packed Cholesky factor L_j
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) Li[i * B + j] = j <= i ? fp[(Fac<B>::LI + q++) * SK] : 0.0;
    if (hasL)
SP_UNROLL
        for (int i = 0; i < B * B; ++i) Y[i] = fp[(Fac<B>::Y + i) * SK];
SP_UNROLL
    for (int i = 0; i < B; ++i) z[i] = fp[(Fac<B>::Z + i) * SK];
}

// Solution sinks for the reverse sweep of levels >= 1.
template <int B>
struct SolSink {  // component-major sol of this level (segment mode: slot -1 = left separator)
    double* sol;
    long long Sn;  // S * (n + segL)
    long long n;
    int segL;
    SP_DEV void put(int s, long long i, const double* x, const double* Cd, bool needC) const {
        const long long k = static_cast<long long>(s) * (n + segL) + segL + i;
SP_UNROLL
        for (int q = 0; q < B; ++q) sol[(Sol<B>::X + q) * Sn + k] = x[q];
        if (needC)
SP_UNROLL
            for (int q = 0; q < B * B; ++q) sol[(Sol<B>::CD + q) * Sn + k] = Cd[q];
    }
    SP_DEV void put_upper(int s, long long i, const double* Cu) const {
        const long long k = static_cast<long long>(s) * (n + segL) + segL + i;
SP_UNROLL
        for (int q = 0; q < B * B; ++q) sol[(Sol<B>::CU + q) * Sn + k] = Cu[q];
    }
};
template <int B>
struct UserSink {  // row-major user outputs (b <= B), any may be null
    double* x;
    double* cdiag;
    double* cupper;
    int b, k, col;
    SP_DEV void put(int, long long i, const double* xv, const double* Cd, bool needC) const {
        if (x)
            for (int p = 0; p < b; ++p) x[(i * b + p) * k + col] = xv[p];
        if (needC && cdiag)
            for (int p = 0; p < b; ++p)
                for (int q = 0; q < b; ++q) cdiag[(i * b + p) * b + q] = Cd[p * B + q];
    }
    SP_DEV void put_upper(int, long long i, const double* Cu) const {
        if (cupper)
            for (int p = 0; p < b; ++p)
                for (int q = 0; q < b; ++q) cupper[(i * b + p) * b + q] = Cu[p * B + q];
    }
};

template <int B, class Src, class Sink>
SP_DEV void revL_item(const Src& src, const Sink& sink, const Geom& geo, int lev, const double* __restrict__ fac,
                      const double* __restrict__ solU, int needC, long long g) {
    const long long K = geo.K[lev], SK = K * geo.S;
    const int s = static_cast<int>(g / K);
    const long long c = g - s * K;
    const long long n = geo.n[lev];
    const int m = geo.m[lev];
    const long long st = c * m, en = min(n, st + m);
    const bool hasL = c > 0 || geo.segL;
    SepData<B> sd;
    load_sep<B>(solU, static_cast<long long>(geo.S) * (geo.n[lev + 1] + geo.segL), g + geo.segL * (s + 1), hasL,
                needC, sd);
    double xn[B], Cnn[B * B], CnL[B * B];
SP_UNROLL
    for (int q = 0; q < B; ++q) xn[q] = sd.xR[q];
    mcopy<B>(Cnn, sd.CRR);
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) CnL[i * B + j] = sd.CLR[j * B + i];
    sink.put(s, en - 1, xn, Cnn, needC);
    if (c == 0 && geo.segL) sink.put(s, -1, sd.xL, sd.CLL, needC);  // propagate the left separator
    double Li[B * B], Y[B * B], z[B], U[B * B];
    if (en - 2 >= st) {
        load_fac<B>(fac + (en - 2 - st) * Fac<B>::N * SK + g, SK, hasL, Li, Y, z);
        src.upper(s, en - 2, U);
    }
    for (long long j = en - 2; j >= st; --j) {
        double X[B * B], Lin[B * B], Yn[B * B], zn[B], Un[B * B];
        if (j - 1 >= st) {  // prefetch the next (lower) block of the reverse sweep
            load_fac<B>(fac + (j - 1 - st) * Fac<B>::N * SK + g, SK, hasL, Lin, Yn, zn);
            src.upper(s, j - 1, Un);
        }
        lsolve<B>(X, Li, U);
        double xj[B], CjL[B * B], Cjn[B * B], Cjj[B * B];
        back_step<B>(Li, Y, z, X, hasL, needC, sd, xn, Cnn, CnL, xj, CjL, Cjn, Cjj);
        sink.put(s, j, xj, Cjj, needC);
        if (needC) sink.put_upper(s, j, Cjn);
SP_UNROLL
        for (int q = 0; q < B; ++q) xn[q] = xj[q];
        if (needC) {
            mcopy<B>(Cnn, Cjj);
            mcopy<B>(CnL, CjL);
        }
        if (j - 1 >= st) {
            mcopy<B>(Li, Lin);
            if (hasL) mcopy<B>(Y, Yn);
            mcopy<B>(U, Un);
SP_UNROLL
            for (int q = 0; q < B; ++q) z[q] = zn[q];
        }
    }
    if (hasL && needC) {  // C_{st-1, st} = C_{st, L}^T
        double X[B * B];
SP_UNROLL
        for (int i = 0; i < B; ++i)
SP_UNROLL
            for (int j = 0; j < B; ++j) X[i * B + j] = CnL[j * B + i];
        sink.put_upper(s, st - 1, X);
    }
}
template <int B, class Src, class Sink>
__global__ void __launch_bounds__(128) k_revL(Src src, Sink sink, Geom geo, int lev,
                                              const double* __restrict__ fac,
                                              const double* __restrict__ solU, int needC) {
    const long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (g >= geo.K[lev] * geo.S) return;
    revL_item<B, Src, Sink>(src, sink, geo, lev, fac, solU, needC, g);
}

// ================================================ fused upper levels (1 launch) ==
// All levels >= 1 in one persistent cooperative kernel: forward levels 1..nlev-1,
// the top inverse, reverse levels nlev-1..1, a grid-wide barrier between phases.
// The per-level work items are exactly those of k_fwdL / k_top / k_revL; what goes
// away is 2(nlev-1)+1 launches of latency-bound chains (the upper
// levels hold ~1/37888 of the points but cost ~35% of the step as separate kernels).
#ifndef SPINGP_HOST_EMU
struct UpperArgs {
    double* rec[kMaxLev];
    double* fac[kMaxLev];
    double* sol[kMaxLev + 1];
    double* toplogdet;
    unsigned long long* status;
    int needC, do_fwd, do_top, do_rev;
    unsigned long long* stamps;  // diagnostics: %globaltimer after every phase (null = off)
};
SP_DEV void upper_stamp(const UpperArgs& a, int& k) {
    if (a.stamps && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.stamps[k] = t;
    }
    ++k;
}
template <int B>
__global__ void __launch_bounds__(128) k_upper(Geom geo, UpperArgs a) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    const long long tid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long nth = static_cast<long long>(gridDim.x) * blockDim.x;
    int ks = 0;
    upper_stamp(a, ks);
    if (a.do_fwd) {
        for (int l = 1; l < geo.nlev; ++l) {
            const RecSource<B> src{a.rec[l - 1], geo.K[l - 1] * geo.S, geo.n[l]};
            const long long SK = geo.K[l] * geo.S;
            for (long long g = tid; g < SK; g += nth) fwdL_item<B, RecSource<B>>(src, geo, l, a.fac[l], a.rec[l], a.status, g);
            grid.sync();
            upper_stamp(a, ks);
        }
    }
    if (a.do_top) {
        for (long long s = tid; s < geo.S; s += nth)
            top_item<B>(geo, a.rec[geo.nlev - 1], a.sol[geo.nlev], a.toplogdet, a.status, static_cast<int>(s));
        grid.sync();
        upper_stamp(a, ks);
    }
    if (a.do_rev) {
        for (int l = geo.nlev - 1; l >= 1; --l) {
            const RecSource<B> src{a.rec[l - 1], geo.K[l - 1] * geo.S, geo.n[l]};
            const SolSink<B> sink{a.sol[l], (geo.n[l] + geo.segL) * geo.S, geo.n[l], geo.segL};
            const long long SK = geo.K[l] * geo.S;
            for (long long g = tid; g < SK; g += nth)
                revL_item<B, RecSource<B>, SolSink<B>>(src, sink, geo, l, a.fac[l], a.sol[l + 1], a.needC, g);
            if (l > 1) grid.sync();
            upper_stamp(a, ks);
        }
    }
}
#endif

// ============================================ level-0 reverse (fused outputs) ==

struct Outs {
    double* mean;
    double* var;
    int include_noise;
    int want_grad;
    int need_c;
};

template <class T>
SP_DEV void point_out(const ModelDesc& md, const Outs& o, long long gi, double yv, double is2,
                      double sig, const double* x, const double* C, double& fy, double& noise,
                      unsigned long long* status, bool ob = true) {
    constexpr int B = T::B;
    double mu = 0.0;
SP_UNROLL
    for (int k = 0; k < B; ++k) mu += T::H(md, k) * x[k];
    const double r = yv - mu;
    if (ob) fy += r * r * is2;
    if (o.mean) o.mean[gi] = mu;
    if (o.need_c) {
        double v = 0.0;
SP_UNROLL
        for (int a = 0; a < B; ++a)
SP_UNROLL
            for (int b2 = 0; b2 < B; ++b2) v += T::H(md, a) * C[a * B + b2] * T::H(md, b2);
        if (ob) noise += r * r + v;
        if (o.var) {
            if (v < -1e-10) report(status, gi, ST_NEG_VAR);
            if (v < 0.0) v = 0.0;  // clamp [-1e-10, 0) -> 0
            o.var[gi] = o.include_noise ? v + sig * sig : v;
        }
    }
}

// Likelihood / gradient terms of step i with transition Φ
// (Φ := 0 at the anchor), L_Q = chol(Q̃), previous block (xp, Cpp) and
// cross-covariance Cpc = C_{i-1,i}:
//   ē = x_c - Φ x_p,  fe += |L_Q^{-1} ē|²
//   E = C_cc - Φ C_pc - (Φ C_pc)^T + Φ C_pp Φ^T + ē ē^T
//   Zc = C_pc - C_pp Φ^T + x_p ē^T
//   M = Q̃^{-1}(E - Q̃)Q̃^{-1},  Bm = Zc Q̃^{-1};  T::grad adds ½Tr(M dQ̃) + Tr(dΦ Bm).
// Every Q̃^{-1} is applied by forward/backward substitution with L_Q.
template <int B>
SP_DEV void qinv_apply_right(double* out, const double* LQ, const double* A) {  // out = A Q̃^{-1}
    double At[B * B], X[B * B], Y[B * B];
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) At[i * B + j] = A[j * B + i];
    lsolve<B>(X, LQ, At);
    ltsolve<B>(Y, LQ, X);  // Q̃^{-1} A^T
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) out[i * B + j] = Y[j * B + i];
}

template <class T>
SP_DEV void step_terms(const ModelDesc& md, const double* rp, double dt, const double* Phi,
                       const double* Qraw, const double* LQ, const double* xc, const double* Ccc,
                       const double* xp, const double* Cpp, const double* Cpc, bool anchor,
                       bool grad, double& fe, double* g) {
    constexpr int B = T::B;
    double e[B], tmp[B];
    if (anchor) {
SP_UNROLL
        for (int i = 0; i < B; ++i) e[i] = xc[i];
    } else {
        mv<B>(tmp, Phi, xp);
SP_UNROLL
        for (int i = 0; i < B; ++i) e[i] = xc[i] - tmp[i];
    }
    lsolve_v<B>(tmp, LQ, e);
    double q = 0.0;
SP_UNROLL
    for (int i = 0; i < B; ++i) q += tmp[i] * tmp[i];
    fe += q;
    if (!grad) return;
    const double jit = rp[1];
    double E[B * B], Bm[B * B], X[B * B], Y[B * B];
    if (anchor) {
SP_UNROLL
        for (int i = 0; i < B; ++i)
SP_UNROLL
            for (int j = 0; j < B; ++j) E[i * B + j] = Ccc[i * B + j] + e[i] * e[j];
        mzero<B>(Bm);
    } else {
        double Z[B * B];
        mm<B>(X, Phi, Cpc);
        mm<B>(Y, Phi, Cpp);
        mmt<B>(Z, Y, Phi);
SP_UNROLL
        for (int i = 0; i < B; ++i)
SP_UNROLL
            for (int j = 0; j < B; ++j)
                E[i * B + j] = Ccc[i * B + j] - X[i * B + j] - X[j * B + i] + Z[i * B + j] + e[i] * e[j];
        // C_pp Φ^T = (Φ C_pp)^T exactly (C_pp is symmetrised): transpose instead of a product
SP_UNROLL
        for (int i = 0; i < B; ++i)
SP_UNROLL
            for (int j = 0; j < i; ++j) {
                const double t2 = Y[i * B + j];
                Y[i * B + j] = Y[j * B + i];
                Y[j * B + i] = t2;
            }
SP_UNROLL
        for (int i = 0; i < B; ++i)
SP_UNROLL
            for (int j = 0; j < B; ++j) Z[i * B + j] = Cpc[i * B + j] - Y[i * B + j] + xp[i] * e[j];
        qinv_apply_right<B>(Bm, LQ, Z);
    }
    // E - Q̃ (padding states have Q̃ = 1 and E = 0; their rows of M are never read)
SP_UNROLL
    for (int i = 0; i < B * B; ++i) E[i] -= Qraw[i];
SP_UNROLL
    for (int i = 0; i < B; ++i)
        if (i < md.b) E[i * B + i] -= jit;
    msym<B>(E);
    // M = Q̃^{-1} (E - Q̃) Q̃^{-1}
    lsolve<B>(X, LQ, E);
    ltsolve<B>(Y, LQ, X);         // Q̃^{-1}(E - Q̃)
    qinv_apply_right<B>(X, LQ, Y);
    msym<B>(X);
    T::grad(md, rp, dt, Phi, Qraw, X, Bm, g);
}

template <class T>
__global__ void __launch_bounds__(128, SP_REV0_MINB) k_rev0(ModelDesc md, const double* __restrict__ params,
                                              const double* __restrict__ t,
                                              const double* __restrict__ y, Geom geo,
                                              const double* __restrict__ fac,
                                              const double* __restrict__ solU,
                                              double* __restrict__ part, Outs outs,
                                              unsigned long long* status,
                                              const double* __restrict__ halo, long long g0, long long g1,
                                              const unsigned char* __restrict__ obs) {
    // chunks [g0, g1) of the S * K level-0 chunks (host-input pipelining launches pieces)
    constexpr int B = T::B;
    const long long K = geo.K[0], SK = K * geo.S;
    const long long g = g0 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (g >= g1) return;
    const int s = static_cast<int>(g / K);
    const long long c = g - s * K;
    const long long n = geo.n[0];
    const int m = geo.m[0];
    const long long st = c * m, en = min(n, st + m);
    const double* ts = t + s * n;
    const double* ys = y + s * n;
    const double* rp = params + static_cast<long long>(s) * md.rec_stride;
    const double sig = rp[0], jit = rp[1], is2 = 1.0 / (sig * sig);
    const long long gbase = static_cast<long long>(s) * n;
    const bool hasL = c > 0 || geo.segL;
    const bool needC = outs.need_c != 0, grad = outs.want_grad != 0;

    SepData<B> sd;
    load_sep<B>(solU, static_cast<long long>(geo.S) * (geo.n[1] + geo.segL), g + geo.segL * (s + 1), hasL, needC,
                sd);
    double xn[B], Cnn[B * B], CnL[B * B];
SP_UNROLL
    for (int q = 0; q < B; ++q) xn[q] = sd.xR[q];
    mcopy<B>(Cnn, sd.CRR);
SP_UNROLL
    for (int i = 0; i < B; ++i)
SP_UNROLL
        for (int j = 0; j < B; ++j) CnL[i * B + j] = sd.CLR[j * B + i];

    double fy = 0.0, fe = 0.0, noise = 0.0;
    LogDetAcc ldq;  // log det of every Q̃ of the chunk
    ldq.init();
    double gr[kMaxTheta];
    for (int p = 0; p < md.nt; ++p) gr[p] = 0.0;

    for (long long j = en - 2; j >= st; --j) {
        const long long nb = j + 1;
        if (m >= 32 && j - 1 >= st) {  // long chunks: the next (lower) step's time and value
            // (prefetching its 18-component factor as well measured slower at b = 3:
            // the 255-register kernel starts to spill)
            prefetch_l1(ts + j - 1);
            prefetch_l1(ys + j - 1);
        }
        const double dt = ts[nb] - ts[j];
        double Phn[B * B], Qn[B * B], Mqn[B * B];
        T::step(md, rp, dt, Phn, Qn);
        qt_factor<B>(Qn, jit, md.b, Mqn, &ldq);
        double Li[B * B], Y[B * B], z[B], U[B * B], X[B * B], PQP[B * B];
        load_fac<B>(fac + (j - st) * Fac<B>::N * SK + g, SK, hasL, Li, Y, z);
        step_assembly<B>(Phn, Mqn, PQP, U);
        lsolve<B>(X, Li, U);
        double xj[B], CjL[B * B], Cjn[B * B], Cjj[B * B];
        back_step<B>(Li, Y, z, X, hasL, needC, sd, xn, Cnn, CnL, xj, CjL, Cjn, Cjj);
        const bool obn = !obs || obs[gbase + nb];
        point_out<T>(md, outs, gbase + nb, obn ? ys[nb] : 0.0, is2, sig, xn, Cnn, fy, noise, status, obn);
        step_terms<T>(md, rp, dt, Phn, Qn, Mqn, xn, Cnn, xj, Cjj, Cjn, false, grad, fe, gr);
SP_UNROLL
        for (int q = 0; q < B; ++q) xn[q] = xj[q];
        if (needC) {
            mcopy<B>(Cnn, Cjj);
            mcopy<B>(CnL, CjL);
        }
    }
    // block st: previous block is the left separator (or the anchor at st = 0)
    const bool obs0 = !obs || obs[gbase + st];
    point_out<T>(md, outs, gbase + st, obs0 ? ys[st] : 0.0, is2, sig, xn, Cnn, fy, noise, status, obs0);
    {
        const bool anchor = st == 0 && !geo.segL;
        const double dt = anchor ? -1.0 : ts[st] - (st > 0 ? ts[st - 1] : halo[2 * s]);
        double Ph[B * B], Qr[B * B], Mq[B * B];
        T::step(md, rp, dt, Ph, Qr);
        qt_factor<B>(Qr, jit, md.b, Mq, &ldq);
        double CLs[B * B];  // C_{L, st} = C_{st, L}^T
SP_UNROLL
        for (int i = 0; i < B; ++i)
SP_UNROLL
            for (int j = 0; j < B; ++j) CLs[i * B + j] = CnL[j * B + i];
        step_terms<T>(md, rp, dt, Ph, Qr, Mq, xn, Cnn, sd.xL, sd.CLL, CLs, anchor, grad, fe, gr);
    }
    part[P_FITY * SK + g] = fy;
    part[P_FITE * SK + g] = fe;
    part[P_LDQ * SK + g] = ldq.logdet();
    part[P_NOISE * SK + g] = noise;
    for (int p = 0; p < md.nt; ++p) part[(P_GRAD + p) * SK + g] = gr[p];
}

// ================================================================ reductions ==

// One launch, two fixed-order stages (bit-reproducible):
//   stage 1  block (seg, s) sums chunks [seg*kSeg, (seg+1)*kSeg) of series s for every
//            partial component: warp w takes components w, w+8, ...; lane l sums
//            chunks l, l+32, ... in order, then a fixed shuffle tree -> seg[s][seg][comp];
//   stage 2  the last block of series s to arrive (per-series counter, self-resetting)
//            sums seg[s][0..nseg) the same way and writes loglik / gradient (or, in
//            segment mode, the raw partial sums).
// The log-determinant of the whole precision is toplogdet[s] (cumulative records).
constexpr int kSeg = 256;  // chunks per stage-1 block (cfg2: 280 blocks)
constexpr int kRedThreads = 256;
constexpr int kMaxNC = P_GRAD + kMaxTheta;

struct FinalArgs {
    const double* part;    // [NC][S*K] level-0 per-chunk partial sums
    long long K;           // chunks per series
    long long S;           // series (grid = nseg * S blocks on x: no 65535 cap on S)
    int NC;
    double* seg;           // [S][nseg][NC] scratch
    unsigned int* arrive;  // [S] zero-initialised counters
    const double* toplogdet;
    const double* params;
    int rec_stride, nt;
    long long n;
    double* loglik;        // [S]
    double* grad;          // [S][nt+1] or null
    double* partials;      // segment mode: raw sums (logdetP, fit_y, fit_e, logdetQ, noise, grad...)
};

SP_DEV double warp_sum(double v) {
#ifndef SPINGP_HOST_EMU
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
#endif
    return v;
}

#ifndef SPINGP_HOST_EMU
static __global__ void __launch_bounds__(kRedThreads) k_reduce(FinalArgs a) {
    __shared__ double acc[kMaxNC];
    __shared__ int last;
    const int nseg = static_cast<int>((a.K + kSeg - 1) / kSeg);
    const int s = static_cast<int>(blockIdx.x / nseg), sg = static_cast<int>(blockIdx.x % nseg);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long SK = a.K * a.S;
    const long long base = static_cast<long long>(s) * a.K + static_cast<long long>(sg) * kSeg;
    const int lim = static_cast<int>(min(static_cast<long long>(kSeg), a.K - static_cast<long long>(sg) * kSeg));
    for (int c = warp; c < a.NC; c += kRedThreads / 32) {
        const double* p = a.part + c * SK + base;
        double v = 0.0;
#pragma unroll 8
        for (int k = lane; k < lim; k += 32) v += p[k];
        v = warp_sum(v);
        if (lane == 0) a.seg[(static_cast<long long>(s) * nseg + sg) * a.NC + c] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&a.arrive[s], 1u) == static_cast<unsigned>(nseg - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int c = warp; c < a.NC; c += kRedThreads / 32) {
        double v = 0.0;
#pragma unroll 8
        for (int k = lane; k < nseg; k += 32) v += __ldcg(a.seg + (static_cast<long long>(s) * nseg + k) * a.NC + c);
        v = warp_sum(v);
        if (lane == 0) acc[c] = v;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    a.arrive[s] = 0u;  // ready for the next launch (stream-ordered)
    const double ldP = a.toplogdet[s];
    if (a.partials) {
        for (int c = 0; c < a.NC; ++c) a.partials[c] = acc[c];
        a.partials[P_LOGDET] = ldP;
        return;
    }
    const double* rp = a.params + static_cast<long long>(s) * a.rec_stride;
    const double sig = rp[0], s2 = sig * sig;
    const double nn = static_cast<double>(a.n);
    const double kLog2Pi = 1.8378770664093454835606594728112;
    a.loglik[s] = -0.5 * (acc[P_FITY] + acc[P_FITE]) - 0.5 * (ldP + acc[P_LDQ] + nn * log(s2)) - 0.5 * nn * kLog2Pi;
    if (a.grad) {
        double* gs = a.grad + static_cast<long long>(s) * (a.nt + 1);
        for (int p = 0; p < a.nt; ++p) gs[p] = acc[P_GRAD + p];
        gs[a.nt] = 2.0 * sig * (-0.5 * nn / s2 + acc[P_NOISE] / (2.0 * s2 * s2));
    }
}
#endif

// ===================================================== multi-GPU reduced system ==
// Segment mode: rank r has reduced its time segment to a 2-separator record
// (left separator = rank r-1's last block, right = its own last block).  Every rank
// solves the P-block BTD of the ranks' last blocks redundantly (P <= a few dozen),
// then keeps x and the selected-inverse blocks it needs for its reverse sweep:
//   sol slot 0 (segL only) = (x_{r-1}, C_{r-1,r-1}), Cu slot 0 = C_{r-1,r}; next slot = (x_r, C_rr).
// recs: P records, each Rec<B>::N contiguous doubles (the K = 1 top-level record).
// scratch: P x (2 B^2 + B) doubles of global memory for the per-block factor (kept out of
// per-thread local arrays: large dynamically indexed local arrays were miscompiled by nvcc
// 12.9 for sm_100a elsewhere in this code).
template <int B>
__global__ void k_seg_solve(int P, int rank, const double* __restrict__ recs, double* __restrict__ sol,
                            double* __restrict__ toplogdet, unsigned long long* status, long long gidx,
                            double* __restrict__ scratch) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    constexpr int NR = Rec<B>::N;
    double S_L[B * B], T[B * B], rc[B];
    auto Ls = [&](int r) { return scratch + static_cast<long long>(r) * (2 * B * B + B); };
    auto Xs = [&](int r) { return scratch + static_cast<long long>(r) * (2 * B * B + B) + B * B; };
    auto Zs = [&](int r) { return scratch + static_cast<long long>(r) * (2 * B * B + B) + 2 * B * B; };
    mzero<B>(T);
    vzero<B>(rc);
    double ld = 0.0;
    for (int r = 0; r < P; ++r) {
        const double* R0 = recs + static_cast<long long>(r) * NR;
        const double* R1 = recs + static_cast<long long>(r + 1) * NR;
        double D[B * B], U[B * B], rhs[B];
        for (int q = 0; q < B * B; ++q)
            D[q] = R0[Rec<B>::RDIAG + q] + (r + 1 < P ? R1[Rec<B>::LDIAG + q] : 0.0) - T[q];
        for (int q = 0; q < B; ++q) rhs[q] = R0[Rec<B>::RRHS + q] + (r + 1 < P ? R1[Rec<B>::LRHS + q] : 0.0) - rc[q];
        msym<B>(D);
        double ldr;
        if (!chol<B>(S_L, D, ldr)) {
            report(status, gidx, ST_NOT_PD);
            return;
        }
        ld += ldr;
        mcopy<B>(Ls(r), S_L);
        double z[B];
        lsolve_v<B>(z, S_L, rhs);
        for (int q = 0; q < B; ++q) Zs(r)[q] = z[q];
        if (r + 1 < P) {
            double X[B * B];
            for (int q = 0; q < B * B; ++q) U[q] = R1[Rec<B>::LR + q];
            lsolve<B>(X, S_L, U);
            mcopy<B>(Xs(r), X);
            mtm_sym<B>(T, X, X);
            mtv<B>(rc, X, z);
        }
    }
    // back substitution + Takahashi down to block rank-1
    double xn[B], Cnn[B * B], xj[B], Cjn[B * B], Cjj[B * B];
    {
        double Lq[B * B], z[B];
        mcopy<B>(Lq, Ls(P - 1));
        for (int q = 0; q < B; ++q) z[q] = Zs(P - 1)[q];
        ltsolve_v<B>(xn, Lq, z);
        chol_inv_solve<B>(Cnn, Lq);
    }
    const int lo = rank > 0 ? rank - 1 : rank;
    double xr[B], Crr[B * B], xl[B], Cll[B * B], Clr[B * B];
    if (P - 1 == rank) {
        for (int q = 0; q < B; ++q) xr[q] = xn[q];
        mcopy<B>(Crr, Cnn);
    }
    for (int j = P - 2; j >= lo; --j) {
        SepData<B> none;
        vzero<B>(none.xL);
        mzero<B>(none.CLL);
        mzero<B>(none.CLR);
        double Y0[B * B], CnL0[B * B], CjL0[B * B];
        mzero<B>(Y0);
        mzero<B>(CnL0);
        double Lj[B * B], Xj[B * B], zj[B];
        mcopy<B>(Lj, Ls(j));
        mcopy<B>(Xj, Xs(j));
        for (int q = 0; q < B; ++q) zj[q] = Zs(j)[q];
        back_step<B>(Lj, Y0, zj, Xj, false, true, none, xn, Cnn, CnL0, xj, CjL0, Cjn, Cjj);
        if (j == rank) {
            for (int q = 0; q < B; ++q) xr[q] = xj[q];
            mcopy<B>(Crr, Cjj);
        }
        if (j == rank - 1) {
            for (int q = 0; q < B; ++q) xl[q] = xj[q];
            mcopy<B>(Cll, Cjj);
            mcopy<B>(Clr, Cjn);
        }
        for (int q = 0; q < B; ++q) xn[q] = xj[q];
        mcopy<B>(Cnn, Cjj);
    }
    const int segL = rank > 0 ? 1 : 0;
    const long long Sn = 1 + segL;
    if (segL) {
        for (int q = 0; q < B; ++q) sol[(Sol<B>::X + q) * Sn + 0] = xl[q];
        for (int q = 0; q < B * B; ++q) sol[(Sol<B>::CD + q) * Sn + 0] = Cll[q];
        for (int q = 0; q < B * B; ++q) sol[(Sol<B>::CU + q) * Sn + 0] = Clr[q];
    }
    for (int q = 0; q < B; ++q) sol[(Sol<B>::X + q) * Sn + segL] = xr[q];
    for (int q = 0; q < B * B; ++q) sol[(Sol<B>::CD + q) * Sn + segL] = Crr[q];
    // this rank's segment log-det (cumulative record) + the reduced system's (rank 0 only)
    toplogdet[0] = (rank == 0 ? ld : 0.0) + recs[static_cast<long long>(rank) * NR + Rec<B>::LOGDET];
}

// After the all-reduce of the ranks' partial sums: loglik and gradient.
struct SegFinalArgs {
    const double* sums;  // [P_GRAD + nt]: (logdetP, fit_y, fit_e, logdetQ, noise, grad...)
    int nt;
    long long n;         // total points over all ranks
    double sigma;
    double* loglik;
    double* grad;
};
static __global__ void k_seg_final(SegFinalArgs a) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double s2 = a.sigma * a.sigma, nn = static_cast<double>(a.n);
    const double kLog2Pi = 1.8378770664093454835606594728112;
    a.loglik[0] = -0.5 * (a.sums[P_FITY] + a.sums[P_FITE]) -
                  0.5 * (a.sums[P_LOGDET] + a.sums[P_LDQ] + nn * log(s2)) - 0.5 * nn * kLog2Pi;
    if (a.grad) {
        for (int p = 0; p < a.nt; ++p) a.grad[p] = a.sums[P_GRAD + p];
        a.grad[a.nt] = 2.0 * a.sigma * (-0.5 * nn / s2 + a.sums[P_NOISE] / (2.0 * s2 * s2));
    }
}

// y = M v for a user SymBTD (one thread per block row).
static __global__ void k_matvec(long long n, int b, const double* __restrict__ diag,
                         const double* __restrict__ up, const double* __restrict__ v,
                         double* __restrict__ out) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    for (int p = 0; p < b; ++p) {
        double s = 0.0;
        for (int q = 0; q < b; ++q) s += diag[(i * b + p) * b + q] * v[i * b + q];
        if (i + 1 < n)
            for (int q = 0; q < b; ++q) s += up[(i * b + p) * b + q] * v[(i + 1) * b + q];
        if (i > 0)
            for (int q = 0; q < b; ++q) s += up[((i - 1) * b + q) * b + p] * v[(i - 1) * b + q];
        out[i * b + p] = s;
    }
}

// assemble_prior_precision + add_observation_term: one thread per
// time point writes D_i, U_i (b_real x b_real) and rhs_i.
template <class T>
__global__ void __launch_bounds__(128) k_assemble(ModelDesc md, const double* __restrict__ params,
                                                  const double* __restrict__ t,
                                                  const double* __restrict__ y, long long n,
                                                  double* __restrict__ diag, double* __restrict__ up,
                                                  double* __restrict__ rhs, unsigned long long* status) {
    constexpr int B = T::B;
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double sig = params[0], jit = params[1], is2 = 1.0 / (sig * sig);
    const int b = md.b;
    double Phi[B * B], Q[B * B], Mq[B * B], D[B * B];
    const double dt = i == 0 ? -1.0 : t[i] - t[i - 1];
    if (i > 0 && (!(dt > 0.0) || !isfinite(dt))) {
        report(status, i, dt == 0.0 ? ST_DUPLICATE : ST_BAD_ARG);
        return;
    }
    T::step(md, params, dt, Phi, Q);
    if (!qt_factor<B>(Q, jit, b, Mq, nullptr)) {
        report(status, i, ST_SINGULAR_Q);
        return;
    }
    chol_inv_solve<B>(D, Mq);
    if (i + 1 < n) {
        const double dtn = t[i + 1] - t[i];
        if (!(dtn > 0.0) || !isfinite(dtn)) {
            report(status, i + 1, dtn == 0.0 ? ST_DUPLICATE : ST_BAD_ARG);
            return;
        }
        double Phn[B * B], Qn[B * B], Mqn[B * B], PQP[B * B], U[B * B];
        T::step(md, params, dtn, Phn, Qn);
        if (!qt_factor<B>(Qn, jit, b, Mqn, nullptr)) {
            report(status, i + 1, ST_SINGULAR_Q);
            return;
        }
        step_assembly<B>(Phn, Mqn, PQP, U);
        for (int q = 0; q < B * B; ++q) D[q] += PQP[q];
        for (int p = 0; p < b; ++p)
            for (int q = 0; q < b; ++q) up[(i * b + p) * b + q] = U[p * B + q];
    }
    for (int p = 0; p < b; ++p)
        for (int q = 0; q < b; ++q)
            diag[(i * b + p) * b + q] = D[p * B + q] + T::H(md, p) * T::H(md, q) * is2;
    if (rhs)
        for (int p = 0; p < b; ++p) rhs[i * b + p] = T::H(md, p) * y[i] * is2;
}

}  // namespace spingp_dev
