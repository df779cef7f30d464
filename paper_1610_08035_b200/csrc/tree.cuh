// tree.cuh — levels >= 1 of the hierarchical elimination as CTA-wide binary trees in
// shared memory (the eval path's replacement for the per-thread record chains of
// k_fwdL / k_revL and the cooperative k_upper).
//
// Why.  Above level 0 there are ~7.6e4 records per GPU; the work is tiny but it is a
// chain: with one thread per 4 records every level costs an L2 round trip per record
// plus a grid-wide barrier, ~10 us a level on B200 (profiles/r01_summary.md: 137 us
// for the 15 upper phases of cfg2, 40% of the step).  Here a CTA owns a *group* of up
// to G(B) consecutive records of one series (G = 512 at b = 3, model_desc.h), stages
// them into shared memory with cp.async and reduces them pairwise: ceil(log2 G) merge
// rounds separated by __syncthreads, no HBM/L2 traffic between rounds.  A level with
// one group per series (always the last) also does the top inverse and the whole
// reverse tree in the same CTA (k_tree_one).
//
// Records (Rec<B>) are 2-separator Schur complements in "split" form: RDIAG / RRHS are
// what the record contributes to its right separator R, LDIAG / LRHS to its left
// separator L, LR is the (L, R) block, LOGDET is cumulative.  The neighbour's
// contribution to a separator is added only when the separator is eliminated, so a
// group depends on nothing outside itself (the level-0 records already have this
// form, engine.cuh write_rec; it is also the segment record of SPEC.md:197-205).
//
// Merge of A = (L, M) and B = (M, R), eliminating M:
//   S = A.RR + B.LL = L_S L_S^T,  r = A.rR + B.rL,
//   Y_L = L_S^{-1} A.LR^T,  Y_R = L_S^{-1} B.LR,  z = L_S^{-1} r
//   C.LL = A.LL - Y_L^T Y_L,  C.RR = B.RR - Y_R^T Y_R,  C.LR = -Y_L^T Y_R,
//   C.rL = A.rL - Y_L^T z,    C.rR = B.rR - Y_R^T z,   C.logdet = A + B + log det S.
// Reverse (selected inverse, SURVEY.md App. B / SPEC.md:170-187): with the node's outer
// separators known (x_L, x_R, C_LL, C_RR, C_LR), engine.cuh back_step gives
//   x_M, C_MM, C_ML, C_MR;  C_{L,M} and C_{M,R} are the separators' "next" covariances
//   at the finer granularity.
//
// Shared-memory layout (bank-conflict free).  Level j of a group holds n_j =
// ceil(cnt / 2^j) records, compacted at slots [0, n_j) of a component-major area
// R[c * RS + slot]: round j -> j+1 merges slots (2k, 2k+1) into slot k (one 16-byte
// load per component per thread, contiguous across the warp) and parks the factor
// (L_S, Y_L, Y_R, z) at slot n_{j+1} + k, which no later round touches.  Separators
// at level j are the n_j + 1 record boundaries E_j[i] = original boundary i * 2^j,
// component-major E[q * ES + i]; the reverse round j+1 -> j expands E_{j+1} into E_j
// in place (E_j[2k] = E_{j+1}[k], E_j[2k+1] = the eliminated M).  Every round reads
// into registers, passes a barrier, then writes.
#pragma once

#include "engine.cuh"

namespace spingp_dev {

// Full unroll of the rectangular component loops below (scratch arrays stay in
// registers); devmat.cuh's triangular loops keep their own (empty) SP_UNROLL.
#ifdef SPINGP_HOST_EMU
#define TR_UNROLL
#else
#define TR_UNROLL _Pragma("unroll")
#endif

template <int B>
struct Tree {
    static constexpr int NR = Rec<B>::N;
    static constexpr int NF = 3 * B * B + B;          // merge factor: L_S, Y_L, Y_R, z
    static constexpr int FL = 0, FYL = B * B, FYR = 2 * B * B, FZ = 3 * B * B;
    static constexpr int NS = Sol<B>::N;              // separator: x, C_diag, C_next
    static constexpr int SX = Sol<B>::X, SCD = Sol<B>::CD, SCU = Sol<B>::CU;
    static_assert(NF <= NR, "merge factor must fit a record slot");
};
constexpr int kTreeMaxThreads = 256;

struct TreeArgs {
    const double* rec_in;  // level l-1 records, component-major, stride SKin
    long long SKin, nin;   // nin records per series
    double* rec_out;       // level l records, stride S * nG
    double* fac;           // merge factors, [S * nG][NF][G]
    const double* solU;    // separators of the level-l records (level above), stride S * (nG + segL)
    double* sol;           // separators of the level-(l-1) records, stride S * (nin + segL)
    double* toplogdet;     // [S] (k_tree_one)
    unsigned long long* status;
    int G, nG, S, segL, needC;
    int RS, ES;            // shared row lengths (records, separators): tree_row(gcap), tree_row(gcap + 1)
    long long span;        // level-0 records per input record (error reports)
    long long K0, n0;
    int m0;
    unsigned long long* stamps;  // diagnostics: %globaltimer per phase of CTA 0 (null = off)
};

struct TreeGroup {
    int s, j, cnt;
    long long k0, gidx;
    bool hasL;
};
SP_DEV TreeGroup tree_group(const TreeArgs& a, long long gidx) {
    TreeGroup t;
    t.gidx = gidx;
    t.s = static_cast<int>(gidx / a.nG);
    t.j = static_cast<int>(gidx - static_cast<long long>(t.s) * a.nG);
    t.k0 = static_cast<long long>(t.j) * a.G;
    t.cnt = static_cast<int>(min(static_cast<long long>(a.G), a.nin - t.k0));
    t.hasL = t.j > 0 || a.segL;
    return t;
}
// level-0 time index of the right separator of input record k of the group's series
SP_DEV long long tree_point(const TreeArgs& a, const TreeGroup& t, long long k) {
    const long long r0 = min(a.K0, (k + 1) * a.span);
    return static_cast<long long>(t.s) * a.n0 + min(a.n0, r0 * a.m0) - 1;
}
SP_DEV int tree_levels(int cnt) {  // merge rounds: ceil(log2 cnt)
    int J = 0;
    while ((1 << J) < cnt) ++J;
    return J;
}
SP_DEV int tree_width(int cnt, int j) { return (cnt + (1 << j) - 1) >> j; }  // n_j

// global -> shared, 8 bytes, asynchronous (cp.async; completes at tree_copy_wait)
SP_DEV void tree_copy(double* dst, const double* src) {
#ifdef SPINGP_HOST_EMU
    *dst = *src;
#else
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
#endif
}
SP_DEV void tree_copy_wait() {
#ifndef SPINGP_HOST_EMU
    asm volatile("cp.async.wait_all;\n" ::: "memory");
#endif
}

// ---------------------------------------------------------------- phases ----
// A phase is executed by every thread (tid < nt) of the CTA between two barriers; the
// host emulation (tests/emu) runs the same phases thread by thread.  Values carried
// across a barrier live in the thread's scratch struct (registers on the device).

template <int B>
SP_DEV void tree_load_recs(const TreeArgs& a, const TreeGroup& t, double* R, int tid, int nt) {
    using TR = Tree<B>;
    const double* src = a.rec_in + static_cast<long long>(t.s) * a.nin + t.k0;
    for (int c = 0; c < TR::NR; ++c)
        for (int i = tid; i < t.cnt; i += nt) tree_copy(R + c * a.RS + i, src + c * a.SKin + i);
    tree_copy_wait();
}

template <int B>
struct TreeFwdScratch {
    double C[Tree<B>::NR];
    double F[Tree<B>::NF];
    bool active, merged, ok;
};

// Merge of two adjacent records held in registers: A = (L, M), Bv = (M, R) -> C = (L, R)
// and the merge factor F = (L_S, Y_L, Y_R, z) of the eliminated separator M.
template <int B>
SP_DEV bool tree_merge(const double* A, const double* Bv, double* C, double* F) {
    using TR = Tree<B>;
    using RC = Rec<B>;
    double S[B * B], r[B], T1[B * B], v[B];
    double* Ls = F + TR::FL;
    double* YL = F + TR::FYL;
    double* YR = F + TR::FYR;
    double* z = F + TR::FZ;
TR_UNROLL
    for (int i = 0; i < B * B; ++i) S[i] = A[RC::RDIAG + i] + Bv[RC::LDIAG + i];
    msym<B>(S);
TR_UNROLL
    for (int i = 0; i < B; ++i) r[i] = A[RC::RRHS + i] + Bv[RC::LRHS + i];
    double ld;
    const bool ok = chol<B>(Ls, S, ld);
    lsolve_v<B>(z, Ls, r);
TR_UNROLL
    for (int i = 0; i < B; ++i)
TR_UNROLL
        for (int j = 0; j < B; ++j) T1[i * B + j] = A[RC::LR + j * B + i];  // P_{M,L} = A.LR^T
    lsolve<B>(YL, Ls, T1);
    lsolve<B>(YR, Ls, Bv + RC::LR);  // P_{M,R} = B.LR
    mtm_sym<B>(T1, YL, YL);
TR_UNROLL
    for (int i = 0; i < B * B; ++i) C[RC::LDIAG + i] = A[RC::LDIAG + i] - T1[i];
    mtm<B>(T1, YL, YR);
TR_UNROLL
    for (int i = 0; i < B * B; ++i) C[RC::LR + i] = -T1[i];
    mtm_sym<B>(T1, YR, YR);
TR_UNROLL
    for (int i = 0; i < B * B; ++i) C[RC::RDIAG + i] = Bv[RC::RDIAG + i] - T1[i];
    mtv<B>(v, YL, z);
TR_UNROLL
    for (int i = 0; i < B; ++i) C[RC::LRHS + i] = A[RC::LRHS + i] - v[i];
    mtv<B>(v, YR, z);
TR_UNROLL
    for (int i = 0; i < B; ++i) C[RC::RRHS + i] = Bv[RC::RRHS + i] - v[i];
    C[RC::LOGDET] = A[RC::LOGDET] + Bv[RC::LOGDET] + ld;
    return ok;
}

// round j -> j+1, compute part: node k (< n_{j+1}) merges slots 2k and 2k+1 of level j
template <int B>
SP_DEV void tree_fwd_compute(const double* R, int RS, int n, int k, TreeFwdScratch<B>& sc) {
    using TR = Tree<B>;
    const int nn = (n + 1) >> 1;
    sc.active = k < nn;
    sc.merged = sc.active && 2 * k + 1 < n;
    sc.ok = true;
    if (!sc.active) return;
    if (!sc.merged) {  // odd level width: the last record passes through
TR_UNROLL
        for (int c = 0; c < TR::NR; ++c) sc.C[c] = R[c * RS + 2 * k];
        return;
    }
    double A[TR::NR], Bv[TR::NR];
TR_UNROLL
    for (int c = 0; c < TR::NR; ++c) {
#ifdef SPINGP_HOST_EMU
        A[c] = R[c * RS + 2 * k];
        Bv[c] = R[c * RS + 2 * k + 1];
#else
        const double2 v = *reinterpret_cast<const double2*>(R + c * RS + 2 * k);
        A[c] = v.x;
        Bv[c] = v.y;
#endif
    }
    sc.ok = tree_merge<B>(A, Bv, sc.C, sc.F);
}
// store part (after the barrier): record -> slot k, factor -> slot n_{j+1} + k
template <int B>
SP_DEV void tree_fwd_store(double* R, int RS, int n, int k, const TreeFwdScratch<B>& sc) {
    using TR = Tree<B>;
    if (!sc.active) return;
    const int nn = (n + 1) >> 1;
TR_UNROLL
    for (int c = 0; c < TR::NR; ++c) R[c * RS + k] = sc.C[c];
    if (sc.merged)
TR_UNROLL
        for (int c = 0; c < TR::NF; ++c) R[c * RS + nn + k] = sc.F[c];
}

template <int B>
SP_DEV void tree_store_fwd(const TreeArgs& a, const TreeGroup& t, const double* R, int tid, int nt) {
    using TR = Tree<B>;
    const long long SKo = static_cast<long long>(a.S) * a.nG;
    for (int c = tid; c < TR::NR; c += nt) a.rec_out[c * SKo + t.gidx] = R[c * a.RS];
    double* f = a.fac + t.gidx * static_cast<long long>(TR::NF) * a.G;
    for (int c = 0; c < TR::NF; ++c)
        for (int i = 1 + tid; i < t.cnt; i += nt) f[c * a.G + i] = R[c * a.RS + i];
}

// reverse: factors of this group's merges + its two outer separators (level above)
// -> E_J = (L, R) at separator slots 0 and 1
template <int B>
SP_DEV void tree_load_rev(const TreeArgs& a, const TreeGroup& t, double* R, double* E, int tid, int nt) {
    using TR = Tree<B>;
    const double* f = a.fac + t.gidx * static_cast<long long>(TR::NF) * a.G;
    for (int c = 0; c < TR::NF; ++c)
        for (int i = 1 + tid; i < t.cnt; i += nt) tree_copy(R + c * a.RS + i, f + c * a.G + i);
    const long long SnU = static_cast<long long>(a.S) * (a.nG + a.segL);
    const long long u = static_cast<long long>(t.s) * (a.nG + a.segL) + a.segL + t.j;
    for (int q = tid; q < TR::NS; q += nt) {
        const bool want = q < B || a.needC;
        // R of the group: x, C_RR (its "next" covariance belongs to the next group)
        E[q * a.ES + 1] = (want && q < TR::SCU) ? a.solU[q * SnU + u] : 0.0;
        // L: x, C_LL and C_{L,R}
        E[q * a.ES] = (want && t.hasL) ? a.solU[q * SnU + u - 1] : 0.0;
    }
    tree_copy_wait();
}

// the single record left of a series (no left separator): invert it -> E_J
template <int B>
SP_DEV void tree_top(const TreeArgs& a, const TreeGroup& t, const double* R, double* E, bool write_ld = true) {
    using TR = Tree<B>;
    using RC = Rec<B>;
    double D[B * B], r[B], Lc[B * B], C[B * B], x[B], z[B], ld;
TR_UNROLL
    for (int q = 0; q < B * B; ++q) D[q] = R[(RC::RDIAG + q) * a.RS];
TR_UNROLL
    for (int q = 0; q < B; ++q) r[q] = R[(RC::RRHS + q) * a.RS];
    msym<B>(D);
    if (!chol<B>(Lc, D, ld) && a.status) report(a.status, tree_point(a, t, t.k0 + t.cnt - 1), ST_NOT_PD);
    chol_inv_solve<B>(C, Lc);
    lsolve_v<B>(z, Lc, r);
    ltsolve_v<B>(x, Lc, z);
    for (int q = 0; q < TR::NS; ++q) E[q * a.ES] = 0.0;
TR_UNROLL
    for (int q = 0; q < B; ++q) E[(TR::SX + q) * a.ES + 1] = x[q];
TR_UNROLL
    for (int q = 0; q < B * B; ++q) E[(TR::SCD + q) * a.ES + 1] = C[q];
TR_UNROLL
    for (int q = 0; q < B * B; ++q) E[(TR::SCU + q) * a.ES + 1] = 0.0;
    if (write_ld) a.toplogdet[t.s] = ld + R[RC::LOGDET * a.RS];
}

template <int B>
struct TreeRevScratch {
    double L[Sol<B>::N];   // E_{j+1}[k]: x, C_diag, C_next (C_next replaced by C_{L,M} if merged)
    double M[Sol<B>::N];   // the eliminated separator: x, C_diag, C_{M,R}
    double Rt[Sol<B>::N];  // the group's right boundary (last node only)
    bool active, merged, last;
};

// round j+1 -> j, compute part: node k of level j+1 (< n_{j+1}) with factor at slot
// n_{j+1} + k un-merges into level-j separators 2k (its L) and 2k + 1 (its M)
template <int B>
SP_DEV void tree_rev_compute(const double* R, const double* E, int RS, int ES, int n, int k, bool needC,
                             TreeRevScratch<B>& sc) {
    using TR = Tree<B>;
    const int nn = (n + 1) >> 1;
    sc.active = k < nn;
    sc.merged = sc.active && 2 * k + 1 < n;
    sc.last = k == nn - 1;
    if (!sc.active) return;
    const int nq = needC ? TR::NS : B;
TR_UNROLL
    for (int q = 0; q < TR::NS; ++q) sc.L[q] = q < nq ? E[q * ES + k] : 0.0;
    if (sc.last)
TR_UNROLL
        for (int q = 0; q < TR::NS; ++q) sc.Rt[q] = q < nq ? E[q * ES + k + 1] : 0.0;
    if (!sc.merged) return;
    double F[TR::NF];
TR_UNROLL
    for (int c = 0; c < TR::NF; ++c) F[c] = R[c * RS + nn + k];
    SepData<B> sd;
    double CRL[B * B];
TR_UNROLL
    for (int i = 0; i < B; ++i) {
        sd.xL[i] = sc.L[TR::SX + i];
        sd.xR[i] = E[(TR::SX + i) * ES + k + 1];
    }
    if (needC) {
TR_UNROLL
        for (int i = 0; i < B * B; ++i) {
            sd.CLL[i] = sc.L[TR::SCD + i];
            sd.CRR[i] = E[(TR::SCD + i) * ES + k + 1];
            sd.CLR[i] = sc.L[TR::SCU + i];
        }
TR_UNROLL
        for (int i = 0; i < B; ++i)
TR_UNROLL
            for (int j = 0; j < B; ++j) CRL[i * B + j] = sd.CLR[j * B + i];
    } else {
        mzero<B>(sd.CLL);
        mzero<B>(sd.CRR);
        mzero<B>(sd.CLR);
        mzero<B>(CRL);
    }
    double CML[B * B];
    back_step<B>(F + TR::FL, F + TR::FYL, F + TR::FZ, F + TR::FYR, true, needC, sd, sd.xR, sd.CRR, CRL,
                 sc.M + TR::SX, CML, sc.M + TR::SCU, sc.M + TR::SCD);
    if (!needC) return;
TR_UNROLL
    for (int i = 0; i < B; ++i)
TR_UNROLL
        for (int j = 0; j < B; ++j) sc.L[TR::SCU + i * B + j] = CML[j * B + i];  // C_{L,M}
}
// store part (after the barrier): E_j[2k] = L, E_j[2k+1] = M, E_j[n_j] = the right boundary
template <int B>
SP_DEV void tree_rev_store(double* E, int ES, int n, int k, bool needC, const TreeRevScratch<B>& sc) {
    using TR = Tree<B>;
    if (!sc.active) return;
    const int nq = needC ? TR::NS : B;
TR_UNROLL
    for (int q = 0; q < TR::NS; ++q) {
        if (q >= nq) break;
        if (sc.merged) {
#ifdef SPINGP_HOST_EMU
            E[q * ES + 2 * k] = sc.L[q];
            E[q * ES + 2 * k + 1] = sc.M[q];
#else
            *reinterpret_cast<double2*>(E + q * ES + 2 * k) = make_double2(sc.L[q], sc.M[q]);
#endif
        } else {
            E[q * ES + 2 * k] = sc.L[q];
        }
        if (sc.last) E[q * ES + n] = sc.Rt[q];
    }
}

// E_0 slot i (1..cnt) is the right separator of input record k0 + i - 1
template <int B>
SP_DEV void tree_store_rev(const TreeArgs& a, const TreeGroup& t, const double* E, int tid, int nt) {
    using TR = Tree<B>;
    const long long Sn = static_cast<long long>(a.S) * (a.nin + a.segL);
    const long long base = static_cast<long long>(t.s) * (a.nin + a.segL) + a.segL + t.k0 - 1;  // + slot
    const int nq = a.needC ? TR::NS : B;
    for (int q = 0; q < nq; ++q) {
        const int hi = q < TR::SCU ? t.cnt : t.cnt - 1;  // C_{R, next} is the next group's
        for (int i = 1 + tid; i <= hi; i += nt) a.sol[q * Sn + base + i] = E[q * a.ES + i];
    }
    if (t.hasL) {  // slot 0: C_{L, first} (and, for a segment's first group, L itself)
        const int q0 = (t.j == 0) ? 0 : TR::SCU;
        for (int q = q0 + tid; q < nq; q += nt) a.sol[q * Sn + base] = E[q * a.ES];
    }
}

#ifndef SPINGP_HOST_EMU
SP_DEV void tree_stamp(const TreeArgs& a, int& k) {
    if (a.stamps && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.stamps[k] = t;
    }
    ++k;
}
template <int B>
SP_DEV void tree_forward_rounds(double* R, int RS, const TreeArgs& a, const TreeGroup& t, int& ks) {
    const int J = tree_levels(t.cnt);
    for (int j = 0; j < J; ++j) {
        const int n = tree_width(t.cnt, j);
        TreeFwdScratch<B> sc;
        tree_fwd_compute<B>(R, RS, n, threadIdx.x, sc);
        if (!sc.ok && a.status) {
            // the origin of the failure if the merged pivot A.RR + B.LL is finite, else the echo of
            // an earlier one (a NaN child record): reported at a lower priority
            const int k2 = 2 * static_cast<int>(threadIdx.x);
            double acc = 0.0;
TR_UNROLL
            for (int i = 0; i < B * B; ++i)
                acc += R[(Rec<B>::RDIAG + i) * RS + k2] + R[(Rec<B>::LDIAG + i) * RS + k2 + 1];
            const long long idx = tree_point(a, t, t.k0 + min(t.cnt, (k2 + 1) << j) - 1);
            if (isfinite(acc)) report(a.status, idx, ST_NOT_PD);
            else report_echo(a.status, idx, ST_NOT_PD);
        }
        __syncthreads();
        tree_fwd_store<B>(R, RS, n, threadIdx.x, sc);
        __syncthreads();
        tree_stamp(a, ks);
    }
}
template <int B>
SP_DEV void tree_reverse_rounds(const double* R, double* E, const TreeArgs& a, const TreeGroup& t, int& ks) {
    for (int j = tree_levels(t.cnt) - 1; j >= 0; --j) {
        const int n = tree_width(t.cnt, j);
        TreeRevScratch<B> sc;
        tree_rev_compute<B>(R, E, a.RS, a.ES, n, threadIdx.x, a.needC != 0, sc);
        __syncthreads();
        tree_rev_store<B>(E, a.ES, n, threadIdx.x, a.needC != 0, sc);
        __syncthreads();
        tree_stamp(a, ks);
    }
}

// blockDim.x >= ceil(gcap / 2): one node per thread in every round
template <int B>
__global__ void __launch_bounds__(kTreeMaxThreads) k_tree_fwd(TreeArgs a) {
    extern __shared__ double2 tsm2[];
    double* R = reinterpret_cast<double*>(tsm2);
    const TreeGroup t = tree_group(a, blockIdx.x);
    int ks = 0;
    tree_stamp(a, ks);
    tree_load_recs<B>(a, t, R, threadIdx.x, blockDim.x);
    __syncthreads();
    tree_stamp(a, ks);
    tree_forward_rounds<B>(R, a.RS, a, t, ks);
    tree_store_fwd<B>(a, t, R, threadIdx.x, blockDim.x);
    tree_stamp(a, ks);
}

template <int B>
__global__ void __launch_bounds__(kTreeMaxThreads) k_tree_rev(TreeArgs a) {
    extern __shared__ double2 tsm2[];
    double* R = reinterpret_cast<double*>(tsm2);
    double* E = R + static_cast<long long>(Tree<B>::NR) * a.RS;
    const TreeGroup t = tree_group(a, blockIdx.x);
    int ks = 0;
    tree_stamp(a, ks);
    tree_load_rev<B>(a, t, R, E, threadIdx.x, blockDim.x);
    __syncthreads();
    tree_stamp(a, ks);
    tree_reverse_rounds<B>(R, E, a, t, ks);
    tree_store_rev<B>(a, t, E, threadIdx.x, blockDim.x);
    tree_stamp(a, ks);
}

// one group per series: forward tree, top inverse, reverse tree in one CTA
template <int B>
__global__ void __launch_bounds__(kTreeMaxThreads) k_tree_one(TreeArgs a) {
    extern __shared__ double2 tsm2[];
    double* R = reinterpret_cast<double*>(tsm2);
    double* E = R + static_cast<long long>(Tree<B>::NR) * a.RS;
    const TreeGroup t = tree_group(a, blockIdx.x);
    int ks = 0;
    tree_stamp(a, ks);
    tree_load_recs<B>(a, t, R, threadIdx.x, blockDim.x);
    __syncthreads();
    tree_stamp(a, ks);
    tree_forward_rounds<B>(R, a.RS, a, t, ks);
    if (threadIdx.x == 0) tree_top<B>(a, t, R, E);
    __syncthreads();
    tree_stamp(a, ks);
    tree_reverse_rounds<B>(R, E, a, t, ks);
    tree_store_rev<B>(a, t, E, threadIdx.x, blockDim.x);
    tree_stamp(a, ks);
}

// The two top levels in one cooperative launch (one CTA per level-(L-1) group, all
// co-resident):  A) every CTA reduces its group, keeping the merge factors in shared
// memory, and publishes its group record;  grid barrier;  B) the first CTA of each
// series reduces the series' group records (the top group, staged in its separator
// area, which is still free), inverts the top block and runs the top reverse tree,
// publishing the group boundaries' separators;  grid barrier;  C) every CTA loads its
// two boundary separators and runs its reverse tree from the factors it kept.
// Saves the factor store/reload of k_tree_fwd/k_tree_rev, the reload of k_tree_one
// and two launch boundaries.  a1 = level L-1 (many groups), a2 = level L (one group
// per series); the top group's capacity must fit a1's separator area.
template <int B>
SP_DEV void tree_load_recs_cg(const TreeArgs& a, const TreeGroup& t, double* R, int tid, int nt) {
    using TR = Tree<B>;  // records written by other CTAs before a grid barrier: L2 loads
    const double* src = a.rec_in + static_cast<long long>(t.s) * a.nin + t.k0;
    constexpr int CB = 8;
    for (int i = tid; i < t.cnt; i += nt)
        for (int c0 = 0; c0 < TR::NR; c0 += CB) {
            double v[CB];
TR_UNROLL
            for (int c = 0; c < CB; ++c)
                if (c0 + c < TR::NR) v[c] = __ldcg(src + (c0 + c) * a.SKin + i);
TR_UNROLL
            for (int c = 0; c < CB; ++c)
                if (c0 + c < TR::NR) R[(c0 + c) * a.RS + i] = v[c];
        }
}
template <int B>
__global__ void __launch_bounds__(kTreeMaxThreads) k_tree_coop(TreeArgs a1, TreeArgs a2) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    using TR = Tree<B>;
    extern __shared__ double2 tsm2[];
    double* R = reinterpret_cast<double*>(tsm2);
    double* E = R + static_cast<long long>(TR::NR) * a1.RS;
    const TreeGroup t = tree_group(a1, blockIdx.x);
    const int tid = threadIdx.x, nt = blockDim.x;
    int ks = 0;
    tree_stamp(a1, ks);
    tree_load_recs<B>(a1, t, R, tid, nt);
    __syncthreads();
    tree_stamp(a1, ks);
    tree_forward_rounds<B>(R, a1.RS, a1, t, ks);
    {
        const long long SKo = static_cast<long long>(a1.S) * a1.nG;
        for (int c = tid; c < TR::NR; c += nt) a1.rec_out[c * SKo + t.gidx] = R[c * a1.RS];
    }
    grid.sync();
    tree_stamp(a1, ks);
    {  // every CTA reduces its series' top group redundantly (in its still-free separator
       // area): its own boundary separators then come out of shared memory, with no second
       // grid barrier and no global round trip
        const TreeGroup t2 = tree_group(a2, t.s);
        double* R2 = E;
        double* E2 = R2 + static_cast<long long>(TR::NR) * a2.RS;
        int ks2 = 0;
        TreeArgs a2q = a2;
        if (t.j != 0) a2q.status = nullptr;  // report failures once per series
        tree_load_recs_cg<B>(a2, t2, R2, tid, nt);
        __syncthreads();
        tree_forward_rounds<B>(R2, a2.RS, a2q, t2, ks2);
        if (tid == 0) tree_top<B>(a2q, t2, R2, E2, t.j == 0);
        __syncthreads();
        tree_reverse_rounds<B>(R2, E2, a2q, t2, ks2);
        // boundaries j (L: x, C_LL, C_{L,R}) and j + 1 (R: x, C_RR) of this group
        constexpr int NPT = (TR::NS + 31) / 32;  // components per thread (>= 32 threads)
        double vL[NPT], vR[NPT];
        for (int r = 0; r < NPT; ++r) {
            vL[r] = vR[r] = 0.0;
            const int q = tid + r * nt;
            if (q >= TR::NS) continue;
            const bool want = q < B || a1.needC;
            vL[r] = (want && t.hasL) ? E2[q * a2.ES + t.j] : 0.0;
            vR[r] = (want && q < TR::SCU) ? E2[q * a2.ES + t.j + 1] : 0.0;
        }
        __syncthreads();
        for (int r = 0; r < NPT; ++r) {
            const int q = tid + r * nt;
            if (q >= TR::NS) break;
            E[q * a1.ES] = vL[r];
            E[q * a1.ES + 1] = vR[r];
        }
    }
    tree_stamp(a1, ks);
    __syncthreads();
    tree_reverse_rounds<B>(R, E, a1, t, ks);
    tree_store_rev<B>(a1, t, E, tid, nt);
    tree_stamp(a1, ks);
}
#endif

}  // namespace spingp_dev
