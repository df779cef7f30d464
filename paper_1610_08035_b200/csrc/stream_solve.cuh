// stream_solve.cuh — cr_solve of a materialised SymBTD as
// ONE persistent kernel that streams contiguous tiles of blocks through shared memory.
//
// Why.  The solve operator is HBM-bound (SURVEY.md §8(d) figure 1: B_solve = 8(2b²+2b)
// bytes per block row).  The thread-per-chunk kernels (btd_ops.cuh) move 2.9x that: every
// thread walks its own strip of diag/upper/rhs (uncoalesced), and the per-block factor
// (L, Y, z: 144 B at b = 3) goes out to HBM and comes back for the back-substitution.
// Here the blocks are only ever read in whole tiles (bulk asynchronous copies, one
// mbarrier per tile), the factor never leaves the SM, and the second sweep re-reads the
// tiles in the reverse order of the first, so most of them are still in the 126 MB L2.
//
//   tile     TB = NT * M consecutive blocks, staged as three contiguous pieces (diag,
//            upper, rhs) by cp.async.bulk.  Thread t owns blocks [t M, (t+1) M) of the
//            tile: M - 1 interior blocks, eliminated in order against the previous
//            thread's last block (left spike) and its own last block, exactly as
//            engine.cuh's elim_block (same record, Rec<B>).  With KEEP the factor is
//            written IN PLACE over the inputs as G = S^{-1}U, V = S^{-1}W, h = S^{-1}r
//            (2b²+b doubles per block, the size of the inputs).
//   tree     the NT chunk records of a tile are merged pairwise in shared memory
//            (tree.cuh's merge) into one tile record; a CTA owns a contiguous range of
//            tiles and chains their records into one CTA record (left separator = the
//            previous CTA's last block).
//   sweep 1  every CTA reduces its tiles in ascending order and publishes its record.
//   top      one grid-wide barrier; CTA 0 solves the G-record reduced system in shared
//            memory (chains of q records per thread + the same tree) and publishes the
//            solution at every CTA boundary and log det.
//   sweep 2  every CTA walks its tiles in DESCENDING order: un-chain the tile's boundary
//            solutions, re-read and re-eliminate the tile (the last tile of sweep 1 is
//            still in shared memory and is not re-read), un-merge the tree, back-
//            substitute x_j = h_j - G_j x_{j+1} - V_j x_L per thread, store x coalesced.
//
// HBM traffic: sweep 1 reads every block once; sweep 2 re-reads what L2 lost and writes x.
#pragma once

#include "tree.cuh"

namespace spingp_dev {

template <int B, int NT_, int M_>
struct SSCfg {
    static constexpr int NT = NT_;            // threads per CTA = chunks per tile
    static constexpr int M = M_;              // blocks per chunk (M - 1 interior + 1 separator)
    static constexpr int TB = NT_ * M_;       // blocks per tile
    static constexpr int BB = B * B;
    static constexpr int NR = Rec<B>::N;      // record components
    static constexpr int NF = Tree<B>::NF;    // merge factor components
    static constexpr int RS = (NT_ + 1) & ~1; // row length of the record area
    static constexpr int ES = (NT_ + 2) & ~1; // row length of the separator area
    // shared memory (doubles): tile | records | separators | chain records | halo | boundary x | barrier
    static constexpr int OFF_D = 0;
    static constexpr int OFF_U = OFF_D + TB * BB;
    static constexpr int OFF_R = OFF_U + TB * BB;
    static constexpr int OFF_REC = OFF_R + TB * B + ((TB * B) & 1);
    static constexpr int OFF_E = OFF_REC + NR * RS;
    static constexpr int OFF_CR = OFF_E + B * ES;
    static constexpr int OFF_UH = OFF_CR + 2 * NR;
    static constexpr int OFF_XB = OFF_UH + BB;           // xL[B], xR[B]
    static constexpr int OFF_BAR = (OFF_XB + 2 * B + 1) & ~1;
    static constexpr int SMEM_DOUBLES = OFF_BAR + 2;
    static constexpr size_t SMEM_BYTES = static_cast<size_t>(SMEM_DOUBLES) * 8;
    static constexpr int TILE_DOUBLES = OFF_REC;          // room for CTA 0's G records
    static_assert(TB % 2 == 0, "tile pieces must be multiples of 16 bytes");
};

struct SSArgs {
    const double* diag;
    const double* up;
    const double* rhs;
    double* x;        // null: log det only (sweep 1 + top)
    double* logdet;   // device scalar or null
    long long n;      // block rows
    long long ntiles;
    int G;            // CTAs (all co-resident), G <= ntiles
    int Tmax;         // max tiles per CTA
    int bulk;         // 1: pointers are 16-byte aligned (bulk copies), 0: plain loads
    int l2mode;       // sweep-1 loads: 0 normal, 1 evict_last (tiles re-read by sweep 2)
    double* crec;     // [NR][G] CTA records, component-major
    double* xsep;     // [G][B] solution at every CTA's last block
    double* cfac;     // [G][Tmax][NF] chain-merge factors of the CTA's tiles
    unsigned long long* sync;  // [0] arrivals (monotonic), [1] release word (monotonic)
    unsigned long long arrive_target, release_target;
    unsigned long long* status;
    unsigned long long* stamps;  // diagnostics: [G][16] %globaltimer per phase (null = off)
};

#ifndef SPINGP_HOST_EMU
SP_DEV void ss_stamp(const SSArgs& a, int k) {
    if (a.stamps && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.stamps[blockIdx.x * 16 + k] = t;
    }
}
// ---- asynchronous bulk copy + mbarrier (PTX) ---------------------------------
SP_DEV unsigned ss_smem(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
SP_DEV void ss_bar_init(void* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ss_smem(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
SP_DEV void ss_bar_expect(void* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ss_smem(bar)), "r"(bytes) : "memory");
}
SP_DEV void ss_bar_wait(void* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(ss_smem(bar)),
        "r"(parity)
        : "memory");
}
SP_DEV void ss_bulk_load(void* dst, const void* src, unsigned bytes, void* bar, unsigned long long policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(ss_smem(dst)), "l"(src), "r"(bytes), "r"(ss_smem(bar)), "l"(policy)
        : "memory");
}
SP_DEV void ss_fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
SP_DEV unsigned long long ss_policy_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
SP_DEV unsigned long long ss_policy_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
SP_DEV unsigned long long ss_policy_normal() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
SP_DEV unsigned long long ss_ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
SP_DEV void ss_st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- one thread's chunk: forward elimination (in place when KEEP) -------------
// Blocks lo .. lo+M-1 of the tile; Uprev = the upper block coupling block lo-1 to lo
// (the previous chunk's separator, or the tile halo).  rec receives the chunk record.
template <class C, int B, bool KEEP>
SP_DEV bool ss_eliminate(double* sD, double* sU, double* sR, const double* Uprev, int lo, double* rec, int& badj) {
    constexpr int BB = B * B;
    constexpr int M = C::M;
    using RC = Rec<B>;
    double T[BB], rc[B], W[BB], accLL[BB], accrL[B];
    LogDetAcc piv;
    piv.init();
TR_UNROLL
    for (int i = 0; i < B; ++i)
TR_UNROLL
        for (int j = 0; j < B; ++j) W[i * B + j] = Uprev[j * B + i];
    mzero<B>(T);
    vzero<B>(rc);
    mzero<B>(accLL);
    vzero<B>(accrL);
    bool ok = true;
    badj = 0;
#pragma unroll 1
    for (int j = 0; j < M - 1; ++j) {
        double* Dp = sD + (lo + j) * BB;
        double* Up = sU + (lo + j) * BB;
        double* rp = sR + (lo + j) * B;
        double S[BB], L[BB], U[BB], r[B], z[B], X[BB], Y[BB], Gm[BB];
TR_UNROLL
        for (int i = 0; i < BB; ++i) S[i] = Dp[i] - T[i];
TR_UNROLL
        for (int i = 0; i < BB; ++i) U[i] = Up[i];
TR_UNROLL
        for (int i = 0; i < B; ++i) r[i] = rp[i] - rc[i];
        msym<B>(S);
        const bool okj = chol<B>(L, S, piv);
        if (!okj && ok) badj = j;
        ok = ok && okj;
        lsolve_v<B>(z, L, r);
        lsolve<B>(X, L, U);
        lsolve<B>(Y, L, W);
        mtm_sym<B>(Gm, Y, Y);
TR_UNROLL
        for (int i = 0; i < BB; ++i) accLL[i] -= Gm[i];
        double yz[B];
        mtv<B>(yz, Y, z);
TR_UNROLL
        for (int i = 0; i < B; ++i) accrL[i] -= yz[i];
        mtm<B>(Gm, X, Y);
TR_UNROLL
        for (int i = 0; i < BB; ++i) W[i] = -Gm[i];
        mtm_sym<B>(T, X, X);
        mtv<B>(rc, X, z);
        if (KEEP) {  // G = L^{-T}X -> upper slot, V = L^{-T}Y -> diag slot, h = L^{-T}z -> rhs slot
            double h[B];
            ltsolve<B>(Gm, L, X);
TR_UNROLL
            for (int i = 0; i < BB; ++i) Up[i] = Gm[i];
            ltsolve<B>(Gm, L, Y);
TR_UNROLL
            for (int i = 0; i < BB; ++i) Dp[i] = Gm[i];
            ltsolve_v<B>(h, L, z);
TR_UNROLL
            for (int i = 0; i < B; ++i) rp[i] = h[i];
        }
    }
    const double* Dp = sD + (lo + M - 1) * BB;
    const double* rp = sR + (lo + M - 1) * B;
TR_UNROLL
    for (int i = 0; i < BB; ++i) rec[RC::RDIAG + i] = Dp[i] - T[i];
TR_UNROLL
    for (int i = 0; i < BB; ++i) rec[RC::LDIAG + i] = accLL[i];
TR_UNROLL
    for (int i = 0; i < B; ++i)
TR_UNROLL
        for (int j = 0; j < B; ++j) rec[RC::LR + i * B + j] = W[j * B + i];
TR_UNROLL
    for (int i = 0; i < B; ++i) rec[RC::RRHS + i] = rp[i] - rc[i];
TR_UNROLL
    for (int i = 0; i < B; ++i) rec[RC::LRHS + i] = accrL[i];
    rec[RC::LOGDET] = piv.logdet();
    return ok;
}

// x of the separator eliminated by a merge with factor F (L_S, Y_L, Y_R, z):
//   x_M = L_S^{-T} (z - Y_L x_L - Y_R x_R)
template <int B>
SP_DEV void ss_unmerge(const double* F, const double* xL, const double* xR, double* xM) {
    using TR = Tree<B>;
    double a[B], t1[B], t2[B];
    mv<B>(t1, F + TR::FYL, xL);
    mv<B>(t2, F + TR::FYR, xR);
TR_UNROLL
    for (int i = 0; i < B; ++i) a[i] = F[TR::FZ + i] - t1[i] - t2[i];
    ltsolve_v<B>(xM, F + TR::FL, a);
}

// Merge of records A = (L, M) and Bv = (M, R) read with strides (shared or global memory)
// -> record at Cp, merge factor at Fp.  A real call: it runs on one thread per CTA (tile
// chain) or per group (top system), outside the hot loops, and its ~130 live doubles must
// not set the register count of the whole kernel.
template <int B>
__device__ __noinline__ bool ss_merge_at(const double* Ap, int As, const double* Bp, int Bs, double* Cp, int Cs,
                                         double* Fp, int Fs) {
    constexpr int NR = Rec<B>::N, NF = Tree<B>::NF;
    double A[NR], Bv[NR], Cm[NR], F[NF];
TR_UNROLL
    for (int c = 0; c < NR; ++c) {
        A[c] = Ap[c * As];
        Bv[c] = Bp[c * Bs];
    }
    const bool ok = tree_merge<B>(A, Bv, Cm, F);
TR_UNROLL
    for (int c = 0; c < NR; ++c) Cp[c * Cs] = Cm[c];
TR_UNROLL
    for (int c = 0; c < NF; ++c) Fp[c * Fs] = F[c];
    return ok;
}

// Forward tree over cnt records at slots [0, cnt) of R (component-major, row RS):
// leaves the merged record at slot 0 and the merge factors parked (tree.cuh layout).
template <class C, int B>
SP_DEV bool ss_tree_up(double* R, int cnt) {
    bool ok = true;
    const int J = tree_levels(cnt);
    for (int j = 0; j < J; ++j) {
        const int n = tree_width(cnt, j);
        TreeFwdScratch<B> sc;
        tree_fwd_compute<B>(R, C::RS, n, threadIdx.x, sc);
        ok = ok && sc.ok;
        __syncthreads();
        tree_fwd_store<B>(R, C::RS, n, threadIdx.x, sc);
        __syncthreads();
    }
    return ok;
}
// Reverse tree, solution only: E[q * ES + i], slots 0 (left) and 1 (right) set by the
// caller; on return E holds x at the cnt + 1 record boundaries.
template <class C, int B>
SP_DEV void ss_tree_down(const double* R, double* E, int cnt) {
    using TR = Tree<B>;
    const int k = threadIdx.x;
    for (int j = tree_levels(cnt) - 1; j >= 0; --j) {
        const int n = tree_width(cnt, j);
        const int nn = (n + 1) >> 1;
        const bool active = k < nn, merged = active && 2 * k + 1 < n, last = k == nn - 1;
        double xL[B], xM[B], xR[B];
        if (active) {
TR_UNROLL
            for (int q = 0; q < B; ++q) {
                xL[q] = E[q * C::ES + k];
                xR[q] = E[q * C::ES + k + 1];
            }
            if (merged) {
                double F[TR::NF];
TR_UNROLL
                for (int c = 0; c < TR::NF; ++c) F[c] = R[c * C::RS + nn + k];
                ss_unmerge<B>(F, xL, xR, xM);
            }
        }
        __syncthreads();
        if (active) {
TR_UNROLL
            for (int q = 0; q < B; ++q) {
                E[q * C::ES + 2 * k] = xL[q];
                if (merged) E[q * C::ES + 2 * k + 1] = xM[q];
                if (last) E[q * C::ES + n] = xR[q];
            }
        }
        __syncthreads();
    }
}

// ---- tile staging ---------------------------------------------------------------
// Full tiles with every upper block present go through three bulk copies (thread 0);
// the last tile(s) and misaligned arrays are staged with plain loads, padded with
// identity blocks past the end (D = I, U = 0, r = 0: x = 0, log det 0).
template <class C, int B>
SP_DEV bool ss_tile_is_bulk(const SSArgs& a, long long tile) {
    return a.bulk && (tile + 1) * C::TB <= a.n - 1;
}
template <class C, int B>
SP_DEV void ss_tile_issue(const SSArgs& a, double* sm, long long tile, unsigned long long policy) {
    constexpr int BB = B * B;
    const long long t0 = tile * C::TB;
    void* bar = sm + C::OFF_BAR;
    if (ss_tile_is_bulk<C, B>(a, tile)) {
        if (threadIdx.x == 0) {
            ss_fence_async();
            constexpr unsigned nbD = C::TB * BB * 8, nbR = C::TB * B * 8;
            ss_bar_expect(bar, 2 * nbD + nbR);
            ss_bulk_load(sm + C::OFF_D, a.diag + t0 * BB, nbD, bar, policy);
            ss_bulk_load(sm + C::OFF_U, a.up + t0 * BB, nbD, bar, policy);
            ss_bulk_load(sm + C::OFF_R, a.rhs + t0 * B, nbR, bar, policy);
        }
    } else {
        const long long nd = a.n * BB, nu = (a.n - 1) * BB, nr = a.n * B;
        for (int i = threadIdx.x; i < C::TB * BB; i += C::NT) {
            const long long gi = t0 * BB + i;
            const int e = i % BB;
            sm[C::OFF_D + i] = gi < nd ? a.diag[gi] : ((e / B == e % B) ? 1.0 : 0.0);
            sm[C::OFF_U + i] = gi < nu ? a.up[gi] : 0.0;
        }
        for (int i = threadIdx.x; i < C::TB * B; i += C::NT) {
            const long long gi = t0 * B + i;
            sm[C::OFF_R + i] = (gi < nr && a.rhs) ? a.rhs[gi] : 0.0;
        }
    }
    if (threadIdx.x < BB) sm[C::OFF_UH + threadIdx.x] = t0 > 0 ? a.up[(t0 - 1) * BB + threadIdx.x] : 0.0;
}
template <class C, int B>
SP_DEV void ss_tile_wait(const SSArgs& a, double* sm, long long tile, unsigned& phase) {
    if (ss_tile_is_bulk<C, B>(a, tile)) {
        ss_bar_wait(sm + C::OFF_BAR, phase);
        phase ^= 1u;
    }
    __syncthreads();  // halo / plain loads visible
}

// eliminate the staged tile and reduce it to one record at slot 0 of the record area
template <class C, int B, bool KEEP>
SP_DEV void ss_tile_reduce(const SSArgs& a, double* sm, long long tile) {
    constexpr int BB = B * B;
    const int t = threadIdx.x;
    double rec[C::NR];
    int badj;
    const double* Uprev = t == 0 ? sm + C::OFF_UH : sm + C::OFF_U + (t * C::M - 1) * BB;
    const bool ok = ss_eliminate<C, B, KEEP>(sm + C::OFF_D, sm + C::OFF_U, sm + C::OFF_R, Uprev, t * C::M, rec, badj);
    if (!ok) report(a.status, min(a.n - 1, tile * C::TB + t * C::M + badj), ST_NOT_PD);
    double* R = sm + C::OFF_REC;
TR_UNROLL
    for (int c = 0; c < C::NR; ++c) R[c * C::RS + t] = rec[c];
    __syncthreads();
}

template <class C, int B>
__global__ void __launch_bounds__(C::NT) k_solve_stream(SSArgs a) {
    extern __shared__ double2 ss_sm2[];
    double* sm = reinterpret_cast<double*>(ss_sm2);
    constexpr int BB = B * B;
    constexpr int NR = C::NR, NF = C::NF;
    using RC = Rec<B>;
    const int t = threadIdx.x;
    const int cta = blockIdx.x;
    const long long tlo = a.ntiles * cta / a.G, thi = a.ntiles * (cta + 1) / a.G;
    const int T = static_cast<int>(thi - tlo);
    double* R = sm + C::OFF_REC;
    double* E = sm + C::OFF_E;
    double* CR = sm + C::OFF_CR;
    double* XB = sm + C::OFF_XB;
    double* cf = a.cfac + static_cast<long long>(cta) * a.Tmax * NF;
    unsigned phase = 0;
    if (t == 0) ss_bar_init(sm + C::OFF_BAR, 1);
    __syncthreads();
    const bool want_x = a.x != nullptr;
    const bool retain = want_x && cta != 0;  // the last tile of sweep 1 stays in shared memory
    const unsigned long long pol_keep = a.l2mode == 1 ? ss_policy_last() : ss_policy_normal();
    const unsigned long long pol_once = ss_policy_first();

    ss_stamp(a, 0);
    // ---- sweep 1: tiles ascending -> CTA record ---------------------------------
    ss_tile_issue<C, B>(a, sm, tlo, T == 1 && retain ? pol_once : pol_keep);
    for (int k = 0; k < T; ++k) {
        const long long tile = tlo + k;
        const bool keep = retain && k == T - 1;
        ss_tile_wait<C, B>(a, sm, tile, phase);
        if (k == 1) ss_stamp(a, 1);
        if (keep) ss_tile_reduce<C, B, true>(a, sm, tile);
        else ss_tile_reduce<C, B, false>(a, sm, tile);
        if (k == 1) ss_stamp(a, 2);
        // the tile area is free again: stage the next tile behind the tree rounds
        if (k + 1 < T) ss_tile_issue<C, B>(a, sm, tile + 1, (retain && k + 2 == T) ? pol_once : pol_keep);
        const bool ok = ss_tree_up<C, B>(R, C::NT);
        if (!ok) report(a.status, min(a.n - 1, tile * C::TB), ST_NOT_PD);
        if (k == 1) ss_stamp(a, 3);
        if (t == 0) {  // chain the tile record into the CTA record
            if (k == 0) {
                for (int c = 0; c < NR; ++c) CR[c] = R[c * C::RS];
            } else if (!ss_merge_at<B>(CR, 1, R, C::RS, CR, 1, cf + k * NF, 1)) {
                report(a.status, min(a.n - 1, tile * C::TB - 1), ST_NOT_PD);
            }
        }
        __syncthreads();
        if (k == 1) ss_stamp(a, 4);
    }
    ss_stamp(a, 5);
    for (int c = t; c < NR; c += C::NT) a.crec[static_cast<long long>(c) * a.G + cta] = CR[c];
    __threadfence();
    __syncthreads();
    if (t == 0) atomicAdd(a.sync, 1ULL);

    // ---- top: CTA 0 solves the G-record reduced system ---------------------------
    if (cta == 0) {
        if (t == 0)
            while (ss_ld_acquire(a.sync) < a.arrive_target) __nanosleep(40);
        __syncthreads();
        const int G = a.G, GS = (G + 1) & ~1;
        double* GR = sm;  // [NR][GS] over the tile area
        for (int c = 0; c < NR; ++c)
            for (int i = t; i < G; i += C::NT) GR[c * GS + i] = __ldcg(a.crec + static_cast<long long>(c) * G + i);
        __syncthreads();
        const int q = (G + C::NT - 1) / C::NT;       // records per thread
        const int NG = (G + q - 1) / q;              // active threads
        const int g0 = t * q, gc = t < NG ? min(q, G - g0) : 0;
        if (gc > 0) {  // chain in place at slot g0; factors parked over the consumed records
            for (int i = 1; i < gc; ++i)
                if (!ss_merge_at<B>(GR + g0, GS, GR + g0 + i, GS, GR + g0, GS, GR + g0 + i, GS))
                    report(a.status, a.n - 1, ST_NOT_PD);
            for (int c = 0; c < NR; ++c) R[c * C::RS + t] = GR[c * GS + g0];
        }
        __syncthreads();
        if (!ss_tree_up<C, B>(R, NG)) report(a.status, a.n - 1, ST_NOT_PD);
        if (t == 0) {  // top block
            double D[BB], r[B], Lc[BB], z[B], xx[B], ld;
TR_UNROLL
            for (int i = 0; i < BB; ++i) D[i] = R[(RC::RDIAG + i) * C::RS];
TR_UNROLL
            for (int i = 0; i < B; ++i) r[i] = R[(RC::RRHS + i) * C::RS];
            msym<B>(D);
            if (!chol<B>(Lc, D, ld)) report(a.status, a.n - 1, ST_NOT_PD);
            lsolve_v<B>(z, Lc, r);
            ltsolve_v<B>(xx, Lc, z);
TR_UNROLL
            for (int i = 0; i < B; ++i) {
                E[i * C::ES] = 0.0;
                E[i * C::ES + 1] = xx[i];
            }
            if (a.logdet) *a.logdet = ld + R[RC::LOGDET * C::RS];
        }
        __syncthreads();
        if (want_x) {
            ss_tree_down<C, B>(R, E, NG);
            if (gc > 0) {  // un-chain: x at the right separator of every record of the group
                double xL[B], xR[B], xM[B];
TR_UNROLL
                for (int i = 0; i < B; ++i) {
                    xL[i] = E[i * C::ES + t];
                    xR[i] = E[i * C::ES + t + 1];
                }
                for (int i = gc - 1; i >= 0; --i) {
TR_UNROLL
                    for (int p = 0; p < B; ++p) a.xsep[static_cast<long long>(g0 + i) * B + p] = xR[p];
                    if (i == 0) break;
                    double F[NF];
TR_UNROLL
                    for (int c = 0; c < NF; ++c) F[c] = GR[c * GS + g0 + i];
                    ss_unmerge<B>(F, xL, xR, xM);
TR_UNROLL
                    for (int p = 0; p < B; ++p) xR[p] = xM[p];
                }
            }
            __threadfence();
            __syncthreads();
            if (t == 0) ss_st_release(a.sync + 1, a.release_target);
        }
    }
    if (!want_x) return;
    if (cta != 0) {
        if (t == 0)
            while (ss_ld_acquire(a.sync + 1) < a.release_target) __nanosleep(40);
    }
    __syncthreads();
    ss_stamp(a, 6);

    // ---- sweep 2: tiles descending -> x -------------------------------------------
    double xLc[B], xRk[B];  // thread 0: the CTA's left boundary, the current tile's right boundary
    if (t == 0) {
TR_UNROLL
        for (int i = 0; i < B; ++i) {
            xLc[i] = cta > 0 ? __ldcg(a.xsep + static_cast<long long>(cta - 1) * B + i) : 0.0;
            xRk[i] = __ldcg(a.xsep + static_cast<long long>(cta) * B + i);
        }
    }
    for (int k = T - 1; k >= 0; --k) {
        const long long tile = tlo + k;
        const bool staged = retain && k == T - 1;
        if (!staged) ss_tile_issue<C, B>(a, sm, tile, pol_once);
        if (t == 0) {  // boundary solutions of this tile (behind the copy)
            double xLk[B];
            if (k > 0) {
                double F[NF];
TR_UNROLL
                for (int c = 0; c < NF; ++c) F[c] = cf[k * NF + c];
                ss_unmerge<B>(F, xLc, xRk, xLk);
            } else {
TR_UNROLL
                for (int i = 0; i < B; ++i) xLk[i] = xLc[i];
            }
TR_UNROLL
            for (int i = 0; i < B; ++i) {
                XB[i] = xLk[i];
                XB[B + i] = xRk[i];
                xRk[i] = xLk[i];
            }
        }
        if (!staged) {
            ss_tile_wait<C, B>(a, sm, tile, phase);
            if (k == 1) ss_stamp(a, 8);
            ss_tile_reduce<C, B, true>(a, sm, tile);
            if (k == 1) ss_stamp(a, 9);
            ss_tree_up<C, B>(R, C::NT);
            if (k == 1) ss_stamp(a, 10);
        } else {
            __syncthreads();
        }
        if (t < B) {
            E[t * C::ES] = XB[t];
            E[t * C::ES + 1] = XB[B + t];
        }
        __syncthreads();
        ss_tree_down<C, B>(R, E, C::NT);
        if (k == 1) ss_stamp(a, 11);
        {  // back-substitution of this thread's chunk, x over the rhs slots
            double xp[B], xn[B];
TR_UNROLL
            for (int i = 0; i < B; ++i) {
                xp[i] = E[i * C::ES + t];
                xn[i] = E[i * C::ES + t + 1];
            }
            const int lo = t * C::M;
            double* sR = sm + C::OFF_R;
TR_UNROLL
            for (int i = 0; i < B; ++i) sR[(lo + C::M - 1) * B + i] = xn[i];
#pragma unroll 1
            for (int j = C::M - 2; j >= 0; --j) {
                const double* Gp = sm + C::OFF_U + (lo + j) * BB;
                const double* Vp = sm + C::OFF_D + (lo + j) * BB;
                double* hp = sR + (lo + j) * B;
                double xj[B];
TR_UNROLL
                for (int i = 0; i < B; ++i) {
                    double s = hp[i];
TR_UNROLL
                    for (int c = 0; c < B; ++c) s = fma(-Gp[i * B + c], xn[c], s);
TR_UNROLL
                    for (int c = 0; c < B; ++c) s = fma(-Vp[i * B + c], xp[c], s);
                    xj[i] = s;
                }
TR_UNROLL
                for (int i = 0; i < B; ++i) {
                    hp[i] = xj[i];
                    xn[i] = xj[i];
                }
            }
        }
        __syncthreads();
        {
            const long long t0 = tile * C::TB;
            const long long lim = min(static_cast<long long>(C::TB), a.n - t0) * B;
            const double* sR = sm + C::OFF_R;
            double* xo = a.x + t0 * B;
            for (int i = t; i < lim; i += C::NT) __stcs(xo + i, sR[i]);
        }
        __syncthreads();
        if (k == 1) ss_stamp(a, 12);
    }
    ss_stamp(a, 7);
}
#endif  // SPINGP_HOST_EMU

}  // namespace spingp_dev
