// stream_solve.cuh — cr_solve of a materialised SymBTD as
// ONE persistent kernel in which every WARP streams its own contiguous run of blocks
// through shared memory, tile by tile.  (The tile kernel: SPINGP_SOLVE_STRIP=0 and systems
// too short for strip_solve.cuh, which shares this file's elimination step, trees, top
// system and barrier.)
//
// Why.  The solve operator is HBM-bound (SURVEY.md §8(d) figure 1: B_solve = 8(2b²+2b)
// bytes per block row).  The thread-per-chunk kernels (btd_ops.cuh) move 2.9x that: every
// thread walks its own strip of diag/upper/rhs (uncoalesced), and the per-block factor
// (L, Y, z: 144 B at b = 3) goes out to HBM and comes back for the back-substitution.
// Here the blocks are only ever read in whole tiles (bulk asynchronous copies, one
// mbarrier per warp), the factor never leaves the SM, and the second sweep re-reads the
// tiles in the reverse order of the first, so most of them are still in the 126 MB L2.
// (A first version with CTA-wide tiles and shared-memory trees spent 66% of every tile in
// barrier-bound tree rounds, profiles/r02_stream_solve.md; the warps are independent now.)
//
//   warp tile  WT = 32 M consecutive blocks, staged as three contiguous pieces (diag,
//              upper, rhs) by cp.async.bulk into the warp's own buffer.  Lane l owns
//              blocks [l M, (l+1) M): M - 1 interior blocks, eliminated in order against
//              the previous lane's last block (left spike) and its own last block, as
//              engine.cuh's elim_block (same record, Rec<B>).  Sweep 1 only reads the tile.
//   warp tree  the 32 lane records are merged pairwise with warp shuffles (5 rounds, no
//              barrier, no shared memory); the merge factor of a pair is shuffled back
//              to the lane whose record was consumed, which stores it for sweep 2.
//   carry      a warp owns a contiguous run of tiles.  The record reduced so far (left
//              separator Z = the block before the run, right = the previous tile's last
//              block P) is carried in lane 0, which eliminates P as one more interior
//              block of its chunk; the warp tree then yields the carry of the next tile.
//   sweep 1    every warp reduces its tiles in ascending order, checkpointing the carry
//              (2b²+b doubles per tile); the NW warp records of a CTA are merged in shared
//              memory (tree.cuh) and the CTA record is published.
//   top        one grid-wide barrier; CTA 0 solves the G-record reduced system in shared
//              memory and publishes the solution at every CTA boundary and log det.
//   sweep 2    every group walks its tiles in DESCENDING order: un-merge the tile's tree from
//              the merge factors sweep 1 stored (30 doubles per lane and tile), which gives
//              every lane the solution at both ends of its chunk; reload the tile (the last
//              tile of sweep 1 is still in shared memory and is not re-read) and solve each
//              chunk as a Dirichlet problem: plain block Thomas, no spike, no tree.
//
// HBM traffic: sweep 1 reads every block once and writes the tree factors (48 B per block
// at b = 3, M = 5, mostly L2-resident until sweep 2 reads them back in reverse order);
// sweep 2 re-reads what L2 lost and writes x.
// A "group" is LPT = 32, 16 or 8 lanes of a warp with their own tile buffer and run: fewer
// lanes per tile means a shallower tree for the same blocks per lane (measured slower than
// 32 lanes: the groups of a warp drift apart; profiles/r02_stream_solve.md).
#pragma once

#include "tree.cuh"

namespace spingp_dev {

constexpr int ss_even(int v) { return (v + 1) & ~1; }

template <int B, int NW_, int M_, int LPT_ = 32>
struct SSCfg {
    static constexpr int LPT = LPT_;          // lanes per tile (a group of lanes of one warp)
    static constexpr int NW = NW_ * (32 / LPT_);  // groups per CTA (independent pipelines)
    static constexpr int NT = 32 * NW_;
    static constexpr int M = M_;              // blocks per lane (M - 1 interior + 1 separator)
    static constexpr int WT = LPT_ * M_;      // blocks per tile
    static constexpr int BB = B * B;
    static constexpr int NR = Rec<B>::N;      // record components
    static constexpr int NF = Tree<B>::NF;    // merge factor components
    static constexpr int NK = 2 * BB + B;     // checkpoint / kept-factor doubles per block
    // per-warp shared memory (doubles): tile | kept factor of the carried block | halo | barrier
    static constexpr int W_D = 0;
    static constexpr int W_U = W_D + WT * BB;
    static constexpr int W_R = W_U + WT * BB;
    static constexpr int W_P = ss_even(W_R + WT * B);
    static constexpr int W_UH = W_P + NK;
    static constexpr int W_BAR = ss_even(W_UH + BB);
    static constexpr int W_SIZE = W_BAR + 2;
    // CTA level: warp records, their separators
    static constexpr int RSW = ss_even(NW);
    static constexpr int ESW = ss_even(NW + 1);
    static constexpr int OFF_WR = NW * W_SIZE;
    static constexpr int OFF_WE = OFF_WR + NR * RSW;
    static constexpr int SMEM_DOUBLES = ss_even(OFF_WE + B * ESW);
    static constexpr size_t SMEM_BYTES = static_cast<size_t>(SMEM_DOUBLES) * 8;
    // top system (CTA 0, over its tile buffers): one record per thread, the NT / 32 warp
    // records [NR][RST] and their separators [B][EST]
    static constexpr int RST = ss_even(NT / 32);
    static constexpr int EST = ss_even(NT / 32 + 1);
    static_assert(WT % 2 == 0, "tile pieces must be multiples of 16 bytes");
    static_assert(NR * RST + B * EST < OFF_WR, "top system does not fit");
    static_assert((M_ & 1) == 1 || B % 2 == 0, "odd M keeps the lane strips off the same banks");
};

struct SSArgs {
    const double* diag;
    const double* up;
    const double* rhs;
    double* x;        // null: log det only (sweep 1 + top)
    double* logdet;   // device scalar or null
    long long n;      // block rows
    long long ntiles; // warp tiles
    int G;            // CTAs (all co-resident); G * NW <= ntiles
    int Tmax;         // max tiles per warp
    int bulk;         // 1: pointers are 16-byte aligned (bulk copies), 0: plain loads
    int l2mode;       // sweep-1 loads: 0 normal, 1 evict_last (tiles re-read by sweep 2)
    int l2keep;       // strip kernel, l2mode 1: sub-tiles (from the end) loaded evict_last in sweep 1
    double* crec;     // [NR][G] CTA records, component-major
    double* xsep;     // [G][B] solution at every CTA's last block
    double* ckpt;     // [G * NW][Tmax][NK] carry checkpoints (S_P, W_P, r_P) per tile
    double* tfac;     // [G * NW][Tmax][NF][LPT] merge factors of every tile's tree
    long long Lc;     // strip kernel: blocks per lane (even)
    int nsub;         // strip kernel: sub-tiles per lane
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
constexpr unsigned kFullWarp = 0xffffffffu;

// ---- one lane's chunk: forward elimination against the left spike ----------------
template <int B>
struct SSElim {
    double T[B * B], rc[B], W[B * B], accLL[B * B], accrL[B];
    LogDetAcc piv;
    unsigned long long* status;
    long long idx, nmax;  // global index of the block being eliminated, n - 1
};
// A pivot failed.  If its inputs were finite it is the origin (priority 1); a NaN pivot
// is most likely the echo of an earlier failure or of a NaN in the caller's arrays
// (priority 2: reported only when nothing else was), so that the smallest index that
// reaches the caller is the block that really is not positive definite.
template <int N>
SP_DEV void ss_report_pivot(unsigned long long* status, long long idx, const double* S) {
    double acc = 0.0;
TR_UNROLL
    for (int i = 0; i < N; ++i) acc += S[i];
    if (isfinite(acc)) report(status, idx, ST_NOT_PD);
    else report_echo(status, idx, ST_NOT_PD);
}
// One interior block with diagonal D, coupling U (to the next block) and rhs r.
template <int B>
SP_DEV void ss_elim_step(SSElim<B>& es, const double* Dp, const double* Up, const double* rp) {
    constexpr int BB = B * B;
    double S[BB], L[BB], U[BB], r[B], z[B], X[BB], Y[BB], Gm[BB];
TR_UNROLL
    for (int i = 0; i < BB; ++i) S[i] = Dp[i] - es.T[i];
TR_UNROLL
    for (int i = 0; i < BB; ++i) U[i] = Up[i];
TR_UNROLL
    for (int i = 0; i < B; ++i) r[i] = rp[i] - es.rc[i];
    msym<B>(S);
    if (!chol<B>(L, S, es.piv)) ss_report_pivot<BB>(es.status, min(es.idx, es.nmax), S);
    ++es.idx;
    lsolve_v<B>(z, L, r);
    lsolve<B>(X, L, U);
    lsolve<B>(Y, L, es.W);
    mtm_sym<B>(Gm, Y, Y);
TR_UNROLL
    for (int i = 0; i < BB; ++i) es.accLL[i] -= Gm[i];
    double yz[B];
    mtv<B>(yz, Y, z);
TR_UNROLL
    for (int i = 0; i < B; ++i) es.accrL[i] -= yz[i];
    mtm<B>(Gm, X, Y);
TR_UNROLL
    for (int i = 0; i < BB; ++i) es.W[i] = -Gm[i];
    mtm_sym<B>(es.T, X, X);
    mtv<B>(es.rc, X, z);
}

// Lane chunk lo .. lo+M-1 of the tile at (sD, sU, sR), read only.  Uprev = the upper block
// that couples block lo-1 to lo.  carry (group leader, tiles after the run's first): the
// checkpoint (S_P, W_P = P_{P,Z}, r_P) of the carried block P, eliminated first, with the
// run's accumulated left-separator terms and log det in rec (LDIAG, LRHS, LOGDET).
// base = the global index of block lo (failed pivots are reported from here).
template <class C, int B>
SP_DEV void ss_eliminate(const double* sD, const double* sU, const double* sR, const double* Uprev, int lo,
                         const double* carry, double* rec, unsigned long long* status, long long base, long long nmax) {
    constexpr int BB = B * B;
    constexpr int M = C::M;
    using RC = Rec<B>;
    SSElim<B> es;
    es.piv.init();
    es.status = status;
    es.idx = base - (carry ? 1 : 0);
    es.nmax = nmax;
    mzero<B>(es.T);
    vzero<B>(es.rc);
    double ld0 = 0.0;
    if (carry) {
TR_UNROLL
        for (int i = 0; i < BB; ++i) es.W[i] = carry[BB + i];
TR_UNROLL
        for (int i = 0; i < BB; ++i) es.accLL[i] = rec[RC::LDIAG + i];
TR_UNROLL
        for (int i = 0; i < B; ++i) es.accrL[i] = rec[RC::LRHS + i];
        ld0 = rec[RC::LOGDET];
        ss_elim_step<B>(es, carry, Uprev, carry + 2 * BB);
    } else {
TR_UNROLL
        for (int i = 0; i < B; ++i)
TR_UNROLL
            for (int j = 0; j < B; ++j) es.W[i * B + j] = Uprev[j * B + i];
        mzero<B>(es.accLL);
        vzero<B>(es.accrL);
    }
#pragma unroll 1
    for (int j = 0; j < M - 1; ++j)
        ss_elim_step<B>(es, sD + (lo + j) * BB, sU + (lo + j) * BB, sR + (lo + j) * B);
    const double* Dp = sD + (lo + M - 1) * BB;
    const double* rp = sR + (lo + M - 1) * B;
TR_UNROLL
    for (int i = 0; i < BB; ++i) rec[RC::RDIAG + i] = Dp[i] - es.T[i];
TR_UNROLL
    for (int i = 0; i < BB; ++i) rec[RC::LDIAG + i] = es.accLL[i];
TR_UNROLL
    for (int i = 0; i < B; ++i)
TR_UNROLL
        for (int j = 0; j < B; ++j) rec[RC::LR + i * B + j] = es.W[j * B + i];
TR_UNROLL
    for (int i = 0; i < B; ++i) rec[RC::RRHS + i] = rp[i] - es.rc[i];
TR_UNROLL
    for (int i = 0; i < B; ++i) rec[RC::LRHS + i] = es.accrL[i];
    rec[RC::LOGDET] = ld0 + es.piv.logdet();
}

// ---- one lane's chunk as a Dirichlet problem (sweep 2) ----------------------------
// Both ends known (xl at the chunk's left separator, xr at its own last block): plain
// block Thomas over the M - 1 interior blocks, L -> diag slot, X = L^{-1}U -> upper slot,
// z -> rhs slot, then x_j = L^{-T}(z_j - X_j x_{j+1}) written over the rhs slots.
// Leader with a carried block P: P is eliminated first from its checkpoint, and x_P (the
// solution at the previous tile's last block) is returned in xP.
template <class C, int B>
SP_DEV void ss_dirichlet(double* sD, double* sU, double* sR, const double* Uprev, int lo, const double* carry,
                         const double* xl, const double* xr, double* xP) {
    constexpr int BB = B * B;
    constexpr int M = C::M;
    double T[BB], rc[B], Lp[BB], Xp[BB], zp[B];
    if (carry) {  // S_P, W_P (coupling to the run's left separator Z, x_Z = xl), r_P
        double S[BB], r[B], t1[B];
TR_UNROLL
        for (int i = 0; i < BB; ++i) S[i] = carry[i];
        mv<B>(t1, carry + BB, xl);
TR_UNROLL
        for (int i = 0; i < B; ++i) r[i] = carry[2 * BB + i] - t1[i];
        msym<B>(S);
        chol_nolog<B>(Lp, S);
        lsolve_v<B>(zp, Lp, r);
        lsolve<B>(Xp, Lp, Uprev);
        mtm_sym<B>(T, Xp, Xp);
        mtv<B>(rc, Xp, zp);
    } else {  // the left separator's x moves to the first block's right-hand side
        mzero<B>(T);
        mtv<B>(rc, Uprev, xl);  // P_{lo,lo-1} x_{lo-1} = Uprev^T xl
    }
#pragma unroll 1
    for (int j = 0; j < M - 1; ++j) {
        double* Dp = sD + (lo + j) * BB;
        double* Up = sU + (lo + j) * BB;
        double* rp = sR + (lo + j) * B;
        double S[BB], L[BB], U[BB], r[B], z[B], X[BB];
TR_UNROLL
        for (int i = 0; i < BB; ++i) S[i] = Dp[i] - T[i];
TR_UNROLL
        for (int i = 0; i < BB; ++i) U[i] = Up[i];
TR_UNROLL
        for (int i = 0; i < B; ++i) r[i] = rp[i] - rc[i];
        msym<B>(S);
        chol_nolog<B>(L, S);
        lsolve_v<B>(z, L, r);
        lsolve<B>(X, L, U);
        mtm_sym<B>(T, X, X);
        mtv<B>(rc, X, z);
TR_UNROLL
        for (int i = 0; i < BB; ++i) Dp[i] = L[i];
TR_UNROLL
        for (int i = 0; i < BB; ++i) Up[i] = X[i];
TR_UNROLL
        for (int i = 0; i < B; ++i) rp[i] = z[i];
    }
    double xn[B];
TR_UNROLL
    for (int i = 0; i < B; ++i) {
        xn[i] = xr[i];
        sR[(lo + M - 1) * B + i] = xr[i];
    }
#pragma unroll 1
    for (int j = M - 2; j >= 0; --j) {
        const double* Lq = sD + (lo + j) * BB;
        const double* Xq = sU + (lo + j) * BB;
        double* zq = sR + (lo + j) * B;
        double L[BB], a[B], t1[B], xj[B];
TR_UNROLL
        for (int i = 0; i < BB; ++i) L[i] = Lq[i];
        mv<B>(t1, Xq, xn);
TR_UNROLL
        for (int i = 0; i < B; ++i) a[i] = zq[i] - t1[i];
        ltsolve_v<B>(xj, L, a);
TR_UNROLL
        for (int i = 0; i < B; ++i) {
            zq[i] = xj[i];
            xn[i] = xj[i];
        }
    }
    if (carry) {
        double a[B], t1[B];
        mv<B>(t1, Xp, xn);
TR_UNROLL
        for (int i = 0; i < B; ++i) a[i] = zp[i] - t1[i];
        ltsolve_v<B>(xP, Lp, a);
    }
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

// ---- group tree (shuffles over W = 32, 16 or 8 lanes) ------------------------------
// In: every lane's record rec.  Out: the group leader's rec = the merged record of the W
// chunks; every other lane holds in F the factor of the merge that consumed its record.
// Fo + c * fs receives component c of the factor (registers: fs = 1; global: fs = lanes).
// mask: the lanes of this group (groups of one warp run independently: their runs may
// differ by a tile, so every warp-level primitive names only the group's own lanes).
// A failed merge pivot is reported at last(lane + stride - 1): the separator it eliminates
// is the last block of that lane's record.
template <int B, int W, class LastFn>
SP_DEV void ss_warp_tree_up(double* rec, double* Fo, int fs, unsigned mask, unsigned long long* status,
                            LastFn last) {
    constexpr int NR = Rec<B>::N, NF = Tree<B>::NF;
    using RC = Rec<B>;
    const int lane = threadIdx.x & (W - 1);
#pragma unroll 1
    for (int s = 1; s < W; s <<= 1) {
        double Bv[NR], Fm[NF];
TR_UNROLL
        for (int c = 0; c < NR; ++c) Bv[c] = __shfl_down_sync(mask, rec[c], s, W);
TR_UNROLL
        for (int c = 0; c < NF; ++c) Fm[c] = 0.0;
        if ((lane & (2 * s - 1)) == 0) {
            double Cm[NR];
            if (!tree_merge<B>(rec, Bv, Cm, Fm)) {  // rare: the pivot block, for origin vs echo
                double Sm[B * B];
TR_UNROLL
                for (int i = 0; i < B * B; ++i) Sm[i] = rec[RC::RDIAG + i] + Bv[RC::LDIAG + i];
                ss_report_pivot<B * B>(status, last(lane + s - 1), Sm);
            }
TR_UNROLL
            for (int c = 0; c < NR; ++c) rec[c] = Cm[c];
        }
TR_UNROLL
        for (int c = 0; c < NF; ++c) {
            const double f = __shfl_up_sync(mask, Fm[c], s, W);
            if ((lane & (2 * s - 1)) == s) Fo[c * fs] = f;
        }
    }
}
// In: the leader's (xL, xR) = the solution at the tile's outer separators.  Out: every
// lane's (xL, xR) = the solution at its chunk's left separator and at its own last block.
template <int B, int W>
SP_DEV void ss_warp_tree_down(const double* F, double* xL, double* xR, unsigned mask) {
    const int lane = threadIdx.x & (W - 1);
#pragma unroll 1
    for (int s = W / 2; s >= 1; s >>= 1) {
        double pL[B], pR[B], xM[B];
TR_UNROLL
        for (int i = 0; i < B; ++i) {
            pL[i] = __shfl_up_sync(mask, xL[i], s, W);
            pR[i] = __shfl_up_sync(mask, xR[i], s, W);
            xM[i] = 0.0;
        }
        const bool consumed = (lane & (2 * s - 1)) == s;
        if (consumed) {
            ss_unmerge<B>(F, pL, pR, xM);
TR_UNROLL
            for (int i = 0; i < B; ++i) {
                xL[i] = xM[i];
                xR[i] = pR[i];
            }
        }
TR_UNROLL
        for (int i = 0; i < B; ++i) {
            const double m = __shfl_down_sync(mask, xM[i], s, W);
            if ((lane & (2 * s - 1)) == 0) xR[i] = m;
        }
    }
}

// ---- CTA-level trees in shared memory (group records; the top's warp records) -------
// Forward tree over cnt records at slots [0, cnt) of R (component-major, row RS): leaves
// the merged record at slot 0 and the merge factors parked (tree.cuh layout).
// A failed merge pivot of node k in round j is reported at last(((2k + 1) << j) - 1).
template <int B, class LastFn>
SP_DEV void ss_tree_up(double* R, int RS, int cnt, unsigned long long* status, LastFn last) {
    const int J = tree_levels(cnt);
    for (int j = 0; j < J; ++j) {
        const int n = tree_width(cnt, j);
        TreeFwdScratch<B> sc;
        tree_fwd_compute<B>(R, RS, n, threadIdx.x, sc);
        if (!sc.ok) {  // origin or echo: the eliminated pivot block is finite or not
            double Sm[B * B];
TR_UNROLL
            for (int i = 0; i < B * B; ++i)
                Sm[i] = R[(Rec<B>::RDIAG + i) * RS + 2 * threadIdx.x] + R[(Rec<B>::LDIAG + i) * RS + 2 * threadIdx.x + 1];
            ss_report_pivot<B * B>(status, last(((2 * static_cast<int>(threadIdx.x) + 1) << j) - 1), Sm);
        }
        __syncthreads();
        tree_fwd_store<B>(R, RS, n, threadIdx.x, sc);
        __syncthreads();
    }
}
// Reverse tree, solution only: E[q * ES + i], slots 0 (left) and 1 (right) set by the
// caller; on return E holds x at the cnt + 1 record boundaries.
template <int B>
SP_DEV void ss_tree_down(const double* R, int RS, double* E, int ES, int cnt) {
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
                xL[q] = E[q * ES + k];
                xR[q] = E[q * ES + k + 1];
            }
            if (merged) {
                double F[TR::NF];
TR_UNROLL
                for (int c = 0; c < TR::NF; ++c) F[c] = R[c * RS + nn + k];
                ss_unmerge<B>(F, xL, xR, xM);
            }
        }
        __syncthreads();
        if (active) {
TR_UNROLL
            for (int q = 0; q < B; ++q) {
                E[q * ES + 2 * k] = xL[q];
                if (merged) E[q * ES + 2 * k + 1] = xM[q];
                if (last) E[q * ES + n] = xR[q];
            }
        }
        __syncthreads();
    }
}

// ---- tile staging ------------------------------------------------------------------
// Three bulk copies per tile (the group leader): diag, upper, rhs, each clipped to the
// blocks that exist and to an even block count (16-byte multiples); the odd block, the
// last upper block's absence and the identity padding past the end (D = I, U = 0, r = 0:
// x = 0, log det 0) are plain accesses.  Misaligned arrays are staged with plain loads.
template <class C, int B>
SP_DEV bool ss_tile_is_bulk(const SSArgs& a, long long tile) {
    return a.bulk && a.n - tile * C::WT >= 2;
}
template <class C, int B>
SP_DEV void ss_tile_issue(const SSArgs& a, double* wm, long long tile, unsigned long long policy, unsigned mask) {
    constexpr int BB = B * B;
    const int lane = threadIdx.x & (C::LPT - 1);
    const long long t0 = tile * C::WT;
    void* bar = wm + C::W_BAR;
    const int cD = static_cast<int>(min(static_cast<long long>(C::WT), a.n - t0));
    const int cU = static_cast<int>(max(0LL, min(static_cast<long long>(C::WT), a.n - 1 - t0)));
    const int bD = a.bulk ? (cD & ~1) : 0, bU = a.bulk ? (cU & ~1) : 0;
    __syncwarp(mask);
    if (lane == 0 && bD > 0) {
        ss_fence_async();
        ss_bar_expect(bar, static_cast<unsigned>((bD * BB + bU * BB + bD * B) * 8));
        ss_bulk_load(wm + C::W_D, a.diag + t0 * BB, static_cast<unsigned>(bD * BB * 8), bar, policy);
        if (bU > 0) ss_bulk_load(wm + C::W_U, a.up + t0 * BB, static_cast<unsigned>(bU * BB * 8), bar, policy);
        ss_bulk_load(wm + C::W_R, a.rhs + t0 * B, static_cast<unsigned>(bD * B * 8), bar, policy);
    }
    if (bD < C::WT || bU < C::WT) {  // ragged end or no bulk copies
        for (int i = bD * BB + lane; i < C::WT * BB; i += C::LPT) {
            const int e = i % BB;
            wm[C::W_D + i] = i < cD * BB ? a.diag[t0 * BB + i] : ((e / B == e % B) ? 1.0 : 0.0);
        }
        for (int i = bU * BB + lane; i < C::WT * BB; i += C::LPT)
            wm[C::W_U + i] = i < cU * BB ? a.up[t0 * BB + i] : 0.0;
        for (int i = bD * B + lane; i < C::WT * B; i += C::LPT)
            wm[C::W_R + i] = (i < cD * B && a.rhs) ? a.rhs[t0 * B + i] : 0.0;
    }
    // halo: the upper block that couples the previous tile's last block to this tile (8 bytes
    // off a 16-byte boundary, so not a bulk copy): asynchronous 8-byte copies, waited for with
    // the tile, so that the issuing lanes do not sit on an L2 / HBM round trip here
    for (int i = lane; i < BB; i += C::LPT) {
        if (t0 > 0) tree_copy(wm + C::W_UH + i, a.up + (t0 - 1) * BB + i);
        else wm[C::W_UH + i] = 0.0;
    }
}
template <class C, int B>
SP_DEV void ss_tile_wait(const SSArgs& a, double* wm, long long tile, unsigned& phase, unsigned mask) {
    if (ss_tile_is_bulk<C, B>(a, tile)) {
        ss_bar_wait(wm + C::W_BAR, phase);
        phase ^= 1u;
    }
    tree_copy_wait();  // the halo's cp.async
    __syncwarp(mask);  // halo / plain loads visible
}

template <class C, int B>
__global__ void __launch_bounds__(C::NT, 1) k_solve_stream(SSArgs a) {
    extern __shared__ double2 ss_sm2[];
    double* sm = reinterpret_cast<double*>(ss_sm2);
    constexpr int BB = B * B;
    constexpr int NR = C::NR, NF = C::NF, NK = C::NK, LPT = C::LPT;
    using RC = Rec<B>;
    const int t = threadIdx.x, lane = t & (LPT - 1), w = t / LPT;  // w: group within the CTA
    const bool lead = lane == 0;
    const unsigned gmask = LPT == 32 ? kFullWarp : (((1u << (LPT & 31)) - 1u) << ((t & 31) / LPT * LPT));
    const int cta = blockIdx.x;
    const long long GW = static_cast<long long>(a.G) * C::NW, gw = static_cast<long long>(cta) * C::NW + w;
    const long long tlo = a.ntiles * gw / GW, thi = a.ntiles * (gw + 1) / GW;
    const int T = static_cast<int>(thi - tlo);
    double* wm = sm + w * C::W_SIZE;
    double* WR = sm + C::OFF_WR;
    double* WE = sm + C::OFF_WE;
    double* ckw = a.ckpt + gw * a.Tmax * NK;
    double* tfw = a.tfac + gw * a.Tmax * (NF * LPT);
    unsigned phase = 0;
    if (lead) ss_bar_init(wm + C::W_BAR, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const bool want_x = a.x != nullptr;
    const bool retain = want_x && cta != 0;  // the last tile of sweep 1 stays on the SM
    const unsigned long long pol_keep = a.l2mode == 1 ? ss_policy_last() : ss_policy_normal();
    const unsigned long long pol_once = ss_policy_first();
    double rec[NR];
    double* ck = wm + C::W_P;  // the carried block's checkpoint (written and read by the leader)
    const double* Uprev = lead ? wm + C::W_UH : wm + C::W_U + (lane * C::M - 1) * BB;

    ss_stamp(a, 0);
    // ---- sweep 1: tiles ascending -> run record --------------------------------------
    ss_tile_issue<C, B>(a, wm, tlo, T == 1 && retain ? pol_once : pol_keep, gmask);
#pragma unroll 1
    for (int k = 0; k < T; ++k) {
        const long long tile = tlo + k;
        const bool keep = retain && k == T - 1;
        if (k > 0 && lead) {  // checkpoint of the carried block: S_P, W_P = LR^T, r_P
TR_UNROLL
            for (int i = 0; i < BB; ++i) ck[i] = rec[RC::RDIAG + i];
TR_UNROLL
            for (int i = 0; i < B; ++i)
TR_UNROLL
                for (int j = 0; j < B; ++j) ck[BB + i * B + j] = rec[RC::LR + j * B + i];
TR_UNROLL
            for (int i = 0; i < B; ++i) ck[2 * BB + i] = rec[RC::RRHS + i];
            if (want_x && !keep)
                for (int i = 0; i < NK; ++i) ckw[k * NK + i] = ck[i];
        }
        __syncwarp(gmask);
        if (k == 2) ss_stamp(a, 7);
        ss_tile_wait<C, B>(a, wm, tile, phase, gmask);
        if (k == 2) ss_stamp(a, 8);
        ss_eliminate<C, B>(wm + C::W_D, wm + C::W_U, wm + C::W_R, Uprev, lane * C::M, (k > 0 && lead) ? ck : nullptr,
                           rec, a.status, tile * C::WT + lane * C::M, a.n - 1);
        if (k == 2) ss_stamp(a, 9);
        // the tile buffer is free again: stage the next tile behind the tree rounds
        if (k + 1 < T) ss_tile_issue<C, B>(a, wm, tile + 1, (retain && k + 2 == T) ? pol_once : pol_keep, gmask);
        // the tree's merge factors go to tfac (L2) for sweep 2
        ss_warp_tree_up<B, LPT>(rec, tfw + static_cast<long long>(k) * (NF * LPT) + lane, LPT, gmask, a.status,
                                [&](int l) { return min(a.n - 1, tile * C::WT + (l + 1) * C::M - 1); });
        if (k == 2) ss_stamp(a, 10);
    }
    ss_stamp(a, 1);
    if (lead)
TR_UNROLL
        for (int c = 0; c < NR; ++c) WR[c * C::RSW + w] = rec[c];
    __syncthreads();
    // last block of the run of group g of this CTA / of CTA c
    auto run_last = [&](int g) {
        return min(a.n - 1, a.ntiles * (static_cast<long long>(cta) * C::NW + g + 1) / GW * C::WT - 1);
    };
    auto cta_last = [&](int c) {
        return min(a.n - 1, a.ntiles * (static_cast<long long>(min(c, a.G - 1) + 1) * C::NW) / GW * C::WT - 1);
    };
    ss_tree_up<B>(WR, C::RSW, C::NW, a.status, run_last);
    for (int c = t; c < NR; c += C::NT) a.crec[static_cast<long long>(c) * a.G + cta] = WR[c * C::RSW];
    __threadfence();
    __syncthreads();
    if (t == 0) atomicAdd(a.sync, 1ULL);
    ss_stamp(a, 2);

    // ---- top: CTA 0 solves the G-record reduced system ---------------------------
    // One record per thread (G <= NT, padded with identity records), a shuffle tree per
    // warp, the NT / 32 warp records through the shared-memory tree, and back down.
    if (cta == 0) {
        if (t == 0)
            while (ss_ld_acquire(a.sync) < a.arrive_target) __nanosleep(40);
        __syncthreads();
        ss_stamp(a, 3);
        const int G = a.G;
        double* TR_ = sm;                      // [NR][RST] over the tile buffers
        double* TE = TR_ + NR * C::RST;        // [B][EST]
        double grec[NR], gF[NF];
TR_UNROLL
        for (int c = 0; c < NR; ++c) {
            const bool diag1 = c >= RC::RDIAG && c < RC::RDIAG + BB && ((c - RC::RDIAG) % (B + 1) == 0);
            grec[c] = t < G ? __ldcg(a.crec + static_cast<long long>(c) * G + t) : (diag1 ? 1.0 : 0.0);
        }
TR_UNROLL
        for (int c = 0; c < NF; ++c) gF[c] = 0.0;
        ss_warp_tree_up<B, 32>(grec, gF, 1, kFullWarp, a.status, [&](int l) { return cta_last((t & ~31) + l); });
        if ((t & 31) == 0)
TR_UNROLL
            for (int c = 0; c < NR; ++c) TR_[c * C::RST + (t >> 5)] = grec[c];
        __syncthreads();
        ss_tree_up<B>(TR_, C::RST, C::NT / 32, a.status, [&](int wv) { return cta_last(32 * wv + 31); });
        if (t == 0) {  // top block
            double D[BB], r[B], Lc[BB], z[B], xx[B], ld;
TR_UNROLL
            for (int i = 0; i < BB; ++i) D[i] = TR_[(RC::RDIAG + i) * C::RST];
TR_UNROLL
            for (int i = 0; i < B; ++i) r[i] = TR_[(RC::RRHS + i) * C::RST];
            msym<B>(D);
            if (!chol<B>(Lc, D, ld)) ss_report_pivot<BB>(a.status, a.n - 1, D);
            lsolve_v<B>(z, Lc, r);
            ltsolve_v<B>(xx, Lc, z);
TR_UNROLL
            for (int i = 0; i < B; ++i) {
                TE[i * C::EST] = 0.0;
                TE[i * C::EST + 1] = xx[i];
            }
            if (a.logdet) *a.logdet = ld + TR_[RC::LOGDET * C::RST];
        }
        __syncthreads();
        if (want_x) {
            ss_tree_down<B>(TR_, C::RST, TE, C::EST, C::NT / 32);
            double xl[B], xr[B];
TR_UNROLL
            for (int i = 0; i < B; ++i) {
                xl[i] = (t & 31) == 0 ? TE[i * C::EST + (t >> 5)] : 0.0;
                xr[i] = (t & 31) == 0 ? TE[i * C::EST + (t >> 5) + 1] : 0.0;
            }
            ss_warp_tree_down<B, 32>(gF, xl, xr, kFullWarp);
            if (t < G)
TR_UNROLL
                for (int p = 0; p < B; ++p) a.xsep[static_cast<long long>(t) * B + p] = xr[p];
            __threadfence();
            __syncthreads();
            if (t == 0) ss_st_release(a.sync + 1, a.release_target);
        }
        ss_stamp(a, 4);
    }
    if (!want_x) return;
    if (cta != 0) {
        if (t == 0)
            while (ss_ld_acquire(a.sync + 1) < a.release_target) __nanosleep(40);
    }
    __syncthreads();
    ss_stamp(a, 5);

    // ---- CTA tree down: the solution at every run's boundaries ----------------------
    if (t < B) {
        WE[t * C::ESW] = cta > 0 ? __ldcg(a.xsep + static_cast<long long>(cta - 1) * B + t) : 0.0;
        WE[t * C::ESW + 1] = __ldcg(a.xsep + static_cast<long long>(cta) * B + t);
    }
    __syncthreads();
    ss_tree_down<B>(WR, C::RSW, WE, C::ESW, C::NW);
    double xZ[B], xRt[B];  // the run's left boundary, the current tile's right boundary
TR_UNROLL
    for (int i = 0; i < B; ++i) {
        xZ[i] = WE[i * C::ESW + w];
        xRt[i] = WE[i * C::ESW + w + 1];
    }

    // ---- sweep 2: tiles descending -> x -------------------------------------------
#pragma unroll 1
    for (int k = T - 1; k >= 0; --k) {
        const long long tile = tlo + k;
        const bool staged = retain && k == T - 1;
        if (!staged) ss_tile_issue<C, B>(a, wm, tile, pol_once, gmask);
        double F[NF];
        {
            const double* tf = tfw + static_cast<long long>(k) * (NF * LPT) + lane;
TR_UNROLL
            for (int c = 0; c < NF; ++c) F[c] = lead ? 0.0 : tf[c * LPT];
        }
        double xl[B], xr[B], xP[B];
TR_UNROLL
        for (int i = 0; i < B; ++i) {
            xl[i] = lead ? xZ[i] : 0.0;
            xr[i] = lead ? xRt[i] : 0.0;
            xP[i] = 0.0;
        }
        if (k == 2) ss_stamp(a, 11);
        ss_warp_tree_down<B, LPT>(F, xl, xr, gmask);
        if (k == 2) ss_stamp(a, 12);
        if (!staged) ss_tile_wait<C, B>(a, wm, tile, phase, gmask);
        if (k == 2) ss_stamp(a, 13);
        ss_dirichlet<C, B>(wm + C::W_D, wm + C::W_U, wm + C::W_R, Uprev, lane * C::M,
                           (k > 0 && lead) ? (staged ? ck : ckw + k * NK) : nullptr, xl, xr, xP);
TR_UNROLL
        for (int i = 0; i < B; ++i) xRt[i] = __shfl_sync(gmask, xP[i], 0, LPT);
        __syncwarp(gmask);
        if (k == 2) ss_stamp(a, 14);
        {
            const long long t0 = tile * C::WT;
            const long long lim = min(static_cast<long long>(C::WT), a.n - t0) * B;
            const double* sR = wm + C::W_R;
            double* xo = a.x + t0 * B;
            for (int i = lane; i < lim; i += LPT) __stcs(xo + i, sR[i]);
        }
        __syncwarp(gmask);
        if (k == 2) ss_stamp(a, 15);
    }
    ss_stamp(a, 6);
}
#endif  // SPINGP_HOST_EMU

}  // namespace spingp_dev
