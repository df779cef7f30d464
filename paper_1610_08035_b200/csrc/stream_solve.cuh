// stream_solve.cuh — cr_solve of a materialised SymBTD as
// ONE persistent kernel in which every WARP streams its own contiguous run of blocks
// through shared memory, tile by tile.
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
//              engine.cuh's elim_block (same record, Rec<B>).  With KEEP the factor is
//              written IN PLACE over the inputs as G = S^{-1}U, V = S^{-1}W, h = S^{-1}r
//              (2b²+b doubles per block, the size of the inputs).
//   warp tree  the 32 lane records are merged pairwise with warp shuffles (5 rounds, no
//              barrier, no shared memory); the merge factor of a pair is shuffled back
//              to the lane whose record was consumed and stays in its registers.
//   carry      a warp owns a contiguous run of tiles.  The record reduced so far (left
//              separator Z = the block before the run, right = the previous tile's last
//              block P) is carried in lane 0, which eliminates P as one more interior
//              block of its chunk; the warp tree then yields the carry of the next tile.
//   sweep 1    every warp reduces its tiles in ascending order, checkpointing the carry
//              (2b²+b doubles per tile); the NW warp records of a CTA are merged in shared
//              memory (tree.cuh) and the CTA record is published.
//   top        one grid-wide barrier; CTA 0 solves the G-record reduced system in shared
//              memory and publishes the solution at every CTA boundary and log det.
//   sweep 2    every warp walks its tiles in DESCENDING order: reload and re-eliminate
//              from the checkpoint (the last tile of sweep 1 is still in shared memory
//              and registers and is not re-read), un-merge the warp tree, back-substitute
//              x_j = h_j - G_j x_{j+1} - V_j x_L per lane, store x coalesced.
//
// HBM traffic: sweep 1 reads every block once; sweep 2 re-reads what L2 lost and writes x.
#pragma once

#include "tree.cuh"

namespace spingp_dev {

constexpr int ss_even(int v) { return (v + 1) & ~1; }

template <int B, int NW_, int M_>
struct SSCfg {
    static constexpr int NW = NW_;            // warps per CTA (independent pipelines)
    static constexpr int NT = 32 * NW_;
    static constexpr int M = M_;              // blocks per lane (M - 1 interior + 1 separator)
    static constexpr int WT = 32 * M_;        // blocks per warp tile
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
    static constexpr int RSW = ss_even(NW_);
    static constexpr int ESW = ss_even(NW_ + 1);
    static constexpr int OFF_WR = NW_ * W_SIZE;
    static constexpr int OFF_WE = OFF_WR + NR * RSW;
    static constexpr int SMEM_DOUBLES = ss_even(OFF_WE + B * ESW);
    static constexpr size_t SMEM_BYTES = static_cast<size_t>(SMEM_DOUBLES) * 8;
    // top system (CTA 0, over its tile buffers): records [NR][GS], tree [NR][RS], separators [B][ES]
    static constexpr int RS = ss_even(NT);
    static constexpr int ES = ss_even(NT + 1);
    static constexpr int TOP_FIXED = NR * RS + B * ES;   // + NR * GS must fit OFF_WR doubles
    static_assert(WT % 2 == 0, "tile pieces must be multiples of 16 bytes");
    static_assert(TOP_FIXED + 2 * NR < OFF_WR, "top system does not fit");
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
    double* crec;     // [NR][G] CTA records, component-major
    double* xsep;     // [G][B] solution at every CTA's last block
    double* ckpt;     // [G * NW][Tmax][NK] carry checkpoints (S_P, W_P, r_P) per tile
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

// ---- one lane's chunk: forward elimination (in place when KEEP) ----------------
template <int B>
struct SSElim {
    double T[B * B], rc[B], W[B * B], accLL[B * B], accrL[B];
    LogDetAcc piv;
    bool ok;
};
// One interior block with diagonal D, coupling U (to the next block) and rhs r; with KEEP
// V = S^{-1}W -> Vo, G = S^{-1}U -> Go, h = S^{-1}r -> ho (they may be D, U, r's own
// storage: everything is read before anything is written).
template <int B, bool KEEP>
SP_DEV void ss_elim_step(SSElim<B>& es, const double* Dp, const double* Up, const double* rp, double* Vo, double* Go,
                         double* ho) {
    constexpr int BB = B * B;
    double S[BB], L[BB], U[BB], r[B], z[B], X[BB], Y[BB], Gm[BB];
TR_UNROLL
    for (int i = 0; i < BB; ++i) S[i] = Dp[i] - es.T[i];
TR_UNROLL
    for (int i = 0; i < BB; ++i) U[i] = Up[i];
TR_UNROLL
    for (int i = 0; i < B; ++i) r[i] = rp[i] - es.rc[i];
    msym<B>(S);
    es.ok = chol<B>(L, S, es.piv) && es.ok;
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
    if (KEEP) {
        double h[B];
        ltsolve<B>(Gm, L, X);
TR_UNROLL
        for (int i = 0; i < BB; ++i) Go[i] = Gm[i];
        ltsolve<B>(Gm, L, Y);
TR_UNROLL
        for (int i = 0; i < BB; ++i) Vo[i] = Gm[i];
        ltsolve_v<B>(h, L, z);
TR_UNROLL
        for (int i = 0; i < B; ++i) ho[i] = h[i];
    }
}

// Lane chunk lo .. lo+M-1 of the warp tile at (sD, sU, sR).  Uprev = the upper block that
// couples block lo-1 to lo.  carry (lane 0, tiles after the warp's first): the checkpoint
// (S_P, W_P = P_{P,Z}, r_P) of the carried block P, eliminated first (kept factor -> sP),
// with the run's accumulated left-separator terms and log det in rec (LDIAG, LRHS, LOGDET).
template <class C, int B, bool KEEP>
SP_DEV bool ss_eliminate(double* sD, double* sU, double* sR, const double* Uprev, int lo, const double* carry,
                         double* sP, double* rec) {
    constexpr int BB = B * B;
    constexpr int M = C::M;
    using RC = Rec<B>;
    SSElim<B> es;
    es.piv.init();
    es.ok = true;
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
        ss_elim_step<B, KEEP>(es, carry, Uprev, carry + 2 * BB, sP, sP + BB, sP + 2 * BB);
    } else {
TR_UNROLL
        for (int i = 0; i < B; ++i)
TR_UNROLL
            for (int j = 0; j < B; ++j) es.W[i * B + j] = Uprev[j * B + i];
        mzero<B>(es.accLL);
        vzero<B>(es.accrL);
    }
#pragma unroll 1
    for (int j = 0; j < M - 1; ++j) {
        double* Dp = sD + (lo + j) * BB;
        double* Up = sU + (lo + j) * BB;
        double* rp = sR + (lo + j) * B;
        ss_elim_step<B, KEEP>(es, Dp, Up, rp, Dp, Up, rp);
    }
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
    return es.ok;
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

// ---- warp tree (shuffles) -------------------------------------------------------
// In: every lane's record rec.  Out: lane 0's rec = the merged record of the 32 chunks;
// lane l > 0 holds in F the factor of the merge that consumed its record (round ctz(l)).
template <int B>
SP_DEV bool ss_warp_tree_up(double* rec, double* F) {
    constexpr int NR = Rec<B>::N, NF = Tree<B>::NF;
    const int lane = threadIdx.x & 31;
    bool ok = true;
#pragma unroll 1
    for (int s = 1; s < 32; s <<= 1) {
        double Bv[NR], Fm[NF];
TR_UNROLL
        for (int c = 0; c < NR; ++c) Bv[c] = __shfl_down_sync(kFullWarp, rec[c], s);
TR_UNROLL
        for (int c = 0; c < NF; ++c) Fm[c] = 0.0;
        if ((lane & (2 * s - 1)) == 0) {
            double Cm[NR];
            ok = tree_merge<B>(rec, Bv, Cm, Fm) && ok;
TR_UNROLL
            for (int c = 0; c < NR; ++c) rec[c] = Cm[c];
        }
TR_UNROLL
        for (int c = 0; c < NF; ++c) {
            const double f = __shfl_up_sync(kFullWarp, Fm[c], s);
            if ((lane & (2 * s - 1)) == s) F[c] = f;
        }
    }
    return ok;
}
// In: lane 0's (xL, xR) = the solution at the tile's outer separators.  Out: every lane's
// (xL, xR) = the solution at its chunk's left separator and at its own last block.
template <int B>
SP_DEV void ss_warp_tree_down(const double* F, double* xL, double* xR) {
    const int lane = threadIdx.x & 31;
#pragma unroll 1
    for (int s = 16; s >= 1; s >>= 1) {
        double pL[B], pR[B], xM[B];
TR_UNROLL
        for (int i = 0; i < B; ++i) {
            pL[i] = __shfl_up_sync(kFullWarp, xL[i], s);
            pR[i] = __shfl_up_sync(kFullWarp, xR[i], s);
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
            const double m = __shfl_down_sync(kFullWarp, xM[i], s);
            if ((lane & (2 * s - 1)) == 0) xR[i] = m;
        }
    }
}

// ---- CTA-level trees in shared memory (warp records; the top system) -------------
// Forward tree over cnt records at slots [0, cnt) of R (component-major, row RS): leaves
// the merged record at slot 0 and the merge factors parked (tree.cuh layout).
template <int B>
SP_DEV bool ss_tree_up(double* R, int RS, int cnt) {
    bool ok = true;
    const int J = tree_levels(cnt);
    for (int j = 0; j < J; ++j) {
        const int n = tree_width(cnt, j);
        TreeFwdScratch<B> sc;
        tree_fwd_compute<B>(R, RS, n, threadIdx.x, sc);
        ok = ok && sc.ok;
        __syncthreads();
        tree_fwd_store<B>(R, RS, n, threadIdx.x, sc);
        __syncthreads();
    }
    return ok;
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
// Merge of records read with strides -> record at Cp, merge factor at Fp.  A real call:
// it runs on a few threads of CTA 0 only, and its ~130 live doubles must not set the
// register count of the whole kernel.
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

// ---- warp tile staging -----------------------------------------------------------
// Full tiles with every upper block present go through three bulk copies (lane 0); the
// last tile(s) and misaligned arrays are staged with plain loads, padded with identity
// blocks past the end (D = I, U = 0, r = 0: x = 0, log det 0).
template <class C, int B>
SP_DEV bool ss_tile_is_bulk(const SSArgs& a, long long tile) {
    return a.bulk && (tile + 1) * C::WT <= a.n - 1;
}
template <class C, int B>
SP_DEV void ss_tile_issue(const SSArgs& a, double* wm, long long tile, unsigned long long policy) {
    constexpr int BB = B * B;
    const int lane = threadIdx.x & 31;
    const long long t0 = tile * C::WT;
    void* bar = wm + C::W_BAR;
    __syncwarp();
    if (ss_tile_is_bulk<C, B>(a, tile)) {
        if (lane == 0) {
            ss_fence_async();
            constexpr unsigned nbD = C::WT * BB * 8, nbR = C::WT * B * 8;
            ss_bar_expect(bar, 2 * nbD + nbR);
            ss_bulk_load(wm + C::W_D, a.diag + t0 * BB, nbD, bar, policy);
            ss_bulk_load(wm + C::W_U, a.up + t0 * BB, nbD, bar, policy);
            ss_bulk_load(wm + C::W_R, a.rhs + t0 * B, nbR, bar, policy);
        }
    } else {
        const long long nd = a.n * BB, nu = (a.n - 1) * BB, nr = a.n * B;
        for (int i = lane; i < C::WT * BB; i += 32) {
            const long long gi = t0 * BB + i;
            const int e = i % BB;
            wm[C::W_D + i] = gi < nd ? a.diag[gi] : ((e / B == e % B) ? 1.0 : 0.0);
            wm[C::W_U + i] = gi < nu ? a.up[gi] : 0.0;
        }
        for (int i = lane; i < C::WT * B; i += 32) {
            const long long gi = t0 * B + i;
            wm[C::W_R + i] = (gi < nr && a.rhs) ? a.rhs[gi] : 0.0;
        }
    }
    if (lane < BB) wm[C::W_UH + lane] = t0 > 0 ? a.up[(t0 - 1) * BB + lane] : 0.0;
}
template <class C, int B>
SP_DEV void ss_tile_wait(const SSArgs& a, double* wm, long long tile, unsigned& phase) {
    if (ss_tile_is_bulk<C, B>(a, tile)) {
        ss_bar_wait(wm + C::W_BAR, phase);
        phase ^= 1u;
    }
    __syncwarp();  // halo / plain loads visible
}

// eliminate the staged tile -> lane records.  ck: lane 0's checkpoint of the carried block
// (has_carry: every tile but the warp's first); lane 0's rec holds the run's record.
template <class C, int B, bool KEEP>
SP_DEV void ss_tile_reduce(const SSArgs& a, double* wm, long long tile, bool has_carry, const double* ck,
                           double* rec) {
    constexpr int BB = B * B;
    const int lane = threadIdx.x & 31;
    const double* Uprev = lane == 0 ? wm + C::W_UH : wm + C::W_U + (lane * C::M - 1) * BB;
    const bool carry = has_carry && lane == 0;
    const bool ok = ss_eliminate<C, B, KEEP>(wm + C::W_D, wm + C::W_U, wm + C::W_R, Uprev, lane * C::M,
                                             carry ? ck : nullptr, wm + C::W_P, rec);
    if (!ok) report(a.status, min(a.n - 1, tile * C::WT + lane * C::M), ST_NOT_PD);
}

template <class C, int B>
__global__ void __launch_bounds__(C::NT, 1) k_solve_stream(SSArgs a) {
    extern __shared__ double2 ss_sm2[];
    double* sm = reinterpret_cast<double*>(ss_sm2);
    constexpr int BB = B * B;
    constexpr int NR = C::NR, NF = C::NF, NK = C::NK;
    using RC = Rec<B>;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int cta = blockIdx.x;
    const long long GW = static_cast<long long>(a.G) * C::NW, gw = static_cast<long long>(cta) * C::NW + w;
    const long long tlo = a.ntiles * gw / GW, thi = a.ntiles * (gw + 1) / GW;
    const int T = static_cast<int>(thi - tlo);
    double* wm = sm + w * C::W_SIZE;
    double* WR = sm + C::OFF_WR;
    double* WE = sm + C::OFF_WE;
    double* ckw = a.ckpt + gw * a.Tmax * NK;
    unsigned phase = 0;
    if (lane == 0) ss_bar_init(wm + C::W_BAR, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const bool want_x = a.x != nullptr;
    const bool retain = want_x && cta != 0;  // the last tile of sweep 1 stays on the SM
    const unsigned long long pol_keep = a.l2mode == 1 ? ss_policy_last() : ss_policy_normal();
    const unsigned long long pol_once = ss_policy_first();
    double rec[NR], F[NF], ck[NK];
TR_UNROLL
    for (int c = 0; c < NF; ++c) F[c] = 0.0;
TR_UNROLL
    for (int c = 0; c < NK; ++c) ck[c] = 0.0;

    ss_stamp(a, 0);
    // ---- sweep 1: tiles ascending -> warp record -----------------------------------
    ss_tile_issue<C, B>(a, wm, tlo, T == 1 && retain ? pol_once : pol_keep);
#pragma unroll 1
    for (int k = 0; k < T; ++k) {
        const long long tile = tlo + k;
        const bool keep = retain && k == T - 1;
        if (k > 0 && lane == 0) {  // checkpoint of the carried block: S_P, W_P = LR^T, r_P
TR_UNROLL
            for (int i = 0; i < BB; ++i) ck[i] = rec[RC::RDIAG + i];
TR_UNROLL
            for (int i = 0; i < B; ++i)
TR_UNROLL
                for (int j = 0; j < B; ++j) ck[BB + i * B + j] = rec[RC::LR + j * B + i];
TR_UNROLL
            for (int i = 0; i < B; ++i) ck[2 * BB + i] = rec[RC::RRHS + i];
            if (want_x)
TR_UNROLL
                for (int i = 0; i < NK; ++i) ckw[k * NK + i] = ck[i];
        }
        ss_tile_wait<C, B>(a, wm, tile, phase);
        if (keep) ss_tile_reduce<C, B, true>(a, wm, tile, k > 0, ck, rec);
        else ss_tile_reduce<C, B, false>(a, wm, tile, k > 0, ck, rec);
        // the tile buffer is free again: stage the next tile behind the tree rounds
        if (k + 1 < T) ss_tile_issue<C, B>(a, wm, tile + 1, (retain && k + 2 == T) ? pol_once : pol_keep);
        if (!ss_warp_tree_up<B>(rec, F)) report(a.status, min(a.n - 1, tile * C::WT), ST_NOT_PD);
    }
    ss_stamp(a, 1);
    if (lane == 0)
TR_UNROLL
        for (int c = 0; c < NR; ++c) WR[c * C::RSW + w] = rec[c];
    __syncthreads();
    if (!ss_tree_up<B>(WR, C::RSW, C::NW)) report(a.status, a.n - 1, ST_NOT_PD);
    for (int c = t; c < NR; c += C::NT) a.crec[static_cast<long long>(c) * a.G + cta] = WR[c * C::RSW];
    __threadfence();
    __syncthreads();
    if (t == 0) atomicAdd(a.sync, 1ULL);
    ss_stamp(a, 2);

    // ---- top: CTA 0 solves the G-record reduced system ---------------------------
    if (cta == 0) {
        if (t == 0)
            while (ss_ld_acquire(a.sync) < a.arrive_target) __nanosleep(40);
        __syncthreads();
        ss_stamp(a, 3);
        const int G = a.G, GS = (G + 1) & ~1;
        double* GR = sm;                 // [NR][GS] over the tile buffers
        double* R = GR + NR * GS;        // [NR][RS]
        double* E = R + NR * C::RS;      // [B][ES]
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
        if (!ss_tree_up<B>(R, C::RS, NG)) report(a.status, a.n - 1, ST_NOT_PD);
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
            ss_tree_down<B>(R, C::RS, E, C::ES, NG);
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
                    double Fg[NF];
TR_UNROLL
                    for (int c = 0; c < NF; ++c) Fg[c] = GR[c * GS + g0 + i];
                    ss_unmerge<B>(Fg, xL, xR, xM);
TR_UNROLL
                    for (int p = 0; p < B; ++p) xR[p] = xM[p];
                }
            }
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

    // ---- CTA tree down: the solution at every warp run's boundaries ---------------
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
        if (!staged) {
            ss_tile_issue<C, B>(a, wm, tile, pol_once);
            if (k > 0 && lane == 0)
TR_UNROLL
                for (int i = 0; i < NK; ++i) ck[i] = ckw[k * NK + i];
            rec[RC::LOGDET] = 0.0;
TR_UNROLL
            for (int i = 0; i < BB; ++i) rec[RC::LDIAG + i] = 0.0;
TR_UNROLL
            for (int i = 0; i < B; ++i) rec[RC::LRHS + i] = 0.0;
            ss_tile_wait<C, B>(a, wm, tile, phase);
            ss_tile_reduce<C, B, true>(a, wm, tile, k > 0, ck, rec);
            ss_warp_tree_up<B>(rec, F);
        }
        double xl[B], xr[B];
TR_UNROLL
        for (int i = 0; i < B; ++i) {
            xl[i] = lane == 0 ? xZ[i] : 0.0;
            xr[i] = lane == 0 ? xRt[i] : 0.0;
        }
        ss_warp_tree_down<B>(F, xl, xr);
        {  // back-substitution of this lane's chunk, x over the rhs slots
            const int lo = lane * C::M;
            double* sR = wm + C::W_R;
            double xn[B];
TR_UNROLL
            for (int i = 0; i < B; ++i) {
                xn[i] = xr[i];
                sR[(lo + C::M - 1) * B + i] = xr[i];
            }
#pragma unroll 1
            for (int j = C::M - 2; j >= 0; --j) {
                const double* Gp = wm + C::W_U + (lo + j) * BB;
                const double* Vp = wm + C::W_D + (lo + j) * BB;
                double* hp = sR + (lo + j) * B;
                double xj[B];
TR_UNROLL
                for (int i = 0; i < B; ++i) {
                    double s = hp[i];
TR_UNROLL
                    for (int c = 0; c < B; ++c) s = fma(-Gp[i * B + c], xn[c], s);
TR_UNROLL
                    for (int c = 0; c < B; ++c) s = fma(-Vp[i * B + c], xl[c], s);
                    xj[i] = s;
                }
TR_UNROLL
                for (int i = 0; i < B; ++i) {
                    hp[i] = xj[i];
                    xn[i] = xj[i];
                }
            }
            // the carried block P (the previous tile's last block): the next right boundary
            double xP[B];
            const double* sP = wm + C::W_P;
TR_UNROLL
            for (int i = 0; i < B; ++i) {
                double s = 0.0;
                if (lane == 0 && k > 0) {
                    s = sP[2 * BB + i];
TR_UNROLL
                    for (int c = 0; c < B; ++c) s = fma(-sP[BB + i * B + c], xn[c], s);
TR_UNROLL
                    for (int c = 0; c < B; ++c) s = fma(-sP[i * B + c], xl[c], s);
                }
                xP[i] = s;
            }
TR_UNROLL
            for (int i = 0; i < B; ++i) xRt[i] = __shfl_sync(kFullWarp, xP[i], 0);
        }
        __syncwarp();
        {
            const long long t0 = tile * C::WT;
            const long long lim = min(static_cast<long long>(C::WT), a.n - t0) * B;
            const double* sR = wm + C::W_R;
            double* xo = a.x + t0 * B;
            for (int i = lane; i < lim; i += 32) __stcs(xo + i, sR[i]);
        }
        __syncwarp();
    }
    ss_stamp(a, 6);
}
#endif  // SPINGP_HOST_EMU

}  // namespace spingp_dev
