// strip_solve.cuh — cr_solve of a materialised SymBTD:
// one persistent kernel, ONE LANE PER LONG CHUNK, the blocks staged strip by strip.
//
// stream_solve.cuh stages contiguous tiles and therefore has to merge the 32 lane records
// of every tile with a shuffle tree: 73% of its first sweep (profiles/r02_stream_solve.md).
// Here lane l of a warp owns one contiguous chunk of Lc blocks (N / #lanes, ~26 at 1 M
// blocks) and walks it in sub-tiles of MB blocks; the warp stages the 32 strips of a
// sub-tile cooperatively: consecutive lanes copy consecutive 16-byte pieces of one strip
// with cp.async (every strip piece is >= 96 contiguous bytes, so the sectors are used in
// full, unlike a thread that walks its own strip).  There is no tree per tile: a lane's
// elimination state simply continues into its next sub-tile.
//
//   sweep 1  spike elimination along the chunk (stream_solve.cuh's ss_elim_step, the
//            records of engine.cuh), the state (T, W, rc) checkpointed at every sub-tile
//            start (2b²+b doubles per MB blocks); one shuffle tree per warp over the 32
//            chunk records, the CTA's 8 warp records in shared memory, one grid barrier,
//            the top system in CTA 0, and back down to (x_left, x_right) of every lane.
//   sweep 2  sub-tiles in descending order: restore the checkpoint, fold x_left into the
//            right-hand side (rc = rc0 + W x_left), plain block Thomas over the MB blocks
//            in place, back-substitute from the block to the right, store x cooperatively.
//            The last sub-tile of sweep 1 is still in shared memory and is not re-read.
#pragma once

#include "stream_solve.cuh"

namespace spingp_dev {

// strip stride in shared memory: even (16-byte pieces) with an odd half, so that the 32
// strips of a warp fall on distinct bank pairs within every group of 8 lanes
constexpr int st_pad(int x) { return ((x / 2) & 1) ? x : x + 2; }

template <int B, int NWARP, int MB_>
struct STCfg {
    static constexpr int NW = NWARP;
    static constexpr int NT = 32 * NWARP;
    static constexpr int MB = MB_;            // blocks per lane and sub-tile (even)
    static constexpr int BB = B * B;
    static constexpr int NR = Rec<B>::N;
    static constexpr int NF = Tree<B>::NF;
    static constexpr int NCK = 2 * BB + B;    // checkpoint: T, W, rc
    static constexpr int SD = st_pad(MB_ * BB);   // strip strides (doubles)
    static constexpr int SR = st_pad(MB_ * B);
    static constexpr int W_D = 0;
    static constexpr int W_U = 32 * SD;
    static constexpr int W_R = 64 * SD;
    static constexpr int W_SIZE = ss_even(64 * SD + 32 * SR);
    static constexpr int RSW = ss_even(NW);
    static constexpr int ESW = ss_even(NW + 1);
    static constexpr int OFF_WR = NW * W_SIZE;
    static constexpr int OFF_WE = OFF_WR + NR * RSW;
    static constexpr int OFF_TOP = ss_even(OFF_WE + B * ESW);  // top system: [NR][RST] + [B][EST]
    static constexpr int RST = ss_even(NT / 32);
    static constexpr int EST = ss_even(NT / 32 + 1);
    static constexpr int SMEM_DOUBLES = ss_even(OFF_TOP + NR * RST + B * EST);
    static constexpr size_t SMEM_BYTES = static_cast<size_t>(SMEM_DOUBLES) * 8;
    static_assert(MB_ % 2 == 0, "strip pieces must be multiples of 16 bytes");
};

#ifndef SPINGP_HOST_EMU
SP_DEV void st_cp16(double* dst, const double* src, unsigned long long policy) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "l"(policy)
                 : "memory");
}
SP_DEV void st_cp_wait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

SP_DEV void st_cp_wait_but_one() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
SP_DEV void st_cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

// Stage blocks [j0, j0 + NB) of sub-tile s of the warp's 32 strips.  wfl = global index of the
// warp's lane 0; strip q belongs to lane q and starts at block (wfl + q) Lc + s MB.  When the
// whole piece lies inside the matrix (all but the last warp with data) every 16-byte piece is
// a cp.async with compile-time piece -> (strip, offset) arithmetic and no bounds checks;
// otherwise strip by strip: inside -> cp.async, past the end -> identity padding (D = I, U = 0,
// r = 0), the strip across the end (or misaligned arrays) element by element.
template <class C, int B, int NB>
SP_DEV void st_stage(const SSArgs& a, double* wm, long long wfl, int qin, int s, int j0, unsigned long long policy) {
    constexpr int BB = B * B, MB = C::MB;
    constexpr int nD = NB * BB / 2, nR = NB * B / 2;  // 16-byte pieces per strip
    static_assert(NB % 2 == 0, "16-byte pieces");
    const int lane = threadIdx.x & 31;
    const long long gb0 = wfl * a.Lc + static_cast<long long>(s) * MB + j0;  // strip 0's first block
    double* wD = wm + C::W_D + j0 * BB;
    double* wU = wm + C::W_U + j0 * BB;
    double* wR = wm + C::W_R + j0 * B;
    if (qin > 0) {  // strips [0, qin): whole chunks inside the matrix, aligned arrays
        const double* dbase = a.diag + gb0 * BB;
        const double* ubase = a.up + gb0 * BB;
        const double* rbase = a.rhs + gb0 * B;
        const int strideD = static_cast<int>(a.Lc) * BB, strideR = static_cast<int>(a.Lc) * B;
TR_UNROLL
        for (int it = 0; it < (32 * nD + 31) / 32; ++it) {
            const int p = it * 32 + lane, q = p / nD, wi = p - q * nD;
            if (q < qin) {
                st_cp16(wD + q * C::SD + 2 * wi, dbase + q * strideD + 2 * wi, policy);
                st_cp16(wU + q * C::SD + 2 * wi, ubase + q * strideD + 2 * wi, policy);
            }
        }
TR_UNROLL
        for (int it = 0; it < (32 * nR + 31) / 32; ++it) {
            const int p = it * 32 + lane, q = p / nR, wi = p - q * nR;
            if (q < qin) st_cp16(wR + q * C::SR + 2 * wi, rbase + q * strideR + 2 * wi, policy);
        }
    }
    if (qin == 32) return;
    // the chunk across the end of the matrix (identity padding past it: D = I, U = 0, r = 0),
    // or every chunk when the arrays are misaligned: element by element.  Chunks that start
    // past the end are never read (their lanes sit the sweeps out).
    const long long nd = a.n * BB, nu = (a.n - 1) * BB, nr = a.n * B;
    const long long own = (a.n + a.Lc - 1) / a.Lc - wfl;  // lanes of this warp that own a block
    const int nq = static_cast<int>(max(0LL, min(32LL, own))) - qin;
    for (int p = lane; p < nq * NB * BB; p += 32) {
        const int q = qin + p / (NB * BB), e = p % (NB * BB);
        const long long gi = (gb0 + q * a.Lc) * BB + e;
        wD[q * C::SD + e] = gi < nd ? a.diag[gi] : (((e % BB) % (B + 1) == 0) ? 1.0 : 0.0);
        wU[q * C::SD + e] = gi < nu ? a.up[gi] : 0.0;
    }
    for (int p = lane; p < nq * NB * B; p += 32) {
        const int q = qin + p / (NB * B), e = p % (NB * B);
        const long long gi = (gb0 + q * a.Lc) * B + e;
        wR[q * C::SR + e] = (gi < nr && a.rhs) ? a.rhs[gi] : 0.0;
    }
}

// Store the sub-tile's solution (the rhs slots of the 32 strips) to x.
template <class C, int B>
SP_DEV void st_store_x(const SSArgs& a, const double* wm, long long wfl, int s) {
    constexpr int MB = C::MB;
    constexpr int nR = MB * B / 2;
    const int lane = threadIdx.x & 31;
    const long long gb0 = wfl * a.Lc + static_cast<long long>(s) * MB;
    const long long last = gb0 + 31 * a.Lc + MB;
    if ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && last <= a.n) {
        double* xbase = a.x + gb0 * B;
        const int strideR = static_cast<int>(a.Lc) * B;
TR_UNROLL
        for (int it = 0; it < (32 * nR + 31) / 32; ++it) {
            const int p = it * 32 + lane, q = p / nR, wi = p - q * nR;
            if (32 * nR % 32 == 0 || p < 32 * nR) {
                const double* src = wm + C::W_R + q * C::SR + 2 * wi;
                __stcs(reinterpret_cast<double2*>(xbase + q * strideR + 2 * wi), make_double2(src[0], src[1]));
            }
        }
        return;
    }
    const long long nr = a.n * B;
    for (int p = lane; p < 32 * MB * B; p += 32) {
        const int q = p / (MB * B), e = p - q * (MB * B);
        const long long gi = (gb0 + q * a.Lc) * B + e;
        if (gi < nr) a.x[gi] = wm[C::W_R + q * C::SR + e];
    }
}

template <class C, int B>
__global__ void __launch_bounds__(C::NT, 1) k_solve_strip(SSArgs a) {
    extern __shared__ double2 st_sm2[];
    double* sm = reinterpret_cast<double*>(st_sm2);
    constexpr int BB = B * B;
    constexpr int NR = C::NR, NF = C::NF, NCK = C::NCK, MB = C::MB;
    using RC = Rec<B>;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int cta = blockIdx.x;
    const long long gwarp = static_cast<long long>(cta) * C::NW + w, wfl = gwarp * 32;
    const long long g0 = (wfl + lane) * a.Lc;  // first block of this lane's chunk
    const int nsub = a.nsub;  // Lc = nsub * MB: every sub-tile is full
    double* wm = sm + w * C::W_SIZE;
    double* sD = wm + C::W_D + lane * C::SD;
    double* sU = wm + C::W_U + lane * C::SD;
    double* sR = wm + C::W_R + lane * C::SR;
    double* WR = sm + C::OFF_WR;
    double* WE = sm + C::OFF_WE;
    double* ckw = a.ckpt + gwarp * nsub * (NCK * 32) + lane;
    double* tfw = a.tfac + gwarp * (NF * 32) + lane;
    const bool want_x = a.x != nullptr;
    const bool empty = wfl * a.Lc >= a.n;  // a warp past the end of the matrix: neutral records
    const bool off = g0 >= a.n;            // a lane whose chunk starts past the end: likewise
    // L2 hints (a.l2mode = 1): sweep 2 re-reads the sub-tiles in reverse order, so the last few
    // of sweep 1 are worth keeping in L2, the first ones are not, and sweep 2's own loads are dead
    const unsigned long long pol_n = ss_policy_normal();
    const unsigned long long pol_first = a.l2mode ? ss_policy_first() : pol_n;
    const unsigned long long pol_last = a.l2mode ? ss_policy_last() : pol_n;
    const int keep_from = nsub - 1 - a.l2keep;  // sub-tiles >= this one: evict_last in sweep 1
    // lanes of this warp whose whole chunk (and its last upper block) lies inside the matrix
    const int qin = a.bulk ? static_cast<int>(max(0LL, min(32LL, (a.n - 1) / a.Lc - wfl))) : 0;

    // the block that couples this chunk to its left separator (the previous lane's last block)
    double Up0[BB];
TR_UNROLL
    for (int i = 0; i < BB; ++i) Up0[i] = (g0 > 0 && g0 < a.n) ? a.up[(g0 - 1) * BB + i] : 0.0;

    ss_stamp(a, 0);
    // ---- sweep 1 ---------------------------------------------------------------------
    double rec[NR];
    {
        SSElim<B> es;
        es.piv.init();
        es.status = a.status;
        es.idx = g0;
        es.nmax = a.n - 1;
        mzero<B>(es.T);
        vzero<B>(es.rc);
        mzero<B>(es.accLL);
        vzero<B>(es.accrL);
TR_UNROLL
        for (int i = 0; i < B; ++i)
TR_UNROLL
            for (int j = 0; j < B; ++j) es.W[i * B + j] = Up0[j * B + i];
        // sub-tiles are staged in halves of MB / 2 blocks, one half ahead of the elimination
        // (the half being filled was eliminated one step earlier)
        constexpr int HB = MB / 2;
        if (!empty) st_stage<C, B, HB>(a, wm, wfl, qin, 0, 0, 0 >= keep_from ? pol_last : pol_first);
        st_cp_commit();
#pragma unroll 1
        for (int sh = 0; sh < 2 * nsub && !empty; ++sh) {
            const int s = sh >> 1, h = sh & 1;
            __syncwarp();
            if (sh + 1 < 2 * nsub)
                st_stage<C, B, HB>(a, wm, wfl, qin, (sh + 1) >> 1, ((sh + 1) & 1) * HB,
                                   ((sh + 1) >> 1) >= keep_from ? pol_last : pol_first);
            st_cp_commit();
            if (want_x && s > 0 && h == 0) {  // the state at the sub-tile's start, for sweep 2
                double* ck = ckw + static_cast<long long>(s) * (NCK * 32);
TR_UNROLL
                for (int i = 0; i < BB; ++i) ck[i * 32] = es.T[i];
TR_UNROLL
                for (int i = 0; i < BB; ++i) ck[(BB + i) * 32] = es.W[i];
TR_UNROLL
                for (int i = 0; i < B; ++i) ck[(2 * BB + i) * 32] = es.rc[i];
            }
            if (sh == 6) ss_stamp(a, 7);
            st_cp_wait_but_one();
            __syncwarp();
            if (sh == 6) ss_stamp(a, 8);
            const int nel = sh == 2 * nsub - 1 ? HB - 1 : HB;
#pragma unroll 1
            for (int j = 0; j < nel && !off; ++j)
                ss_elim_step<B>(es, sD + (h * HB + j) * BB, sU + (h * HB + j) * BB, sR + (h * HB + j) * B);
            if (sh == 6) ss_stamp(a, 9);
            if (sh == 7) ss_stamp(a, 10);
        }
        // the chunk's record: its last block is the separator
        const double* Dp = sD + (MB - 1) * BB;
        const double* rp = sR + (MB - 1) * B;
TR_UNROLL
        for (int i = 0; i < BB; ++i) rec[RC::RDIAG + i] = (empty || off) ? ((i % (B + 1) == 0) ? 1.0 : 0.0) : Dp[i] - es.T[i];
TR_UNROLL
        for (int i = 0; i < BB; ++i) rec[RC::LDIAG + i] = es.accLL[i];
TR_UNROLL
        for (int i = 0; i < B; ++i)
TR_UNROLL
            for (int j = 0; j < B; ++j) rec[RC::LR + i * B + j] = es.W[j * B + i];
TR_UNROLL
        for (int i = 0; i < B; ++i) rec[RC::RRHS + i] = (empty || off) ? 0.0 : rp[i] - es.rc[i];
TR_UNROLL
        for (int i = 0; i < B; ++i) rec[RC::LRHS + i] = es.accrL[i];
        rec[RC::LOGDET] = es.piv.logdet();
    }
    ss_stamp(a, 1);
    // last block of lane l of this warp / of warp g of this CTA / of CTA c
    auto lane_last = [&](int l) { return min(a.n - 1, (wfl + l + 1) * a.Lc - 1); };
    auto warp_last = [&](int g) { return min(a.n - 1, (static_cast<long long>(cta) * C::NW + g + 1) * 32 * a.Lc - 1); };
    auto cta_last = [&](int c) {
        return min(a.n - 1, static_cast<long long>(min(c, a.G - 1) + 1) * C::NT * a.Lc - 1);
    };
    ss_warp_tree_up<B, 32>(rec, tfw, 32, kFullWarp, a.status, lane_last);
    if (lane == 0)
TR_UNROLL
        for (int c = 0; c < NR; ++c) WR[c * C::RSW + w] = rec[c];
    __syncthreads();
    ss_tree_up<B>(WR, C::RSW, C::NW, a.status, warp_last);
    for (int c = t; c < NR; c += C::NT) a.crec[static_cast<long long>(c) * a.G + cta] = WR[c * C::RSW];
    __threadfence();
    __syncthreads();
    if (t == 0) atomicAdd(a.sync, 1ULL);
    ss_stamp(a, 2);

    // ---- top: CTA 0 solves the G-record reduced system (as in stream_solve.cuh) ----------
    if (cta == 0) {
        if (t == 0)
            while (ss_ld_acquire(a.sync) < a.arrive_target) __nanosleep(40);
        __syncthreads();
        ss_stamp(a, 3);
        const int G = a.G;
        double* TR_ = sm + C::OFF_TOP;         // [NR][RST]
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
        if (lane == 0)
TR_UNROLL
            for (int c = 0; c < NR; ++c) TR_[c * C::RST + w] = grec[c];
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
                xl[i] = lane == 0 ? TE[i * C::EST + w] : 0.0;
                xr[i] = lane == 0 ? TE[i * C::EST + w + 1] : 0.0;
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

    // ---- down: CTA boundaries -> warp boundaries -> lane boundaries ----------------------
    if (t < B) {
        WE[t * C::ESW] = cta > 0 ? __ldcg(a.xsep + static_cast<long long>(cta - 1) * B + t) : 0.0;
        WE[t * C::ESW + 1] = __ldcg(a.xsep + static_cast<long long>(cta) * B + t);
    }
    __syncthreads();
    ss_tree_down<B>(WR, C::RSW, WE, C::ESW, C::NW);
    double xl[B], xn[B];  // x at the chunk's left separator; x of the block to the right
    {
        double F[NF], xr[B];
TR_UNROLL
        for (int c = 0; c < NF; ++c) F[c] = lane == 0 ? 0.0 : tfw[c * 32];
TR_UNROLL
        for (int i = 0; i < B; ++i) {
            xl[i] = lane == 0 ? WE[i * C::ESW + w] : 0.0;
            xr[i] = lane == 0 ? WE[i * C::ESW + w + 1] : 0.0;
        }
        ss_warp_tree_down<B, 32>(F, xl, xr, kFullWarp);
TR_UNROLL
        for (int i = 0; i < B; ++i) xn[i] = xr[i];
    }

    // ---- sweep 2: sub-tiles descending ---------------------------------------------------
#pragma unroll 1
    for (int s = nsub - 1; s >= 0 && !empty; --s) {
        double T[BB], rc[B];
        if (s < nsub - 1) {  // (the last sub-tile of sweep 1 is still staged)
            __syncwarp();
            st_stage<C, B, MB>(a, wm, wfl, qin, s, 0, pol_first);
        }
        if (s > 0) {
            const double* ck = ckw + static_cast<long long>(s) * (NCK * 32);
            double Wk[BB], t1[B];
TR_UNROLL
            for (int i = 0; i < BB; ++i) T[i] = ck[i * 32];
TR_UNROLL
            for (int i = 0; i < BB; ++i) Wk[i] = ck[(BB + i) * 32];
TR_UNROLL
            for (int i = 0; i < B; ++i) rc[i] = ck[(2 * BB + i) * 32];
            mv<B>(t1, Wk, xl);  // the left separator's x, folded into the right-hand side
TR_UNROLL
            for (int i = 0; i < B; ++i) rc[i] += t1[i];
        } else {
            mzero<B>(T);
            mtv<B>(rc, Up0, xl);
        }
        if (s == 2) ss_stamp(a, 11);
        st_cp_wait();
        __syncwarp();
        if (s == 2) ss_stamp(a, 12);
        const int nel = off ? 0 : (s == nsub - 1 ? MB - 1 : MB);
#pragma unroll 1
        for (int j = 0; j < nel; ++j) {
            double* Dp = sD + j * BB;
            double* Up = sU + j * BB;
            double* rp = sR + j * B;
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
        if (s == nsub - 1)
TR_UNROLL
            for (int i = 0; i < B; ++i) sR[(MB - 1) * B + i] = xn[i];  // the separator's own x
#pragma unroll 1
        for (int j = nel - 1; j >= 0; --j) {
            const double* Lq = sD + j * BB;
            const double* Xq = sU + j * BB;
            double* zq = sR + j * B;
            double L[BB], av[B], t1[B], xj[B];
TR_UNROLL
            for (int i = 0; i < BB; ++i) L[i] = Lq[i];
            mv<B>(t1, Xq, xn);
TR_UNROLL
            for (int i = 0; i < B; ++i) av[i] = zq[i] - t1[i];
            ltsolve_v<B>(xj, L, av);
TR_UNROLL
            for (int i = 0; i < B; ++i) {
                zq[i] = xj[i];
                xn[i] = xj[i];
            }
        }
        __syncwarp();
        if (s == 2) ss_stamp(a, 13);
        st_store_x<C, B>(a, wm, wfl, s);
        if (s == 2) ss_stamp(a, 14);
    }
    ss_stamp(a, 6);
}
#endif  // SPINGP_HOST_EMU

}  // namespace spingp_dev
