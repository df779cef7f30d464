// team.cuh — level-0 kernels for the large state dimensions (b >= 6): one TEAM of
// TS lanes per chunk instead of one thread per chunk.
//
// Why.  A b x b block costs b^2 doubles; with one thread per chunk the ~12 live blocks
// of the elimination (S, L, X, Y, T, W, accLL, Φ, Q̃, L_Q, ...) need 400 (b = 6) to
// 3000 (b = 16) doubles per thread, i.e. local memory: the round-1 kernels ran 18.5 k
// LDL/STL against 3.2 k DFMA (k_revL<16>) and cfg4 / cfg5 reached 1.2 % / 0.5 % of the
// FP64 peak.  Here lane l of a team owns COLUMN l of every working block (b doubles in
// registers), and the blocks that serve as the broadcast operand of a product or a
// triangular solve are staged in shared memory:
//
//   y = A c        lane l: y = A (c = column l of the right operand)      A broadcast
//   y = A^T c      lane l: y = A^T c                                      A broadcast
//   c <- L^{-1} c  forward substitution on the lane's own column          L broadcast
//   chol(S)        right-looking: lane k scales column k, the other lanes
//                  update theirs from it (one team barrier per column)
//   transpose      column put, team barrier, row get (odd row stride b+1:
//                  both column and row accesses are bank-conflict free)
//
// Every per-block operation of the thread-per-chunk kernels (engine.cuh: elim_block,
// step_assembly, back_step, step_terms, point_out) is restated column by column, in
// the same arithmetic order (fma chains over k ascending, inverted Cholesky pivots,
// pivot / covariance symmetrisation), so results agree with them to rounding.
// The level-0 record, solution and partial-sum layouts are the ones engine.cuh's upper
// levels and k_reduce read; only the level-0 factor layout is private:
//   fac[(chunk * m0 + step) * NF + comp],  NF = b(b+1)/2 (L, inverted diagonal) + b^2 (Y) + b (z)
//
// References: SPEC.md:143-205 (btd_core factorize / solve / selective_inverse),
// :262-306 (assembly, MLL, gradient, posterior); SURVEY.md App. B (formulas).
#pragma once

#include "engine.cuh"

namespace spingp_dev {

#define TP_INL __device__ __forceinline__

// occupancy knobs (minimum resident CTAs for b <= 8; CTA size for b > 8), tuned on B200
// (measured, cfg4 at 4 M / cfg5 at 2 M points: fwd 5.62 -> 4.36 ms and 44.6 -> 39.2 ms,
// rev 10.36 -> 9.81 ms and 82.6 -> 74.3 ms against minB 1 / 64-thread CTAs)
#ifndef SP_TEAM_FWD_MINB
#define SP_TEAM_FWD_MINB 4
#endif
#ifndef SP_TEAM_REV_MINB
#define SP_TEAM_REV_MINB 3
#endif
#ifndef SP_TEAM_CTA16
#define SP_TEAM_CTA16 32
#endif

template <int B>
struct TeamCfg {
    // lanes per team, one per column: the reverse packs b = 6 as 5 teams of 6 lanes per
    // warp; the forward (fewer live columns, register-capped) keeps 8-lane teams there
    // (measured, cfg4 16 M: rev 38.6 -> 31.5 ms with 6-lane teams, fwd 17.1 -> 19.7 ms)
    static constexpr int TSR = B <= 8 ? B : 16;
    static constexpr int TSF = B <= 8 ? 8 : 16;
    static constexpr int LD = B + 1;             // odd smem row stride
    static constexpr int MAT = B * LD;           // doubles per staged block
    static constexpr int VEC = (B + 1) & ~1;
    // per-team smem (doubles), padded so that team t of a warp starts 2 TS t words into the
    // bank ring: the TS columns a team touches at once (2 words each) then tile the 32
    // banks of a half-warp without overlap (ncu: 2.7e9 bank conflicts in the b = 6
    // reverse with unpadded teams)
    static constexpr int pad_to(int raw, int ts) { return raw + ((ts % 16) - raw % 16 + 16) % 16; }
    static constexpr int CTA = B <= 8 ? 128 : SP_TEAM_CTA16;  // threads per CTA
    static constexpr int FWD_MINB = B <= 8 ? SP_TEAM_FWD_MINB : 1;
    static constexpr int REV_MINB = B <= 8 ? SP_TEAM_REV_MINB : 1;
    static constexpr int FWD = pad_to(10 * MAT + VEC, TSF);
    static constexpr int REV = pad_to(10 * MAT + 4 * VEC, TSR);
    static constexpr int TPCR = (CTA / 32) * (32 / TSR);  // teams per CTA, reverse
    static constexpr int TPCF = (CTA / 32) * (32 / TSF);  // teams per CTA, forward
};

struct Team {
    int l;          // column owned (lane within the team)
    int base;       // first lane of the team in the warp
    unsigned mask;  // the team's lanes
    int n;          // lanes in the team
};

template <int TS>
TP_INL Team make_team() {  // teams are TS consecutive lanes; lanes past the last whole team idle
    const int lane = threadIdx.x & 31;
    Team t;
    t.l = lane % TS;
    t.base = lane - t.l;
    t.mask = (TS == 32 ? 0xffffffffu : ((1u << TS) - 1u)) << t.base;
    t.n = TS;
    return t;
}
// team index of this thread within its CTA (>= teams per CTA for the idle lanes)
template <int TS>
TP_INL int team_in_cta() {
    const int lane = threadIdx.x & 31;
    const int tw = lane / TS;
    return tw < 32 / TS ? (threadIdx.x >> 5) * (32 / TS) + tw : 1 << 20;
}
TP_INL void tsync(const Team& t) { __syncwarp(t.mask); }
TP_INL double tshfl(const Team& t, double v, int src) { return __shfl_sync(t.mask, v, t.base + src); }
TP_INL double tsum(const Team& t, double v) {
    if ((t.n & (t.n - 1)) == 0) {
        for (int o = t.n / 2; o > 0; o >>= 1) v += __shfl_xor_sync(t.mask, v, o);
        return v;
    }
    double s = 0.0;  // non-power-of-two team: every lane sums the n values in lane order
    for (int k = 0; k < t.n; ++k) s += __shfl_sync(t.mask, v, t.base + k);
    return s;
}

// ---- column primitives (stride S of the staged block: LD, or B for model blocks) ----
template <int B, int S>
TP_INL void colget(double (&c)[B], const double* M, int l) {
#pragma unroll
    for (int i = 0; i < B; ++i) c[i] = l < B ? M[i * S + l] : 0.0;
}
template <int B, int S>
TP_INL void colput(double* M, const double (&c)[B], int l) {
    if (l < B)
#pragma unroll
        for (int i = 0; i < B; ++i) M[i * S + l] = c[i];
}
template <int B, int S>
TP_INL void rowget(double (&c)[B], const double* M, int l) {
#pragma unroll
    for (int i = 0; i < B; ++i) c[i] = l < B ? M[l * S + i] : 0.0;
}
template <int B, int S>
TP_INL void rowput(double* M, const double (&c)[B], int l) {
    if (l < B)
#pragma unroll
        for (int i = 0; i < B; ++i) M[l * S + i] = c[i];
}
template <int B>
TP_INL void unitcol(double (&c)[B], int l) {
#pragma unroll
    for (int i = 0; i < B; ++i) c[i] = i == l ? 1.0 : 0.0;
}
template <int B>
TP_INL double pick(const double (&c)[B], int l) {  // c[l] without dynamic register indexing
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < B; ++i) v = i == l ? c[i] : v;
    return v;
}
// o = A c
template <int B, int S>
TP_INL void tmv(double (&o)[B], const double* A, const double (&c)[B]) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < B; ++k) s = fma(A[i * S + k], c[k], s);
        o[i] = s;
    }
}
// o = A^T c
template <int B, int S>
TP_INL void tmtv(double (&o)[B], const double* A, const double (&c)[B]) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < B; ++k) s = fma(A[k * S + i], c[k], s);
        o[i] = s;
    }
}
// c <- L^{-1} c  (L lower, inverted pivots on the diagonal; devmat.cuh lsolve order)
template <int B, int S>
TP_INL void tlsolve(double (&c)[B], const double* L) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
        double s = c[i];
#pragma unroll
        for (int k = 0; k < i; ++k) s = fma(-L[i * S + k], c[k], s);
        c[i] = s * L[i * S + i];
    }
}
// c <- L^{-T} c  (devmat.cuh ltsolve order)
template <int B, int S>
TP_INL void tltsolve(double (&c)[B], const double* L) {
#pragma unroll
    for (int i = B - 1; i >= 0; --i) {
        double s = c[i];
#pragma unroll
        for (int k = i + 1; k < B; ++k) s = fma(-L[k * S + i], c[k], s);
        c[i] = s * L[i * S + i];
    }
}
// Solves and products with the MODEL blocks (L_Q, Φ).  D2 = the model is block diagonal
// in aligned 2 x 2 blocks (Matérn-3/2 + quasi-periodic sums, T::kDiag2): only the two
// in-block terms of every sum are formed.  The dense loops would add exact zeros in the
// same order, so both branches give identical results on such models.
template <int B, bool D2>
TP_INL void mlsolve(double (&c)[B], const double* L) {
    constexpr int LD = TeamCfg<B>::LD;
    if constexpr (D2) {
#pragma unroll
        for (int p = 0; p < B / 2; ++p) {
            const int i = 2 * p;
            c[i] = c[i] * L[i * LD + i];
            c[i + 1] = fma(-L[(i + 1) * LD + i], c[i], c[i + 1]) * L[(i + 1) * LD + i + 1];
        }
    } else {
        tlsolve<B, LD>(c, L);
    }
}
template <int B, bool D2>
TP_INL void mltsolve(double (&c)[B], const double* L) {
    constexpr int LD = TeamCfg<B>::LD;
    if constexpr (D2) {
#pragma unroll
        for (int p = 0; p < B / 2; ++p) {
            const int i = 2 * p;
            c[i + 1] = c[i + 1] * L[(i + 1) * LD + i + 1];
            c[i] = fma(-L[(i + 1) * LD + i], c[i + 1], c[i]) * L[i * LD + i];
        }
    } else {
        tltsolve<B, LD>(c, L);
    }
}
template <int B, bool D2>
TP_INL void mmv(double (&o)[B], const double* Phi, const double (&c)[B]) {  // o = Φ c
    constexpr int LD = TeamCfg<B>::LD;
    if constexpr (D2) {
#pragma unroll
        for (int p = 0; p < B / 2; ++p) {
            const int i = 2 * p;
            o[i] = fma(Phi[i * LD + i + 1], c[i + 1], Phi[i * LD + i] * c[i]);
            o[i + 1] = fma(Phi[(i + 1) * LD + i + 1], c[i + 1], Phi[(i + 1) * LD + i] * c[i]);
        }
    } else {
        tmv<B, LD>(o, Phi, c);
    }
}

// Cholesky of the symmetric block whose column l is c (lower part read): L (inverted
// pivots, devmat.cuh chol_nolog arithmetic) staged at Ls; team-uniform success flag.
// The per-element fma order (k ascending from S[i][l]) equals the left-looking one.
template <int B>
TP_INL bool tchol(const Team& tm, double (&c)[B], double* Ls, LogDetAcc* acc) {
    constexpr int LD = TeamCfg<B>::LD;
    const int l = tm.l;
    bool ok = true;
    double p4 = 1.0;
#pragma unroll
    for (int k = 0; k < B; ++k) {
        const double piv = tshfl(tm, c[k], k);
        ok = ok && (piv > 0.0) && isfinite(piv);
        const double inv = rsqrt(piv);
        if (l == k) {
            Ls[k * LD + k] = inv;
#pragma unroll
            for (int i = k + 1; i < B; ++i) Ls[i * LD + k] = c[i] * inv;
        }
        tsync(tm);
        if (l > k && l < B) {
            const double lk = Ls[l * LD + k];
#pragma unroll
            for (int i = k + 1; i < B; ++i) c[i] = fma(-Ls[i * LD + k], lk, c[i]);
        }
        p4 *= inv;
        if (acc && ((k & 3) == 3 || k == B - 1)) {
            acc->mul(p4);
            p4 = 1.0;
        }
    }
    return ok;
}
// symmetrise the block whose column l is c: c <- (c + row l) / 2 through the scratch block
template <int B>
TP_INL void tsym(const Team& tm, double (&c)[B], double* scratch) {
    constexpr int LD = TeamCfg<B>::LD;
    tsync(tm);
    colput<B, LD>(scratch, c, tm.l);
    tsync(tm);
    double r[B];
    rowget<B, LD>(r, scratch, tm.l);
#pragma unroll
    for (int i = 0; i < B; ++i) c[i] = 0.5 * (c[i] + r[i]);
}
// column l of the transpose of the block whose column l is c
template <int B>
TP_INL void ttrans(const Team& tm, double (&o)[B], const double (&c)[B], double* scratch) {
    constexpr int LD = TeamCfg<B>::LD;
    tsync(tm);
    colput<B, LD>(scratch, c, tm.l);
    tsync(tm);
    rowget<B, LD>(o, scratch, tm.l);
}

// Φ, Q for step dt into PhiS, QS (row stride B, written by the model code of lane 0),
// then L_Q = chol(Q + jit I) into LQ.  Team-uniform success.
template <class T>
TP_INL bool tmodel(const Team& tm, const ModelDesc& md, const double* rp, double dt, double jit, double* PhiS,
                   double* QS, double* LQ, LogDetAcc* ldq) {
    constexpr int B = T::B;
    constexpr int LD = TeamCfg<B>::LD;
    T::template step_team<LD>(md, rp, dt, PhiS, QS, tm.l, tm.n, tm.mask);
    tsync(tm);
    if constexpr (T::kDiag2) {
        // 2 x 2 pivots of the block-diagonal Q̃, every lane all of them (the dense tchol's
        // arithmetic and log-det grouping); lane 2p stores block p of L_Q
        bool ok = true;
        double p4 = 1.0;
#pragma unroll
        for (int p = 0; p < B / 2; ++p) {
            const int i = 2 * p;
            const double a = QS[i * LD + i] + (i < md.b ? jit : 0.0);
            const double bq = QS[(i + 1) * LD + i];
            const double cq = QS[(i + 1) * LD + i + 1] + (i + 1 < md.b ? jit : 0.0);
            const double inv0 = rsqrt(a);
            const double l10 = bq * inv0;
            const double d = fma(-l10, l10, cq);
            const double inv1 = rsqrt(d);
            ok = ok && (a > 0.0) && isfinite(a) && (d > 0.0) && isfinite(d);
            if (tm.l == i) {
                LQ[i * LD + i] = inv0;
                LQ[(i + 1) * LD + i] = l10;
                LQ[(i + 1) * LD + i + 1] = inv1;
            }
            if (ldq) {
                p4 *= inv0;
                if (((i) & 3) == 3) { ldq->mul(p4); p4 = 1.0; }
                p4 *= inv1;
                if (((i + 1) & 3) == 3 || i + 1 == B - 1) { ldq->mul(p4); p4 = 1.0; }
            }
        }
        tsync(tm);
        return ok;
    }
    double c[B];
    colget<B, TeamCfg<B>::LD>(c, QS, tm.l);
#pragma unroll
    for (int i = 0; i < B; ++i)
        if (i == tm.l && i < md.b) c[i] += jit;
    return tchol<B>(tm, c, LQ, ldq);
}

// Assembly pieces of one step (engine.cuh step_assembly): column l of
//   PQP = Φ^T Q̃^{-1} Φ = Z^T Z (Z = L_Q^{-1} Φ)   and   U = -Φ^T Q̃^{-1} = -(L_Q^{-T} Z)^T;
// optionally column l of W0 = U^T = -Q̃^{-1} Φ (the first block's left coupling).
template <int B, bool D2 = false>
TP_INL void tassembly(const Team& tm, const double* PhiS, const double* LQ, double* ZS, double* WS, double* pqp,
                      double (&U)[B], double* W0) {
    constexpr int LD = TeamCfg<B>::LD;
    if constexpr (D2) {
        // Z = L_Q^{-1} Φ, Z^T Z and Q̃^{-1} Φ are block diagonal: column l has entries only
        // in its block (2p, 2p+1); the partner column comes from lane l ^ 1
        const int l = tm.l, i0 = l & ~1;
        double z[B];
        colget<B, LD>(z, PhiS, l);
        mlsolve<B, true>(z, LQ);
        const double z0 = pick<B>(z, i0), z1 = pick<B>(z, i0 + 1);
        const double y0 = __shfl_xor_sync(tm.mask, z0, 1), y1 = __shfl_xor_sync(tm.mask, z1, 1);
        const double e0 = (l & 1) ? y0 : z0, e1 = (l & 1) ? y1 : z1;  // column i0 of Z
        const double o0 = (l & 1) ? z0 : y0, o1 = (l & 1) ? z1 : y1;  // column i0 + 1 of Z
        if (pqp) {
#pragma unroll
            for (int i = 0; i < B; ++i) pqp[i] = 0.0;
            const double v0 = fma(e1, z1, e0 * z0), v1 = fma(o1, z1, o0 * z0);
#pragma unroll
            for (int i = 0; i < B; ++i) {
                if (i == i0) pqp[i] = v0;
                if (i == i0 + 1) pqp[i] = v1;
            }
        }
        mltsolve<B, true>(z, LQ);  // column l of Q̃^{-1} Φ
        if (W0)
#pragma unroll
            for (int i = 0; i < B; ++i) W0[i] = -z[i];
        // U = -(Q̃^{-1} Φ)^T: column l = -(row l), whose block entries are column i0's and
        // column i0+1's element l
        const double own = pick<B>(z, l), oth = __shfl_xor_sync(tm.mask, pick<B>(z, l ^ 1), 1);
        const double a0 = (l & 1) ? oth : own, a1 = (l & 1) ? own : oth;
#pragma unroll
        for (int i = 0; i < B; ++i) U[i] = i == i0 ? -a0 : (i == i0 + 1 ? -a1 : 0.0);
        return;
    }
    double z[B];
    colget<B, LD>(z, PhiS, tm.l);
    tlsolve<B, LD>(z, LQ);
    if (pqp) {
        colput<B, LD>(ZS, z, tm.l);
        tsync(tm);
        double q[B];
        tmtv<B, LD>(q, ZS, z);
#pragma unroll
        for (int i = 0; i < B; ++i) pqp[i] = q[i];
    }
    tltsolve<B, LD>(z, LQ);  // column l of Q̃^{-1} Φ
    if (W0)
#pragma unroll
        for (int i = 0; i < B; ++i) W0[i] = -z[i];
    colput<B, LD>(WS, z, tm.l);
    tsync(tm);
    rowget<B, LD>(U, WS, tm.l);
#pragma unroll
    for (int i = 0; i < B; ++i) U[i] = -U[i];
}

// column l of Q̃^{-1} (engine.cuh chol_inv_solve, symmetrised)
template <int B, bool D2 = false>
TP_INL void tqinv(const Team& tm, double (&q)[B], const double* LQ, double* scratch) {
    constexpr int LD = TeamCfg<B>::LD;
    unitcol<B>(q, tm.l);
    if constexpr (D2) {
        mlsolve<B, true>(q, LQ);
        mltsolve<B, true>(q, LQ);
        // symmetrise the in-block pair with the partner column
        const int l = tm.l;
        const double mine = pick<B>(q, l ^ 1), theirs = __shfl_xor_sync(tm.mask, mine, 1);
#pragma unroll
        for (int i = 0; i < B; ++i)
            if (i == (l ^ 1)) q[i] = 0.5 * (q[i] + theirs);
        return;
    }
    tlsolve<B, LD>(q, LQ);
    tltsolve<B, LD>(q, LQ);
    tsym<B>(tm, q, scratch);
}

// A lane-private column kept in shared memory between uses (frees registers; lane l
// only ever touches column l, so no team barrier is needed around these)
template <int B>
TP_INL void pget(double (&c)[B], const double* M, int l) {
    colget<B, TeamCfg<B>::LD>(c, M, l);
}
template <int B>
TP_INL void pput(double* M, const double (&c)[B], int l) {
    colput<B, TeamCfg<B>::LD>(M, c, l);
}

// ======================================================== forward, level 0 ====
template <class T>
__global__ void __launch_bounds__(TeamCfg<T::B>::CTA, TeamCfg<T::B>::FWD_MINB) k_fwd0_team(
    ModelDesc md, const double* __restrict__ params, const double* __restrict__ t, const double* __restrict__ y,
    Geom geo, double* __restrict__ fac, double* __restrict__ rec, double* __restrict__ part,
    unsigned long long* status, const double* __restrict__ halo, long long g0, long long g1,
    const unsigned char* __restrict__ obs) {
    constexpr int B = T::B;
    using C = TeamCfg<B>;
    constexpr int LD = C::LD;
    constexpr int NLI = B * (B + 1) / 2, NF = NLI + B * B + B;
    extern __shared__ double smem_team[];
    const Team tm = make_team<C::TSF>();
    const int tid = team_in_cta<C::TSF>();
    if (tid >= C::TPCF) return;
    double* R = smem_team + static_cast<size_t>(tid) * C::FWD;
    double* PhiS = R;               // model blocks
    double* QS = R + C::MAT;
    double* LQ = R + 2 * C::MAT;    // chol(Q̃)
    double* LS = R + 3 * C::MAT;    // chol(S)
    double* XS = R + 4 * C::MAT;
    double* YS = R + 5 * C::MAT;
    double* QiS = R + 6 * C::MAT;   // lane-private carried columns: Q̃^{-1} of the current block,
    double* WS = R + 7 * C::MAT;    //   the left coupling W,
    double* TcS = R + 8 * C::MAT;   //   the Schur update T = X^T X,
    double* AcS = R + 9 * C::MAT;   //   acc_LL
    double* vS = R + 10 * C::MAT;   // rc (vector)
    const long long g = g0 + static_cast<long long>(blockIdx.x) * C::TPCF + tid;
    if (g >= g1) return;
    const int l = tm.l;
    const long long K = geo.K[0], SK = K * geo.S;
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
    const double Hl = l < B ? T::H(md, l) : 0.0;

    double dt = -1.0;
    if (st > 0 || geo.segL) {
        dt = ts[st] - (st > 0 ? ts[st - 1] : halo[2 * s]);
        if (!(dt > 0.0) || !isfinite(dt)) {
            if (l == 0) report(status, gbase + st, dt == 0.0 ? ST_DUPLICATE : ST_BAD_ARG);
            return;
        }
    }
    if (!tmodel<T>(tm, md, rp, dt, jit, PhiS, QS, LQ, nullptr)) {
        if (l == 0) report(status, gbase + st, ST_SINGULAR_Q);
        return;
    }
    {
        double q[B];
        tqinv<B, T::kDiag2>(tm, q, LQ, XS);
        pput<B>(QiS, q, l);
#pragma unroll
        for (int i = 0; i < B; ++i) q[i] = 0.0;
        pput<B>(TcS, q, l);
        pput<B>(AcS, q, l);
        if (hasL) {  // P_{st, st-1} = U_{st-1}^T = -Q̃_st^{-1} Φ_st
            double U[B], W[B];
            tassembly<B, T::kDiag2>(tm, PhiS, LQ, XS, YS, nullptr, U, W);
            pput<B>(WS, W, l);
        } else {
            pput<B>(WS, q, l);
        }
        if (l < B) vS[l] = 0.0;
    }
    double accrL = 0.0;  // component l of the carried left rhs
    LogDetAcc piv;
    piv.init();

    for (long long j = st; j < en - 1; ++j) {
        const double dtn = ts[j + 1] - ts[j];
        if (!(dtn > 0.0) || !isfinite(dtn)) {
            if (l == 0) report(status, gbase + j + 1, dtn == 0.0 ? ST_DUPLICATE : ST_BAD_ARG);
            return;
        }
        tsync(tm);  // the previous step's reads of the staged blocks are done
        if (!tmodel<T>(tm, md, rp, dtn, jit, PhiS, QS, LQ, nullptr)) {
            if (l == 0) report(status, gbase + j + 1, ST_SINGULAR_Q);
            return;
        }
        double D[B], U[B];
        tassembly<B, T::kDiag2>(tm, PhiS, LQ, XS, YS, D, U, nullptr);
        const double wo = (!obs || obs[gbase + j]) ? 1.0 : 0.0;
        const double yj = wo != 0.0 ? ys[j] : 0.0;
        if (!isfinite(yj)) {
            if (l == 0) report(status, gbase + j, ST_BAD_ARG);
            return;
        }
        {
            double q[B], tc[B];
            pget<B>(q, QiS, l);
            pget<B>(tc, TcS, l);
#pragma unroll
            for (int i = 0; i < B; ++i) D[i] = (D[i] + (q[i] + wo * (T::H(md, i) * Hl * is2))) - tc[i];
        }
        // S = D - T (Q̃^{-1} symmetrised by tqinv; PQP and T exactly symmetric)
        if (!tchol<B>(tm, D, LS, &piv)) {
            if (l == 0) report(status, gbase + j, ST_NOT_PD);
            return;
        }
        {
            double q[B];
            tqinv<B, T::kDiag2>(tm, q, LQ, PhiS);  // Q̃_{j+1}^{-1}: the next block's diagonal term
            pput<B>(QiS, q, l);
        }
        double z[B];
#pragma unroll
        for (int i = 0; i < B; ++i) z[i] = T::H(md, i) * yj * is2 - vS[i];
        tlsolve<B, LD>(z, LS);
        tlsolve<B, LD>(U, LS);  // X = L^{-1} U
        double Y[B];
        if (hasL) {
            pget<B>(Y, WS, l);
            tlsolve<B, LD>(Y, LS);  // Y = L^{-1} W
        }
        tsync(tm);
        colput<B, LD>(XS, U, l);
        if (hasL) colput<B, LD>(YS, Y, l);
        tsync(tm);
        {
            double tc[B];
            tmtv<B, LD>(tc, XS, U);  // T' = X^T X
            pput<B>(TcS, tc, l);
        }
        double rcl = 0.0;
#pragma unroll
        for (int i = 0; i < B; ++i) rcl = fma(U[i], z[i], rcl);  // (X^T z)_l
        // factor of step j for the reverse sweep: L (packed, inverted pivots), Y, z
        double* fp = fac + (g * m + (j - st)) * static_cast<long long>(NF);
        if (l < B) {
#pragma unroll
            for (int i = 0; i < B; ++i)
                if (i >= l) fp[i * (i + 1) / 2 + l] = LS[i * LD + l];
            if (hasL)
#pragma unroll
                for (int i = 0; i < B; ++i) fp[NLI + i * B + l] = Y[i];
            fp[NLI + B * B + l] = pick<B>(z, l);
        }
        if (hasL) {
            double G[B], a[B];
            tmtv<B, LD>(G, YS, Y);  // acc_LL -= Y^T Y
            pget<B>(a, AcS, l);
#pragma unroll
            for (int i = 0; i < B; ++i) a[i] -= G[i];
            pput<B>(AcS, a, l);
            double yz = 0.0;
#pragma unroll
            for (int i = 0; i < B; ++i) yz = fma(Y[i], z[i], yz);
            accrL -= yz;
            tmtv<B, LD>(G, XS, Y);  // W' = -X^T Y
#pragma unroll
            for (int i = 0; i < B; ++i) G[i] = -G[i];
            pput<B>(WS, G, l);
        }
        tsync(tm);
        if (l < B) vS[l] = rcl;
        tsync(tm);
    }
    // separator R = en - 1
    const double woR = (!obs || obs[gbase + en - 1]) ? 1.0 : 0.0;
    double D[B];
    pget<B>(D, QiS, l);
#pragma unroll
    for (int i = 0; i < B; ++i) D[i] += woR * (T::H(md, i) * Hl * is2);
    if (en < n || geo.segR) {
        const double dte = (en < n ? ts[en] : halo[2 * s + 1]) - ts[en - 1];
        if (!(dte > 0.0) || !isfinite(dte)) {
            if (l == 0) report(status, gbase + en, dte == 0.0 ? ST_DUPLICATE : ST_BAD_ARG);
            return;
        }
        tsync(tm);
        if (!tmodel<T>(tm, md, rp, dte, jit, PhiS, QS, LQ, nullptr)) {
            if (l == 0) report(status, gbase + en, ST_SINGULAR_Q);
            return;
        }
        double pqp[B], U[B];
        tassembly<B, T::kDiag2>(tm, PhiS, LQ, XS, YS, pqp, U, nullptr);
#pragma unroll
        for (int i = 0; i < B; ++i) D[i] += pqp[i];
    }
    const double yR = woR != 0.0 ? ys[en - 1] : 0.0;
    if (!isfinite(yR)) {
        if (l == 0) report(status, gbase + en - 1, ST_BAD_ARG);
        return;
    }
    // record (engine.cuh write_rec layout, component-major over chunks)
    double* r = rec + g;
    if (l < B) {
        double tc[B], a[B], w[B];
        pget<B>(tc, TcS, l);
        pget<B>(a, AcS, l);
        pget<B>(w, WS, l);
#pragma unroll
        for (int i = 0; i < B; ++i) {
            r[(Rec<B>::RDIAG + i * B + l) * SK] = D[i] - tc[i];
            r[(Rec<B>::LDIAG + i * B + l) * SK] = a[i];
            r[(Rec<B>::LR + l * B + i) * SK] = hasL ? w[i] : 0.0;  // LR = W^T
        }
        r[(Rec<B>::RRHS + l) * SK] = Hl * yR * is2 - vS[l];
        r[(Rec<B>::LRHS + l) * SK] = accrL;
    }
    if (l == 0) {
        r[Rec<B>::LOGDET * SK] = piv.logdet();
        part[P_LOGDET * SK + g] = piv.logdet();
    }
}

// ======================================================== reverse, level 0 ====

// Likelihood / gradient terms of one step (engine.cuh step_terms) for the team: the
// current block (xc, column l of Ccc), the previous block (xp, column l of Cpp) and
// column l of Cpc = C_{p,c}; Φ, Q (raw) at PhiS, QS (stride B), L_Q at LQ; xc, xp are
// smem vectors.  Scratch blocks S0..S3 (S0, S1 also the stride-B M and Bm handed to
// T::grad).  fe and g are accumulated by lane 0.
template <class T>
TP_INL void tstep_terms(const Team& tm, const ModelDesc& md, const double* rp, double dt, const double* PhiS,
                        const double* QS, const double* LQ, const double* xcS, const double (&Ccc)[T::B],
                        const double* xpS, const double (&Cpp)[T::B], const double (&Cpc)[T::B], bool anchor,
                        bool grad, double& fe, double* g, double* S0, double* S1, double* S2, double* S3) {
    constexpr int B = T::B;
    constexpr int LD = TeamCfg<B>::LD;
    constexpr bool D2 = T::kDiag2;
    const int l = tm.l;
    double e[B];
    if (anchor) {
#pragma unroll
        for (int i = 0; i < B; ++i) e[i] = xcS[i];
    } else {
        double xp[B];
#pragma unroll
        for (int i = 0; i < B; ++i) xp[i] = xpS[i];
        mmv<B, D2>(e, PhiS, xp);
#pragma unroll
        for (int i = 0; i < B; ++i) e[i] = xcS[i] - e[i];
    }
    {
        double u[B];
#pragma unroll
        for (int i = 0; i < B; ++i) u[i] = e[i];
        mlsolve<B, D2>(u, LQ);
        double q = 0.0;
#pragma unroll
        for (int i = 0; i < B; ++i) q += u[i] * u[i];
        if (l == 0) fe += q;
    }
    if (!grad) return;
    const double jit = rp[1];
    const double el = pick<B>(e, l);
    double E[B];
    if (anchor) {
#pragma unroll
        for (int i = 0; i < B; ++i) E[i] = Ccc[i] + e[i] * el;
    } else {
        {
            double X1[B], Y1[B];
            mmv<B, D2>(X1, PhiS, Cpc);  // Φ C_pc
            mmv<B, D2>(Y1, PhiS, Cpp);  // Φ C_pp
            tsync(tm);
            colput<B, LD>(S2, X1, l);
            colput<B, LD>(S3, Y1, l);
#pragma unroll
            for (int i = 0; i < B; ++i) E[i] = Ccc[i] - X1[i];
        }
        tsync(tm);
        double r[B], ph[B];
        rowget<B, LD>(r, S2, l);
        rowget<B, LD>(ph, PhiS, l);
#pragma unroll
        for (int i = 0; i < B; ++i) E[i] -= r[i];
        if constexpr (D2) {  // row l of Φ has its two entries in block (i0, i0+1)
            const int i0 = l & ~1;
            const double p0 = pick<B>(ph, i0), p1 = pick<B>(ph, i0 + 1);
#pragma unroll
            for (int i = 0; i < B; ++i) {
                double a0 = 0.0, a1 = 0.0;
#pragma unroll
                for (int k = 0; k < B; k += 2)
                    if (k == i0) {
                        a0 = S3[i * LD + k];
                        a1 = S3[i * LD + k + 1];
                    }
                r[i] = fma(a1, p1, a0 * p0);
            }
        } else {
            tmv<B, LD>(r, S3, ph);  // Φ C_pp Φ^T
        }
#pragma unroll
        for (int i = 0; i < B; ++i) E[i] = (E[i] + r[i]) + e[i] * el;
    }
    // E - Q̃ (padding states have Q̃ = 1 and E = 0; their rows of M are never read)
    {
        double q[B];
        colget<B, LD>(q, QS, l);
#pragma unroll
        for (int i = 0; i < B; ++i) E[i] -= q[i];
#pragma unroll
        for (int i = 0; i < B; ++i)
            if (i == l && i < md.b) E[i] -= jit;
    }
    tsym<B>(tm, E, S0);
    // M = Q̃^{-1}(E - Q̃)Q̃^{-1}: G = Q̃^{-1}(E - Q̃) by columns, then M = (Q̃^{-1} G^T)^T by rows
    mlsolve<B, D2>(E, LQ);
    mltsolve<B, D2>(E, LQ);
    {
        double v[B];
        ttrans<B>(tm, v, E, S1);  // column l of G^T
        mlsolve<B, D2>(v, LQ);
        mltsolve<B, D2>(v, LQ);   // = row l of M
        // symmetrise M (row l in v) and hand it to T::grad at row stride B
        tsync(tm);
        rowput<B, LD>(S0, v, l);
        tsync(tm);
        double cm[B];
        colget<B, LD>(cm, S0, l);
#pragma unroll
        for (int i = 0; i < B; ++i) v[i] = 0.5 * (v[i] + cm[i]);
        tsync(tm);
        rowput<B, LD>(S0, v, l);
    }
    // Bm = Z Q̃^{-1} = (Q̃^{-1} Z^T)^T with Z = C_pc - C_pp Φ^T + x_p e^T: row l of Bm
    // from column l of Z^T = row l of Z
    {
        double v[B];
        if (anchor) {
#pragma unroll
            for (int i = 0; i < B; ++i) v[i] = 0.0;
        } else {
            double y1r[B];
            rowget<B, LD>(y1r, S3, l);  // C_pp Φ^T = (Φ C_pp)^T: column l = row l of Φ C_pp
#pragma unroll
            for (int i = 0; i < B; ++i) v[i] = Cpc[i] - y1r[i] + xpS[i] * el;
            ttrans<B>(tm, v, v, S2);
            mlsolve<B, D2>(v, LQ);
            mltsolve<B, D2>(v, LQ);
        }
        rowput<B, LD>(S1, v, l);
    }
    tsync(tm);
    double gp[T::NP];
#pragma unroll
    for (int p = 0; p < T::NP; ++p) gp[p] = 0.0;
    T::template grad_team<LD>(md, rp, dt, PhiS, QS, S0, S1, l, tm.n, gp);
#pragma unroll
    for (int p = 0; p < T::NP; ++p) {
        const double v = tsum(tm, gp[p]);
        if (l == 0 && p < md.nt) g[p] += v;
    }
}

template <class T>
__global__ void __launch_bounds__(TeamCfg<T::B>::CTA, TeamCfg<T::B>::REV_MINB) k_rev0_team(
    ModelDesc md, const double* __restrict__ params, const double* __restrict__ t, const double* __restrict__ y,
    Geom geo, const double* __restrict__ fac, const double* __restrict__ solU, double* __restrict__ part, Outs outs,
    unsigned long long* status, const double* __restrict__ halo, long long g0, long long g1,
    const unsigned char* __restrict__ obs) {
    constexpr int B = T::B;
    using C = TeamCfg<B>;
    constexpr int LD = C::LD;
    constexpr int NLI = B * (B + 1) / 2, NF = NLI + B * B + B;
    extern __shared__ double smem_team[];
    const Team tm = make_team<C::TSR>();
    const int tid = team_in_cta<C::TSR>();
    if (tid >= C::TPCR) return;
    double* R = smem_team + static_cast<size_t>(tid) * C::REV;
    double* PhiS = R;
    double* QS = R + C::MAT;
    double* LQ = R + 2 * C::MAT;
    double* LS = R + 3 * C::MAT;
    double* XS = R + 4 * C::MAT;
    double* YS = R + 5 * C::MAT;
    double* S6 = R + 6 * C::MAT;
    double* S7 = R + 7 * C::MAT;
    double* CnnS = R + 8 * C::MAT;  // C_{n,n}: lane-private columns
    double* CnLS = R + 9 * C::MAT;  // C_{n,L}: columns written lane-privately, rows read after a barrier
    double* xnS = R + 10 * C::MAT;  // x_n, x_j (swapped every step), x_L, z (vectors)
    double* xjS = xnS + C::VEC;
    double* xLS = xjS + C::VEC;
    double* zS = xLS + C::VEC;
    const long long g = g0 + static_cast<long long>(blockIdx.x) * C::TPCR + tid;
    if (g >= g1) return;
    const int l = tm.l;
    const long long K = geo.K[0], SK = K * geo.S;
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
    const double Hl = l < B ? T::H(md, l) : 0.0;

    // separators (engine.cuh load_sep): right = this chunk's last block, left = the
    // previous chunk's (x, C_LL, C_LR)
    const long long SnU = static_cast<long long>(geo.S) * (geo.n[1] + geo.segL), iR = g + geo.segL * (s + 1);
    if (l < B) {
        xnS[l] = solU[(Sol<B>::X + l) * SnU + iR];
        xLS[l] = hasL ? solU[(Sol<B>::X + l) * SnU + iR - 1] : 0.0;
#pragma unroll
        for (int i = 0; i < B; ++i) {
            CnnS[i * LD + l] = needC ? solU[(Sol<B>::CD + i * B + l) * SnU + iR] : 0.0;
            // C_{n,L} = C_LR^T: column l = row l of C_LR
            CnLS[i * LD + l] = (hasL && needC) ? solU[(Sol<B>::CU + l * B + i) * SnU + iR - 1] : 0.0;
        }
    }
    const double* CLLg = solU + Sol<B>::CD * SnU + iR - 1;  // C_LL[i][l] at CLLg[(i * B + l) * SnU]
    tsync(tm);

    double fy = 0.0, fe = 0.0, noise = 0.0;
    LogDetAcc ldq;  // log det of every Q̃ of the chunk
    ldq.init();
    double gr[kMaxTheta];
    for (int p = 0; p < md.nt; ++p) gr[p] = 0.0;

    // engine.cuh point_out for block i0 with mean x (smem vector) and column l of C
    auto point = [&](long long i0, const double* xS, const double (&Cc)[B]) {
        const bool ob = !obs || obs[gbase + i0];
        const double yv = ob ? ys[i0] : 0.0;
        double mu = 0.0;
#pragma unroll
        for (int k = 0; k < B; ++k) mu += T::H(md, k) * xS[k];
        const double rr = yv - mu;
        if (l == 0 && ob) fy += rr * rr * is2;
        if (l == 0 && outs.mean) outs.mean[gbase + i0] = mu;
        if (outs.need_c) {
            double hc = 0.0;
#pragma unroll
            for (int a = 0; a < B; ++a) hc += T::H(md, a) * Cc[a];
            double v = tsum(tm, Hl * hc);
            if (l == 0) {
                if (ob) noise += rr * rr + v;
                if (outs.var) {
                    if (v < -1e-10) report(status, gbase + i0, ST_NEG_VAR);
                    if (v < 0.0) v = 0.0;  // clamp [-1e-10, 0) -> 0
                    outs.var[gbase + i0] = outs.include_noise ? v + sig * sig : v;
                }
            }
        }
    };

    for (long long j = en - 2; j >= st; --j) {
        const long long nb = j + 1;
        const double dt = ts[nb] - ts[j];
        tsync(tm);
        tmodel<T>(tm, md, rp, dt, jit, PhiS, QS, LQ, &ldq);
        double X[B];
        tassembly<B, T::kDiag2>(tm, PhiS, LQ, XS, S6, nullptr, X, nullptr);  // X <- U
        // factor of step j
        const double* fp = fac + (g * m + (j - st)) * static_cast<long long>(NF);
        double Y[B];
        if (l < B) {
#pragma unroll
            for (int i = 0; i < B; ++i) {
                if (i >= l) LS[i * LD + l] = fp[i * (i + 1) / 2 + l];
                Y[i] = hasL ? fp[NLI + i * B + l] : 0.0;
            }
            zS[l] = fp[NLI + B * B + l];
        } else {
#pragma unroll
            for (int i = 0; i < B; ++i) Y[i] = 0.0;
        }
        tsync(tm);
        tlsolve<B, LD>(X, LS);  // X = L^{-1} U
        colput<B, LD>(XS, X, l);
        if (hasL) colput<B, LD>(YS, Y, l);
        tsync(tm);
        // back substitution: x_j = L^{-T}(z - X x_n - Y x_L)
        {
            // lane l forms component l (row l of X and Y), then every lane solves
            double r[B];
            if (l < B) {
                double sx = 0.0, sy = 0.0;
                rowget<B, LD>(r, XS, l);
#pragma unroll
                for (int k = 0; k < B; ++k) sx = fma(r[k], xnS[k], sx);
                double al = zS[l] - sx;
                if (hasL) {
                    rowget<B, LD>(r, YS, l);
#pragma unroll
                    for (int k = 0; k < B; ++k) sy = fma(r[k], xLS[k], sy);
                    al -= sy;
                }
                zS[l] = al;
            }
            tsync(tm);
            double a[B];
#pragma unroll
            for (int i = 0; i < B; ++i) a[i] = zS[i];
            tltsolve<B, LD>(a, LS);
            if (l < B) xjS[l] = pick<B>(a, l);
        }
        double Cjn[B], Cjj[B];
        if (needC) {
            // P1 = X C_nL + Y C_LL,  P2 = X C_nn + Y C_Ln   (engine.cuh back_step)
            double P[B], tmp[B], q[B];
            pget<B>(q, CnLS, l);
            tmv<B, LD>(P, XS, q);
            if (hasL) {
#pragma unroll
                for (int i = 0; i < B; ++i) q[i] = l < B ? CLLg[(i * B + l) * SnU] : 0.0;
                tmv<B, LD>(tmp, YS, q);
#pragma unroll
                for (int i = 0; i < B; ++i) P[i] += tmp[i];
            }
            colput<B, LD>(S7, P, l);  // P1 (S7 free: its last readers passed two barriers)
            pget<B>(q, CnnS, l);
            tmv<B, LD>(Cjn, XS, q);
            if (hasL) {
                rowget<B, LD>(q, CnLS, l);  // column l of C_{L,n} = row l of C_{n,L}
                tmv<B, LD>(tmp, YS, q);
#pragma unroll
                for (int i = 0; i < B; ++i) Cjn[i] += tmp[i];
            }
            colput<B, LD>(S6, Cjn, l);  // P2
            tsync(tm);                  // all rows of C_{n,L} read; P1, P2 staged
            tltsolve<B, LD>(P, LS);
#pragma unroll
            for (int i = 0; i < B; ++i) P[i] = -P[i];
            pput<B>(CnLS, P, l);  // C_{j,L}: the next step's C_{n,L}
            tltsolve<B, LD>(Cjn, LS);
#pragma unroll
            for (int i = 0; i < B; ++i) Cjn[i] = -Cjn[i];
            // M = I + P2 X^T + P1 Y^T (column l: P2 (row l of X) + P1 (row l of Y))
            double M[B];
            rowget<B, LD>(q, XS, l);
            tmv<B, LD>(M, S6, q);
            if (hasL) {
                rowget<B, LD>(q, YS, l);
                tmv<B, LD>(tmp, S7, q);
#pragma unroll
                for (int i = 0; i < B; ++i) M[i] += tmp[i];
            }
#pragma unroll
            for (int i = 0; i < B; ++i)
                if (i == l) M[i] += 1.0;
            tsym<B>(tm, M, S6);
            // C_jj = L^{-T} M L^{-1} = L^{-T} (L^{-T} M)^T
            tltsolve<B, LD>(M, LS);
            ttrans<B>(tm, Cjj, M, S7);
            tltsolve<B, LD>(Cjj, LS);
            tsym<B>(tm, Cjj, S6);
        } else {
#pragma unroll
            for (int i = 0; i < B; ++i) {
                Cjn[i] = 0.0;
                Cjj[i] = 0.0;
            }
        }
        tsync(tm);
        {
            double q[B];
            pget<B>(q, CnnS, l);
            point(nb, xnS, q);
            tstep_terms<T>(tm, md, rp, dt, PhiS, QS, LQ, xnS, q, xjS, Cjj, Cjn, false, grad, fe, gr, XS, YS, S6, S7);
        }
        pput<B>(CnnS, Cjj, l);
        tsync(tm);
        double* sw = xnS;  // x_n <- x_j
        xnS = xjS;
        xjS = sw;
    }
    // block st: previous block is the left separator (or the anchor at st = 0)
    {
        double q[B];
        pget<B>(q, CnnS, l);
        point(st, xnS, q);
        const bool anchor = st == 0 && !geo.segL;
        const double dt = anchor ? -1.0 : ts[st] - (st > 0 ? ts[st - 1] : halo[2 * s]);
        tsync(tm);
        tmodel<T>(tm, md, rp, dt, jit, PhiS, QS, LQ, &ldq);
        double CLL[B], CLs[B];
#pragma unroll
        for (int i = 0; i < B; ++i) CLL[i] = (hasL && needC && l < B) ? CLLg[(i * B + l) * SnU] : 0.0;
        rowget<B, LD>(CLs, CnLS, l);  // C_{L,st} = C_{st,L}^T: column l = row l of C_{st,L}
        tstep_terms<T>(tm, md, rp, dt, PhiS, QS, LQ, xnS, q, xLS, CLL, CLs, anchor, grad, fe, gr, XS, YS, S6, S7);
    }
    if (l == 0) {
        part[P_FITY * SK + g] = fy;
        part[P_FITE * SK + g] = fe;
        part[P_LDQ * SK + g] = ldq.logdet();
        part[P_NOISE * SK + g] = noise;
        for (int p = 0; p < md.nt; ++p) part[(P_GRAD + p) * SK + g] = gr[p];
    }
}

// ================================================== upper levels (b >= 6) ====
// Levels >= 1 with a team per chunk of m_l records (engine.cuh fwdL_item / revL_item,
// the same arithmetic): the blocks come from the level-(l-1) records (RecSource
// semantics) instead of the model.  Per-thread chains kept every b x b block of these
// levels in local memory (k_upper<16>: 18 GB of DRAM traffic per cfg5 evaluation).
// Factor layout of level l: fac[(chunk * m_l + step) * NF + comp], NF = b(b+1)/2 + b^2 + b.
template <int B>
struct TeamUpper {
    static constexpr int TS = TeamCfg<B>::TSF;
    static constexpr int CTA = TeamCfg<B>::CTA;
    static constexpr int TPC = (CTA / 32) * (32 / TS);
    static constexpr int LD = TeamCfg<B>::LD;
    static constexpr int SMF = TeamCfg<B>::pad_to(3 * TeamCfg<B>::MAT + TeamCfg<B>::VEC, TS);      // per team, fwd
    static constexpr int SMR = TeamCfg<B>::pad_to(5 * TeamCfg<B>::MAT + 2 * TeamCfg<B>::VEC, TS);  // per team, rev
};

template <int B>
__global__ void __launch_bounds__(TeamUpper<B>::CTA) k_fwdL_team(RecSource<B> src, Geom geo, int lev,
                                                               double* __restrict__ fac, double* __restrict__ rec,
                                                               unsigned long long* status) {
    using U_ = TeamUpper<B>;
    constexpr int LD = U_::LD;
    constexpr int NLI = B * (B + 1) / 2, NF = NLI + B * B + B;
    extern __shared__ double smem_team[];
    const Team tm = make_team<U_::TS>();
    const int tid = team_in_cta<U_::TS>();
    if (tid >= U_::TPC) return;
    double* R = smem_team + static_cast<size_t>(tid) * U_::SMF;
    double* LS = R;
    double* XS = R + TeamCfg<B>::MAT;
    double* YS = R + 2 * TeamCfg<B>::MAT;
    double* vS = R + 3 * TeamCfg<B>::MAT;  // rc gather
    const long long g = static_cast<long long>(blockIdx.x) * U_::TPC + tid;
    const long long K = geo.K[lev], SK = K * geo.S;
    if (g >= SK) return;
    const int l = tm.l;
    const int s = static_cast<int>(g / K);
    const long long c = g - s * K;
    const long long n = geo.n[lev];
    const int m = geo.m[lev];
    const long long st = c * m, en = min(n, st + m);
    const bool hasL = c > 0 || geo.segL;
    const long long gbase = static_cast<long long>(s) * geo.n[0];
    const long long base = static_cast<long long>(s) * n;  // this series' first record
    const double* rr = src.rec;
    const long long SKp = src.SKp;
    auto dcol = [&](long long k, double (&D)[B]) {  // column l of D_k = R-part of k + L-part of k+1
        const bool nx = k + 1 < n;
#pragma unroll
        for (int i = 0; i < B; ++i)
            D[i] = l < B ? rr[(Rec<B>::RDIAG + i * B + l) * SKp + base + k] +
                               (nx ? rr[(Rec<B>::LDIAG + i * B + l) * SKp + base + k + 1] : 0.0)
                         : 0.0;
    };
    auto rvec = [&](long long k, double (&r)[B]) {
        const bool nx = k + 1 < n;
#pragma unroll
        for (int i = 0; i < B; ++i)
            r[i] = rr[(Rec<B>::RRHS + i) * SKp + base + k] + (nx ? rr[(Rec<B>::LRHS + i) * SKp + base + k + 1] : 0.0);
    };
    auto ucol = [&](long long k, double (&U)[B]) {  // column l of the (k, k+1) block
#pragma unroll
        for (int i = 0; i < B; ++i) U[i] = l < B ? rr[(Rec<B>::LR + i * B + l) * SKp + base + k + 1] : 0.0;
    };
    double Tc[B], acc[B], W[B], rc[B];
    double accrL = 0.0, cld = 0.0;
#pragma unroll
    for (int i = 0; i < B; ++i) {
        Tc[i] = 0.0;
        acc[i] = 0.0;
        W[i] = 0.0;
        rc[i] = 0.0;
    }
    if (c == 0 && geo.segL) {  // carried to the segment's L
#pragma unroll
        for (int i = 0; i < B; ++i) acc[i] = l < B ? rr[(Rec<B>::LDIAG + i * B + l) * SKp + base] : 0.0;
        accrL = l < B ? rr[(Rec<B>::LRHS + l) * SKp + base] : 0.0;
    }
    if (hasL)  // P_{st, st-1} = upper(st-1)^T: column l = row l of upper(st-1)
#pragma unroll
        for (int i = 0; i < B; ++i) W[i] = l < B ? rr[(Rec<B>::LR + l * B + i) * SKp + base + st] : 0.0;
    LogDetAcc piv;
    piv.init();
    for (long long j = st; j < en - 1; ++j) {
        double D[B], U[B], r[B];
        dcol(j, D);
        ucol(j, U);
        rvec(j, r);
#pragma unroll
        for (int i = 0; i < B; ++i) D[i] -= Tc[i];
        tsync(tm);
        if (!tchol<B>(tm, D, LS, &piv)) {
            if (l == 0) report(status, gbase + to_global(geo, lev, j), ST_NOT_PD);
            return;
        }
        double z[B];
#pragma unroll
        for (int i = 0; i < B; ++i) z[i] = r[i] - rc[i];
        tlsolve<B, LD>(z, LS);
        tlsolve<B, LD>(U, LS);
        if (hasL) tlsolve<B, LD>(W, LS);
        colput<B, LD>(XS, U, l);
        if (hasL) colput<B, LD>(YS, W, l);
        tsync(tm);
        tmtv<B, LD>(Tc, XS, U);
        double rcl = 0.0;
#pragma unroll
        for (int i = 0; i < B; ++i) rcl = fma(U[i], z[i], rcl);
        double* fp = fac + (g * m + (j - st)) * static_cast<long long>(NF);
        if (l < B) {
#pragma unroll
            for (int i = 0; i < B; ++i)
                if (i >= l) fp[i * (i + 1) / 2 + l] = LS[i * LD + l];
            if (hasL)
#pragma unroll
                for (int i = 0; i < B; ++i) fp[NLI + i * B + l] = W[i];
            fp[NLI + B * B + l] = pick<B>(z, l);
        }
        if (hasL) {
            double G[B];
            tmtv<B, LD>(G, YS, W);
#pragma unroll
            for (int i = 0; i < B; ++i) acc[i] -= G[i];
            double yz = 0.0;
#pragma unroll
            for (int i = 0; i < B; ++i) yz = fma(W[i], z[i], yz);
            accrL -= yz;
            tmtv<B, LD>(G, XS, W);
#pragma unroll
            for (int i = 0; i < B; ++i) W[i] = -G[i];
        }
        tsync(tm);
        if (l < B) vS[l] = rcl;
        tsync(tm);
#pragma unroll
        for (int i = 0; i < B; ++i) rc[i] = vS[i];
    }
    double D[B], r[B];
    dcol(en - 1, D);
    rvec(en - 1, r);
    for (long long j = st; j < en; ++j) cld += rr[Rec<B>::LOGDET * SKp + base + j];
    double* ro = rec + g;
    if (l < B) {
#pragma unroll
        for (int i = 0; i < B; ++i) {
            ro[(Rec<B>::RDIAG + i * B + l) * SK] = D[i] - Tc[i];
            ro[(Rec<B>::LDIAG + i * B + l) * SK] = acc[i];
            ro[(Rec<B>::LR + l * B + i) * SK] = hasL ? W[i] : 0.0;
        }
        ro[(Rec<B>::RRHS + l) * SK] = pick<B>(r, l) - pick<B>(rc, l);
        ro[(Rec<B>::LRHS + l) * SK] = accrL;
    }
    if (l == 0) ro[Rec<B>::LOGDET * SK] = cld + piv.logdet();
}

template <int B>
__global__ void __launch_bounds__(TeamUpper<B>::CTA) k_revL_team(RecSource<B> src, SolSink<B> sink, Geom geo, int lev,
                                                               const double* __restrict__ fac,
                                                               const double* __restrict__ solU, int needC) {
    using U_ = TeamUpper<B>;
    constexpr int LD = U_::LD;
    constexpr int NLI = B * (B + 1) / 2, NF = NLI + B * B + B;
    extern __shared__ double smem_team[];
    const Team tm = make_team<U_::TS>();
    const int tid = team_in_cta<U_::TS>();
    if (tid >= U_::TPC) return;
    double* R = smem_team + static_cast<size_t>(tid) * U_::SMR;
    double* LS = R;
    double* XS = R + TeamCfg<B>::MAT;
    double* YS = R + 2 * TeamCfg<B>::MAT;
    double* vS = R + 3 * TeamCfg<B>::MAT;  // z / x_L
    double* wS = vS + TeamCfg<B>::VEC;      // a -> x_j
    const long long g = static_cast<long long>(blockIdx.x) * U_::TPC + tid;
    const long long K = geo.K[lev], SK = K * geo.S;
    if (g >= SK) return;
    const int l = tm.l;
    const int s = static_cast<int>(g / K);
    const long long c = g - s * K;
    const long long n = geo.n[lev];
    const int m = geo.m[lev];
    const long long st = c * m, en = min(n, st + m);
    const bool hasL = c > 0 || geo.segL;
    const bool nC = needC != 0;
    const long long base = static_cast<long long>(s) * n;
    const double* rr = src.rec;
    const long long SKp = src.SKp;
    const long long SnU = static_cast<long long>(geo.S) * (geo.n[lev + 1] + geo.segL), iR = g + geo.segL * (s + 1);
    // separators: x vectors every lane, C blocks by columns
    double xn[B], xL[B], Cnn[B], CnL[B], CLL[B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
        xn[i] = solU[(Sol<B>::X + i) * SnU + iR];
        xL[i] = hasL ? solU[(Sol<B>::X + i) * SnU + iR - 1] : 0.0;
        Cnn[i] = (nC && l < B) ? solU[(Sol<B>::CD + i * B + l) * SnU + iR] : 0.0;
        CLL[i] = (nC && hasL && l < B) ? solU[(Sol<B>::CD + i * B + l) * SnU + iR - 1] : 0.0;
        CnL[i] = (nC && hasL && l < B) ? solU[(Sol<B>::CU + l * B + i) * SnU + iR - 1] : 0.0;
    }
    auto put = [&](long long i, const double (&x)[B], const double (&Cc)[B]) {  // SolSink::put, column l
        const long long k = static_cast<long long>(s) * (sink.n + sink.segL) + sink.segL + i;
        if (l < B) {
            sink.sol[(Sol<B>::X + l) * sink.Sn + k] = pick<B>(x, l);
            if (nC)
#pragma unroll
                for (int q = 0; q < B; ++q) sink.sol[(Sol<B>::CD + q * B + l) * sink.Sn + k] = Cc[q];
        }
    };
    auto put_upper = [&](long long i, const double (&Cu)[B]) {  // column l of C_{i,i+1}
        const long long k = static_cast<long long>(s) * (sink.n + sink.segL) + sink.segL + i;
        if (l < B)
#pragma unroll
            for (int q = 0; q < B; ++q) sink.sol[(Sol<B>::CU + q * B + l) * sink.Sn + k] = Cu[q];
    };
    put(en - 1, xn, Cnn);
    if (c == 0 && geo.segL) put(-1, xL, CLL);
    for (long long j = en - 2; j >= st; --j) {
        const double* fp = fac + (g * m + (j - st)) * static_cast<long long>(NF);
        double Y[B], X[B];
        tsync(tm);
        if (l < B) {
#pragma unroll
            for (int i = 0; i < B; ++i) {
                if (i >= l) LS[i * LD + l] = fp[i * (i + 1) / 2 + l];
                Y[i] = hasL ? fp[NLI + i * B + l] : 0.0;
                X[i] = rr[(Rec<B>::LR + i * B + l) * SKp + base + j + 1];  // column l of upper(j)
            }
            vS[l] = fp[NLI + B * B + l];
        } else {
#pragma unroll
            for (int i = 0; i < B; ++i) {
                Y[i] = 0.0;
                X[i] = 0.0;
            }
        }
        tsync(tm);
        tlsolve<B, LD>(X, LS);
        colput<B, LD>(XS, X, l);
        if (hasL) colput<B, LD>(YS, Y, l);
        tsync(tm);
        {  // x_j = L^{-T}(z - X x_n - Y x_L), component l per lane
            double r[B];
            if (l < B) {
                double sx = 0.0, sy = 0.0;
                rowget<B, LD>(r, XS, l);
#pragma unroll
                for (int k = 0; k < B; ++k) sx = fma(r[k], xn[k], sx);
                double al = vS[l] - sx;
                if (hasL) {
                    rowget<B, LD>(r, YS, l);
#pragma unroll
                    for (int k = 0; k < B; ++k) sy = fma(r[k], xL[k], sy);
                    al -= sy;
                }
                wS[l] = al;
            }
            tsync(tm);
        }
        double xj[B];
#pragma unroll
        for (int i = 0; i < B; ++i) xj[i] = wS[i];
        tltsolve<B, LD>(xj, LS);
        double Cjj[B], CjL[B], Cjn[B];
        if (nC) {
            double P[B], tmp[B], q[B];
            tmv<B, LD>(P, XS, CnL);
            if (hasL) {
                tmv<B, LD>(tmp, YS, CLL);
#pragma unroll
                for (int i = 0; i < B; ++i) P[i] += tmp[i];
            }
            tmv<B, LD>(Cjn, XS, Cnn);
            if (hasL) {
                ttrans<B>(tm, q, CnL, vS + 2 * TeamCfg<B>::VEC);  // column l of C_{L,n}
                tmv<B, LD>(tmp, YS, q);
#pragma unroll
                for (int i = 0; i < B; ++i) Cjn[i] += tmp[i];
            }
            (void)tmp;
#pragma unroll
            for (int i = 0; i < B; ++i) {
                CjL[i] = P[i];
                Cjj[i] = Cjn[i];
            }
            tltsolve<B, LD>(CjL, LS);
            tltsolve<B, LD>(Cjn, LS);
#pragma unroll
            for (int i = 0; i < B; ++i) {
                CjL[i] = -CjL[i];
                Cjn[i] = -Cjn[i];
            }
            // M = I + P2 X^T + P1 Y^T with P2 = (pre-solve Cjn) in Cjj, P1 in P
            double* S6 = vS + 2 * TeamCfg<B>::VEC;
            double* S7 = S6 + TeamCfg<B>::MAT;
            tsync(tm);
            colput<B, LD>(S6, Cjj, l);
            colput<B, LD>(S7, P, l);
            tsync(tm);
            double M[B], rw[B];
            rowget<B, LD>(rw, XS, l);
            tmv<B, LD>(M, S6, rw);
            if (hasL) {
                rowget<B, LD>(rw, YS, l);
                tmv<B, LD>(tmp, S7, rw);
#pragma unroll
                for (int i = 0; i < B; ++i) M[i] += tmp[i];
            }
#pragma unroll
            for (int i = 0; i < B; ++i)
                if (i == l) M[i] += 1.0;
            tsym<B>(tm, M, S6);
            tltsolve<B, LD>(M, LS);
            ttrans<B>(tm, Cjj, M, S7);
            tltsolve<B, LD>(Cjj, LS);
            tsym<B>(tm, Cjj, S6);
        } else {
#pragma unroll
            for (int i = 0; i < B; ++i) {
                Cjj[i] = 0.0;
                CjL[i] = 0.0;
                Cjn[i] = 0.0;
            }
        }
        put(j, xj, Cjj);
        if (nC) put_upper(j, Cjn);
#pragma unroll
        for (int i = 0; i < B; ++i) {
            xn[i] = xj[i];
            Cnn[i] = Cjj[i];
            CnL[i] = CjL[i];
        }
    }
    if (hasL && nC) {  // C_{st-1, st} = C_{st, L}^T: column l = row l of C_{st, L}
        double q[B];
        ttrans<B>(tm, q, CnL, vS + 2 * TeamCfg<B>::VEC);
        put_upper(st - 1, q);
    }
}

}  // namespace spingp_dev
