// btd_ops.cuh — btd_core on a materialised symmetric BTD:
// cr_solve / solve / logdet / selective_inverse through the same hierarchical
// partitioned elimination as the fused path, with the level-0 blocks read from
// the caller's diag/upper/rhs arrays (padded to the instantiated B).
#pragma once

#include "launch_eval.cuh"  // EvalBufs, tree_args, launch_tree, launch_tree_coop


namespace spingp_dev {

// Level 0 of the materialised solve (cr_solve with the selected inverse off, b = B <= 4):
// the same elimination as fwdL_item / revL_item over UserSource, with the caller's
// row-major blocks streamed through a per-thread shared-memory ring of kSolveDepth blocks
// filled by asynchronous 8-byte copies (cp.async): the strided per-chunk reads of a warp
// are in flight several blocks ahead instead of one (round 1: k_fwdL<UserSource> at 2.3
// TB/s, latency-bound).  Ring layout ring[slot][component][thread] (conflict-free).
constexpr int kSolveDepth = 3;
constexpr int kSolveTpb = 128;

SP_DEVM void async8(double* dst, const double* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}
SP_DEVM void async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
SP_DEVM void async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int B>
__global__ void __launch_bounds__(kSolveTpb, 3) k_fwd0_solve(UserSource<B> src, Geom geo, double* __restrict__ fac,
                                                              double* __restrict__ rec, unsigned long long* status) {
    constexpr int NW = 2 * B * B + B;  // D, U, r of one block
    extern __shared__ double ring_solve[];
    const long long K = geo.K[0], SK = K;
    const long long g = blockIdx.x * static_cast<long long>(kSolveTpb) + threadIdx.x;
    if (g >= SK) return;
    const int tid = threadIdx.x;
    const long long n = geo.n[0];
    const int m = geo.m[0];
    const long long st = g * m, en = min(n, st + m);
    const bool hasL = g > 0;
    auto slot = [&](int k, int w) -> double* { return ring_solve + (static_cast<size_t>(k) * NW + w) * kSolveTpb + tid; };
    auto fetch = [&](long long j) {  // block j (D, U if j < n - 1, r) into its ring slot
        const int k = static_cast<int>((j - st) % kSolveDepth);
        const double* d = src.diag + j * B * B;
#pragma unroll
        for (int q = 0; q < B * B; ++q) async8(slot(k, q), d + q);
        if (j + 1 < n) {
            const double* u = src.up + j * B * B;
#pragma unroll
            for (int q = 0; q < B * B; ++q) async8(slot(k, B * B + q), u + q);
        }
#pragma unroll
        for (int q = 0; q < B; ++q) async8(slot(k, 2 * B * B + q), src.rhs + (j * B + q) * src.k + src.col);
    };
    for (int p = 0; p < kSolveDepth; ++p) {
        if (st + p < en) fetch(st + p);
        async_commit();
    }
    ElimState<B> es;
    elim_init<B>(es);
    if (hasL) {  // P_{st, st-1} = upper(st-1)^T
        double U[B * B];
        src.upper(0, st - 1, U);
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
            for (int j = 0; j < B; ++j) es.W[i * B + j] = U[j * B + i];
    }
    double D[B * B], U[B * B], r[B];
    for (long long j = st; j < en; ++j) {
        async_wait<kSolveDepth - 1>();  // block j has landed (groups complete in order)
        const int k = static_cast<int>((j - st) % kSolveDepth);
#pragma unroll
        for (int q = 0; q < B * B; ++q) D[q] = *slot(k, q);
#pragma unroll
        for (int q = 0; q < B * B; ++q) U[q] = (j + 1 < n) ? *slot(k, B * B + q) : 0.0;
#pragma unroll
        for (int q = 0; q < B; ++q) r[q] = *slot(k, 2 * B * B + q);
        if (j + kSolveDepth < en) fetch(j + kSolveDepth);  // the slot just read
        async_commit();
        if (j == en - 1) break;
        double* fp = fac + (j - st) * Fac<B>::N * SK + g;
        if (!elim_block<B>(es, D, U, r, hasL, fp, SK)) {
            report(status, j, ST_NOT_PD);
            return;
        }
    }
    async_wait<0>();
#pragma unroll
    for (int i = 0; i < B * B; ++i) D[i] -= es.T[i];
#pragma unroll
    for (int i = 0; i < B; ++i) r[i] -= es.rc[i];
    write_rec<B>(rec, SK, g, es, D, r, hasL);
}

template <int B>
__global__ void __launch_bounds__(kSolveTpb, 2) k_rev0_solve(UserSource<B> src, UserSink<B> sink, Geom geo,
                                                              const double* __restrict__ fac,
                                                              const double* __restrict__ solU) {
    extern __shared__ double ring_solve[];
    const long long K = geo.K[0], SK = K;
    const long long g = blockIdx.x * static_cast<long long>(kSolveTpb) + threadIdx.x;
    if (g >= SK) return;
    const int tid = threadIdx.x;
    const long long n = geo.n[0];
    const int m = geo.m[0];
    const long long st = g * m, en = min(n, st + m);
    const bool hasL = g > 0;
    auto slot = [&](int k, int w) -> double* {
        return ring_solve + (static_cast<size_t>(k) * B * B + w) * kSolveTpb + tid;
    };
    // U blocks en-2 down to st, streamed in that order
    auto fetch = [&](long long j) {
        const int k = static_cast<int>((en - 2 - j) % kSolveDepth);
        const double* u = src.up + j * B * B;
#pragma unroll
        for (int q = 0; q < B * B; ++q) async8(slot(k, q), u + q);
    };
    for (int p = 0; p < kSolveDepth; ++p) {
        if (en - 2 - p >= st) fetch(en - 2 - p);
        async_commit();
    }
    SepData<B> sd;
    load_sep<B>(solU, static_cast<long long>(geo.n[1]), g, hasL, false, sd);
    double xn[B];
#pragma unroll
    for (int q = 0; q < B; ++q) xn[q] = sd.xR[q];
    double Cz[B * B];
    mzero<B>(Cz);
    sink.put(0, en - 1, xn, Cz, false);
    for (long long j = en - 2; j >= st; --j) {
        async_wait<kSolveDepth - 1>();
        const int k = static_cast<int>((en - 2 - j) % kSolveDepth);
        double U[B * B], Li[B * B], Y[B * B], z[B], X[B * B];
#pragma unroll
        for (int q = 0; q < B * B; ++q) U[q] = *slot(k, q);
        if (j - kSolveDepth >= st) fetch(j - kSolveDepth);
        async_commit();
        load_fac<B>(fac + (j - st) * Fac<B>::N * SK + g, SK, hasL, Li, Y, z);
        lsolve<B>(X, Li, U);
        double xj[B], CjL[B * B], Cjn[B * B], Cjj[B * B];
        back_step<B>(Li, Y, z, X, hasL, false, sd, xn, Cz, Cz, xj, CjL, Cjn, Cjj);
        sink.put(0, j, xj, Cz, false);
#pragma unroll
        for (int q = 0; q < B; ++q) xn[q] = xj[q];
    }
    async_wait<0>();
}

}  // namespace spingp_dev

namespace spingp_host {

using namespace spingp_dev;

template <int B>
void launch_btd(spingp_ctx* ctx, int64_t n, int b, const double* d_diag, const double* d_upper,
                const double* d_rhs, int k, int col, double* d_x, double* d_cdiag, double* d_cupper,
                double* d_logdet, bool needC) {
    const Plan plan = make_plan(n, 1, B, ctx->m0_override, -1, ctx->g_override);
    const Geom& g = plan.geo;
    size_t tot = 4096;
    for (int l = 0; l < g.nlev; ++l)
        tot += arena_bytes(static_cast<size_t>(g.m[l]) * (l ? Tree<B>::NF : Fac<B>::N) * g.K[l]) +
               arena_bytes(Rec<B>::N * g.K[l]);
    for (int l = 1; l <= g.nlev; ++l) tot += arena_bytes(Sol<B>::N * static_cast<size_t>(g.n[l]));
    tot += arena_bytes(1);
    ctx->ensure_ws(tot);
    ctx->ws.reset();
    EvalBufs eb{};
    double* fac[kMaxLev];
    double* rec[kMaxLev];
    double* sol[kMaxLev + 1];
    for (int l = 0; l < g.nlev; ++l) {
        fac[l] = eb.fac[l] = ctx->ws.take<double>(static_cast<size_t>(g.m[l]) * (l ? Tree<B>::NF : Fac<B>::N) * g.K[l]);
        rec[l] = eb.rec[l] = ctx->ws.take<double>(Rec<B>::N * g.K[l]);
    }
    for (int l = 1; l <= g.nlev; ++l) sol[l] = eb.sol[l] = ctx->ws.take<double>(Sol<B>::N * static_cast<size_t>(g.n[l]));
    double* toplogdet = eb.toplogdet = ctx->ws.take<double>(1);
    const int tpb = 128;
    UserSource<B> usrc{d_diag, d_upper, d_rhs, n, b, k, col};
    // solve only (no selected inverse), unpadded blocks with a right-hand side: the
    // cp.async-staged level-0 kernels (SPINGP_SOLVE_STAGED=0 selects the generic ones)
    static const bool staged_on = [] {
        const char* e = std::getenv("SPINGP_SOLVE_STAGED");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    const bool staged = staged_on && !needC && b == B && B <= 4 && d_rhs && n > 1;
    ctx->pre();
    if (staged) {
        if constexpr (B <= 4) {
            const int smem = kSolveDepth * (2 * B * B + B) * kSolveTpb * static_cast<int>(sizeof(double));
            static unsigned long long attr = 0;
            opt_in_smem(reinterpret_cast<const void*>(k_fwd0_solve<B>), attr, ctx->device, smem);
            k_fwd0_solve<B><<<blocks_for(g.K[0], kSolveTpb), kSolveTpb, smem, ctx->stream>>>(usrc, g, fac[0], rec[0],
                                                                                        ctx->d_status);
        }
    } else {
        k_fwdL<B, UserSource<B>><<<blocks_for(g.K[0], tpb), tpb, 0, ctx->stream>>>(usrc, g, 0, fac[0], rec[0],
                                                                                   ctx->d_status);
    }
    ctx->launched(staged ? "k_fwd0_solve" : "k_fwd");
    constexpr bool kTree = B <= 4;  // tree levels are built for b <= 4 only
    if (kTree && plan.tree) {  // levels >= 1 as shared-memory trees (tree.cuh), as in launch_eval
        if constexpr (kTree) {
            int l = g.nlev - 1;
            bool coop = false;
            if (g.nlev >= 3) {
                for (int f = 1; f <= g.nlev - 3; ++f) {
                    TreeArgs ta = tree_args<B>(ctx, g, eb, f, needC);
                    launch_tree<B>(ctx, TREE_FWD, ta);
                }
                TreeArgs t1 = tree_args<B>(ctx, g, eb, g.nlev - 2, needC);
                TreeArgs t2 = tree_args<B>(ctx, g, eb, g.nlev - 1, needC);
                coop = launch_tree_coop<B>(ctx, t1, t2);
                if (!coop) launch_tree<B>(ctx, TREE_FWD, t1);
            }
            if (coop) {
                l = g.nlev - 3;
            } else {
                TreeArgs ta = tree_args<B>(ctx, g, eb, l, needC);
                launch_tree<B>(ctx, TREE_ONE, ta);
                --l;
            }
            for (; l >= 1; --l) {
                TreeArgs ta = tree_args<B>(ctx, g, eb, l, needC);
                launch_tree<B>(ctx, TREE_REV, ta);
            }
            }
    } else {
    for (int l = 1; l < g.nlev; ++l) {
        RecSource<B> src{rec[l - 1], g.K[l - 1], g.n[l]};
        ctx->pre();
        k_fwdL<B, RecSource<B>><<<blocks_for(g.K[l], tpb), tpb, 0, ctx->stream>>>(src, g, l, fac[l], rec[l],
                                                                                 ctx->d_status);
        ctx->launched("k_fwd");
    }
    ctx->pre();
    k_top<B><<<1, 32, 0, ctx->stream>>>(g, rec[g.nlev - 1], sol[g.nlev], toplogdet, ctx->d_status);
    ctx->launched("k_top");
    for (int l = g.nlev - 1; l >= 1; --l) {
        RecSource<B> src{rec[l - 1], g.K[l - 1], g.n[l]};
        SolSink<B> sink{sol[l], g.n[l], g.n[l], 0};
        ctx->pre();
        k_revL<B, RecSource<B>, SolSink<B>><<<blocks_for(g.K[l], tpb), tpb, 0, ctx->stream>>>(
            src, sink, g, l, fac[l], sol[l + 1], needC ? 1 : 0);
        ctx->launched("k_rev");
    }
    }
    if (d_x || needC) {
        UserSink<B> usink{d_x, d_cdiag, d_cupper, b, k, col};
        ctx->pre();
        if (staged && d_x) {
            if constexpr (B <= 4) {
                const int smem = kSolveDepth * B * B * kSolveTpb * static_cast<int>(sizeof(double));
                k_rev0_solve<B><<<blocks_for(g.K[0], kSolveTpb), kSolveTpb, smem, ctx->stream>>>(usrc, usink, g,
                                                                                            fac[0], sol[1]);
            }
        } else {
            k_revL<B, UserSource<B>, UserSink<B>><<<blocks_for(g.K[0], tpb), tpb, 0, ctx->stream>>>(
                usrc, usink, g, 0, fac[0], sol[1], needC ? 1 : 0);
        }
        ctx->launched(staged && d_x ? "k_rev0_solve" : "k_rev");
    }
    if (d_logdet)  // toplogdet is the whole log-determinant (cumulative records)
        CUDA_OK(cudaMemcpyAsync(d_logdet, toplogdet, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
}

}  // namespace spingp_host
