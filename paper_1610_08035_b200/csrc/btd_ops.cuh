// btd_ops.cuh — btd_core on a materialised symmetric BTD:
// cr_solve / solve / logdet / selective_inverse through the same hierarchical
// partitioned elimination as the fused path, with the level-0 blocks read from
// the caller's diag/upper/rhs arrays (padded to the instantiated B).
#pragma once

#include "launch_eval.cuh"  // EvalBufs, tree_args, launch_tree, launch_tree_coop

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
    ctx->pre();
    k_fwdL<B, UserSource<B>><<<blocks_for(g.K[0], tpb), tpb, 0, ctx->stream>>>(usrc, g, 0, fac[0], rec[0],
                                                                               ctx->d_status);
    ctx->launched("k_fwd");
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
        k_revL<B, UserSource<B>, UserSink<B>><<<blocks_for(g.K[0], tpb), tpb, 0, ctx->stream>>>(
            usrc, usink, g, 0, fac[0], sol[1], needC ? 1 : 0);
        ctx->launched("k_rev");
    }
    if (d_logdet)  // toplogdet is the whole log-determinant (cumulative records)
        CUDA_OK(cudaMemcpyAsync(d_logdet, toplogdet, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
}

}  // namespace spingp_host
