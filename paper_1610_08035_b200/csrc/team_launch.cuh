// team_launch.cuh — host launchers of the b >= 6 team kernels (team.cuh).  Included
// only by the team_*.cu units, which are built fully inlined (no SP_DEV_NOINLINE): the
// team kernels keep their blocks in registers and shared memory, and a real call to the
// model code inside the step loop would spill every live register column to the stack.
#pragma once

#include "launch_eval.cuh"
#include "team.cuh"

namespace spingp_host {

template <class T>
void launch_fwd0_team(spingp_ctx* ctx, const ModelDesc& md, const EvalBufs& eb, const EvalArgs& a, const Geom& g,
                      const double* halo, long long c0, long long c1) {
    using C = TeamCfg<T::B>;
    static unsigned long long attr = 0;
    const int smem = C::TPCF * C::FWD * static_cast<int>(sizeof(double));
    opt_in_smem(reinterpret_cast<const void*>(k_fwd0_team<T>), attr, ctx->device, smem);
    const unsigned grid = static_cast<unsigned>((c1 - c0 + C::TPCF - 1) / C::TPCF);
    ctx->pre();
    k_fwd0_team<T><<<grid, C::CTA, smem, ctx->stream>>>(md, eb.params, a.d_t, a.d_y, g, eb.fac[0], eb.rec[0], eb.part,
                                                        ctx->d_status, halo, c0, c1, a.d_obs);
    ctx->launched("k_fwd0_team");
}

template <class T>
void launch_rev0_team(spingp_ctx* ctx, const ModelDesc& md, const EvalBufs& eb, const EvalArgs& a, const Geom& g,
                      const double* halo, const Outs& outs, long long c0, long long c1) {
    using C = TeamCfg<T::B>;
    static unsigned long long attr = 0;
    const int smem = C::TPCR * C::REV * static_cast<int>(sizeof(double));
    opt_in_smem(reinterpret_cast<const void*>(k_rev0_team<T>), attr, ctx->device, smem);
    const unsigned grid = static_cast<unsigned>((c1 - c0 + C::TPCR - 1) / C::TPCR);
    ctx->pre();
    k_rev0_team<T><<<grid, C::CTA, smem, ctx->stream>>>(md, eb.params, a.d_t, a.d_y, g, eb.fac[0], eb.sol[1], eb.part,
                                                        outs, ctx->d_status, halo, c0, c1, a.d_obs);
    ctx->launched("k_rev0_team");
}

// levels >= 1 for b >= 6 with team kernels: forward levels [1, lev_end), the top inverse
// (mode 0), reverse levels [1, nlev) (do_rev)
template <int B>
void launch_upper_team(spingp_ctx* ctx, const Geom& g, const EvalBufs& eb, bool do_fwd, bool do_top, bool do_rev,
                       bool needC) {
    using U_ = TeamUpper<B>;
    static unsigned long long attr_f = 0, attr_r = 0;
    const int smf = U_::TPC * U_::SMF * static_cast<int>(sizeof(double));
    const int smr = U_::TPC * U_::SMR * static_cast<int>(sizeof(double));
    opt_in_smem(reinterpret_cast<const void*>(k_fwdL_team<B>), attr_f, ctx->device, smf);
    opt_in_smem(reinterpret_cast<const void*>(k_revL_team<B>), attr_r, ctx->device, smr);
    if (do_fwd)
        for (int l = 1; l < g.nlev; ++l) {
            RecSource<B> src{eb.rec[l - 1], g.K[l - 1] * g.S, g.n[l]};
            const unsigned grid = static_cast<unsigned>((g.K[l] * g.S + U_::TPC - 1) / U_::TPC);
            ctx->pre();
            k_fwdL_team<B><<<grid, U_::CTA, smf, ctx->stream>>>(src, g, l, eb.fac[l], eb.rec[l], ctx->d_status);
            ctx->launched("k_fwdL_team");
        }
    if (do_top) {
        ctx->pre();
        k_top<B><<<blocks_for(g.S, 128), 128, 0, ctx->stream>>>(g, eb.rec[g.nlev - 1], eb.sol[g.nlev], eb.toplogdet,
                                                               ctx->d_status);
        ctx->launched("k_top");
    }
    if (do_rev)
        for (int l = g.nlev - 1; l >= 1; --l) {
            RecSource<B> src{eb.rec[l - 1], g.K[l - 1] * g.S, g.n[l]};
            SolSink<B> sink{eb.sol[l], (g.n[l] + g.segL) * g.S, g.n[l], g.segL};
            const unsigned grid = static_cast<unsigned>((g.K[l] * g.S + U_::TPC - 1) / U_::TPC);
            ctx->pre();
            k_revL_team<B><<<grid, U_::CTA, smr, ctx->stream>>>(src, sink, g, l, eb.fac[l], eb.sol[l + 1],
                                                                needC ? 1 : 0);
            ctx->launched("k_revL_team");
        }
}

}  // namespace spingp_host

#define SPINGP_TEAM_UPPER_INST(B)                                                                             \
    template void spingp_host::launch_upper_team<B>(spingp_ctx*, const Geom&, const EvalBufs&, bool, bool, bool, bool);
#define SPINGP_TEAM_INST(...)                                                                                  \
    template void spingp_host::launch_fwd0_team<__VA_ARGS__>(spingp_ctx*, const ModelDesc&, const EvalBufs&, const EvalArgs&, \
                                                   const Geom&, const double*, long long, long long);             \
    template void spingp_host::launch_rev0_team<__VA_ARGS__>(spingp_ctx*, const ModelDesc&, const EvalBufs&, const EvalArgs&, \
                                                   const Geom&, const double*, const Outs&, long long, long long);
