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

}  // namespace spingp_host

#define SPINGP_TEAM_INST(...)                                                                                  \
    template void spingp_host::launch_fwd0_team<__VA_ARGS__>(spingp_ctx*, const ModelDesc&, const EvalBufs&, const EvalArgs&, \
                                                   const Geom&, const double*, long long, long long);             \
    template void spingp_host::launch_rev0_team<__VA_ARGS__>(spingp_ctx*, const ModelDesc&, const EvalBufs&, const EvalArgs&, \
                                                   const Geom&, const double*, const Outs&, long long, long long);
