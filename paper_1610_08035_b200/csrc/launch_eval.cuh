// launch_eval.cuh — the fused evaluation pipeline for one kernel-traits type:
// level-0 fused forward -> upper-level forwards -> top inverse -> upper-level
// reverses -> level-0 fused reverse (outputs, loglik terms, gradient) ->
// deterministic two-stage reduction.  Included by the inst_*.cu files only.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ctx.hpp"

namespace spingp_host {

using namespace spingp_dev;

struct EvalBufs {
    double* params;
    double* fac[kMaxLev];
    double* rec[kMaxLev];
    double* sol[kMaxLev + 1];
    double* toplogdet;
    double* part;
    double* seg;
    int nseg;
    double* segscratch;
    unsigned int* arrive;  // per-series counters of k_reduce (zeroed at workspace creation)
};

template <int B>
EvalBufs carve_eval(spingp_ctx* ctx, const Plan& p, int nt, size_t params_count) {
    const Geom& g = p.geo;
    size_t tot = arena_bytes(params_count) + 4096;
    for (int l = 0; l < g.nlev; ++l) {
        const size_t SK = static_cast<size_t>(g.K[l]) * g.S;
        tot += arena_bytes(static_cast<size_t>(g.m[l]) * Fac<B>::N * SK) + arena_bytes(Rec<B>::N * SK);
    }
    for (int l = 1; l <= g.nlev; ++l) tot += arena_bytes(Sol<B>::N * static_cast<size_t>(g.n[l] + g.segL) * g.S);
    const size_t SK0 = static_cast<size_t>(g.K[0]) * g.S;
    const int nseg = static_cast<int>((g.K[0] + kSeg - 1) / kSeg);
    tot += arena_bytes(g.S) + arena_bytes((P_GRAD + nt) * SK0) +
           arena_bytes(static_cast<size_t>(nseg) * g.S * (P_GRAD + nt)) + arena_bytes(64 * (2 * B * B + B));
    ctx->ensure_ws(tot);
    ctx->ws.reset();
    EvalBufs eb{};
    eb.params = ctx->ws.take<double>(params_count);
    for (int l = 0; l < g.nlev; ++l) {
        const size_t SK = static_cast<size_t>(g.K[l]) * g.S;
        eb.fac[l] = ctx->ws.take<double>(static_cast<size_t>(g.m[l]) * Fac<B>::N * SK);
        eb.rec[l] = ctx->ws.take<double>(Rec<B>::N * SK);
    }
    for (int l = 1; l <= g.nlev; ++l)
        eb.sol[l] = ctx->ws.take<double>(Sol<B>::N * static_cast<size_t>(g.n[l] + g.segL) * g.S);
    eb.toplogdet = ctx->ws.take<double>(g.S);
    eb.part = ctx->ws.take<double>((P_GRAD + nt) * SK0);
    eb.nseg = nseg;
    eb.seg = ctx->ws.take<double>(static_cast<size_t>(nseg) * g.S * (P_GRAD + nt));
    eb.segscratch = ctx->ws.take<double>(64 * (2 * B * B + B));
    eb.arrive = ctx->counters(g.S);
    return eb;
}

// Levels >= 1 as one cooperative launch (default) or as per-level kernels
// (SPINGP_UPPER=levels: A/B comparison knob).
inline bool upper_fused() {
    static const bool f = [] {
        const char* e = std::getenv("SPINGP_UPPER");
        return !(e && std::strcmp(e, "levels") == 0);
    }();
    return f;
}

template <int B>
void launch_upper(spingp_ctx* ctx, const Geom& g, UpperArgs& ua) {
    constexpr int tpb = 128;
    static int resident = 0;  // co-resident CTAs of k_upper<B> on this device type
    if (!resident) {
        int per = 0, dev = 0, sms = 0;
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_upper<B>, tpb, 0));
        CUDA_OK(cudaGetDevice(&dev));
        CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        resident = std::max(1, per) * sms;
    }
    long long work = g.S;
    for (int l = 1; l < g.nlev; ++l) work = std::max(work, g.K[l] * g.S);
    const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>(resident, (work + tpb - 1) / tpb)));
    Geom geo = g;
    void* args[] = {&geo, &ua};
    ctx->pre();
    CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_upper<B>), dim3(grid), dim3(tpb), args, 0,
                                        ctx->stream));
    ctx->launched("k_upper");
}

template <class T>
void launch_eval(spingp_ctx* ctx, const EvalArgs& a) {
    constexpr int B = T::B;
    const HostModel& hm = *a.hm;
    const Geom& g = a.plan->geo;
    const int nt = hm.nt;
    const size_t ncount = a.nparams + hm.eqconst.size();
    EvalBufs eb = carve_eval<B>(ctx, *a.plan, nt, ncount);
    // parameters + EQ constants: one upload through the pinned stage
    double* st = ctx->stage(ncount);
    std::memcpy(st, a.h_params, a.nparams * sizeof(double));
    if (!hm.eqconst.empty()) std::memcpy(st + a.nparams, hm.eqconst.data(), hm.eqconst.size() * sizeof(double));
    CUDA_OK(cudaMemcpyAsync(eb.params, st, ncount * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ctx->stage_done();
    ModelDesc md = hm.desc;
    md.eqconst = eb.params + a.nparams;
    // segment halo times (t_left, t_right) are the last two doubles of h_params' tail
    const double* halo = (a.mode >= 2) ? eb.params + a.nparams - 2 : nullptr;

    const int tpb = 128;
    if (a.mode == 1) {
        ctx->pre();
        k_assemble<T><<<blocks_for(g.n[0], tpb), tpb, 0, ctx->stream>>>(md, eb.params, a.d_t, a.d_y, g.n[0], a.d_diag,
                                                                       a.d_upper, a.d_rhs, ctx->d_status);
        ctx->launched("k_assemble");
        return;
    }
    const long long SK0 = g.K[0] * g.S;
    const bool grad = a.flags & SPINGP_WANT_GRAD;
    const bool needC = grad || (a.flags & SPINGP_WANT_VAR);
    const bool fused = upper_fused();
    if (a.mode != 3) {
        ctx->pre();
        k_fwd0<T><<<blocks_for(SK0, tpb), tpb, 0, ctx->stream>>>(md, eb.params, a.d_t, a.d_y, g, eb.fac[0],
                                                                 eb.rec[0], eb.part, ctx->d_status, halo);
        ctx->launched("k_fwd0");
        if (!fused || a.mode == 2) {
            for (int l = 1; l < g.nlev; ++l) {
                RecSource<B> src{eb.rec[l - 1], g.K[l - 1] * g.S, g.n[l]};
                ctx->pre();
                k_fwdL<B, RecSource<B>><<<blocks_for(g.K[l] * g.S, tpb), tpb, 0, ctx->stream>>>(
                    src, g, l, eb.fac[l], eb.rec[l], ctx->d_status);
                ctx->launched("k_fwd");
            }
        }
    }
    if (a.mode == 2) {  // segment forward: hand this rank's top-level record to the caller
        CUDA_OK(cudaMemcpyAsync(a.d_seg_out, eb.rec[g.nlev - 1], Rec<B>::N * sizeof(double),
                                cudaMemcpyDeviceToDevice, ctx->stream));
        return;
    }
    if (a.mode == 3) {
        ctx->pre();
        k_seg_solve<B><<<1, 1, 0, ctx->stream>>>(a.nranks, a.rank, a.d_seg_in, eb.sol[g.nlev], eb.toplogdet,
                                                 ctx->d_status, g.n[0] - 1, eb.segscratch);
        ctx->launched("k_seg_solve");
    }
    if (fused && (a.mode == 0 || g.nlev > 1)) {
        UpperArgs ua{};
        for (int l = 0; l < g.nlev; ++l) {
            ua.rec[l] = eb.rec[l];
            ua.fac[l] = eb.fac[l];
        }
        for (int l = 1; l <= g.nlev; ++l) ua.sol[l] = eb.sol[l];
        ua.toplogdet = eb.toplogdet;
        ua.status = ctx->d_status;
        ua.needC = needC ? 1 : 0;
        ua.do_fwd = a.mode == 0;
        ua.do_top = a.mode == 0;
        ua.do_rev = 1;
        ua.stamps = ctx->upper_stamps;
        launch_upper<B>(ctx, g, ua);
    } else {
        if (a.mode != 3) {
            ctx->pre();
            k_top<B><<<blocks_for(g.S, 128), 128, 0, ctx->stream>>>(g, eb.rec[g.nlev - 1], eb.sol[g.nlev],
                                                                   eb.toplogdet, ctx->d_status);
            ctx->launched("k_top");
        }
        for (int l = g.nlev - 1; l >= 1; --l) {
            RecSource<B> src{eb.rec[l - 1], g.K[l - 1] * g.S, g.n[l]};
            SolSink<B> sink{eb.sol[l], (g.n[l] + g.segL) * g.S, g.n[l], g.segL};
            ctx->pre();
            k_revL<B, RecSource<B>, SolSink<B>><<<blocks_for(g.K[l] * g.S, tpb), tpb, 0, ctx->stream>>>(
                src, sink, g, l, eb.fac[l], eb.sol[l + 1], needC ? 1 : 0);
            ctx->launched("k_rev");
        }
    }
    Outs outs{(a.flags & SPINGP_WANT_MEAN) ? a.d_mean : nullptr, (a.flags & SPINGP_WANT_VAR) ? a.d_var : nullptr,
              (a.flags & SPINGP_INCLUDE_NOISE) ? 1 : 0, grad ? 1 : 0, needC ? 1 : 0};
    ctx->pre();
    k_rev0<T><<<blocks_for(SK0, tpb), tpb, 0, ctx->stream>>>(md, eb.params, a.d_t, a.d_y, g, eb.fac[0],
                                                             eb.sol[1], eb.part, outs, ctx->d_status, halo);
    ctx->launched("k_rev0");
    FinalArgs fa{};
    fa.part = eb.part;
    fa.K = g.K[0];
    fa.NC = P_GRAD + nt;
    fa.seg = eb.seg;
    fa.arrive = eb.arrive;
    fa.toplogdet = eb.toplogdet;
    fa.params = eb.params;
    fa.rec_stride = hm.rec_stride;
    fa.nt = nt;
    fa.n = g.n[0];
    fa.loglik = a.d_loglik;
    fa.grad = grad ? a.d_grad : nullptr;
    fa.partials = a.mode == 3 ? a.d_seg_out : nullptr;
    ctx->pre();
    k_reduce<<<dim3(eb.nseg, g.S), kRedThreads, 0, ctx->stream>>>(fa);
    ctx->launched("k_reduce");
}

}  // namespace spingp_host
