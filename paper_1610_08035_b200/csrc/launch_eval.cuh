// launch_eval.cuh — the fused evaluation pipeline for one kernel-traits type:
// level-0 fused forward -> upper-level forwards -> top inverse -> upper-level
// reverses -> level-0 fused reverse (outputs, loglik terms, gradient) ->
// deterministic two-stage reduction.  Included by the inst_*.cu files only.
// Upper levels: shared-memory tree groups (tree.cuh; default), or the per-thread
// 4-record chains as one cooperative kernel (SPINGP_UPPER=coop) or one kernel per
// level (SPINGP_UPPER=levels).
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ctx.hpp"
#include "tree.cuh"

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
        tot += arena_bytes(static_cast<size_t>(g.m[l]) * (l ? Tree<B>::NF : Fac<B>::N) * SK) + arena_bytes(Rec<B>::N * SK);
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
        eb.fac[l] = ctx->ws.take<double>(static_cast<size_t>(g.m[l]) * (l ? Tree<B>::NF : Fac<B>::N) * SK);
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
    static int resident_dev[64] = {};  // co-resident CTAs of k_upper<B>, per device
    int& resident = resident_dev[ctx->device & 63];
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

// Tree level l (>= 1): groups of m[l] records of level l-1.
template <int B>
TreeArgs tree_args(spingp_ctx* ctx, const Geom& g, const EvalBufs& eb, int l, bool needC) {
    TreeArgs ta{};
    ta.rec_in = eb.rec[l - 1];
    ta.SKin = g.K[l - 1] * g.S;
    ta.nin = g.n[l];
    ta.rec_out = eb.rec[l];
    ta.fac = eb.fac[l];
    ta.solU = eb.sol[l + 1];
    ta.sol = eb.sol[l];
    ta.toplogdet = eb.toplogdet;
    ta.status = ctx->d_status;
    ta.G = g.m[l];
    ta.nG = static_cast<int>(g.K[l]);
    ta.S = g.S;
    ta.segL = g.segL;
    ta.needC = needC ? 1 : 0;
    const long long gcap = std::min<long long>(g.m[l], g.n[l]);
    ta.RS = static_cast<int>(tree_row(gcap));
    ta.ES = static_cast<int>(tree_row(gcap + 1));
    ta.span = 1;
    for (int i = 1; i < l; ++i) ta.span *= g.m[i];
    ta.K0 = g.K[0];
    ta.n0 = g.n[0];
    ta.m0 = g.m[0];
    return ta;
}

enum TreeKind { TREE_FWD = 0, TREE_REV = 1, TREE_ONE = 2 };

template <int B>
void launch_tree(spingp_ctx* ctx, TreeKind kind, TreeArgs& ta) {
    using TR = Tree<B>;
    void (*kern)(TreeArgs) = kind == TREE_FWD ? k_tree_fwd<B> : kind == TREE_REV ? k_tree_rev<B> : k_tree_one<B>;
    static unsigned long long attr[3] = {0, 0, 0};  // opt in to 227 KB of shared memory per device
    opt_in_smem(reinterpret_cast<const void*>(kern), attr[kind], ctx->device,
                static_cast<int>(tree_smem_bytes(B, tree_group_size(B))));
    const size_t smem = 8 * (static_cast<size_t>(TR::NR) * ta.RS + (kind == TREE_FWD ? 0 : static_cast<size_t>(TR::NS) * ta.ES));
    const int half = std::min(ta.G, static_cast<int>(ta.RS)) / 2 + 1;  // nodes of the first round
    const int tpb = std::min(kTreeMaxThreads, std::max(32, (half + 31) / 32 * 32));
    const long long groups = static_cast<long long>(ta.S) * ta.nG;
    // diagnostics: stamps of CTA 0 at [0,16) k_tree_fwd, [16,48) k_tree_one, [48,64) k_tree_rev
    ta.stamps = ctx->upper_stamps ? ctx->upper_stamps + (kind == TREE_FWD ? 0 : kind == TREE_ONE ? 16 : 48) : nullptr;
    ctx->pre();
    kern<<<static_cast<unsigned>(groups), tpb, smem, ctx->stream>>>(ta);
    ctx->launched(kind == TREE_FWD ? "k_tree_fwd" : kind == TREE_REV ? "k_tree_rev" : "k_tree_one");
}

// Levels L-1 and L (= nlev-1, one group per series) as one cooperative launch when
// every level-(L-1) group gets a co-resident CTA and the top group fits the
// separator area (SPINGP_TREE_COOP=0 disables).
template <int B>
bool launch_tree_coop(spingp_ctx* ctx, TreeArgs& a1, TreeArgs& a2) {
    using TR = Tree<B>;
    static const bool enabled = [] {
        const char* e = std::getenv("SPINGP_TREE_COOP");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    if (!enabled) return false;
    const size_t smem = 8 * (static_cast<size_t>(TR::NR) * a1.RS + static_cast<size_t>(TR::NS) * a1.ES);
    if (static_cast<size_t>(TR::NR) * a2.RS + static_cast<size_t>(TR::NS) * a2.ES >
        static_cast<size_t>(TR::NS) * a1.ES)
        return false;
    const int half = std::min(a1.G, static_cast<int>(a1.RS)) / 2 + 1;
    const int half2 = static_cast<int>(a2.RS) / 2 + 1;
    const int tpb = std::min(kTreeMaxThreads, std::max(32, (std::max(half, half2) + 31) / 32 * 32));
    if ((a2.RS + 1) / 2 > tpb) return false;
    static unsigned long long set = 0;
    opt_in_smem(reinterpret_cast<const void*>(k_tree_coop<B>), set, ctx->device,
                static_cast<int>(tree_smem_bytes(B, tree_group_size(B))));
    int sms = 0, per = 0;  // device SMs, co-resident CTAs of this shape (cheap queries)
    CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_tree_coop<B>, tpb, smem));
    const long long groups = static_cast<long long>(a1.S) * a1.nG;
    if (groups > static_cast<long long>(per) * sms) return false;
    a1.stamps = ctx->upper_stamps;
    a2.stamps = nullptr;
    void* args[] = {&a1, &a2};
    ctx->pre();
    CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_tree_coop<B>), dim3(static_cast<unsigned>(groups)),
                                        dim3(tpb), args, smem, ctx->stream));
    ctx->launched("k_tree_coop");
    return true;
}

// b >= 6: the level-0 kernels run one team of lanes per chunk (team.cuh);
// SPINGP_TEAM=0 selects the thread-per-chunk kernels (A/B knob).
inline bool team_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SPINGP_TEAM");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    return on;
}

// b >= 6 team kernels: launchers defined in the fully inlined team_*.cu units (team_launch.cuh)
template <class T>
void launch_fwd0_team(spingp_ctx* ctx, const ModelDesc& md, const EvalBufs& eb, const EvalArgs& a, const Geom& g,
                      const double* halo, long long c0, long long c1);
template <class T>
void launch_rev0_team(spingp_ctx* ctx, const ModelDesc& md, const EvalBufs& eb, const EvalArgs& a, const Geom& g,
                      const double* halo, const Outs& outs, long long c0, long long c1);
template <int B>
void launch_upper_team(spingp_ctx* ctx, const Geom& g, const EvalBufs& eb, bool do_fwd, bool do_top, bool do_rev,
                       bool needC);

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
    const bool grad = a.flags & SPINGP_WANT_GRAD;
    const bool needC = grad || (a.flags & SPINGP_WANT_VAR);
    if (a.mode == 1) {
        ctx->pre();
        k_assemble<T><<<blocks_for(g.n[0], tpb), tpb, 0, ctx->stream>>>(md, eb.params, a.d_t, a.d_y, g.n[0], a.d_diag,
                                                                       a.d_upper, a.d_rhs, ctx->d_status);
        ctx->launched("k_assemble");
        return;
    }
    const long long SK0 = g.K[0] * g.S;
    // tree levels are built for b <= 4 only (make_plan never plans them above)
    constexpr bool kTree = B <= 4;
    const bool tree = kTree && a.plan->tree;
    bool coop = false;  // top two tree levels in one cooperative launch
    const bool fused = upper_fused();
    if (a.mode != 3) {
        const int np = a.in_pieces > 0 ? a.in_pieces : 1;
        for (int p = 0; p < np; ++p) {
            const long long c0 = a.in_pieces > 0 ? a.in_chunk[p] : 0, c1 = a.in_pieces > 0 ? a.in_chunk[p + 1] : SK0;
            if (a.in_pieces > 0) CUDA_OK(cudaStreamWaitEvent(ctx->stream, a.in_ready[p], 0));
            if (c1 <= c0) continue;
            if constexpr (B >= 6) {
                if (team_enabled()) {
                    launch_fwd0_team<T>(ctx, md, eb, a, g, halo, c0, c1);
                    continue;
                }
            }
            ctx->pre();
            k_fwd0<T><<<blocks_for(c1 - c0, tpb), tpb, 0, ctx->stream>>>(md, eb.params, a.d_t, a.d_y, g, eb.fac[0],
                                                                         eb.rec[0], eb.part, ctx->d_status, halo,
                                                                         c0, c1, a.d_obs);
            ctx->launched("k_fwd0");
        }
        if (tree) {
            if constexpr (kTree) {
                // mode 0: the last level (one group per series) is k_tree_one, or the two
                // top levels k_tree_coop, below
                coop = a.mode == 0 && g.nlev >= 3;
                if (coop) {
                    TreeArgs t1 = tree_args<B>(ctx, g, eb, g.nlev - 2, needC);
                    TreeArgs t2 = tree_args<B>(ctx, g, eb, g.nlev - 1, needC);
                    const int lowf = g.nlev - 3;
                    for (int l = 1; l <= lowf; ++l) {
                        TreeArgs ta = tree_args<B>(ctx, g, eb, l, needC);
                        launch_tree<B>(ctx, TREE_FWD, ta);
                    }
                    coop = launch_tree_coop<B>(ctx, t1, t2);
                    if (!coop) {
                        launch_tree<B>(ctx, TREE_FWD, t1);
                    }
                }
                const int lastf = a.mode == 0 ? g.nlev - 2 : g.nlev - 1;
                for (int l = (a.mode == 0 && g.nlev >= 3) ? lastf + 1 : 1; l <= lastf; ++l) {
                    TreeArgs ta = tree_args<B>(ctx, g, eb, l, needC);
                    launch_tree<B>(ctx, TREE_FWD, ta);
                }
                    }
        } else if (B >= 6 && team_enabled()) {
            if constexpr (B >= 6) launch_upper_team<B>(ctx, g, eb, true, false, false, needC);
        } else if (!fused || a.mode == 2) {
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
    if (tree) {
        if constexpr (kTree) {
            int l = g.nlev - 1;
            if (coop) {
                l = g.nlev - 3;
            } else if (a.mode == 0) {
                TreeArgs ta = tree_args<B>(ctx, g, eb, l, needC);
                launch_tree<B>(ctx, TREE_ONE, ta);
                --l;
            }
            for (; l >= 1; --l) {
                TreeArgs ta = tree_args<B>(ctx, g, eb, l, needC);
                launch_tree<B>(ctx, TREE_REV, ta);
            }
            }
    } else if (B >= 6 && team_enabled()) {
        if constexpr (B >= 6) launch_upper_team<B>(ctx, g, eb, false, a.mode == 0, true, needC);
    } else if (fused && (a.mode == 0 || g.nlev > 1)) {
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
    const int nq = a.out_pieces > 0 ? a.out_pieces : 1;
    for (int q = 0; q < nq; ++q) {
        const long long c0 = a.out_pieces > 0 ? a.out_chunk[q] : 0, c1 = a.out_pieces > 0 ? a.out_chunk[q + 1] : SK0;
        bool done = false;
        if constexpr (B >= 6) {
            if (c1 > c0 && team_enabled()) {
                launch_rev0_team<T>(ctx, md, eb, a, g, halo, outs, c0, c1);
                done = true;
            }
        }
        if (c1 > c0 && !done) {
            ctx->pre();
            k_rev0<T><<<blocks_for(c1 - c0, tpb), tpb, 0, ctx->stream>>>(md, eb.params, a.d_t, a.d_y, g, eb.fac[0],
                                                                         eb.sol[1], eb.part, outs, ctx->d_status,
                                                                         halo, c0, c1, a.d_obs);
            ctx->launched("k_rev0");
        }
        if (a.out_pieces > 0) CUDA_OK(cudaEventRecord(a.out_ready[q], ctx->stream));
    }
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
    fa.n = a.n_obs >= 0 ? a.n_obs : g.n[0];
    fa.loglik = a.d_loglik;
    fa.grad = grad ? a.d_grad : nullptr;
    fa.partials = a.mode == 3 ? a.d_seg_out : nullptr;
    ctx->pre();
    fa.S = g.S;
    k_reduce<<<static_cast<unsigned>(static_cast<long long>(eb.nseg) * g.S), kRedThreads, 0, ctx->stream>>>(fa);
    ctx->launched("k_reduce");
}

}  // namespace spingp_host
