// stream_solve.cu — host side of the tile-streaming cr_solve (stream_solve.cuh): one
// cooperative launch of G co-resident CTAs per solve.  Used by spingp_btd_cr_solve[_device]
// for b <= 4 with at most one right-hand side; everything else keeps the partitioned
// kernels of btd_ops.cuh.  SPINGP_SOLVE_STREAM=0 disables it (A/B knob).
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "ctx.hpp"
#include "stream_solve.cuh"
#include "strip_solve.cuh"

// b = 3 shape: warps per CTA (one CTA per SM), blocks per lane
#ifndef SP_SS3_NW
#define SP_SS3_NW 8
#endif
#ifndef SP_SS3_M
#define SP_SS3_M 5
#endif
#ifndef SP_SS3_LPT
#define SP_SS3_LPT 32
#endif
// strip kernel, b = 3: blocks per lane and sub-tile, warps per CTA
#ifndef SP_ST3_MB
#define SP_ST3_MB 4
#endif
#ifndef SP_ST3_NW
#define SP_ST3_NW 8
#endif

namespace spingp_host {

using namespace spingp_dev;

namespace {

// read on every call (cheap): tests and A/B runs toggle them inside one process
bool stream_enabled() {
    const char* e = std::getenv("SPINGP_SOLVE_STREAM");
    return !(e && std::strcmp(e, "0") == 0);
}
int stream_l2mode() {
    const char* e = std::getenv("SPINGP_SS_L2");
    return e ? std::atoi(e) : 0;
}

// diagnostics (SPINGP_SS_STAMPS=1): per-phase %globaltimer of every CTA, summarised on stderr
void ss_print_stamps(spingp_ctx* ctx, unsigned long long* d, int G) {
    std::vector<unsigned long long> h(static_cast<size_t>(G) * 16);
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    CUDA_OK(cudaMemcpy(h.data(), d, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    CUDA_OK(cudaFree(d));
    unsigned long long t0 = ~0ULL;
    for (int g = 0; g < G; ++g) t0 = std::min(t0, h[g * 16]);
    // 0-6: the phases common to both kernels; 7-15: one sub-tile / tile of each sweep (strip
    // kernel: half-tile 6 of sweep 1 before / after its wait, after its elimination, after the
    // next half; sub-tile 2 of sweep 2 before / after its wait, solved, stored.  tile kernel:
    // tile 2 of sweep 1 start / staged / eliminated / tree up; sweep 2 factors loaded / tree
    // down / staged / solved / stored)
    static const char* names[16] = {"start", "sweep 1 (warp 0)", "CTA record out", "top: all arrived", "top: released",
                                    "release seen", "end (warp 0)", "detail 7", "detail 8", "detail 9", "detail 10",
                                    "detail 11", "detail 12", "detail 13", "detail 14", "detail 15"};
    for (int k = 0; k < 16; ++k) {
        std::vector<double> v;
        for (int g = 0; g < G; ++g)
            if (h[g * 16 + k]) v.push_back((h[g * 16 + k] - t0) * 1e-3);
        if (v.empty()) continue;
        std::sort(v.begin(), v.end());
        std::fprintf(stderr, "[ss] %-18s min %8.2f  med %8.2f  max %8.2f us  (cta0 %8.2f)\n", names[k], v.front(),
                     v[v.size() / 2], v.back(), h[k] ? (h[k] - t0) * 1e-3 : -1.0);
    }
}

template <int B, int NWARP, int M, int LPT>
bool ss_launch(spingp_ctx* ctx, int64_t n, const double* diag, const double* upper, const double* rhs, double* x,
               double* logdet) {
    using C = SSCfg<B, NWARP, M, LPT>;
    constexpr int NR = C::NR, NK = C::NK, NF = C::NF, NW = C::NW;
    const long long ntiles = (n + C::WT - 1) / C::WT;
    if (ntiles < NW) return false;  // every warp of a CTA needs a tile
    auto kern = k_solve_stream<C, B>;
    static unsigned long long attr = 0;
    opt_in_smem(reinterpret_cast<const void*>(kern), attr, ctx->device, static_cast<int>(C::SMEM_BYTES));
    static int resident_dev[64] = {};
    int& resident = resident_dev[ctx->device & 63];
    if (!resident) {
        int per = 0, sms = 0;
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, C::NT, C::SMEM_BYTES));
        CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        resident = std::max(1, per) * sms;
    }
    long long G = std::min<long long>(resident, ntiles / NW);
    G = std::min<long long>(G, C::NT);  // the top system: one CTA record per thread of CTA 0
    if (const char* e = std::getenv("SPINGP_SS_CTAS")) G = std::max<long long>(1, std::min<long long>(G, std::atoll(e)));
    const long long GW = G * NW;
    const int Tmax = static_cast<int>((ntiles + GW - 1) / GW);
    ctx->ensure_ws(arena_bytes(NR * G) + arena_bytes(G * B) + arena_bytes(GW * Tmax * NK) +
                   arena_bytes(GW * Tmax * NF * LPT) + 4096);
    ctx->ws.reset();
    SSArgs a{};
    a.diag = diag;
    a.up = upper;
    a.rhs = rhs;
    a.x = x;
    a.logdet = logdet;
    a.n = n;
    a.ntiles = ntiles;
    a.G = static_cast<int>(G);
    a.Tmax = Tmax;
    auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    a.bulk = (rhs && aligned(diag) && aligned(upper) && aligned(rhs)) ? 1 : 0;
    a.l2mode = stream_l2mode();
    a.crec = ctx->ws.take<double>(NR * G);
    a.xsep = ctx->ws.take<double>(G * B);
    a.ckpt = ctx->ws.take<double>(GW * Tmax * NK);
    a.tfac = ctx->ws.take<double>(GW * Tmax * NF * LPT);
    if (!ctx->d_ss_sync) {
        CUDA_OK(cudaMalloc(&ctx->d_ss_sync, 2 * sizeof(unsigned long long)));
        CUDA_OK(cudaMemsetAsync(ctx->d_ss_sync, 0, 2 * sizeof(unsigned long long), ctx->stream));
        ctx->ss_arrivals = ctx->ss_releases = 0;
    }
    a.sync = ctx->d_ss_sync;
    a.arrive_target = ctx->ss_arrivals + static_cast<unsigned long long>(G);
    a.release_target = ctx->ss_releases + 1;
    a.status = ctx->d_status;
    const bool stamps = std::getenv("SPINGP_SS_STAMPS") != nullptr;
    a.stamps = nullptr;
    if (stamps) {
        CUDA_OK(cudaMalloc(&a.stamps, G * 16 * sizeof(unsigned long long)));
        CUDA_OK(cudaMemsetAsync(a.stamps, 0, G * 16 * sizeof(unsigned long long), ctx->stream));
    }
    void* args[] = {&a};
    ctx->pre();
    CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(static_cast<unsigned>(G)), dim3(C::NT),
                                        args, C::SMEM_BYTES, ctx->stream));
    ctx->launched("k_solve_stream");
    ctx->ss_arrivals = a.arrive_target;
    if (x) ctx->ss_releases = a.release_target;
    if (stamps) ss_print_stamps(ctx, a.stamps, static_cast<int>(G));
    return true;
}

// The strip kernel (strip_solve.cuh): one lane per long chunk, cooperative cp.async staging.
template <int B, int NWARP, int MB>
bool st_launch(spingp_ctx* ctx, int64_t n, const double* diag, const double* upper, const double* rhs, double* x,
               double* logdet) {
    using C = STCfg<B, NWARP, MB>;
    constexpr int NR = C::NR, NCK = C::NCK, NF = C::NF, NW = C::NW, NT = C::NT;
    if (n < static_cast<int64_t>(NT) * 2 * MB) return false;  // at least two sub-tiles per lane of one CTA
    auto kern = k_solve_strip<C, B>;
    static unsigned long long attr = 0;
    opt_in_smem(reinterpret_cast<const void*>(kern), attr, ctx->device, static_cast<int>(C::SMEM_BYTES));
    static int resident_dev[64] = {};
    int& resident = resident_dev[ctx->device & 63];
    if (!resident) {
        int per = 0, sms = 0;
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, NT, C::SMEM_BYTES));
        CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        resident = std::max(1, per) * sms;
    }
    long long G = std::min<long long>(resident, n / (static_cast<long long>(NT) * 2 * MB));
    G = std::min<long long>(G, NT);  // the top system: one CTA record per thread of CTA 0
    if (const char* e = std::getenv("SPINGP_SS_CTAS")) G = std::max<long long>(1, std::min<long long>(G, std::atoll(e)));
    const long long GL = G * NT, GW = G * NW;
    const int nsub = static_cast<int>((n + MB * GL - 1) / (MB * GL));  // sub-tiles per lane, all full
    const long long Lc = static_cast<long long>(nsub) * MB;
    ctx->ensure_ws(arena_bytes(NR * G) + arena_bytes(G * B) + arena_bytes(GW * nsub * NCK * 32) +
                   arena_bytes(GW * NF * 32) + 4096);
    ctx->ws.reset();
    SSArgs a{};
    a.diag = diag;
    a.up = upper;
    a.rhs = rhs;
    a.x = x;
    a.logdet = logdet;
    a.n = n;
    a.G = static_cast<int>(G);
    a.Lc = Lc;
    a.nsub = nsub;
    auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    a.bulk = (rhs && aligned(diag) && aligned(upper) && aligned(rhs)) ? 1 : 0;
    a.l2mode = stream_l2mode();
    if (const char* e = std::getenv("SPINGP_SS_L2KEEP")) a.l2keep = std::atoi(e);
    else a.l2keep = 3;
    a.crec = ctx->ws.take<double>(NR * G);
    a.xsep = ctx->ws.take<double>(G * B);
    a.ckpt = ctx->ws.take<double>(GW * nsub * NCK * 32);
    a.tfac = ctx->ws.take<double>(GW * NF * 32);
    if (!ctx->d_ss_sync) {
        CUDA_OK(cudaMalloc(&ctx->d_ss_sync, 2 * sizeof(unsigned long long)));
        CUDA_OK(cudaMemsetAsync(ctx->d_ss_sync, 0, 2 * sizeof(unsigned long long), ctx->stream));
        ctx->ss_arrivals = ctx->ss_releases = 0;
    }
    a.sync = ctx->d_ss_sync;
    a.arrive_target = ctx->ss_arrivals + static_cast<unsigned long long>(G);
    a.release_target = ctx->ss_releases + 1;
    a.status = ctx->d_status;
    const bool stamps = std::getenv("SPINGP_SS_STAMPS") != nullptr;
    a.stamps = nullptr;
    if (stamps) {
        CUDA_OK(cudaMalloc(&a.stamps, G * 16 * sizeof(unsigned long long)));
        CUDA_OK(cudaMemsetAsync(a.stamps, 0, G * 16 * sizeof(unsigned long long), ctx->stream));
    }
    void* args[] = {&a};
    ctx->pre();
    CUDA_OK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(static_cast<unsigned>(G)), dim3(NT), args,
                                        C::SMEM_BYTES, ctx->stream));
    ctx->launched("k_solve_strip");
    ctx->ss_arrivals = a.arrive_target;
    if (x) ctx->ss_releases = a.release_target;
    if (stamps) ss_print_stamps(ctx, a.stamps, static_cast<int>(G));
    return true;
}

bool strip_enabled() {
    const char* e = std::getenv("SPINGP_SOLVE_STRIP");
    return !(e && std::strcmp(e, "0") == 0);
}

}  // namespace

// x = M^{-1} rhs (one right-hand side, or none: log det only) by the tile-streaming kernel;
// false when the case is not covered (b > 4, too few blocks, disabled).
bool stream_solve(spingp_ctx* ctx, int64_t n, int b, const double* diag, const double* upper, const double* rhs,
                  double* x, double* logdet) {
    if (!stream_enabled() || n < 2 || !upper) return false;
    {  // both kernels are cooperative launches (a grid-wide barrier between the sweeps)
        static int coop_dev[64] = {};
        int& coop = coop_dev[ctx->device & 63];
        if (!coop) {
            int v = 0;
            CUDA_OK(cudaDeviceGetAttribute(&v, cudaDevAttrCooperativeLaunch, ctx->device));
            coop = v ? 1 : -1;
        }
        if (coop < 0) return false;
    }
    if (strip_enabled()) {  // one lane per long chunk (strip_solve.cuh); else contiguous tiles
        bool done = false;
        switch (b) {
            case 1: done = st_launch<1, 8, 8>(ctx, n, diag, upper, rhs, x, logdet); break;
            case 2: done = st_launch<2, 8, 4>(ctx, n, diag, upper, rhs, x, logdet); break;
            case 3: done = st_launch<3, SP_ST3_NW, SP_ST3_MB>(ctx, n, diag, upper, rhs, x, logdet); break;
            case 4: done = st_launch<4, 4, 4>(ctx, n, diag, upper, rhs, x, logdet); break;
            default: break;
        }
        if (done) return true;
    }
    switch (b) {
        case 1: return ss_launch<1, 8, 7, 32>(ctx, n, diag, upper, rhs, x, logdet);
        case 2: return ss_launch<2, 8, 5, 32>(ctx, n, diag, upper, rhs, x, logdet);
        case 3: return ss_launch<3, SP_SS3_NW, SP_SS3_M, SP_SS3_LPT>(ctx, n, diag, upper, rhs, x, logdet);
        case 4: return ss_launch<4, 8, 3, 32>(ctx, n, diag, upper, rhs, x, logdet);
        default: return false;
    }
}

}  // namespace spingp_host
