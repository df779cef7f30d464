// capi.cu — the C ABI of include/spingp_c.h: context lifetime, planning,
// host<->device staging and dispatch to the kernel instantiations
// (inst_*.cu, btd_*.cu).  Every per-point computation runs in the sm_100a
// kernels of engine.cuh; there is no CPU fallback — without a CUDA device the
// computing entry points return SPINGP_CUDA_ERR.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ctx.hpp"

using namespace spingp_dev;
using namespace spingp_host;

namespace spingp_host {

std::string& last_error() {
    thread_local std::string s;
    return s;
}


int take_status(spingp_ctx* ctx, int64_t* fail_block) {
    // status word -> pinned host slot and reset, both stream-ordered; one synchronisation
    if (!ctx->h_status) CUDA_OK(cudaMallocHost(&ctx->h_status, sizeof(unsigned long long)));
    CUDA_OK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            ctx->stream));
    CUDA_OK(cudaMemsetAsync(ctx->d_status, 0xFF, sizeof(unsigned long long), ctx->stream));
    CUDA_OK(cudaStreamSynchronize(ctx->stream));
    const unsigned long long h = *ctx->h_status;
    if (h == ~0ULL) return SPINGP_OK;
    if (fail_block) *fail_block = static_cast<int64_t>((h >> 4) & ((1ULL << 56) - 1));
    const int code = static_cast<int>(h & 15ULL);
    static const char* what[] = {"", "pivot block is not positive definite",
                                 "process noise block singular after jitter", "invalid input value",
                                 "", "", "duplicate training timestamp", "", "negative posterior variance"};
    last_error() = what[code < 9 ? code : 0];
    return code;
}

void upload(spingp_ctx* ctx, double* dst, const double* src, size_t count) {
    double* st = ctx->stage(count);
    std::memcpy(st, src, count * sizeof(double));
    CUDA_OK(cudaMemcpyAsync(dst, st, count * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ctx->stage_done();
}

}  // namespace spingp_host

namespace {

void dispatch_eval(spingp_ctx* ctx, const EvalArgs& a) {
    const HostModel& hm = *a.hm;
    if (hm.single_matern) {
        switch (hm.b) {
            case 1: return eval_matern_1(ctx, a);
            case 2: return eval_matern_2(ctx, a);
            case 3: return eval_matern_3(ctx, a);
        }
    }
    switch (static_model(hm)) {
        case SM_EQ6: return eval_s_eq6(ctx, a);
        case SM_EQ10: return eval_s_eq10(ctx, a);
        case SM_M32_QP6: return eval_s_m32qp6(ctx, a);
        case SM_M32_EQ10: return eval_s_m32eq10(ctx, a);
        default: break;
    }
    switch (pad_b(hm.b)) {
        case 1: case 2: case 3: return eval_generic_3(ctx, a);
        case 4: return eval_generic_4(ctx, a);
        case 6: return eval_generic_6(ctx, a);
        case 8: return eval_generic_8(ctx, a);
        case 12: return eval_generic_12(ctx, a);
        case 16: return eval_generic_16(ctx, a);
    }
    throw ApiError{SPINGP_UNSUPPORTED, -1, "no kernel instantiation for this state dimension"};
}

int plan_bsize(const HostModel& hm) {
    return (hm.single_matern || static_model(hm) != SM_NONE) ? hm.b : std::max(3, pad_b(hm.b));
}

void btd_dispatch(spingp_ctx* ctx, int64_t n, int b, const double* diag, const double* upper,
                  const double* rhs, int k, int col, double* x, double* cdiag, double* cupper,
                  double* logdet, bool needC) {
    if (n < 1 || b < 1) throw std::invalid_argument("empty block-tridiagonal matrix");
#define R(B) btd_run_##B(ctx, n, b, diag, upper, rhs, k, col, x, cdiag, cupper, logdet, needC)
    switch (pad_b(b)) {
        case 1: R(1); break;
        case 2: R(2); break;
        case 3: R(3); break;
        case 4: R(4); break;
        case 6: R(6); break;
        case 8: R(8); break;
        case 12: R(12); break;
        case 16: R(16); break;
    }
#undef R
}

spingp_ctx* checked(spingp_ctx* ctx) {
    if (!ctx) throw std::invalid_argument("null context");
    CUDA_OK(cudaSetDevice(ctx->device));
    return ctx;
}

}  // namespace

// ---- multi-GPU partition of one long series (segment mode) -------

int spingp_seg_sizes(const spingp_leaf* leaves, int32_t n_leaves, int32_t* n_record, int32_t* n_partials) {
    return guarded(nullptr, [&] {
        int32_t b = 0, nt = 0;
        const int st = spingp_kernel_dims(leaves, n_leaves, &b, &nt);
        if (st != SPINGP_OK) return st;
        const HostModel hm = build_model(leaves, n_leaves, nt);
        const int B = plan_bsize(hm);
        if (n_record) *n_record = 3 * B * B + 2 * B + 1;  // Rec<B>::N
        if (n_partials) *n_partials = 5 + nt;             // P_GRAD + nt
        return static_cast<int>(SPINGP_OK);
    });
}

// build_model for a ctx, reusing the last result while the structure repeats (call with
// ctx->mu held)
static const HostModel& ctx_model(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves, int32_t n_theta) {
    std::vector<int32_t> key{n_leaves, n_theta};
    for (int32_t l = 0; l < n_leaves && leaves; ++l) {
        key.push_back(static_cast<int32_t>(leaves[l].type));
        key.push_back(leaves[l].order);
    }
    if (key != ctx->model_key || ctx->model_key.empty()) {
        ctx->model = build_model(leaves, n_leaves, n_theta);
        ctx->model_key = std::move(key);
    }
    return ctx->model;
}

// SPINGP_PIPELINE=0 disables host-input pipelining (A/B knob)
static bool pipeline_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SPINGP_PIPELINE");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    return on;
}

static int seg_run(spingp_ctx* ctx, int mode, const spingp_leaf* leaves, int32_t n_leaves, const double* theta,
                   int32_t n_theta, const double* d_t, const double* d_y, int64_t n_local, double t_left,
                   double t_right, int32_t rank, int32_t nranks, double sigma, uint32_t flags,
                   const double* d_in, double* d_out, double* d_mean, double* d_var) {
    return guarded(nullptr, [&] {
        checked(ctx);
        if (!theta || !d_t || !d_y || !d_out || (mode == 3 && !d_in)) throw std::invalid_argument("null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks || nranks > 64) throw std::invalid_argument("bad rank / nranks");
        if (rank > 0 && !(t_left < 0.0 || t_left >= 0.0)) throw std::invalid_argument("missing left halo time");
        if (rank + 1 < nranks && !(t_right < 0.0 || t_right >= 0.0)) throw std::invalid_argument("missing right halo time");
        std::lock_guard<std::mutex> lk(ctx->mu);
        const HostModel& hm = ctx_model(ctx, leaves, n_leaves, n_theta);
        Plan plan = make_plan(n_local, 1, plan_bsize(hm), ctx->m0_override, -1, ctx->g_override);
        plan.geo.segL = rank > 0 ? 1 : 0;
        plan.geo.segR = rank + 1 < nranks ? 1 : 0;
        std::vector<double> params(hm.rec_stride + 2, 0.0);
        fill_record(hm, theta, sigma, params.data());
        params[hm.rec_stride] = t_left;
        params[hm.rec_stride + 1] = t_right;
        EvalArgs a{&hm, &plan, params.data(), params.size(), d_t, d_y, flags, nullptr, nullptr,
                   (flags & SPINGP_WANT_MEAN) ? d_mean : nullptr, (flags & SPINGP_WANT_VAR) ? d_var : nullptr,
                   mode, nullptr, nullptr, nullptr, rank, nranks, d_in, d_out};
        dispatch_eval(ctx, a);
        return SPINGP_OK;
    });
}

extern "C" {

int spingp_abi_version(void) { return SPINGP_ABI_VERSION; }

const char* spingp_status_string(int status) {
    switch (status) {
        case SPINGP_OK: return "ok";
        case SPINGP_NOT_PD: return "not positive definite";
        case SPINGP_SINGULAR_Q: return "singular process noise";
        case SPINGP_BAD_ARG: return "bad argument";
        case SPINGP_CUDA_ERR: return "cuda error";
        case SPINGP_NCCL_ERR: return "nccl error";
        case SPINGP_DUPLICATE_TIME: return "duplicate timestamp";
        case SPINGP_UNSUPPORTED: return "unsupported";
        case SPINGP_NEG_VARIANCE: return "negative variance";
    }
    return "unknown status";
}

const char* spingp_last_error(void) { return last_error().c_str(); }

int spingp_ctx_create(int32_t device, spingp_ctx** out) {
    return guarded(nullptr, [&] {
        if (!out) throw std::invalid_argument("null output");
        *out = nullptr;
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
            throw ApiError{SPINGP_CUDA_ERR, -1, "no CUDA device available (this build has no CPU fallback)"};
        if (device < 0 || device >= count) throw std::invalid_argument("device index out of range");
        CUDA_OK(cudaSetDevice(device));
        auto* c = new spingp_ctx();
        c->device = device;
        CUDA_OK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
        CUDA_OK(cudaMalloc(&c->d_status, sizeof(unsigned long long)));
        CUDA_OK(cudaMemset(c->d_status, 0xFF, sizeof(unsigned long long)));
        CUDA_OK(cudaEventCreateWithFlags(&c->stage_ev[0], cudaEventDisableTiming));
        CUDA_OK(cudaEventCreateWithFlags(&c->stage_ev[1], cudaEventDisableTiming));
        set_plan_wave(rev0_wave_threads_m3());
        *out = c;
        return SPINGP_OK;
    });
}

int spingp_ctx_destroy(spingp_ctx* ctx) {
    if (!ctx) return SPINGP_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->ws.base) cudaFree(ctx->ws.base);
    ctx->host_io.release();
    if (ctx->d_status) cudaFree(ctx->d_status);
    if (ctx->d_arrive) cudaFree(ctx->d_arrive);
    if (ctx->d_ss_sync) cudaFree(ctx->d_ss_sync);
    for (int k = 0; k < 2; ++k) {
        if (ctx->h_stage[k]) cudaFreeHost(ctx->h_stage[k]);
        if (ctx->stage_ev[k]) cudaEventDestroy(ctx->stage_ev[k]);
    }
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->h_status) cudaFreeHost(ctx->h_status);
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        for (cudaEvent_t e : ctx->pipe_ev) cudaEventDestroy(e);
        cudaStreamDestroy(ctx->copy_stream);
    }
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return SPINGP_OK;
}

int spingp_ctx_set_stream(spingp_ctx* ctx, void* stream) {
    return guarded(nullptr, [&] {
        checked(ctx);
        std::lock_guard<std::mutex> lk(ctx->mu);
        CUDA_OK(cudaStreamSynchronize(ctx->stream));
        if (ctx->own_stream) CUDA_OK(cudaStreamDestroy(ctx->stream));
        ctx->stream = static_cast<cudaStream_t>(stream);  // NULL = legacy default stream
        ctx->own_stream = false;
        return SPINGP_OK;
    });
}

int spingp_ctx_use_own_stream(spingp_ctx* ctx) {
    return guarded(nullptr, [&] {
        checked(ctx);
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (ctx->own_stream) return static_cast<int>(SPINGP_OK);
        CUDA_OK(cudaStreamSynchronize(ctx->stream));
        CUDA_OK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
        return static_cast<int>(SPINGP_OK);
    });
}

void* spingp_ctx_get_stream(spingp_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int spingp_ctx_set_chunk(spingp_ctx* ctx, int64_t m0) {
    if (!ctx || m0 < 0) return SPINGP_BAD_ARG;
    ctx->m0_override = m0;
    return SPINGP_OK;
}

int spingp_ctx_set_tree_group(spingp_ctx* ctx, int64_t g) {
    if (!ctx || g < 0 || g == 1) return SPINGP_BAD_ARG;
    ctx->g_override = g;
    return SPINGP_OK;
}

int spingp_ctx_status(spingp_ctx* ctx, int64_t* fail_block) {
    return guarded(fail_block, [&] {
        checked(ctx);
        std::lock_guard<std::mutex> lk(ctx->mu);
        return take_status(ctx, fail_block);
    });
}

int64_t spingp_ctx_launch_count(spingp_ctx* ctx) { return ctx ? ctx->launches : 0; }

int spingp_ctx_set_phase_stamps(spingp_ctx* ctx, void* d_stamps) {
    return guarded(nullptr, [&] {
        checked(ctx);
        std::lock_guard<std::mutex> lk(ctx->mu);
        ctx->upper_stamps = static_cast<unsigned long long*>(d_stamps);
        return static_cast<int>(SPINGP_OK);
    });
}

int spingp_ctx_set_profiling(spingp_ctx* ctx, int on) {
    if (!ctx) return SPINGP_BAD_ARG;
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->profiling = on != 0;
    ctx->timed.clear();
    ctx->ev_used = 0;
    return SPINGP_OK;
}

int spingp_ctx_kernel_times(spingp_ctx* ctx, const char** names, double* ms, int32_t cap,
                            int32_t* count) {
    return guarded(nullptr, [&] {
        checked(ctx);
        std::lock_guard<std::mutex> lk(ctx->mu);
        CUDA_OK(cudaStreamSynchronize(ctx->stream));
        const int n = static_cast<int>(ctx->timed.size());
        if (count) *count = n;
        for (int i = 0; i < n && i < cap; ++i) {
            float t = 0.f;
            CUDA_OK(cudaEventElapsedTime(&t, ctx->timed[i].a, ctx->timed[i].b));
            if (names) names[i] = ctx->timed[i].name;
            if (ms) ms[i] = t;
        }
        ctx->timed.clear();
        ctx->ev_used = 0;
        return SPINGP_OK;
    });
}

static void eval_batched_locked(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves, const double* theta,
                                int32_t n_theta, int64_t S, int64_t n, const double* d_t, const double* d_y,
                                const double* sigma, uint32_t flags, double* d_loglik, double* d_grad,
                                double* d_mean, double* d_var) {
    // caller holds ctx->mu
    if (!theta || !sigma || !d_t || !d_y || !d_loglik) throw std::invalid_argument("null argument");
    if (S < 1 || n < 1) throw std::invalid_argument("need at least one point and one series");
    if ((flags & SPINGP_WANT_GRAD) && !d_grad) throw std::invalid_argument("gradient output is null");
    if ((flags & SPINGP_WANT_MEAN) && !d_mean) throw std::invalid_argument("mean output is null");
    if ((flags & SPINGP_WANT_VAR) && !d_var) throw std::invalid_argument("variance output is null");
    const HostModel& hm = ctx_model(ctx, leaves, n_leaves, n_theta);
    const Plan plan = make_plan(n, S, plan_bsize(hm), ctx->m0_override, -1, ctx->g_override);
    std::vector<double> params(static_cast<size_t>(S) * hm.rec_stride, 0.0);
    for (int64_t s = 0; s < S; ++s)
        fill_record(hm, theta + s * n_theta, sigma[s], params.data() + s * hm.rec_stride);
    EvalArgs a{&hm, &plan, params.data(), params.size(), d_t, d_y, flags, d_loglik, d_grad, d_mean, d_var,
               0, nullptr, nullptr, nullptr};
    dispatch_eval(ctx, a);
}

int spingp_eval_batched_device(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                               const double* theta, int32_t n_theta, int64_t S, int64_t n,
                               const double* d_t, const double* d_y, const double* sigma,
                               uint32_t flags, double* d_loglik, double* d_grad, double* d_mean,
                               double* d_var) {
    return guarded(nullptr, [&] {
        checked(ctx);
        std::lock_guard<std::mutex> lk(ctx->mu);
        eval_batched_locked(ctx, leaves, n_leaves, theta, n_theta, S, n, d_t, d_y, sigma, flags, d_loglik, d_grad,
                            d_mean, d_var);
        return SPINGP_OK;
    });
}

int spingp_eval_device(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                       const double* theta, int32_t n_theta, const double* d_t, const double* d_y,
                       int64_t n, double sigma, uint32_t flags, double* d_loglik, double* d_grad,
                       double* d_mean, double* d_var) {
    return spingp_eval_batched_device(ctx, leaves, n_leaves, theta, n_theta, 1, n, d_t, d_y, &sigma,
                                      flags, d_loglik, d_grad, d_mean, d_var);
}

// Host-input pipelining for one long series (S = 1, n >= kPipeMin): the H2D of t, y runs
// on a copy stream in kPipeIn pieces of level-0 chunks and k_fwd0 starts on each piece as
// soon as it has landed; k_rev0 runs in kPipeOut pieces and each piece's mean/var is copied
// back while the next piece computes.  Results are identical to the unpipelined call (the
// kernels and their per-chunk arithmetic do not change; only launch boundaries do).
constexpr int64_t kPipeMin = 1 << 18;
constexpr int kPipeMax = 16;
// pieces of the input / output pipeline (SPINGP_PIPE_IN / SPINGP_PIPE_OUT override, <= kPipeMax)
static int pipe_pieces(const char* env, int dflt) {
    const char* e = std::getenv(env);
    const int v = e ? std::atoi(e) : dflt;
    return std::max(1, std::min(kPipeMax, v));
}

static int eval_host_pipelined(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves, const double* theta,
                               int32_t n_theta, int64_t n, const double* t, const double* y, double sigma,
                               uint32_t flags, double* out_loglik, double* out_grad, double* out_mean,
                               double* out_var, int64_t* fail_block) {
    // caller holds ctx->mu
    const size_t nt1 = static_cast<size_t>(n_theta) + 1;
    const size_t ng = (flags & SPINGP_WANT_GRAD) ? nt1 : 0;
    const size_t nm = (flags & SPINGP_WANT_MEAN) ? n : 0;
    const size_t nv = (flags & SPINGP_WANT_VAR) ? n : 0;
    double* base = ctx->host_io.get(2 * static_cast<size_t>(n) + 1 + ng + nm + nv);
    double* d_t = base;
    double* d_y = d_t + n;
    double* d_ll = d_y + n;
    double* d_g = d_ll + 1;
    double* d_m = d_g + ng;
    double* d_v = d_m + nm;
    {
        const HostModel& hm = ctx_model(ctx, leaves, n_leaves, n_theta);
        const Plan plan = make_plan(n, 1, plan_bsize(hm), ctx->m0_override, -1, ctx->g_override);
        std::vector<double> params(hm.rec_stride, 0.0);
        fill_record(hm, theta, sigma, params.data());
        const long long K0 = plan.geo.K[0], m0 = plan.geo.m[0];
        static const int kPipeIn = pipe_pieces("SPINGP_PIPE_IN", 4), kPipeOut = pipe_pieces("SPINGP_PIPE_OUT", 2);
        long long ic[kPipeMax + 1], oc[kPipeMax + 1];
        for (int p = 0; p <= kPipeIn; ++p) ic[p] = K0 * p / kPipeIn;
        for (int q = 0; q <= kPipeOut; ++q) oc[q] = K0 * q / kPipeOut;
        if (!ctx->copy_stream) {
            CUDA_OK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
            for (auto& e : ctx->pipe_ev) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        cudaEvent_t* in_ev = ctx->pipe_ev;
        cudaEvent_t* out_ev = ctx->pipe_ev + kPipeIn;
        cudaEvent_t ev_start = ctx->pipe_ev[kPipeIn + kPipeOut], ev_done = ctx->pipe_ev[kPipeIn + kPipeOut + 1];
        cudaStream_t cs = ctx->copy_stream;
        CUDA_OK(cudaEventRecord(ev_start, ctx->stream));  // earlier work on d_t, d_y is done first
        CUDA_OK(cudaStreamWaitEvent(cs, ev_start, 0));
        for (int p = 0; p < kPipeIn; ++p) {
            // piece p: the points of its chunks plus the next time (the last separator's step)
            const long long lo = ic[p] * m0, hi = std::min<long long>(n, ic[p + 1] * m0 + 1);
            if (hi > lo) {
                CUDA_OK(cudaMemcpyAsync(d_t + lo, t + lo, (hi - lo) * sizeof(double), cudaMemcpyHostToDevice, cs));
                CUDA_OK(cudaMemcpyAsync(d_y + lo, y + lo, (hi - lo) * sizeof(double), cudaMemcpyHostToDevice, cs));
            }
            CUDA_OK(cudaEventRecord(in_ev[p], cs));
        }
        EvalArgs a{&hm, &plan, params.data(), params.size(), d_t, d_y, flags, d_ll, d_g, d_m, d_v,
                   0, nullptr, nullptr, nullptr};
        a.in_pieces = kPipeIn;
        a.in_chunk = ic;
        a.in_ready = in_ev;
        if (nm || nv) {
            a.out_pieces = kPipeOut;
            a.out_chunk = oc;
            a.out_ready = out_ev;
        }
        dispatch_eval(ctx, a);
        if (nm || nv) {
            for (int q = 0; q < kPipeOut; ++q) {
                const long long lo = oc[q] * m0, hi = std::min<long long>(n, oc[q + 1] * m0);
                CUDA_OK(cudaStreamWaitEvent(cs, out_ev[q], 0));
                if (hi <= lo) continue;
                if (nm)
                    CUDA_OK(cudaMemcpyAsync(out_mean + lo, d_m + lo, (hi - lo) * sizeof(double),
                                            cudaMemcpyDeviceToHost, cs));
                if (nv)
                    CUDA_OK(cudaMemcpyAsync(out_var + lo, d_v + lo, (hi - lo) * sizeof(double),
                                            cudaMemcpyDeviceToHost, cs));
            }
        }
        CUDA_OK(cudaEventRecord(ev_done, cs));
        CUDA_OK(cudaMemcpyAsync(out_loglik, d_ll, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (ng) CUDA_OK(cudaMemcpyAsync(out_grad, d_g, ng * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_OK(cudaStreamWaitEvent(ctx->stream, ev_done, 0));
        return take_status(ctx, fail_block);
    }
}

int spingp_eval_batched(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                        const double* theta, int32_t n_theta, int64_t S, int64_t n, const double* t,
                        const double* y, const double* sigma, uint32_t flags, double* out_loglik,
                        double* out_grad, double* out_mean, double* out_var, int64_t* fail_block) {
    return guarded(fail_block, [&] {
        checked(ctx);
        if (!theta || !sigma || !t || !y || !out_loglik || S < 1 || n < 1) throw std::invalid_argument("bad argument");
        if ((flags & SPINGP_WANT_GRAD) && !out_grad) throw std::invalid_argument("gradient output is null");
        if ((flags & SPINGP_WANT_MEAN) && !out_mean) throw std::invalid_argument("mean output is null");
        if ((flags & SPINGP_WANT_VAR) && !out_var) throw std::invalid_argument("variance output is null");
        // one lock from upload to status: the scratch buffers and the status word are the ctx's
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (S == 1 && n >= kPipeMin && pipeline_enabled())
            return eval_host_pipelined(ctx, leaves, n_leaves, theta, n_theta, n, t, y, sigma[0], flags, out_loglik,
                                       out_grad, out_mean, out_var, fail_block);
        const size_t N = static_cast<size_t>(S) * n;
        const size_t nt1 = static_cast<size_t>(n_theta) + 1;
        const size_t ng = (flags & SPINGP_WANT_GRAD) ? S * nt1 : 0;
        const size_t nm = (flags & SPINGP_WANT_MEAN) ? N : 0;
        const size_t nv = (flags & SPINGP_WANT_VAR) ? N : 0;
        double* base = ctx->host_io.get(2 * N + S + ng + nm + nv);
        double* d_t = base;
        double* d_y = d_t + N;
        double* d_ll = d_y + N;
        double* d_g = d_ll + S;
        double* d_m = d_g + ng;
        double* d_v = d_m + nm;
        CUDA_OK(cudaMemcpyAsync(d_t, t, N * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CUDA_OK(cudaMemcpyAsync(d_y, y, N * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        eval_batched_locked(ctx, leaves, n_leaves, theta, n_theta, S, n, d_t, d_y, sigma, flags, d_ll,
                            ng ? d_g : nullptr, nm ? d_m : nullptr, nv ? d_v : nullptr);
        CUDA_OK(cudaMemcpyAsync(out_loglik, d_ll, S * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (ng) CUDA_OK(cudaMemcpyAsync(out_grad, d_g, ng * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (nm) CUDA_OK(cudaMemcpyAsync(out_mean, d_m, nm * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (nv) CUDA_OK(cudaMemcpyAsync(out_var, d_v, nv * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        return take_status(ctx, fail_block);
    });
}

// K hyperparameter vectors on ONE series (line-search probes of the optimizer):
// t, y go up once and are replicated on the device, then one batched evaluation.
int spingp_eval_multi_theta(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves, const double* theta,
                            int32_t n_theta, int64_t K, const double* t, const double* y, int64_t n,
                            const double* sigma, uint32_t flags, double* out_loglik, double* out_grad,
                            int64_t* fail_series) {
    return guarded(fail_series, [&] {
        checked(ctx);
        if (!theta || !sigma || !t || !y || !out_loglik || K < 1 || n < 1) throw std::invalid_argument("bad argument");
        if ((flags & SPINGP_WANT_GRAD) && !out_grad) throw std::invalid_argument("gradient output is null");
        flags &= SPINGP_WANT_GRAD;  // per-point outputs are not returned here
        std::lock_guard<std::mutex> lk(ctx->mu);
        const size_t N = static_cast<size_t>(K) * n;
        const size_t ng = (flags & SPINGP_WANT_GRAD) ? K * (static_cast<size_t>(n_theta) + 1) : 0;
        double* d_t = ctx->host_io.get(2 * N + K + ng);
        double* d_y = d_t + N;
        double* d_ll = d_y + N;
        double* d_g = d_ll + K;
        CUDA_OK(cudaMemcpyAsync(d_t, t, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CUDA_OK(cudaMemcpyAsync(d_y, y, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        for (int64_t k = 1; k < K; ++k) {
            CUDA_OK(cudaMemcpyAsync(d_t + k * n, d_t, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
            CUDA_OK(cudaMemcpyAsync(d_y + k * n, d_y, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        }
        eval_batched_locked(ctx, leaves, n_leaves, theta, n_theta, K, n, d_t, d_y, sigma, flags, d_ll,
                            ng ? d_g : nullptr, nullptr, nullptr);
        CUDA_OK(cudaMemcpyAsync(out_loglik, d_ll, K * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (ng) CUDA_OK(cudaMemcpyAsync(out_grad, d_g, ng * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        int64_t fb = -1;
        const int st = take_status(ctx, &fb);
        if (fail_series) *fail_series = fb >= 0 ? fb / n : -1;  // the (first) failing probe
        return st;
    });
}

int spingp_predict(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves, const double* theta,
                   int32_t n_theta, const double* t, const double* y, int64_t n, const double* test_t, int64_t m,
                   double sigma, uint32_t flags, double* out_loglik, double* out_grad, double* out_mean,
                   double* out_var, int64_t* fail_block) {
    return guarded(fail_block, [&] {
        checked(ctx);
        if (!out_loglik || (m > 0 && (!out_mean || !out_var))) throw std::invalid_argument("null argument");
        if ((flags & SPINGP_WANT_GRAD) && !out_grad) throw std::invalid_argument("gradient output is null");
        const PredictGrid pg = predict_grid(t, y, n, test_t, m);
        const int64_t L = n + m;
        std::lock_guard<std::mutex> lk(ctx->mu);
        const size_t nt1 = static_cast<size_t>(n_theta) + 1;
        // t, y, mean, var (L each), loglik, grad, then the mask bytes
        double* base = ctx->host_io.get(4 * static_cast<size_t>(L) + 1 + nt1 + (static_cast<size_t>(L) + 7) / 8);
        double* d_t = base;
        double* d_y = d_t + L;
        double* d_m = d_y + L;
        double* d_v = d_m + L;
        double* d_ll = d_v + L;
        double* d_g = d_ll + 1;
        unsigned char* d_obs = reinterpret_cast<unsigned char*>(d_g + nt1);
        const HostModel& hm = ctx_model(ctx, leaves, n_leaves, n_theta);
        const Plan plan = make_plan(L, 1, plan_bsize(hm), ctx->m0_override, -1, ctx->g_override);
        std::vector<double> params(hm.rec_stride, 0.0);
        fill_record(hm, theta, sigma, params.data());
        CUDA_OK(cudaMemcpyAsync(d_t, pg.t.data(), L * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CUDA_OK(cudaMemcpyAsync(d_y, pg.y.data(), L * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CUDA_OK(cudaMemcpyAsync(d_obs, pg.obs.data(), L, cudaMemcpyHostToDevice, ctx->stream));
        const uint32_t f = (flags & (SPINGP_WANT_GRAD | SPINGP_INCLUDE_NOISE)) | SPINGP_WANT_MEAN | SPINGP_WANT_VAR;
        EvalArgs a{&hm, &plan, params.data(), params.size(), d_t, d_y, f, d_ll, d_g, d_m, d_v, 0, nullptr, nullptr,
                   nullptr};
        a.d_obs = d_obs;
        a.n_obs = n;
        dispatch_eval(ctx, a);
        std::vector<double> mean(static_cast<size_t>(L)), var(static_cast<size_t>(L));
        CUDA_OK(cudaMemcpyAsync(mean.data(), d_m, L * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_OK(cudaMemcpyAsync(var.data(), d_v, L * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_OK(cudaMemcpyAsync(out_loglik, d_ll, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (flags & SPINGP_WANT_GRAD)
            CUDA_OK(cudaMemcpyAsync(out_grad, d_g, nt1 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        const int st = take_status(ctx, fail_block);
        for (int64_t k = 0; k < m; ++k) {
            out_mean[k] = mean[static_cast<size_t>(pg.test_pos[static_cast<size_t>(k)])];
            out_var[k] = var[static_cast<size_t>(pg.test_pos[static_cast<size_t>(k)])];
        }
        return st;
    });
}

int spingp_eval(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves, const double* theta,
                int32_t n_theta, const double* t, const double* y, int64_t n, double sigma,
                uint32_t flags, double* out_loglik, double* out_grad, double* out_mean,
                double* out_var, int64_t* fail_block) {
    return spingp_eval_batched(ctx, leaves, n_leaves, theta, n_theta, 1, n, t, y, &sigma, flags, out_loglik,
                               out_grad, out_mean, out_var, fail_block);
}

int spingp_assemble(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                    const double* theta, int32_t n_theta, const double* t, const double* y,
                    int64_t n, double sigma, double* diag, double* upper, double* rhs,
                    int64_t* fail_block) {
    return guarded(fail_block, [&] {
        checked(ctx);
        if (!t || !y || !diag || n < 1) throw std::invalid_argument("bad argument");
        std::lock_guard<std::mutex> lk(ctx->mu);
        const HostModel& hm = ctx_model(ctx, leaves, n_leaves, n_theta);
        const int b = hm.b;
        const size_t nd = static_cast<size_t>(n) * b * b, nu = static_cast<size_t>(n > 1 ? n - 1 : 0) * b * b;
        double* d_t = ctx->host_io.get(2 * n + nd + nu + n * b);
        double* d_y = d_t + n;
        double* d_d = d_y + n;
        double* d_u = d_d + nd;
        double* d_r = d_u + nu;
        CUDA_OK(cudaMemcpyAsync(d_t, t, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CUDA_OK(cudaMemcpyAsync(d_y, y, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        const Plan plan = make_plan(n, 1, plan_bsize(hm), 0);
        std::vector<double> params(hm.rec_stride, 0.0);
        fill_record(hm, theta, sigma, params.data());
        EvalArgs a{&hm, &plan, params.data(), params.size(), d_t, d_y, 0, nullptr, nullptr, nullptr, nullptr,
                   1, d_d, d_u, d_r};
        dispatch_eval(ctx, a);
        CUDA_OK(cudaMemcpyAsync(diag, d_d, nd * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (upper && nu) CUDA_OK(cudaMemcpyAsync(upper, d_u, nu * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (rhs) CUDA_OK(cudaMemcpyAsync(rhs, d_r, n * b * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        return take_status(ctx, fail_block);
    });
}

int spingp_seg_forward_device(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                              const double* theta, int32_t n_theta, const double* d_t, const double* d_y,
                              int64_t n_local, double t_left, double t_right, int32_t rank, int32_t nranks,
                              double sigma, uint32_t flags, double* d_record) {
    return seg_run(ctx, 2, leaves, n_leaves, theta, n_theta, d_t, d_y, n_local, t_left, t_right, rank, nranks,
                   sigma, flags, nullptr, d_record, nullptr, nullptr);
}

int spingp_seg_reverse_device(spingp_ctx* ctx, const spingp_leaf* leaves, int32_t n_leaves,
                              const double* theta, int32_t n_theta, const double* d_t, const double* d_y,
                              int64_t n_local, double t_left, double t_right, int32_t rank, int32_t nranks,
                              double sigma, uint32_t flags, const double* d_records, double* d_partials,
                              double* d_mean, double* d_var) {
    return seg_run(ctx, 3, leaves, n_leaves, theta, n_theta, d_t, d_y, n_local, t_left, t_right, rank, nranks,
                   sigma, flags, d_records, d_partials, d_mean, d_var);
}

int spingp_seg_finalize_device(spingp_ctx* ctx, int32_t n_theta, int64_t n_total, double sigma, uint32_t flags,
                               const double* d_partials, double* d_loglik, double* d_grad) {
    return guarded(nullptr, [&] {
        checked(ctx);
        if (!d_partials || !d_loglik || ((flags & SPINGP_WANT_GRAD) && !d_grad)) throw std::invalid_argument("null argument");
        std::lock_guard<std::mutex> lk(ctx->mu);
        SegFinalArgs fa{d_partials, n_theta, n_total, sigma, d_loglik, (flags & SPINGP_WANT_GRAD) ? d_grad : nullptr};
        ctx->pre();
        k_seg_final<<<1, 32, 0, ctx->stream>>>(fa);
        ctx->launched("k_seg_final");
        return SPINGP_OK;
    });
}

static void cr_solve_locked(spingp_ctx* ctx, int64_t n, int32_t b, const double* d_diag, const double* d_upper,
                            const double* d_rhs, int32_t k, double* d_x, double* d_logdet) {
    if (!d_diag || (n > 1 && !d_upper) || k < 0 || (k > 0 && (!d_rhs || !d_x)))
        throw std::invalid_argument("bad argument");
    // b <= 4, at most one right-hand side: the tile-streaming kernel (stream_solve.cuh)
    if (k <= 1 && stream_solve(ctx, n, b, d_diag, d_upper, k ? d_rhs : nullptr, k ? d_x : nullptr, d_logdet)) return;
    if (k == 0) {
        btd_dispatch(ctx, n, b, d_diag, d_upper, nullptr, 1, 0, nullptr, nullptr, nullptr, d_logdet, false);
        return;
    }
    for (int col = 0; col < k; ++col)
        btd_dispatch(ctx, n, b, d_diag, d_upper, d_rhs, k, col, d_x, nullptr, nullptr, col == 0 ? d_logdet : nullptr,
                     false);
}

int spingp_btd_cr_solve_device(spingp_ctx* ctx, int64_t n, int32_t b, const double* d_diag,
                               const double* d_upper, const double* d_rhs, int32_t k, double* d_x,
                               double* d_logdet) {
    return guarded(nullptr, [&] {
        checked(ctx);
        std::lock_guard<std::mutex> lk(ctx->mu);
        cr_solve_locked(ctx, n, b, d_diag, d_upper, d_rhs, k, d_x, d_logdet);
        return SPINGP_OK;
    });
}

int spingp_btd_cr_solve(spingp_ctx* ctx, int64_t n, int32_t b, const double* diag,
                        const double* upper, const double* rhs, int32_t k, double* x,
                        double* logdet, int64_t* fail_block) {
    return guarded(fail_block, [&] {
        checked(ctx);
        if (!diag || n < 1 || b < 1 || k < 0 || (n > 1 && !upper) || (k > 0 && !rhs))
            throw std::invalid_argument("bad argument");
        std::lock_guard<std::mutex> lk(ctx->mu);
        const size_t nd = static_cast<size_t>(n) * b * b, nu = static_cast<size_t>(n - 1) * b * b;
        const size_t nr = static_cast<size_t>(n) * b * k;
        // every array on a 16-byte boundary (even offsets): the streaming solve's bulk copies
        auto even = [](size_t c) { return (c + 1) & ~size_t(1); };
        double* d_d = ctx->host_io.get(even(nd) + even(nu) + 2 * even(nr) + 2);
        double* d_u = d_d + even(nd);
        double* d_r = d_u + even(nu);
        double* d_x = d_r + even(nr);
        double* d_ld = d_x + even(nr);
        CUDA_OK(cudaMemcpyAsync(d_d, diag, nd * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        if (nu) CUDA_OK(cudaMemcpyAsync(d_u, upper, nu * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        if (nr) CUDA_OK(cudaMemcpyAsync(d_r, rhs, nr * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        cr_solve_locked(ctx, n, b, d_d, d_u, nr ? d_r : nullptr, k, nr ? d_x : nullptr, d_ld);
        if (nr && x) CUDA_OK(cudaMemcpyAsync(x, d_x, nr * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (logdet) CUDA_OK(cudaMemcpyAsync(logdet, d_ld, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        return take_status(ctx, fail_block);
    });
}

static void selinv_locked(spingp_ctx* ctx, int64_t n, int32_t b, const double* d_diag, const double* d_upper,
                          double* d_cdiag, double* d_cupper, double* d_logdet) {
    if (!d_diag || !d_cdiag || (n > 1 && (!d_upper || !d_cupper))) throw std::invalid_argument("bad argument");
    btd_dispatch(ctx, n, b, d_diag, d_upper, nullptr, 1, 0, nullptr, d_cdiag, d_cupper, d_logdet, true);
}

int spingp_btd_selinv_device(spingp_ctx* ctx, int64_t n, int32_t b, const double* d_diag,
                             const double* d_upper, double* d_cdiag, double* d_cupper,
                             double* d_logdet) {
    return guarded(nullptr, [&] {
        checked(ctx);
        std::lock_guard<std::mutex> lk(ctx->mu);
        selinv_locked(ctx, n, b, d_diag, d_upper, d_cdiag, d_cupper, d_logdet);
        return SPINGP_OK;
    });
}

int spingp_btd_selinv(spingp_ctx* ctx, int64_t n, int32_t b, const double* diag,
                      const double* upper, double* cdiag, double* cupper, double* logdet,
                      int64_t* fail_block) {
    return guarded(fail_block, [&] {
        checked(ctx);
        if (!diag || !cdiag || n < 1 || b < 1 || (n > 1 && !upper)) throw std::invalid_argument("bad argument");
        std::lock_guard<std::mutex> lk(ctx->mu);
        const size_t nd = static_cast<size_t>(n) * b * b, nu = static_cast<size_t>(n - 1) * b * b;
        double* d_d = ctx->host_io.get(2 * nd + 2 * nu + 1);
        double* d_u = d_d + nd;
        double* d_cd = d_u + nu;
        double* d_cu = d_cd + nd;
        double* d_ld = d_cu + nu;
        CUDA_OK(cudaMemcpyAsync(d_d, diag, nd * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        if (nu) CUDA_OK(cudaMemcpyAsync(d_u, upper, nu * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        selinv_locked(ctx, n, b, d_d, d_u, d_cd, d_cu, d_ld);
        CUDA_OK(cudaMemcpyAsync(cdiag, d_cd, nd * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (nu && cupper) CUDA_OK(cudaMemcpyAsync(cupper, d_cu, nu * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (logdet) CUDA_OK(cudaMemcpyAsync(logdet, d_ld, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        return take_status(ctx, fail_block);
    });
}

int spingp_btd_matvec(spingp_ctx* ctx, int64_t n, int32_t b, const double* diag,
                      const double* upper, const double* v, double* out) {
    return guarded(nullptr, [&] {
        checked(ctx);
        if (!diag || !v || !out || n < 1 || b < 1) throw std::invalid_argument("bad argument");
        std::lock_guard<std::mutex> lk(ctx->mu);
        const size_t nd = static_cast<size_t>(n) * b * b, nu = static_cast<size_t>(n - 1) * b * b;
        const size_t nv = static_cast<size_t>(n) * b;
        double* d_d = ctx->host_io.get(nd + nu + 2 * nv);
        double* d_u = d_d + nd;
        double* d_v = d_u + nu;
        double* d_o = d_v + nv;
        CUDA_OK(cudaMemcpyAsync(d_d, diag, nd * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        if (nu) CUDA_OK(cudaMemcpyAsync(d_u, upper, nu * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        CUDA_OK(cudaMemcpyAsync(d_v, v, nv * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        k_matvec<<<blocks_for(n, 128), 128, 0, ctx->stream>>>(n, b, d_d, d_u, d_v, d_o);
        ctx->launched();
        CUDA_OK(cudaMemcpyAsync(out, d_o, nv * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_OK(cudaStreamSynchronize(ctx->stream));
        return SPINGP_OK;
    });
}

}  // extern "C"
