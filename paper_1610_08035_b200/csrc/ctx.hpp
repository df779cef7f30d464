// ctx.hpp — the context behind the C ABI (device, stream, workspace, status word)
// and the host-side reduction plan.  Shared by the nvcc translation units.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.cuh"
#include "host_model.hpp"
#include "spingp_c.h"

namespace spingp_host {

#define CUDA_OK(expr)                                                                          \
    do {                                                                                       \
        cudaError_t e_ = (expr);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            throw ::spingp_host::ApiError{SPINGP_CUDA_ERR, -1,                                 \
                                          std::string(#expr) + ": " + cudaGetErrorString(e_)}; \
    } while (0)

std::string& last_error();

template <class F>
int guarded(int64_t* fail_block, F&& body) {
    if (fail_block) *fail_block = -1;
    try {
        return body();
    } catch (const ApiError& e) {
        if (fail_block) *fail_block = e.block;
        last_error() = e.what;
        return e.status;
    } catch (const std::invalid_argument& e) {
        last_error() = e.what();
        return SPINGP_BAD_ARG;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return SPINGP_UNSUPPORTED;
    }
}

struct Arena {
    char* base = nullptr;
    size_t size = 0, used = 0;
    void reset() { used = 0; }
    template <class T>
    T* take(size_t count) {
        const size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
        if (used + bytes > size) throw ApiError{SPINGP_CUDA_ERR, -1, "workspace overflow"};
        T* p = reinterpret_cast<T*>(base + used);
        used += bytes;
        return p;
    }
};

inline size_t arena_bytes(size_t count) { return (count * sizeof(double) + 255) & ~size_t(255); }

inline unsigned blocks_for(long long n, int tpb) { return static_cast<unsigned>((n + tpb - 1) / tpb); }

// device scratch of the host-pointer entry points (owned by the context, used under its mutex)
struct DeviceVec {
    double* p = nullptr;
    size_t n = 0;
    double* get(size_t count) {
        if (count > n) {
            if (p) cudaFree(p);
            p = nullptr;
            n = 0;
            CUDA_OK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(double)));
            n = count;
        }
        return p;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

}  // namespace spingp_host

struct spingp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    spingp_host::Arena ws;
    spingp_host::DeviceVec host_io;  // H2D/D2H landing buffers of the host-pointer entry points
    unsigned long long* d_status = nullptr;
    unsigned long long* h_status = nullptr;  // pinned landing slot of the status word
    double* h_stage[2] = {nullptr, nullptr};
    size_t h_stage_cap[2] = {0, 0};
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    int stage_slot = 0, cur_slot = 0;
    int64_t launches = 0;
    int64_t m0_override = 0;  // testing knob: force the level-0 chunk length
    int64_t g_override = 0;   // testing knob: force a smaller tree group (more tree levels)
    // last model built (build_model is per-structure host work: EQ roots in long double,
    // the reference state_space_of); reused while the leaves and theta count repeat
    std::vector<int32_t> model_key;
    spingp_host::HostModel model;
    // host-input pipelining: copy stream + events (created on first use)
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t pipe_ev[40] = {};
    std::mutex mu;
    // optional per-launch CUDA-event timing (spingp_ctx_set_profiling)
    bool profiling = false;
    struct Timed {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Timed> timed;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    cudaEvent_t next_event() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            CUDA_OK(cudaEventCreate(&e));
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }
    // bracket one kernel launch: pre() before, launched(name) after
    cudaEvent_t pending = nullptr;
    void pre() {
        if (!profiling) return;
        pending = next_event();
        CUDA_OK(cudaEventRecord(pending, stream));
    }

    // self-resetting per-series arrival counters of k_reduce (kept out of the arena so
    // their zero state survives between calls; grown on demand, zeroed when allocated)
    unsigned int* d_arrive = nullptr;
    // grid barrier words of the tile-streaming solve (stream_solve.cu): monotonic counters
    unsigned long long* d_ss_sync = nullptr;
    unsigned long long ss_arrivals = 0, ss_releases = 0;
    unsigned long long* upper_stamps = nullptr;  // diagnostics (spingp_ctx_upper_stamps)
    long long arrive_cap = 0;
    unsigned int* counters(long long S) {
        if (S > arrive_cap) {
            if (d_arrive) {
                CUDA_OK(cudaStreamSynchronize(stream));
                CUDA_OK(cudaFree(d_arrive));
            }
            const long long cap = std::max<long long>(S, 1024);
            CUDA_OK(cudaMalloc(&d_arrive, cap * sizeof(unsigned int)));
            CUDA_OK(cudaMemset(d_arrive, 0, cap * sizeof(unsigned int)));
            arrive_cap = cap;
        }
        return d_arrive;
    }

    void ensure_ws(size_t bytes) {
        if (bytes <= ws.size) return;
        if (ws.base) {
            CUDA_OK(cudaStreamSynchronize(stream));
            CUDA_OK(cudaFree(ws.base));
            ws.base = nullptr;
            ws.size = 0;
        }
        const size_t cap = std::max(bytes, ws.size + ws.size / 2);
        CUDA_OK(cudaMalloc(&ws.base, cap));
        ws.size = cap;
    }
    // pinned staging slot for small host->device parameter uploads (double-buffered;
    // a slot is reused only after the copy that read it has executed)
    double* stage(size_t count) {
        const int k = stage_slot;
        stage_slot ^= 1;
        CUDA_OK(cudaEventSynchronize(stage_ev[k]));
        if (count > h_stage_cap[k]) {
            if (h_stage[k]) CUDA_OK(cudaFreeHost(h_stage[k]));
            const size_t cap = std::max<size_t>(count, 4096);
            CUDA_OK(cudaMallocHost(&h_stage[k], cap * sizeof(double)));
            h_stage_cap[k] = cap;
        }
        cur_slot = k;
        return h_stage[k];
    }
    void stage_done() { CUDA_OK(cudaEventRecord(stage_ev[cur_slot], stream)); }
    void launched(const char* name = "kernel") {
        launches++;
        CUDA_OK(cudaGetLastError());
        if (profiling && pending) {
            cudaEvent_t e = next_event();
            CUDA_OK(cudaEventRecord(e, stream));
            timed.push_back(Timed{name, pending, e});
            pending = nullptr;
        }
    }
};

namespace spingp_host {

// Synchronise and collect (then clear) the device status word.
int take_status(spingp_ctx* ctx, int64_t* fail_block);

// Upload `count` doubles from host memory through the context's pinned stage.
void upload(spingp_ctx* ctx, double* dst, const double* src, size_t count);

// One evaluation (S series) on device-resident t, y: entry points per kernel
// instantiation family live in separate translation units.
struct EvalArgs {
    const HostModel* hm;
    const Plan* plan;
    const double* h_params;
    size_t nparams;
    const double* d_t;
    const double* d_y;
    uint32_t flags;
    double* d_loglik;
    double* d_grad;
    double* d_mean;
    double* d_var;
    // mode 1: assemble only into d_diag / d_upper / d_rhs (S = 1)
    // mode 2: segment forward -> d_seg_out (this rank's top-level record)
    // mode 3: segment reverse from d_seg_in (all ranks' records) -> d_seg_out (partial sums)
    int mode;
    double* d_diag;
    double* d_upper;
    double* d_rhs;
    int rank = 0, nranks = 1;
    const double* d_seg_in = nullptr;
    double* d_seg_out = nullptr;
    // host-input pipelining (spingp_eval_batched, S = 1): k_fwd0 runs in pieces of level-0
    // chunks [in_chunk[p], in_chunk[p+1]), each after in_ready[p] (its inputs' H2D);
    // k_rev0 runs in pieces [out_chunk[q], out_chunk[q+1]) and records out_ready[q]
    // after each (its points' mean/var may then be copied back)
    // observation mask (predict at test times): d_obs[S*n] 1 = observed (null = all);
    // n_obs = observed points per series (the loglik's N; < 0 = n)
    const unsigned char* d_obs = nullptr;
    long long n_obs = -1;
    int in_pieces = 0;
    const long long* in_chunk = nullptr;
    const cudaEvent_t* in_ready = nullptr;
    int out_pieces = 0;
    const long long* out_chunk = nullptr;
    const cudaEvent_t* out_ready = nullptr;
};
// one translation unit per instantiation (inst_*.cu, btd_b*.cu) so they build in parallel
void eval_matern_1(spingp_ctx* ctx, const EvalArgs& a);
void eval_matern_2(spingp_ctx* ctx, const EvalArgs& a);
void eval_matern_3(spingp_ctx* ctx, const EvalArgs& a);
void eval_generic_3(spingp_ctx* ctx, const EvalArgs& a);
void eval_generic_4(spingp_ctx* ctx, const EvalArgs& a);
void eval_generic_6(spingp_ctx* ctx, const EvalArgs& a);
void eval_generic_8(spingp_ctx* ctx, const EvalArgs& a);
void eval_generic_12(spingp_ctx* ctx, const EvalArgs& a);
void eval_generic_16(spingp_ctx* ctx, const EvalArgs& a);
int64_t rev0_wave_threads_m3();  // inst_m3.cu
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the attribute
// is per device, so the cache is a per-kernel bitmask of devices
inline void opt_in_smem(const void* kern, unsigned long long& done_mask, int device, int bytes) {
    const unsigned long long bit = 1ULL << (device & 63);
    if (done_mask & bit) return;
    CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done_mask |= bit;
}
void eval_s_eq6(spingp_ctx* ctx, const EvalArgs& a);       // inst_s_eq6.cu
void eval_s_eq10(spingp_ctx* ctx, const EvalArgs& a);      // inst_s_eq10.cu
void eval_s_m32qp6(spingp_ctx* ctx, const EvalArgs& a);    // inst_s_m32qp6.cu
void eval_s_m32eq10(spingp_ctx* ctx, const EvalArgs& a);   // inst_s_m32eq10.cu
#define SPINGP_BTD_DECL(B)                                                                          \
    void btd_run_##B(spingp_ctx* ctx, int64_t n, int b, const double* diag, const double* upper, \
                     const double* rhs, int k, int col, double* x, double* cdiag, double* cupper, \
                     double* logdet, bool needC);
bool stream_solve(spingp_ctx* ctx, int64_t n, int b, const double* diag, const double* upper, const double* rhs,
                  double* x, double* logdet);  // stream_solve.cu
SPINGP_BTD_DECL(1)
SPINGP_BTD_DECL(2)
SPINGP_BTD_DECL(3)
SPINGP_BTD_DECL(4)
SPINGP_BTD_DECL(6)
SPINGP_BTD_DECL(8)
SPINGP_BTD_DECL(12)
SPINGP_BTD_DECL(16)
#undef SPINGP_BTD_DECL

}  // namespace spingp_host
