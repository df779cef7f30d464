// multi.cu — multi-GPU evaluation inside the library: one host
// thread drives P devices of one box, each with its own spingp_ctx (stream, workspace),
// joined by an NCCL communicator (ncclCommInitAll).  One long series is cut into P
// contiguous time segments (segment r owns points [b_r, b_{r+1}) and sees its
// neighbours' adjacent times as halos); per evaluation:
//
//   spingp_seg_forward_device   on every device (segment -> 2-separator Schur record)
//   ncclAllGather               of the P records (3b^2 + 2b + 1 doubles each)
//   spingp_seg_reverse_device   on every device (reduced P-block system solved redundantly,
//                               back substitution, selected inverse, gradient terms)
//   ncclAllReduce               of the 5 + n_theta partial sums
//   spingp_seg_finalize_device  -> loglik, gradient
//
// The collectives are enqueued on the devices' own streams inside ncclGroupStart/End,
// so the whole evaluation is asynchronous until the final D2H.  NCCL is loaded with
// dlopen on first use: the single-GPU library has no NCCL dependency, and without NCCL
// the multi-GPU entry points return SPINGP_NCCL_ERR.
//
// Replaces the data-parallel cr_solve contract of SPEC.md:200,224 ("independent
// eliminations within a level may execute concurrently") at the scale of a box.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "ctx.hpp"

using namespace spingp_host;

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("NCCL not found: ") + dlerror();
            return a;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
        a.commInitAll = reinterpret_cast<decltype(a.commInitAll)>(sym("ncclCommInitAll"));
        a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(sym("ncclCommDestroy"));
        a.allGather = reinterpret_cast<decltype(a.allGather)>(sym("ncclAllGather"));
        a.allReduce = reinterpret_cast<decltype(a.allReduce)>(sym("ncclAllReduce"));
        a.groupStart = reinterpret_cast<decltype(a.groupStart)>(sym("ncclGroupStart"));
        a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(sym("ncclGroupEnd"));
        a.errStr = reinterpret_cast<decltype(a.errStr)>(sym("ncclGetErrorString"));
        a.ok = a.commInitAll && a.commDestroy && a.allGather && a.allReduce && a.groupStart && a.groupEnd && a.errStr;
        if (!a.ok) a.why = "NCCL symbols missing";
        return a;
    }();
    return api;
}

#define NCCL_OK(expr)                                                                                   \
    do {                                                                                                \
        ncclResult_t r_ = (expr);                                                                       \
        if (r_ != ncclSuccess)                                                                          \
            throw ApiError{SPINGP_NCCL_ERR, -1, std::string(#expr) + ": " + nccl().errStr(r_)};         \
    } while (0)

}  // namespace

struct spingp_mctx {
    int P = 0;
    std::vector<int> dev;
    std::vector<spingp_ctx*> ctx;
    std::vector<ncclComm_t> comm;
    // per-rank device buffers (grown on demand): t, y, mean, var segments; record,
    // records (P x nrec), partials, loglik, grad
    std::vector<spingp_host::DeviceVec> seg, small;
    std::mutex mu;
};

extern "C" {

int spingp_mctx_create(int32_t n_gpus, const int32_t* device_ids, spingp_mctx** out) {
    return guarded(nullptr, [&] {
        if (!out || n_gpus < 1 || n_gpus > 64) throw std::invalid_argument("bad argument");
        *out = nullptr;
        const NcclApi& api = nccl();
        if (!api.ok) throw ApiError{SPINGP_NCCL_ERR, -1, api.why};
        auto* m = new spingp_mctx();
        m->P = n_gpus;
        for (int r = 0; r < n_gpus; ++r) m->dev.push_back(device_ids ? device_ids[r] : r);
        try {
            for (int r = 0; r < n_gpus; ++r) {
                spingp_ctx* c = nullptr;
                const int st = spingp_ctx_create(m->dev[r], &c);
                if (st != SPINGP_OK) throw ApiError{st, -1, spingp_last_error()};
                m->ctx.push_back(c);
            }
            m->comm.resize(n_gpus);
            NCCL_OK(api.commInitAll(m->comm.data(), n_gpus, m->dev.data()));
        } catch (...) {
            spingp_mctx_destroy(m);
            throw;
        }
        m->seg.resize(n_gpus);
        m->small.resize(n_gpus);
        *out = m;
        return SPINGP_OK;
    });
}

int spingp_mctx_destroy(spingp_mctx* m) {
    if (!m) return SPINGP_OK;
    for (size_t r = 0; r < m->comm.size(); ++r)
        if (m->comm[r]) nccl().commDestroy(m->comm[r]);
    for (size_t r = 0; r < m->ctx.size(); ++r) {
        cudaSetDevice(m->dev[r]);
        if (r < m->seg.size()) m->seg[r].release();
        if (r < m->small.size()) m->small[r].release();
        spingp_ctx_destroy(m->ctx[r]);
    }
    delete m;
    return SPINGP_OK;
}

int32_t spingp_mctx_size(const spingp_mctx* m) { return m ? m->P : 0; }

spingp_ctx* spingp_mctx_rank_ctx(spingp_mctx* m, int32_t rank) {
    return (m && rank >= 0 && rank < m->P) ? m->ctx[rank] : nullptr;
}

int spingp_eval_partitioned(spingp_mctx* m, const spingp_leaf* leaves, int32_t n_leaves, const double* theta,
                            int32_t n_theta, const double* t, const double* y, int64_t n, double sigma,
                            uint32_t flags, double* out_loglik, double* out_grad, double* out_mean, double* out_var,
                            int64_t* fail_block) {
    return guarded(fail_block, [&] {
        if (!m || !theta || !t || !y || !out_loglik || n < 1) throw std::invalid_argument("bad argument");
        if ((flags & SPINGP_WANT_GRAD) && !out_grad) throw std::invalid_argument("gradient output is null");
        if ((flags & SPINGP_WANT_MEAN) && !out_mean) throw std::invalid_argument("mean output is null");
        if ((flags & SPINGP_WANT_VAR) && !out_var) throw std::invalid_argument("variance output is null");
        const int P = m->P;
        if (n < P) throw std::invalid_argument("need at least one point per device");
        std::lock_guard<std::mutex> lk(m->mu);
        const NcclApi& api = nccl();
        int32_t nrec = 0, npart = 0;
        {
            const int st = spingp_seg_sizes(leaves, n_leaves, &nrec, &npart);
            if (st != SPINGP_OK) throw ApiError{st, -1, spingp_last_error()};
        }
        std::vector<int64_t> bnd(P + 1);
        for (int r = 0; r <= P; ++r) bnd[r] = static_cast<int64_t>(std::llround(static_cast<double>(r) * n / P));
        const bool wm = flags & SPINGP_WANT_MEAN, wv = flags & SPINGP_WANT_VAR;
        const size_t nt1 = static_cast<size_t>(n_theta) + 1;
        struct Bufs {
            double *t, *y, *mean, *var, *rec, *recs, *part, *ll, *g;
            int64_t nl;
        };
        std::vector<Bufs> b(P);
        for (int r = 0; r < P; ++r) {
            CUDA_OK(cudaSetDevice(m->dev[r]));
            const int64_t nl = bnd[r + 1] - bnd[r];
            double* s = m->seg[r].get(static_cast<size_t>(nl) * (2 + wm + wv));
            double* q = m->small[r].get(static_cast<size_t>(nrec) * (P + 1) + npart + 1 + nt1);
            b[r] = Bufs{s, s + nl, wm ? s + 2 * nl : nullptr, wv ? s + (2 + wm) * nl : nullptr, q, q + nrec,
                        q + nrec * (P + 1), q + nrec * (P + 1) + npart, q + nrec * (P + 1) + npart + 1, nl};
            cudaStream_t st = m->ctx[r]->stream;
            CUDA_OK(cudaMemcpyAsync(b[r].t, t + bnd[r], nl * sizeof(double), cudaMemcpyHostToDevice, st));
            CUDA_OK(cudaMemcpyAsync(b[r].y, y + bnd[r], nl * sizeof(double), cudaMemcpyHostToDevice, st));
        }
        auto halo_l = [&](int r) { return r > 0 ? t[bnd[r] - 1] : std::nan(""); };
        auto halo_r = [&](int r) { return r + 1 < P ? t[bnd[r + 1]] : std::nan(""); };
        auto chk = [&](int st) {
            if (st != SPINGP_OK) throw ApiError{st, -1, spingp_last_error()};
        };
        for (int r = 0; r < P; ++r)
            chk(spingp_seg_forward_device(m->ctx[r], leaves, n_leaves, theta, n_theta, b[r].t, b[r].y, b[r].nl,
                                          halo_l(r), halo_r(r), r, P, sigma, flags, b[r].rec));
        NCCL_OK(api.groupStart());
        for (int r = 0; r < P; ++r) {
            CUDA_OK(cudaSetDevice(m->dev[r]));
            NCCL_OK(api.allGather(b[r].rec, b[r].recs, static_cast<size_t>(nrec), ncclDouble, m->comm[r],
                                  m->ctx[r]->stream));
        }
        NCCL_OK(api.groupEnd());
        for (int r = 0; r < P; ++r)
            chk(spingp_seg_reverse_device(m->ctx[r], leaves, n_leaves, theta, n_theta, b[r].t, b[r].y, b[r].nl,
                                          halo_l(r), halo_r(r), r, P, sigma, flags, b[r].recs, b[r].part, b[r].mean,
                                          b[r].var));
        NCCL_OK(api.groupStart());
        for (int r = 0; r < P; ++r) {
            CUDA_OK(cudaSetDevice(m->dev[r]));
            NCCL_OK(api.allReduce(b[r].part, b[r].part, static_cast<size_t>(npart), ncclDouble, ncclSum, m->comm[r],
                                  m->ctx[r]->stream));
        }
        NCCL_OK(api.groupEnd());
        chk(spingp_seg_finalize_device(m->ctx[0], n_theta, n, sigma, flags, b[0].part, b[0].ll, b[0].g));
        CUDA_OK(cudaSetDevice(m->dev[0]));
        CUDA_OK(cudaMemcpyAsync(out_loglik, b[0].ll, sizeof(double), cudaMemcpyDeviceToHost, m->ctx[0]->stream));
        if (flags & SPINGP_WANT_GRAD)
            CUDA_OK(cudaMemcpyAsync(out_grad, b[0].g, nt1 * sizeof(double), cudaMemcpyDeviceToHost, m->ctx[0]->stream));
        for (int r = 0; r < P; ++r) {
            CUDA_OK(cudaSetDevice(m->dev[r]));
            if (wm)
                CUDA_OK(cudaMemcpyAsync(out_mean + bnd[r], b[r].mean, b[r].nl * sizeof(double), cudaMemcpyDeviceToHost,
                                        m->ctx[r]->stream));
            if (wv)
                CUDA_OK(cudaMemcpyAsync(out_var + bnd[r], b[r].var, b[r].nl * sizeof(double), cudaMemcpyDeviceToHost,
                                        m->ctx[r]->stream));
        }
        int first = SPINGP_OK;
        int64_t fb_first = -1;
        for (int r = 0; r < P; ++r) {  // every device's status word (a segment's block index is local)
            int64_t fb = -1;
            const int st = spingp_ctx_status(m->ctx[r], &fb);
            if (st != SPINGP_OK && first == SPINGP_OK) {
                first = st;
                fb_first = fb >= 0 ? fb + bnd[r] : fb;
            }
        }
        if (first != SPINGP_OK) throw ApiError{first, fb_first, spingp_last_error()};
        return SPINGP_OK;
    });
}

}  // extern "C"
