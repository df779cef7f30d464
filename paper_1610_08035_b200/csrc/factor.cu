// factor.cu — the device-resident BTDFactor of SPEC.md:135-140 (btd_core):
// factorize once, then solve / selective_inverse / logdet without re-factorising.
//
// factorize(m).  The partitioned elimination (btd_ops.cuh, the cr_solve machinery) runs
// once with the selected inverse switched on: it yields log det and the BTD blocks
// C_ii, C_{i,i+1} of m^{-1}.  The SPEC's Thomas-form factor then follows block by block
// IN PARALLEL from the Takahashi identities (C_{n-1,n-1} = S_{n-1}^{-1},
// C_{i,i+1} = -G_i C_{i+1,i+1}, C_ii = S_i^{-1} + G_i C_{i+1,i+1} G_i^T, G_i = S_i^{-1} U_i):
//     S_i^{-1} = C_ii - C_{i,i+1} C_{i+1,i+1}^{-1} C_{i,i+1}^T,   L_i = chol(S_i),
//     M_i = U_i^T S_i^{-1}                                          (k_factor_blocks)
// so every pivot block of the sequential recursion is available without running it.
//
// solve(f, rhs).  The block substitutions of the LDL^T factor,
//     forward  y_0 = r_0,  y_i = r_i - M_{i-1} y_{i-1}
//     backward x_{n-1} = S_{n-1}^{-1} y_{n-1},  x_i = S_i^{-1} y_i - M_i^T x_{i+1},
// are linear recurrences, run as chunk-parallel passes: every chunk of kChunk blocks
// computes its local solution from a zero boundary plus its b x b transfer matrix
// (k_sub_local), one thread chains the chunk boundaries (k_sub_scan, K = n / kChunk
// b x b products), and every chunk recomputes with its true boundary (k_sub_final).
// selective_inverse(f) returns the stored blocks; logdet(f) the stored value.
//
// Block size is a runtime b <= 16 (per-thread b x b arrays): this is the API path
// (SPEC-sized problems); the throughput paths are cr_solve and the fused evaluation.
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "ctx.hpp"

using namespace spingp_host;

struct spingp_btd_factor {
    int device = 0;
    int64_t n = 0;
    int b = 0;
    double logdet = 0.0;
    double* d_L = nullptr;   // [n][b][b] lower, positive diagonal
    double* d_M = nullptr;   // [n-1][b][b]
    double* d_Cd = nullptr;  // [n][b][b]  diag blocks of m^{-1}
    double* d_Cu = nullptr;  // [n-1][b][b] upper blocks of m^{-1}
};

namespace {

constexpr int kMaxb = 16;
constexpr int kChunk = 64;
constexpr int kMaxK = 16;  // right-hand sides per substitution pass

__device__ bool dchol(double* L, const double* A, int b) {  // A = L L^T, L lower, diag > 0
    for (int j = 0; j < b; ++j) {
        double d = A[j * b + j];
        for (int k = 0; k < j; ++k) d -= L[j * b + k] * L[j * b + k];
        if (!(d > 0.0) || !isfinite(d)) return false;
        const double l = sqrt(d);
        L[j * b + j] = l;
        for (int i = j + 1; i < b; ++i) {
            double s = A[i * b + j];
            for (int k = 0; k < j; ++k) s -= L[i * b + k] * L[j * b + k];
            L[i * b + j] = s / l;
        }
        for (int i = 0; i < j; ++i) L[i * b + j] = 0.0;
    }
    return true;
}
__device__ void dlsolve(double* x, const double* L, int b) {  // x <- L^{-1} x
    for (int i = 0; i < b; ++i) {
        double s = x[i];
        for (int k = 0; k < i; ++k) s -= L[i * b + k] * x[k];
        x[i] = s / L[i * b + i];
    }
}
__device__ void dltsolve(double* x, const double* L, int b) {  // x <- L^{-T} x
    for (int i = b - 1; i >= 0; --i) {
        double s = x[i];
        for (int k = i + 1; k < b; ++k) s -= L[k * b + i] * x[k];
        x[i] = s / L[i * b + i];
    }
}
__device__ bool dspd_inverse(double* Ai, const double* A, int b, double* work) {  // Ai = A^{-1}, symmetric
    if (!dchol(work, A, b)) return false;
    double e[kMaxb];
    for (int j = 0; j < b; ++j) {
        for (int i = 0; i < b; ++i) e[i] = i == j ? 1.0 : 0.0;
        dlsolve(e, work, b);
        dltsolve(e, work, b);
        for (int i = 0; i < b; ++i) Ai[i * b + j] = e[i];
    }
    for (int i = 0; i < b; ++i)
        for (int j = 0; j < i; ++j) {
            const double v = 0.5 * (Ai[i * b + j] + Ai[j * b + i]);
            Ai[i * b + j] = v;
            Ai[j * b + i] = v;
        }
    return true;
}

// one thread per block row i: S_i^{-1}, L_i = chol(S_i), M_i = U_i^T S_i^{-1}
__global__ void k_factor_blocks(int64_t n, int b, const double* __restrict__ upper, const double* __restrict__ Cd,
                                const double* __restrict__ Cu, double* __restrict__ Lo, double* __restrict__ Mo,
                                unsigned long long* status) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int bb = b * b;
    double Si[kMaxb * kMaxb], W[kMaxb * kMaxb], T[kMaxb * kMaxb], work[kMaxb * kMaxb];
    for (int q = 0; q < bb; ++q) Si[q] = Cd[i * bb + q];
    if (i + 1 < n) {
        if (!dspd_inverse(W, Cd + (i + 1) * bb, b, work)) {
            spingp_dev::report(status, i + 1, spingp_dev::ST_NOT_PD);
            return;
        }
        const double* C = Cu + i * bb;  // C_{i,i+1}
        for (int r = 0; r < b; ++r)      // T = C W
            for (int c = 0; c < b; ++c) {
                double s = 0.0;
                for (int k = 0; k < b; ++k) s += C[r * b + k] * W[k * b + c];
                T[r * b + c] = s;
            }
        for (int r = 0; r < b; ++r)      // S^{-1} = C_ii - T C^T
            for (int c = 0; c < b; ++c) {
                double s = 0.0;
                for (int k = 0; k < b; ++k) s += T[r * b + k] * C[c * b + k];
                Si[r * b + c] -= s;
            }
    }
    for (int r = 0; r < b; ++r)
        for (int c = 0; c < r; ++c) {
            const double v = 0.5 * (Si[r * b + c] + Si[c * b + r]);
            Si[r * b + c] = v;
            Si[c * b + r] = v;
        }
    if (!dspd_inverse(W, Si, b, work) || !dchol(T, W, b)) {  // W = S_i, T = L_i
        spingp_dev::report(status, i, spingp_dev::ST_NOT_PD);
        return;
    }
    for (int q = 0; q < bb; ++q) Lo[i * bb + q] = T[q];
    if (i + 1 < n) {
        const double* U = upper + i * bb;
        for (int r = 0; r < b; ++r)      // M = U^T S^{-1}
            for (int c = 0; c < b; ++c) {
                double s = 0.0;
                for (int k = 0; k < b; ++k) s += U[k * b + r] * Si[k * b + c];
                Mo[i * bb + r * b + c] = s;
            }
    }
}

// Chunk-parallel block substitution.  dir = 0 forward (y), dir = 1 backward (x; y is read
// from x in place).  mode 0: local pass from a zero boundary -> the chunk's exit value
// (b x k at ends) and transfer matrix (b x b at trans); mode 1: final pass from the true
// boundary bnd (b x k) -> x.
__device__ void sub_step(int dir, int64_t i, int64_t n, int b, int k, const double* L, const double* M, double* v,
                         const double* in_v, double* out_x) {
    // forward : v_i = r_i - M_{i-1} v_{i-1}        (in_v = v_{i-1}, r_i from out_x row i)
    // backward: v_i = S_i^{-1} y_i - M_i^T v_{i+1}  (in_v = v_{i+1}, y_i from out_x row i)
    const int bb = b * b;
    for (int c = 0; c < k; ++c) {
        double r[kMaxb], t[kMaxb];
        for (int a = 0; a < b; ++a) r[a] = out_x[(i * b + a) * k + c];
        if (dir == 0) {
            if (i > 0)
                for (int a = 0; a < b; ++a) {
                    double s = 0.0;
                    for (int q = 0; q < b; ++q) s += M[(i - 1) * bb + a * b + q] * in_v[q * k + c];
                    r[a] -= s;
                }
        } else {
            dlsolve(r, L + i * bb, b);
            dltsolve(r, L + i * bb, b);
            if (i + 1 < n)
                for (int a = 0; a < b; ++a) {
                    double s = 0.0;
                    for (int q = 0; q < b; ++q) s += M[i * bb + q * b + a] * in_v[q * k + c];
                    r[a] -= s;
                }
        }
        for (int a = 0; a < b; ++a) t[a] = r[a];
        for (int a = 0; a < b; ++a) v[a * k + c] = t[a];
    }
}

__global__ void k_sub_pass(int dir, int mode, int64_t n, int b, int k, const double* __restrict__ L,
                           const double* __restrict__ M, double* __restrict__ x, double* __restrict__ ends,
                           double* __restrict__ trans, const double* __restrict__ bnd) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t K = (n + kChunk - 1) / kChunk;
    if (c >= K) return;
    const int64_t st = c * kChunk, en = min(n, st + kChunk);
    const int bb = b * b;
    double prev[kMaxb * kMaxK], cur[kMaxb * kMaxK];
    for (int q = 0; q < b * k; ++q) prev[q] = mode == 1 ? bnd[c * b * k + q] : 0.0;
    for (int64_t s = 0; s < en - st; ++s) {
        const int64_t i = dir == 0 ? st + s : en - 1 - s;
        // the boundary value enters only at the chunk's first step
        sub_step(dir, i, n, b, k, L, M, cur, prev, x);
        if (mode == 1)
            for (int a = 0; a < b; ++a)
                for (int q = 0; q < k; ++q) x[(i * b + a) * k + q] = cur[a * k + q];
        for (int q = 0; q < b * k; ++q) prev[q] = cur[q];
    }
    if (mode == 1) return;
    for (int q = 0; q < b * k; ++q) ends[c * b * k + q] = prev[q];
    // transfer matrix of the homogeneous recurrence across the chunk: forward
    // T = (-M_{en-2}) ... (-M_{st-1}), backward T = (-M_st^T) ... (-M_{en-1}^T)
    double T[kMaxb * kMaxb], P[kMaxb * kMaxb];
    for (int q = 0; q < bb; ++q) T[q] = (q % (b + 1) == 0) ? 1.0 : 0.0;
    for (int64_t s = 0; s < en - st; ++s) {
        const int64_t i = dir == 0 ? st + s : en - 1 - s;
        const bool has = dir == 0 ? i > 0 : i + 1 < n;
        for (int r = 0; r < b; ++r)
            for (int cc = 0; cc < b; ++cc) {
                double acc = 0.0;
                if (has)
                    for (int q = 0; q < b; ++q) {
                        const double m = dir == 0 ? M[(i - 1) * bb + r * b + q] : M[i * bb + q * b + r];
                        acc -= m * T[q * b + cc];
                    }
                P[r * b + cc] = acc;
            }
        for (int q = 0; q < bb; ++q) T[q] = P[q];
    }
    for (int q = 0; q < bb; ++q) trans[c * bb + q] = T[q];
}

// chain the chunk boundaries: bnd[c] = true incoming value of chunk c
__global__ void k_sub_scan(int dir, int64_t n, int b, int k, const double* __restrict__ ends,
                           const double* __restrict__ trans, double* __restrict__ bnd) {
    if (blockIdx.x || threadIdx.x) return;
    const int64_t K = (n + kChunk - 1) / kChunk;
    const int bb = b * b, bk = b * k;
    double v[kMaxb * kMaxK], w[kMaxb * kMaxK];
    for (int q = 0; q < bk; ++q) v[q] = 0.0;
    for (int64_t s = 0; s < K; ++s) {
        const int64_t c = dir == 0 ? s : K - 1 - s;
        for (int q = 0; q < bk; ++q) bnd[c * bk + q] = v[q];
        // exit value of chunk c = local exit + T_c (incoming)
        for (int a = 0; a < b; ++a)
            for (int q = 0; q < k; ++q) {
                double acc = ends[c * bk + a * k + q];
                for (int r = 0; r < b; ++r) acc += trans[c * bb + a * b + r] * v[r * k + q];
                w[a * k + q] = acc;
            }
        for (int q = 0; q < bk; ++q) v[q] = w[q];
    }
}

spingp_ctx* checked_ctx(spingp_ctx* ctx) {
    if (!ctx) throw std::invalid_argument("null context");
    CUDA_OK(cudaSetDevice(ctx->device));
    return ctx;
}

void factor_solve_device(spingp_ctx* ctx, const spingp_btd_factor* f, double* d_x, int k) {
    const int64_t K = (f->n + kChunk - 1) / kChunk;
    const int b = f->b;
    double* ends = ctx->host_io.get(static_cast<size_t>(K) * (2 * b * k + b * b));  // scratch (caller holds mu)
    double* trans = ends + K * b * k;
    double* bnd = trans + K * b * b;
    const unsigned grid = blocks_for(K, 128);
    for (int dir = 0; dir < 2; ++dir) {
        k_sub_pass<<<grid, 128, 0, ctx->stream>>>(dir, 0, f->n, b, k, f->d_L, f->d_M, d_x, ends, trans, nullptr);
        k_sub_scan<<<1, 1, 0, ctx->stream>>>(dir, f->n, b, k, ends, trans, bnd);
        k_sub_pass<<<grid, 128, 0, ctx->stream>>>(dir, 1, f->n, b, k, f->d_L, f->d_M, d_x, ends, trans, bnd);
        ctx->launches += 3;
        CUDA_OK(cudaGetLastError());
    }
}

}  // namespace

extern "C" {

int spingp_btd_factorize(spingp_ctx* ctx, int64_t n, int32_t b, const double* diag, const double* upper,
                         spingp_btd_factor** out, double* logdet, int64_t* fail_block) {
    return guarded(fail_block, [&] {
        checked_ctx(ctx);
        if (!out || !diag || n < 1 || b < 1 || b > kMaxb || (n > 1 && !upper)) throw std::invalid_argument("bad argument");
        *out = nullptr;
        auto* f = new spingp_btd_factor();
        f->device = ctx->device;
        f->n = n;
        f->b = b;
        const size_t bb = static_cast<size_t>(b) * b, nd = n * bb, nu = (n - 1) * bb;
        try {
            double* d_in = nullptr;
            CUDA_OK(cudaMalloc(&f->d_L, (2 * nd + 2 * nu + 1) * sizeof(double)));
            f->d_Cd = f->d_L + nd;
            f->d_M = f->d_Cd + nd;
            f->d_Cu = f->d_M + nu;
            CUDA_OK(cudaMalloc(&d_in, (nd + nu + 1) * sizeof(double)));
            double* d_up = d_in + nd;
            int st;
            {
                std::lock_guard<std::mutex> lk(ctx->mu);
                CUDA_OK(cudaMemcpyAsync(d_in, diag, nd * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
                if (nu) CUDA_OK(cudaMemcpyAsync(d_up, upper, nu * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
            }
            // the partitioned elimination with the selected inverse (one pass)
            double* d_ld = f->d_Cu + nu;
            st = spingp_btd_selinv_device(ctx, n, b, d_in, d_up, f->d_Cd, f->d_Cu, d_ld);
            if (st != SPINGP_OK) throw ApiError{st, -1, spingp_last_error()};
            {
                std::lock_guard<std::mutex> lk(ctx->mu);
                k_factor_blocks<<<blocks_for(n, 64), 64, 0, ctx->stream>>>(n, b, d_up, f->d_Cd, f->d_Cu, f->d_L, f->d_M,
                                                                         ctx->d_status);
                ctx->launched("k_factor_blocks");
                CUDA_OK(cudaMemcpyAsync(&f->logdet, d_ld, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
                st = take_status(ctx, fail_block);
            }
            cudaFree(d_in);
            if (st != SPINGP_OK) throw ApiError{st, fail_block ? *fail_block : -1, spingp_last_error()};
        } catch (...) {
            spingp_btd_factor_destroy(f);
            throw;
        }
        if (logdet) *logdet = f->logdet;
        *out = f;
        return SPINGP_OK;
    });
}

int spingp_btd_factor_destroy(spingp_btd_factor* f) {
    if (!f) return SPINGP_OK;
    cudaSetDevice(f->device);
    if (f->d_L) cudaFree(f->d_L);
    delete f;
    return SPINGP_OK;
}

int spingp_btd_factor_info(const spingp_btd_factor* f, int64_t* n, int32_t* b, double* logdet) {
    if (!f) return SPINGP_BAD_ARG;
    if (n) *n = f->n;
    if (b) *b = f->b;
    if (logdet) *logdet = f->logdet;
    return SPINGP_OK;
}

int spingp_btd_factor_blocks(spingp_ctx* ctx, const spingp_btd_factor* f, double* L, double* M) {
    return guarded(nullptr, [&] {
        checked_ctx(ctx);
        if (!f) throw std::invalid_argument("null factor");
        const size_t bb = static_cast<size_t>(f->b) * f->b;
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (L) CUDA_OK(cudaMemcpyAsync(L, f->d_L, f->n * bb * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (M && f->n > 1)
            CUDA_OK(cudaMemcpyAsync(M, f->d_M, (f->n - 1) * bb * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_OK(cudaStreamSynchronize(ctx->stream));
        return SPINGP_OK;
    });
}

int spingp_btd_factor_solve(spingp_ctx* ctx, const spingp_btd_factor* f, const double* rhs, int32_t k, double* x) {
    return guarded(nullptr, [&] {
        checked_ctx(ctx);
        if (!f || !rhs || !x || k < 1) throw std::invalid_argument("bad argument");
        const size_t nr = static_cast<size_t>(f->n) * f->b * k;
        double* d_x = nullptr;
        CUDA_OK(cudaMalloc(&d_x, nr * sizeof(double)));
        std::lock_guard<std::mutex> lk(ctx->mu);
        CUDA_OK(cudaMemcpyAsync(d_x, rhs, nr * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        for (int c0 = 0; c0 < k; c0 += kMaxK) {  // k columns in groups of kMaxK, one pass each
            const int kk = std::min(kMaxK, k - c0);
            if (kk == k) {
                factor_solve_device(ctx, f, d_x, k);
            } else {  // strided column groups: solve a packed copy
                std::vector<double> h(nr), g(static_cast<size_t>(f->n) * f->b * kk);
                CUDA_OK(cudaMemcpyAsync(h.data(), d_x, nr * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
                CUDA_OK(cudaStreamSynchronize(ctx->stream));
                for (size_t r = 0; r < static_cast<size_t>(f->n) * f->b; ++r)
                    for (int c = 0; c < kk; ++c) g[r * kk + c] = h[r * k + c0 + c];
                double* d_g = nullptr;
                CUDA_OK(cudaMalloc(&d_g, g.size() * sizeof(double)));
                CUDA_OK(cudaMemcpyAsync(d_g, g.data(), g.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
                factor_solve_device(ctx, f, d_g, kk);
                CUDA_OK(cudaMemcpyAsync(g.data(), d_g, g.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
                CUDA_OK(cudaStreamSynchronize(ctx->stream));
                cudaFree(d_g);
                for (size_t r = 0; r < static_cast<size_t>(f->n) * f->b; ++r)
                    for (int c = 0; c < kk; ++c) x[r * k + c0 + c] = g[r * kk + c];
            }
        }
        if (k <= kMaxK) CUDA_OK(cudaMemcpyAsync(x, d_x, nr * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_OK(cudaStreamSynchronize(ctx->stream));
        cudaFree(d_x);
        return SPINGP_OK;
    });
}

int spingp_btd_factor_selinv(spingp_ctx* ctx, const spingp_btd_factor* f, double* cdiag, double* cupper) {
    return guarded(nullptr, [&] {
        checked_ctx(ctx);
        if (!f || !cdiag) throw std::invalid_argument("bad argument");
        const size_t bb = static_cast<size_t>(f->b) * f->b;
        std::lock_guard<std::mutex> lk(ctx->mu);
        CUDA_OK(cudaMemcpyAsync(cdiag, f->d_Cd, f->n * bb * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        if (cupper && f->n > 1)
            CUDA_OK(cudaMemcpyAsync(cupper, f->d_Cu, (f->n - 1) * bb * sizeof(double), cudaMemcpyDeviceToHost,
                                    ctx->stream));
        CUDA_OK(cudaStreamSynchronize(ctx->stream));
        return SPINGP_OK;
    });
}

}  // extern "C"
