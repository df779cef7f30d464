#pragma once
// btd_core — symmetric block-tridiagonal algebra, drop-in C++ API
// backed by the B200 kernels through the C ABI (include/spingp_c.h).
//
//   SymBTD                 SPEC.md:129-134 (storage SPEC.md:220)
//   BTDFactor / factorize  SPEC.md:135-151   (device partitioned LDL^T; cached logdet)
//   solve
//   logdet
//   selective_inverse
//   trace_btd_product
//   matvec
//   cr_solve
// Errors: NotPositiveDefinite(block) for a failed pivot, std::invalid_argument for
// dimension mismatches, DeviceError for CUDA failures.
//
// Link with paper_1610_08035_b200/libspingp_b200.so.

#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "spingp/errors.hpp"
#include "spingp/matrix.hpp"
#include "spingp_c.h"

namespace spingp {

// A CUDA device context (device, stream, workspace).  One per host thread.
class Device {
public:
    explicit Device(int device = 0) {
        spingp_ctx* c = nullptr;
        check(spingp_ctx_create(device, &c), -1);
        ctx_.reset(c);
    }
    spingp_ctx* get() const { return ctx_.get(); }

    // Translate a C-ABI status into the reference exception hierarchy (errors.hpp).
    static void check(int st, int64_t block) {
        if (st == SPINGP_OK) return;
        const char* msg = spingp_last_error();
        switch (st) {
            case SPINGP_NOT_PD: throw NotPositiveDefinite(msg, static_cast<std::ptrdiff_t>(block));
            case SPINGP_SINGULAR_Q: throw SingularProcessNoise(msg, static_cast<std::ptrdiff_t>(block));
            case SPINGP_DUPLICATE_TIME: throw DuplicateTimestamp(msg);
            case SPINGP_BAD_ARG: throw std::invalid_argument(msg);
            default: throw DeviceError(std::string(spingp_status_string(st)) + ": " + msg);
        }
    }

private:
    struct Del {
        void operator()(spingp_ctx* c) const { spingp_ctx_destroy(c); }
    };
    std::unique_ptr<spingp_ctx, Del> ctx_;
};

// Several devices of one box joined by NCCL (spingp_mctx_create): the engine functions
// taking a MultiDevice partition one long series into contiguous time segments, one per
// device (spingp_eval_partitioned).
class MultiDevice {
public:
    explicit MultiDevice(const std::vector<int>& devices) {
        std::vector<int32_t> ids(devices.begin(), devices.end());
        spingp_mctx* m = nullptr;
        Device::check(spingp_mctx_create(static_cast<int32_t>(ids.size()), ids.data(), &m), -1);
        m_.reset(m);
    }
    spingp_mctx* get() const { return m_.get(); }
    int size() const { return spingp_mctx_size(m_.get()); }

private:
    struct Del {
        void operator()(spingp_mctx* m) const { spingp_mctx_destroy(m); }
    };
    std::unique_ptr<spingp_mctx, Del> m_;
};

// Per-thread default device (cuda:0), created on first use.
inline Device& default_device() {
    thread_local Device d(0);
    return d;
}

struct SymBTD {
    Index n_blocks = 0;
    Index block_dim = 0;
    std::vector<Matrix> diag;   // n b x b
    std::vector<Matrix> upper;  // n-1 b x b, (i, i+1) blocks

    SymBTD() = default;
    SymBTD(Index n, Index b)
        : n_blocks(n), block_dim(b), diag(static_cast<size_t>(n), Matrix(b, b)),
          upper(static_cast<size_t>(n > 0 ? n - 1 : 0), Matrix(b, b)) {}
};

namespace detail {
inline void pack(const SymBTD& m, std::vector<double>& d, std::vector<double>& u) {
    const Index n = m.n_blocks, b = m.block_dim;
    if (n < 1 || b < 1 || static_cast<Index>(m.diag.size()) != n ||
        static_cast<Index>(m.upper.size()) != (n > 0 ? n - 1 : 0))
        throw std::invalid_argument("SymBTD: inconsistent dimensions");
    d.resize(static_cast<size_t>(n * b * b));
    u.resize(static_cast<size_t>((n - 1) * b * b));
    for (Index i = 0; i < n; ++i) {
        if (m.diag[i].rows() != b || m.diag[i].cols() != b) throw std::invalid_argument("SymBTD: block size");
        std::copy(m.diag[i].data(), m.diag[i].data() + b * b, d.begin() + i * b * b);
    }
    for (Index i = 0; i + 1 < n; ++i) {
        if (m.upper[i].rows() != b || m.upper[i].cols() != b) throw std::invalid_argument("SymBTD: block size");
        std::copy(m.upper[i].data(), m.upper[i].data() + b * b, u.begin() + i * b * b);
    }
}
}  // namespace detail

// The factor of a SymBTD: pivot Cholesky factors L_i (lower, positive
// diagonal), multipliers M_i = U_i^T S_i^{-1}, the cached log-determinant — and the
// device-resident factor they were read from (spingp_btd_factorize), which solve and
// selective_inverse reuse without re-factorising.
struct BTDFactor {
    Index n_blocks = 0;
    Index block_dim = 0;
    std::vector<Matrix> L;  // n
    std::vector<Matrix> M;  // n - 1
    double logdet = 0.0;
    std::shared_ptr<spingp_btd_factor> device;
};

inline BTDFactor factorize(const SymBTD& m, Device& dev = default_device()) {
    std::vector<double> d, u;
    detail::pack(m, d, u);
    const Index n = m.n_blocks, b = m.block_dim;
    spingp_btd_factor* raw = nullptr;
    BTDFactor f;
    int64_t fb = -1;
    // status first, then the failing block it set (argument evaluation order is unspecified)
    const int st_ = spingp_btd_factorize(dev.get(), n, static_cast<int32_t>(b), d.data(), n > 1 ? u.data() : nullptr,
                                         &raw, &f.logdet, &fb);
    Device::check(st_, fb);
    f.device.reset(raw, [](spingp_btd_factor* p) { spingp_btd_factor_destroy(p); });
    f.n_blocks = n;
    f.block_dim = b;
    std::vector<double> L(static_cast<size_t>(n * b * b)), M(static_cast<size_t>((n - 1) * b * b));
    Device::check(spingp_btd_factor_blocks(dev.get(), raw, L.data(), n > 1 ? M.data() : nullptr), -1);
    f.L.assign(static_cast<size_t>(n), Matrix(b, b));
    f.M.assign(static_cast<size_t>(n - 1), Matrix(b, b));
    for (Index i = 0; i < n; ++i) std::copy(L.begin() + i * b * b, L.begin() + (i + 1) * b * b, f.L[i].data());
    for (Index i = 0; i + 1 < n; ++i) std::copy(M.begin() + i * b * b, M.begin() + (i + 1) * b * b, f.M[i].data());
    return f;
}

inline double logdet(const BTDFactor& f) { return f.logdet; }

// X = M^{-1} rhs for an (n b) x k right-hand side, from the kept factor.
inline Matrix solve(const BTDFactor& f, const Matrix& rhs, Device& dev = default_device()) {
    if (!f.device) throw std::invalid_argument("solve: factor has no device state (use factorize)");
    if (rhs.rows() != f.n_blocks * f.block_dim) throw std::invalid_argument("solve: rhs row count must be n*b");
    Matrix x(rhs.rows(), rhs.cols());
    Device::check(spingp_btd_factor_solve(dev.get(), f.device.get(), rhs.data(), static_cast<int32_t>(rhs.cols()),
                                          x.data()),
                  -1);
    return x;
}

struct CrSolveResult {
    Matrix x;
    double logdet;
};

// cr_solve: one partitioned-elimination pass gives x and log det.
inline CrSolveResult cr_solve(const SymBTD& m, const Matrix& rhs, Device& dev = default_device()) {
    const Index n = m.n_blocks, b = m.block_dim;
    if (rhs.rows() != n * b) throw std::invalid_argument("cr_solve: rhs row count must be n*b");
    std::vector<double> d, u;
    detail::pack(m, d, u);
    CrSolveResult r{Matrix(rhs.rows(), rhs.cols()), 0.0};
    int64_t fb = -1;
    const int st_ = spingp_btd_cr_solve(dev.get(), n, static_cast<int32_t>(b), d.data(), u.data(), rhs.data(),
                                        static_cast<int32_t>(rhs.cols()), r.x.data(), &r.logdet, &fb);
    Device::check(st_, fb);
    return r;
}

// The BTD-pattern blocks of M^{-1}, kept by factorize.
inline SymBTD selective_inverse(const BTDFactor& f, Device& dev = default_device()) {
    if (!f.device) throw std::invalid_argument("selective_inverse: factor has no device state (use factorize)");
    const Index n = f.n_blocks, b = f.block_dim;
    std::vector<double> cd(static_cast<size_t>(n * b * b)), cu(static_cast<size_t>((n - 1) * b * b));
    Device::check(spingp_btd_factor_selinv(dev.get(), f.device.get(), cd.data(), n > 1 ? cu.data() : nullptr), -1);
    SymBTD out(n, b);
    for (Index i = 0; i < n; ++i) std::copy(cd.begin() + i * b * b, cd.begin() + (i + 1) * b * b, out.diag[i].data());
    for (Index i = 0; i + 1 < n; ++i)
        std::copy(cu.begin() + i * b * b, cu.begin() + (i + 1) * b * b, out.upper[i].data());
    return out;
}

// Tr(S M) from the BTD blocks only.
inline double trace_btd_product(const SymBTD& s, const SymBTD& m) {
    if (s.n_blocks != m.n_blocks || s.block_dim != m.block_dim)
        throw std::invalid_argument("trace_btd_product: dimension mismatch");
    double tr = 0.0;
    for (Index i = 0; i < s.n_blocks; ++i) tr += (s.diag[i] * m.diag[i]).trace();
    for (Index i = 0; i + 1 < s.n_blocks; ++i) tr += 2.0 * (s.upper[i].transpose() * m.upper[i]).trace();
    return tr;
}

inline Matrix matvec(const SymBTD& m, const Matrix& v, Device& dev = default_device()) {
    const Index n = m.n_blocks, b = m.block_dim;
    if (v.size() != n * b) throw std::invalid_argument("matvec: length mismatch");
    std::vector<double> d, u;
    detail::pack(m, d, u);
    Matrix out(v.rows(), v.cols());
    const int st_ = spingp_btd_matvec(dev.get(), n, static_cast<int32_t>(b), d.data(), u.data(), v.data(), out.data());
    Device::check(st_, -1);
    return out;
}

}  // namespace spingp
