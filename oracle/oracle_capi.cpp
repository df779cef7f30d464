// oracle_capi.cpp — extern "C" surface of the CPU oracle (TEST INFRASTRUCTURE ONLY).
//
// Loaded through ctypes by tests/ and by bench.py's CPU-baseline leg only.  The
// product library never links this.  Every entry point takes `precision`:
// 0 = IEEE double (the restatement proper), 1 = x87 long double (arbiter).
#include <chrono>
#include <cstdio>

#include "spingp_oracle.hpp"

using oracle::Failure;
using oracle::Leaf;
using oracle::Mat;

namespace {

thread_local char g_err[512];

template <class F>
int guarded(int64_t* fail_block, F&& body) {
    if (fail_block) *fail_block = -1;
    try {
        body();
        return 0;
    } catch (const Failure& f) {
        if (fail_block) *fail_block = f.block;
        std::snprintf(g_err, sizeof g_err, "%s", f.what.c_str());
        return f.status;
    } catch (const std::invalid_argument& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return oracle::BAD_ARG;
    } catch (const std::exception& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return oracle::UNSUPPORTED;
    }
}

std::vector<Leaf> leaves_of(const int32_t* lv, int32_t nl) {
    std::vector<Leaf> v;
    for (int i = 0; i < nl; ++i) v.push_back({lv[2 * i], lv[2 * i + 1]});
    return v;
}

template <class R>
std::vector<R> vec_of(const double* p, int64_t n) {
    std::vector<R> v(n);
    for (int64_t i = 0; i < n; ++i) v[i] = R(p[i]);
    return v;
}

template <class R>
void put(const Mat<R>& m, double* out) {
    if (!out) return;
    for (size_t i = 0; i < m.a.size(); ++i) out[i] = static_cast<double>(m.a[i]);
}

template <class R>
Mat<R> mat_of(const double* p, int r, int c) {
    Mat<R> m(r, c);
    for (int i = 0; i < r * c; ++i) m.a[i] = R(p[i]);
    return m;
}

template <class R>
oracle::SymBTD<R> btd_of(int64_t n, int b, const double* diag, const double* upper) {
    oracle::SymBTD<R> m;
    m.n = n;
    m.b = b;
    for (int64_t i = 0; i < n; ++i) m.diag.push_back(mat_of<R>(diag + i * b * b, b, b));
    for (int64_t i = 0; i + 1 < n; ++i) m.upper.push_back(mat_of<R>(upper + i * b * b, b, b));
    return m;
}

template <class R>
void state_space_impl(const int32_t* lv, int32_t nl, const double* theta, int32_t nt, double* F,
                      double* H, double* Pinf, double* dF, double* dPinf, int32_t* fconst) {
    const auto m = oracle::state_space_of<R>(leaves_of(lv, nl), vec_of<R>(theta, nt));
    const int b = m.b;
    put(m.F, F);
    put(m.Pinf, Pinf);
    if (H)
        for (int i = 0; i < b; ++i) H[i] = static_cast<double>(m.H[i]);
    for (int p = 0; p < m.ntheta(); ++p) {
        if (dF) put(m.dF[p], dF + static_cast<size_t>(p) * b * b);
        if (dPinf) put(m.dPinf[p], dPinf + static_cast<size_t>(p) * b * b);
        if (fconst) fconst[p] = m.fconst[p];
    }
}

template <class R>
void discretize_impl(const int32_t* lv, int32_t nl, const double* theta, int32_t nt, double dt,
                     int grad, double* Phi, double* Q, double* dPhi, double* dQ) {
    const auto m = oracle::state_space_of<R>(leaves_of(lv, nl), vec_of<R>(theta, nt));
    const auto st = oracle::discretize(m, R(dt), grad != 0);
    put(st.Phi, Phi);
    put(st.Q, Q);
    const int b = m.b;
    if (grad)
        for (int p = 0; p < m.ntheta(); ++p) {
            put(st.dPhi[p], dPhi ? dPhi + static_cast<size_t>(p) * b * b : nullptr);
            put(st.dQ[p], dQ ? dQ + static_cast<size_t>(p) * b * b : nullptr);
        }
}

template <class R>
void eval_impl(const int32_t* lv, int32_t nl, const double* theta, int32_t nt, const double* t,
               const double* y, int64_t n, double sigma, uint32_t flags, double* loglik,
               double* grad, double* mean, double* var, double* diag4, int threads) {
    const auto m = oracle::state_space_of<R>(leaves_of(lv, nl), vec_of<R>(theta, nt));
    oracle::EvalFlags fl;
    fl.grad = flags & 1u;
    fl.mean = flags & 2u;
    fl.var = flags & 4u;
    fl.include_noise = flags & 8u;
    const auto out = oracle::evaluate(m, t, y, n, R(sigma), fl, threads);
    if (loglik) *loglik = static_cast<double>(out.loglik);
    if (grad && fl.grad)
        for (size_t i = 0; i < out.grad.size(); ++i) grad[i] = static_cast<double>(out.grad[i]);
    if (mean && fl.mean)
        for (int64_t i = 0; i < n; ++i) mean[i] = static_cast<double>(out.mean[i]);
    if (var && fl.var)
        for (int64_t i = 0; i < n; ++i) var[i] = static_cast<double>(out.var[i]);
    if (diag4) {
        diag4[0] = static_cast<double>(out.logdetP);
        diag4[1] = static_cast<double>(out.logdetQ);
        diag4[2] = static_cast<double>(out.fit_y);
        diag4[3] = static_cast<double>(out.fit_e);
    }
}

template <class R>
void assemble_impl(const int32_t* lv, int32_t nl, const double* theta, int32_t nt,
                   const double* t, const double* y, int64_t n, double sigma, double* diag,
                   double* upper, double* rhs, int threads) {
    const auto m = oracle::state_space_of<R>(leaves_of(lv, nl), vec_of<R>(theta, nt));
    oracle::check_times<R>(t, n);
    const auto d = oracle::discretise_all(m, t, n, false, threads);
    const auto P = oracle::assemble(m, d, n, R(sigma), nullptr, threads);
    const int b = m.b;
    for (int64_t i = 0; i < n; ++i) put(P.diag[i], diag + i * b * b);
    for (int64_t i = 0; i + 1 < n; ++i) put(P.upper[i], upper + i * b * b);
    if (rhs)
        for (int64_t i = 0; i < n; ++i)
            for (int a = 0; a < b; ++a)
                rhs[i * b + a] = static_cast<double>(m.H[a] * R(y[i]) / (R(sigma) * R(sigma)));
}

template <class R>
void btd_solve_impl(int64_t n, int b, const double* diag, const double* upper, const double* rhs,
                    int k, double* x, double* logdet) {
    const auto M = btd_of<R>(n, b, diag, upper);
    const auto f = oracle::thomas_factor(M);
    if (logdet) *logdet = static_cast<double>(f.logdet);
    if (rhs && x) {
        std::vector<Mat<R>> z;
        for (int64_t i = 0; i < n; ++i) z.push_back(mat_of<R>(rhs + i * b * k, b, k));
        z = oracle::thomas_solve(M, f, z);
        for (int64_t i = 0; i < n; ++i) put(z[i], x + i * b * k);
    }
}

template <class R>
void btd_selinv_impl(int64_t n, int b, const double* diag, const double* upper, double* cdiag,
                     double* cupper, double* logdet) {
    const auto M = btd_of<R>(n, b, diag, upper);
    const auto f = oracle::thomas_factor(M);
    std::vector<Mat<R>> Cd, Cu;
    oracle::takahashi(M, f, Cd, Cu);
    if (logdet) *logdet = static_cast<double>(f.logdet);
    for (int64_t i = 0; i < n; ++i) put(Cd[i], cdiag + i * b * b);
    for (int64_t i = 0; i + 1 < n; ++i) put(Cu[i], cupper + i * b * b);
}

}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err; }

int oracle_state_space(const int32_t* leaves, int32_t n_leaves, const double* theta,
                       int32_t n_theta, double* F, double* H, double* Pinf, double* dF,
                       double* dPinf, int32_t* fconst, int32_t* b_out, int precision) {
    return guarded(nullptr, [&] {
        int b = 0;
        for (int i = 0; i < n_leaves; ++i) b += oracle::leaf_dim({leaves[2 * i], leaves[2 * i + 1]});
        if (b_out) *b_out = b;
        if (!F && !H && !Pinf && !dF && !dPinf && !fconst) return;
        if (precision) state_space_impl<long double>(leaves, n_leaves, theta, n_theta, F, H, Pinf, dF, dPinf, fconst);
        else state_space_impl<double>(leaves, n_leaves, theta, n_theta, F, H, Pinf, dF, dPinf, fconst);
    });
}

int oracle_discretize(const int32_t* leaves, int32_t n_leaves, const double* theta,
                      int32_t n_theta, double dt, int grad, double* Phi, double* Q, double* dPhi,
                      double* dQ, int precision) {
    return guarded(nullptr, [&] {
        if (precision) discretize_impl<long double>(leaves, n_leaves, theta, n_theta, dt, grad, Phi, Q, dPhi, dQ);
        else discretize_impl<double>(leaves, n_leaves, theta, n_theta, dt, grad, Phi, Q, dPhi, dQ);
    });
}

double oracle_implied_covariance(const int32_t* leaves, int32_t n_leaves, const double* theta,
                                 int32_t n_theta, double tau) {
    double out = 0;
    guarded(nullptr, [&] {
        const auto m = oracle::state_space_of<double>(leaves_of(leaves, n_leaves),
                                                      vec_of<double>(theta, n_theta));
        out = oracle::implied_covariance(m, tau);
    });
    return out;
}

int oracle_eval(const int32_t* leaves, int32_t n_leaves, const double* theta, int32_t n_theta,
                const double* t, const double* y, int64_t n, double sigma, uint32_t flags,
                double* loglik, double* grad, double* mean, double* var, double* diag4,
                int64_t* fail_block, int precision, int threads) {
    return guarded(fail_block, [&] {
        if (precision) eval_impl<long double>(leaves, n_leaves, theta, n_theta, t, y, n, sigma, flags, loglik, grad, mean, var, diag4, threads);
        else eval_impl<double>(leaves, n_leaves, theta, n_theta, t, y, n, sigma, flags, loglik, grad, mean, var, diag4, threads);
    });
}

// Batched: S independent series (series-parallel over `threads`).  Each series is
// evaluated sequentially (the reference algorithm); series are independent units.
int oracle_eval_batched(const int32_t* leaves, int32_t n_leaves, const double* theta,
                        int32_t n_theta, int64_t S, int64_t n, const double* t, const double* y,
                        const double* sigma, uint32_t flags, double* loglik, double* grad,
                        int64_t* fail_series, int precision, int threads) {
    std::vector<int> st(S, 0);
    oracle::parallel_for(S, threads, [&](int64_t lo, int64_t hi) {
        for (int64_t s = lo; s < hi; ++s) {
            int64_t fb;
            st[s] = oracle_eval(leaves, n_leaves, theta + s * n_theta, n_theta, t + s * n,
                                y + s * n, n, sigma[s], flags & 1u, loglik + s,
                                grad ? grad + s * (n_theta + 1) : nullptr, nullptr, nullptr,
                                nullptr, &fb, precision, 1);
        }
    });
    if (fail_series) *fail_series = -1;
    for (int64_t s = 0; s < S; ++s)
        if (st[s]) {
            if (fail_series) *fail_series = s;
            return st[s];
        }
    return 0;
}

int oracle_assemble(const int32_t* leaves, int32_t n_leaves, const double* theta,
                    int32_t n_theta, const double* t, const double* y, int64_t n, double sigma,
                    double* diag, double* upper, double* rhs, int64_t* fail_block, int precision,
                    int threads) {
    return guarded(fail_block, [&] {
        if (precision) assemble_impl<long double>(leaves, n_leaves, theta, n_theta, t, y, n, sigma, diag, upper, rhs, threads);
        else assemble_impl<double>(leaves, n_leaves, theta, n_theta, t, y, n, sigma, diag, upper, rhs, threads);
    });
}

int oracle_btd_solve(int64_t n, int32_t b, const double* diag, const double* upper,
                     const double* rhs, int32_t k, double* x, double* logdet,
                     int64_t* fail_block, int precision) {
    return guarded(fail_block, [&] {
        if (n < 1 || b < 1) throw std::invalid_argument("empty BTD");
        if (precision) btd_solve_impl<long double>(n, b, diag, upper, rhs, k, x, logdet);
        else btd_solve_impl<double>(n, b, diag, upper, rhs, k, x, logdet);
    });
}

int oracle_btd_selinv(int64_t n, int32_t b, const double* diag, const double* upper,
                      double* cdiag, double* cupper, double* logdet, int64_t* fail_block,
                      int precision) {
    return guarded(fail_block, [&] {
        if (n < 1 || b < 1) throw std::invalid_argument("empty BTD");
        if (precision) btd_selinv_impl<long double>(n, b, diag, upper, cdiag, cupper, logdet);
        else btd_selinv_impl<double>(n, b, diag, upper, cdiag, cupper, logdet);
    });
}

// expm through the oracle's Padé path (for the ported reference tests).
// Kalman filter + RTS smoother over a (merged, observation-masked) grid: SPEC.md:379-396.
int oracle_kf_rts(const int32_t* leaves, int32_t n_leaves, const double* theta, int32_t n_theta,
                  const double* t, const double* y, const unsigned char* observed, int64_t n, double sigma,
                  double* loglik, double* mean, double* var, double* fvar, int64_t* fail_block, int precision) {
    return guarded(fail_block, [&] {
        auto run = [&](auto tag) {
            using R = decltype(tag);
            oracle::check_times<R>(t, n);
            const auto m = oracle::state_space_of<R>(leaves_of(leaves, n_leaves), vec_of<R>(theta, n_theta));
            const auto o = oracle::kf_rts(m, t, y, observed, n, R(sigma));
            if (loglik) *loglik = static_cast<double>(o.loglik);
            for (int64_t i = 0; i < n; ++i) {
                if (mean) mean[i] = static_cast<double>(o.mean[i]);
                if (var) var[i] = static_cast<double>(o.var[i]);
                if (fvar) fvar[i] = static_cast<double>(o.fvar[i]);
            }
        };
        if (precision) run((long double)0);
        else run(0.0);
    });
}

int oracle_expm(int32_t b, const double* A, double* out, int precision) {
    return guarded(nullptr, [&] {
        if (precision) put(oracle::expm(mat_of<long double>(A, b, b)), out);
        else put(oracle::expm(mat_of<double>(A, b, b)), out);
    });
}

}  // extern "C"
