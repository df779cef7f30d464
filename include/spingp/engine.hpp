#pragma once
// spingp_engine — marginal likelihood, gradient and training-point posterior
// (SPEC.md:236-344), drop-in C++ API over the fused B200 evaluation
// (spingp_eval in include/spingp_c.h).
//
//   Dataset, NoiseModel, PosteriorSummary
//   assemble_prior_precision                   SPEC.md:262-270 (Q_0 := Pinf :326, jitter :328)
//   add_observation_term
//   log_marginal_likelihood
//   mll_gradient                               SPEC.md:289-297 (raw θ, then ∂/∂σ_n, σ_n = std-dev)
//   predict (at the training times)            SPEC.md:298-306 (clamp :329)
//   predict (at arbitrary test times)          SPEC.md:298-306, nudge :327 (spingp_predict)
//   optimize_hyperparameters                   SPEC.md:307-315 (spingp/optimize.hpp)

#include <cmath>
#include <limits>
#include <vector>

#include "spingp/btd.hpp"
#include "spingp/kernels.hpp"

namespace spingp {

struct Dataset {
    std::vector<double> times;   // strictly increasing
    std::vector<double> values;
};

struct NoiseModel {
    double sigma_n2 = 1.0;  // observation noise variance σ_n²
};

struct PosteriorSummary {
    std::vector<double> times;
    std::vector<double> mean;
    std::vector<double> variance;
    double mll = 0.0;
    std::vector<double> mll_grad;  // per kernel hyperparameter, then σ_n
};

namespace detail {

inline std::vector<spingp_leaf> leaves_of(const KernelSpec& spec) {
    std::vector<spingp_leaf> out;
    for (const KernelSpec* l : kernel_leaves(spec)) {
        spingp_leaf lf{0, l->order};
        switch (l->type) {
            case KernelType::Matern12: lf.type = SPINGP_MATERN12; break;
            case KernelType::Matern32: lf.type = SPINGP_MATERN32; break;
            case KernelType::Matern52: lf.type = SPINGP_MATERN52; break;
            case KernelType::EQApprox: lf.type = SPINGP_EQ; break;
            case KernelType::QuasiPeriodic: lf.type = SPINGP_QP; break;
            default: throw std::invalid_argument("unknown kernel variant");
        }
        out.push_back(lf);
    }
    return out;
}

inline void check_data(const Dataset& d, const NoiseModel& noise) {
    if (d.times.empty() || d.times.size() != d.values.size())
        throw std::invalid_argument("dataset: need N >= 1 equal-length times and values");
    if (!(noise.sigma_n2 > 0.0)) throw std::invalid_argument("noise variance must be positive");
}

struct EvalOut {
    double loglik = 0.0;
    std::vector<double> grad, mean, var;
};

inline EvalOut eval(const Dataset& d, const KernelSpec& spec, const HyperparameterSet& theta,
                    const NoiseModel& noise, uint32_t flags, Device& dev) {
    check_data(d, noise);
    const auto lv = leaves_of(spec);
    EvalOut o;
    const size_t n = d.times.size();
    if (flags & SPINGP_WANT_GRAD) o.grad.resize(theta.size() + 1);
    if (flags & SPINGP_WANT_MEAN) o.mean.resize(n);
    if (flags & SPINGP_WANT_VAR) o.var.resize(n);
    int64_t fb = -1;
    const int st_ = spingp_eval(dev.get(), lv.data(), static_cast<int32_t>(lv.size()), theta.data(),
                              static_cast<int32_t>(theta.size()), d.times.data(), d.values.data(),
                              static_cast<int64_t>(n), std::sqrt(noise.sigma_n2), flags, &o.loglik,
                              o.grad.empty() ? nullptr : o.grad.data(), o.mean.empty() ? nullptr : o.mean.data(),
                              o.var.empty() ? nullptr : o.var.data(), &fb);
    Device::check(st_, fb);
    return o;
}

// the same evaluation partitioned over the devices of a MultiDevice (spingp_eval_partitioned)
inline EvalOut eval(const Dataset& d, const KernelSpec& spec, const HyperparameterSet& theta,
                    const NoiseModel& noise, uint32_t flags, MultiDevice& md) {
    check_data(d, noise);
    const auto lv = leaves_of(spec);
    EvalOut o;
    const size_t n = d.times.size();
    if (flags & SPINGP_WANT_GRAD) o.grad.resize(theta.size() + 1);
    if (flags & SPINGP_WANT_MEAN) o.mean.resize(n);
    if (flags & SPINGP_WANT_VAR) o.var.resize(n);
    int64_t fb = -1;
    const int st_ = spingp_eval_partitioned(md.get(), lv.data(), static_cast<int32_t>(lv.size()), theta.data(),
                                            static_cast<int32_t>(theta.size()), d.times.data(), d.values.data(),
                                            static_cast<int64_t>(n), std::sqrt(noise.sigma_n2), flags, &o.loglik,
                                            o.grad.empty() ? nullptr : o.grad.data(),
                                            o.mean.empty() ? nullptr : o.mean.data(),
                                            o.var.empty() ? nullptr : o.var.data(), &fb);
    Device::check(st_, fb);
    return o;
}
}  // namespace detail

// Multi-GPU overloads: one long series partitioned over the devices.
inline double log_marginal_likelihood(const Dataset& data, const KernelSpec& spec, const HyperparameterSet& theta,
                                      const NoiseModel& noise, MultiDevice& md) {
    return detail::eval(data, spec, theta, noise, 0u, md).loglik;
}
inline std::vector<double> mll_gradient(const Dataset& data, const KernelSpec& spec, const HyperparameterSet& theta,
                                        const NoiseModel& noise, MultiDevice& md) {
    return detail::eval(data, spec, theta, noise, SPINGP_WANT_GRAD, md).grad;
}
inline PosteriorSummary predict(const Dataset& data, const KernelSpec& spec, const HyperparameterSet& theta,
                                const NoiseModel& noise, MultiDevice& md) {
    auto o = detail::eval(data, spec, theta, noise, SPINGP_WANT_GRAD | SPINGP_WANT_MEAN | SPINGP_WANT_VAR, md);
    PosteriorSummary p;
    p.times = data.times;
    p.mean = std::move(o.mean);
    p.variance = std::move(o.var);
    p.mll = o.loglik;
    p.mll_grad = std::move(o.grad);
    return p;
}

// 𝒦^{-1}: the prior precision over the N state blocks (no observation term).
inline SymBTD assemble_prior_precision(const std::vector<double>& times, const KernelSpec& spec,
                                       const HyperparameterSet& theta, Device& dev = default_device()) {
    const auto lv = detail::leaves_of(spec);
    int32_t b = 0, nt = 0;
    Device::check(spingp_kernel_dims(lv.data(), static_cast<int32_t>(lv.size()), &b, &nt), -1);
    const int64_t n = static_cast<int64_t>(times.size());
    if (n < 1) throw std::invalid_argument("need at least one time");
    std::vector<double> d(static_cast<size_t>(n) * b * b), u(static_cast<size_t>(n - 1) * b * b), y(n, 0.0);
    int64_t fb = -1;
    const int st_ = spingp_assemble(dev.get(), lv.data(), static_cast<int32_t>(lv.size()), theta.data(),
                                  static_cast<int32_t>(theta.size()), times.data(), y.data(), n,
                                  std::numeric_limits<double>::infinity(), d.data(), n > 1 ? u.data() : nullptr,
                                  nullptr, &fb);
    Device::check(st_, fb);
    SymBTD m(n, b);
    for (int64_t i = 0; i < n; ++i) std::copy(d.begin() + i * b * b, d.begin() + (i + 1) * b * b, m.diag[i].data());
    for (int64_t i = 0; i + 1 < n; ++i) std::copy(u.begin() + i * b * b, u.begin() + (i + 1) * b * b, m.upper[i].data());
    return m;
}

// diag_i += H^T H / σ_n² for every observed block.
inline SymBTD add_observation_term(SymBTD prior, const StateSpaceModel& ssm, const NoiseModel& noise,
                                   const std::vector<bool>& observed) {
    if (static_cast<Index>(observed.size()) != prior.n_blocks) throw std::invalid_argument("mask length");
    const Index b = prior.block_dim;
    for (Index i = 0; i < prior.n_blocks; ++i)
        if (observed[static_cast<size_t>(i)])
            for (Index a = 0; a < b; ++a)
                for (Index c = 0; c < b; ++c) prior.diag[i](a, c) += ssm.H(a) * ssm.H(c) / noise.sigma_n2;
    return prior;
}

inline double log_marginal_likelihood(const Dataset& data, const KernelSpec& spec,
                                      const HyperparameterSet& theta, const NoiseModel& noise,
                                      Device& dev = default_device()) {
    return detail::eval(data, spec, theta, noise, 0u, dev).loglik;
}

// d MLL / d(θ..., σ_n) in raw parameters (σ_n the noise standard deviation).
inline std::vector<double> mll_gradient(const Dataset& data, const KernelSpec& spec,
                                        const HyperparameterSet& theta, const NoiseModel& noise,
                                        Device& dev = default_device()) {
    return detail::eval(data, spec, theta, noise, SPINGP_WANT_GRAD, dev).grad;
}

// Posterior at the training times (SPEC.md:298-306 restricted to test = train).
inline PosteriorSummary predict(const Dataset& data, const KernelSpec& spec, const HyperparameterSet& theta,
                                const NoiseModel& noise, bool include_noise, Device& dev = default_device()) {
    auto o = detail::eval(data, spec, theta, noise,
                          SPINGP_WANT_GRAD | SPINGP_WANT_MEAN | SPINGP_WANT_VAR |
                              (include_noise ? SPINGP_INCLUDE_NOISE : 0u),
                          dev);
    return PosteriorSummary{data.times, std::move(o.mean), std::move(o.var), o.loglik, std::move(o.grad)};
}

// Posterior at arbitrary test times: the test points join the training
// grid without an observation term; test times colliding with earlier grid times are
// nudged by 1e-9 x span.  PosteriorSummary.times are the test times in the
// caller's order; mll / mll_grad are the training data's.
inline PosteriorSummary predict(const Dataset& data, const KernelSpec& spec, const HyperparameterSet& theta,
                                const NoiseModel& noise, const std::vector<double>& test_times, bool include_noise,
                                Device& dev = default_device()) {
    detail::check_data(data, noise);
    const auto lv = detail::leaves_of(spec);
    const size_t m = test_times.size();
    PosteriorSummary out{test_times, std::vector<double>(m), std::vector<double>(m), 0.0,
                         std::vector<double>(theta.size() + 1)};
    int64_t fb = -1;
    const int st_ = spingp_predict(dev.get(), lv.data(), static_cast<int32_t>(lv.size()), theta.data(),
                                   static_cast<int32_t>(theta.size()), data.times.data(), data.values.data(),
                                   static_cast<int64_t>(data.times.size()), test_times.data(),
                                   static_cast<int64_t>(m), std::sqrt(noise.sigma_n2),
                                   SPINGP_WANT_GRAD | (include_noise ? SPINGP_INCLUDE_NOISE : 0u), &out.mll,
                                   out.mll_grad.data(), out.mean.data(), out.variance.data(), &fb);
    Device::check(st_, fb);
    return out;
}

}  // namespace spingp
