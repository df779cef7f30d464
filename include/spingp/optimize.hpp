#pragma once
// optimize_hyperparameters: the caller that
// makes throughput matter — every iteration is one or more fused loglik + gradient
// evaluations on the B200 (spingp_eval through engine.hpp).
//
// SPEC contract:
//   quasi-Newton ascent on the MLL in log-parameter space with backtracking line search;
//   returns the best-seen parameters; the MLL trace is non-decreasing over accepted
//   steps; terminates on gradient inf-norm < 1e-6, relative MLL change < 1e-10, or the
//   iteration budget.  InfeasibleStart if theta0 yields NotPositiveDefinite; a line-search
//   failure returns the best-seen point with a warning flag.
// Here: L-BFGS (memory 8) on x = log(theta..., sigma_n) with an Armijo backtracking line
// search (c1 = 1e-4, halving, <= 40 trials; trial points that fail to factorise count as
// rejected).  sigma_n is the noise standard deviation (NoiseModel holds sigma_n^2).
// The backtracking trials go to the GPU kProbes at a time (step a, a/2, a/4, a/8 in one
// batched evaluation, spingp_eval_multi_theta: the series is uploaded once and the
// probes run as independent series); the first trial, in that order, that satisfies
// Armijo is accepted, exactly as with one trial per call.

#include <algorithm>
#include <cmath>
#include <deque>
#include <limits>
#include <vector>

#include "spingp/engine.hpp"
#include "spingp/errors.hpp"

namespace spingp {

struct OptimizeResult {
    HyperparameterSet theta;                      // best seen
    NoiseModel noise;                             // best seen
    std::vector<double> trace;                    // MLL of the start and of every accepted step
    std::vector<std::vector<double>> trace_params;  // (theta..., sigma_n) of each trace entry
    int iterations = 0;
    bool line_search_failed = false;              // warning flag
};

namespace detail {

struct Probe {
    double f = -std::numeric_limits<double>::infinity();  // MLL (-inf = could not factorise)
    std::vector<double> g;                                 // d MLL / d log(param)
};

inline Probe mll_probe(const Dataset& data, const KernelSpec& spec, const std::vector<double>& x, Device& dev) {
    const size_t p = x.size() - 1;
    HyperparameterSet theta(p);
    for (size_t i = 0; i < p; ++i) theta[i] = std::exp(x[i]);
    const double sigma = std::exp(x[p]);
    Probe pr;
    auto o = eval(data, spec, theta, NoiseModel{sigma * sigma}, SPINGP_WANT_GRAD, dev);
    pr.f = o.loglik;
    pr.g.resize(p + 1);
    for (size_t i = 0; i < p; ++i) pr.g[i] = o.grad[i] * theta[i];  // chain rule to log space
    pr.g[p] = o.grad[p] * sigma;
    return pr;
}

constexpr int kProbes = 4;

// kProbes (or fewer) trial points in one batched GPU evaluation.  Probes from the first
// one that did not factorise on are left at f = -inf (the status word names only the
// first failing probe).
inline std::vector<Probe> mll_probes(const Dataset& data, const KernelSpec& spec,
                                     const std::vector<std::vector<double>>& xs, Device& dev) {
    check_data(data, NoiseModel{1.0});
    const size_t K = xs.size(), d = xs[0].size(), p = d - 1;
    const auto lv = leaves_of(spec);
    std::vector<double> theta(K * p), sigma(K), ll(K), g(K * d);
    for (size_t k = 0; k < K; ++k) {
        for (size_t i = 0; i < p; ++i) theta[k * p + i] = std::exp(xs[k][i]);
        sigma[k] = std::exp(xs[k][p]);
    }
    int64_t bad = -1;
    const int st = spingp_eval_multi_theta(dev.get(), lv.data(), static_cast<int32_t>(lv.size()), theta.data(),
                                           static_cast<int32_t>(p), static_cast<int64_t>(K), data.times.data(),
                                           data.values.data(), static_cast<int64_t>(data.times.size()), sigma.data(),
                                           SPINGP_WANT_GRAD, ll.data(), g.data(), &bad);
    size_t valid = K;
    if (st == SPINGP_NOT_PD || st == SPINGP_SINGULAR_Q) valid = bad >= 0 ? static_cast<size_t>(bad) : 0;
    else Device::check(st, bad);
    std::vector<Probe> out(K);
    for (size_t k = 0; k < valid && k < K; ++k) {
        out[k].f = ll[k];
        out[k].g.resize(d);
        for (size_t i = 0; i < p; ++i) out[k].g[i] = g[k * d + i] * theta[k * p + i];  // to log space
        out[k].g[p] = g[k * d + p] * sigma[k];
    }
    return out;
}

}  // namespace detail

inline OptimizeResult optimize_hyperparameters(const Dataset& data, const KernelSpec& spec,
                                               const HyperparameterSet& theta0, const NoiseModel& noise0,
                                               int budget, Device& dev = default_device()) {
    if (budget < 1) throw std::invalid_argument("budget must be >= 1 iteration");
    for (double v : theta0)
        if (!(v > 0.0)) throw std::invalid_argument("theta0 must be positive");
    if (!(noise0.sigma_n2 > 0.0)) throw std::invalid_argument("noise0 must be positive");
    const size_t p = theta0.size(), d = p + 1;
    std::vector<double> x(d);
    for (size_t i = 0; i < p; ++i) x[i] = std::log(theta0[i]);
    x[p] = 0.5 * std::log(noise0.sigma_n2);
    detail::Probe cur;
    try {
        cur = detail::mll_probe(data, spec, x, dev);
    } catch (const NotPositiveDefinite& e) {
        throw InfeasibleStart(std::string("theta0 does not factorise: ") + e.what());
    }
    if (!std::isfinite(cur.f)) throw InfeasibleStart("theta0 gives a non-finite marginal likelihood");

    OptimizeResult res;
    auto params_of = [&](const std::vector<double>& xx) {
        std::vector<double> v(d);
        for (size_t i = 0; i < d; ++i) v[i] = std::exp(xx[i]);
        return v;
    };
    res.trace.push_back(cur.f);
    res.trace_params.push_back(params_of(x));

    // minimise F = -MLL; G = -g
    auto dot = [&](const std::vector<double>& a, const std::vector<double>& b) {
        double s = 0.0;
        for (size_t i = 0; i < d; ++i) s += a[i] * b[i];
        return s;
    };
    std::deque<std::pair<std::vector<double>, std::vector<double>>> mem;  // (s, y) pairs
    constexpr size_t kMem = 8;
    std::vector<double> G(d);
    for (size_t i = 0; i < d; ++i) G[i] = -cur.g[i];
    for (int it = 0; it < budget; ++it) {
        double ginf = 0.0;
        for (double v : G) ginf = std::max(ginf, std::abs(v));
        if (ginf < 1e-6) break;
        // two-loop recursion: dir = -H G
        std::vector<double> q = G;
        std::vector<double> alpha(mem.size());
        for (size_t k = mem.size(); k-- > 0;) {
            const auto& [s, y] = mem[k];
            alpha[k] = dot(s, q) / dot(y, s);
            for (size_t i = 0; i < d; ++i) q[i] -= alpha[k] * y[i];
        }
        double gamma = 1.0 / std::max(1.0, ginf);  // first step: at most 1 in log space
        if (!mem.empty()) gamma = dot(mem.back().first, mem.back().second) / dot(mem.back().second, mem.back().second);
        for (double& v : q) v *= gamma;
        for (size_t k = 0; k < mem.size(); ++k) {
            const auto& [s, y] = mem[k];
            const double beta = dot(y, q) / dot(y, s);
            for (size_t i = 0; i < d; ++i) q[i] += (alpha[k] - beta) * s[i];
        }
        std::vector<double> dir(d);
        for (size_t i = 0; i < d; ++i) dir[i] = -q[i];
        double slope = dot(G, dir);
        if (!(slope < 0.0)) {  // not a descent direction: restart from steepest descent
            mem.clear();
            for (size_t i = 0; i < d; ++i) dir[i] = -G[i] / std::max(1.0, ginf);
            slope = dot(G, dir);
        }
        double dinf = 0.0;
        for (double v : dir) dinf = std::max(dinf, std::abs(v));
        double a = dinf > 2.0 ? 2.0 / dinf : 1.0;  // never more than e^2 per parameter per step
        bool accepted = false;
        std::vector<double> xn(d);
        detail::Probe nxt;
        for (int tr = 0; tr < 40 && !accepted;) {
            const int K = std::min(detail::kProbes, 40 - tr);
            std::vector<std::vector<double>> xs(static_cast<size_t>(K), std::vector<double>(d));
            std::vector<double> as(static_cast<size_t>(K));
            for (int k = 0; k < K; ++k, a *= 0.5) {
                as[static_cast<size_t>(k)] = a;
                for (size_t i = 0; i < d; ++i) xs[static_cast<size_t>(k)][i] = x[i] + a * dir[i];
            }
            const auto pr = detail::mll_probes(data, spec, xs, dev);
            for (int k = 0; k < K; ++k) {
                const auto& q = pr[static_cast<size_t>(k)];
                if (!std::isfinite(q.f)) {  // did not factorise: rejected; later probes re-run
                    a = as[static_cast<size_t>(k)] * 0.5;
                    tr += k + 1;
                    break;
                }
                if (-q.f <= -cur.f + 1e-4 * as[static_cast<size_t>(k)] * slope) {
                    accepted = true;
                    xn = xs[static_cast<size_t>(k)];
                    nxt = q;
                    break;
                }
                if (k == K - 1) tr += K;
            }
        }
        if (!accepted) {
            res.line_search_failed = true;
            break;
        }
        std::vector<double> s(d), y(d), Gn(d);
        for (size_t i = 0; i < d; ++i) {
            Gn[i] = -nxt.g[i];
            s[i] = xn[i] - x[i];
            y[i] = Gn[i] - G[i];
        }
        if (dot(s, y) > 1e-12 * std::sqrt(dot(s, s) * dot(y, y))) {
            mem.emplace_back(s, y);
            if (mem.size() > kMem) mem.pop_front();
        }
        const double rel = std::abs(nxt.f - cur.f) / std::max(1.0, std::abs(cur.f));
        x = xn;
        cur = nxt;
        G = Gn;
        res.trace.push_back(cur.f);
        res.trace_params.push_back(params_of(x));
        res.iterations = it + 1;
        if (rel < 1e-10) break;
    }
    // best seen = last accepted (the accepted MLL sequence is non-decreasing)
    const auto& best = res.trace_params.back();
    res.theta.assign(best.begin(), best.begin() + static_cast<std::ptrdiff_t>(p));
    res.noise = NoiseModel{best[p] * best[p]};
    return res;
}

}  // namespace spingp
