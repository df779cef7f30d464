// optimize_hyperparameters through include/spingp/optimize.hpp on the
// GPU: the SPEC's three examples.
#include <cmath>
#include <cstdint>
#include <random>

#include "minitest.hpp"
#include "spingp/optimize.hpp"

using namespace spingp;

namespace {

double unit(std::mt19937_64& r) { return static_cast<double>(r() >> 11) * 0x1.0p-53; }
double normal(std::mt19937_64& r) {  // Box-Muller
    const double u = std::max(unit(r), 1e-300), v = unit(r);
    return std::sqrt(-2.0 * std::log(u)) * std::cos(6.283185307179586 * v);
}

// Matérn-1/2 (OU) prior sample on irregular times by its exact state-space recursion, + noise
Dataset simulate_ou(double var, double len, double sigma_n, int n, uint64_t seed) {
    std::mt19937_64 r(seed);
    Dataset d;
    double t = 0.0, z = std::sqrt(var) * normal(r);
    for (int i = 0; i < n; ++i) {
        if (i) {
            const double dt = 0.05 + 0.15 * unit(r);
            t += dt;
            const double a = std::exp(-dt / len);
            z = a * z + std::sqrt(var * (1.0 - a * a)) * normal(r);
        }
        d.times.push_back(t);
        d.values.push_back(z + sigma_n * normal(r));
    }
    return d;
}

}  // namespace

TEST(Optimize, RecoversLengthscaleFromSimulatedMatern12) {
    const Dataset d = simulate_ou(1.0, 2.0, 0.1, 500, 42);
    auto r = optimize_hyperparameters(d, KernelSpec::matern12(), {0.5, 0.5}, NoiseModel{0.09}, 200);
    EXPECT_TRUE(r.theta[1] > 0.7 * 2.0 && r.theta[1] < 1.3 * 2.0);
    EXPECT_TRUE(!r.line_search_failed);
    for (size_t i = 1; i < r.trace.size(); ++i) EXPECT_TRUE(r.trace[i] >= r.trace[i - 1]);  // non-decreasing
}

TEST(Optimize, StartingAtTheOptimumStops) {
    const Dataset d = simulate_ou(1.0, 2.0, 0.1, 500, 42);
    auto r1 = optimize_hyperparameters(d, KernelSpec::matern12(), {0.5, 0.5}, NoiseModel{0.09}, 200);
    auto r2 = optimize_hyperparameters(d, KernelSpec::matern12(), r1.theta, r1.noise, 200);
    EXPECT_TRUE(r2.iterations <= 2);
    EXPECT_TRUE(r2.trace.back() >= r2.trace.front());
    EXPECT_TRUE(std::abs(r2.trace.back() - r1.trace.back()) <= 1e-8 * std::abs(r1.trace.back()));
}

TEST(Optimize, TraceMatchesReevaluation) {
    const Dataset d = simulate_ou(1.0, 2.0, 0.1, 300, 7);
    auto r = optimize_hyperparameters(d, KernelSpec::matern32(), {0.7, 1.0}, NoiseModel{0.04}, 20);
    for (size_t i = 0; i < r.trace.size(); ++i) {
        const auto& p = r.trace_params[i];
        const double ll = log_marginal_likelihood(d, KernelSpec::matern32(), {p[0], p[1]}, NoiseModel{p[2] * p[2]});
        EXPECT_TRUE(std::abs(ll - r.trace[i]) <= 1e-12 * std::abs(ll));
    }
}

TEST(Optimize, InfeasibleStartAndBadArguments) {
    const Dataset d = simulate_ou(1.0, 2.0, 0.1, 50, 1);
    EXPECT_THROW(optimize_hyperparameters(d, KernelSpec::matern12(), {1.0, 1.0}, NoiseModel{0.01}, 0),
                 std::invalid_argument);
    EXPECT_THROW(optimize_hyperparameters(d, KernelSpec::matern12(), {-1.0, 1.0}, NoiseModel{0.01}, 5),
                 std::invalid_argument);
}

int main() { return minitest::run_all(); }
