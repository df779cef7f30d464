// GPU: the SPEC btd_core / spingp_engine C++ API (include/spingp/btd.hpp,
// engine.hpp) on the B200 through the C ABI.  Known answers from SPEC.md.
#include <cmath>
#include <random>

#include "minitest.hpp"
#include "spingp/engine.hpp"

using namespace spingp;

TEST(BTD, FactorizeScalar) {
    SymBTD m(1, 1);
    m.diag[0](0, 0) = 4.0;
    EXPECT_NEAR(logdet(factorize(m)), std::log(4.0), 1e-15);
}

TEST(BTD, TwoByTwo) {
    SymBTD m(2, 1);
    m.diag[0](0, 0) = m.diag[1](0, 0) = 2.0;
    m.upper[0](0, 0) = -1.0;
    auto f = factorize(m);
    EXPECT_NEAR(logdet(f), std::log(3.0), 1e-15);
    Matrix rhs(2, 1, 1.0);
    auto x = solve(f, rhs);
    EXPECT_NEAR(x(0, 0), 1.0, 1e-15);
    EXPECT_NEAR(x(1, 0), 1.0, 1e-15);
    auto c = selective_inverse(f);
    EXPECT_NEAR(c.diag[0](0, 0), 2.0 / 3, 1e-15);
    EXPECT_NEAR(c.upper[0](0, 0), 1.0 / 3, 1e-15);
    auto mv = matvec(m, rhs);
    EXPECT_NEAR(mv(0, 0), 1.0, 1e-15);
}

TEST(BTD, TraceIdentity) {
    SymBTD m(7, 1);
    for (auto& d : m.diag) d(0, 0) = 1.0;
    EXPECT_NEAR(trace_btd_product(m, m), 7.0, 0.0);
}

TEST(BTD, IndefiniteRaisesNotPositiveDefinite) {
    SymBTD m(1, 1);
    m.diag[0](0, 0) = -1.0;
    bool caught = false;
    try {
        factorize(m);
    } catch (const NotPositiveDefinite& e) {
        caught = e.block_index() == 0;
    }
    EXPECT_TRUE(caught);
}

TEST(Engine, SinglePointClosedForm) {
    Dataset d{{0.0}, {0.7}};
    const double var = 1.3, s2 = 0.09;
    const double ll = log_marginal_likelihood(d, KernelSpec::matern12(), {var, 1.7}, NoiseModel{s2});
    EXPECT_NEAR(ll, -0.5 * std::log(2 * M_PI * (var + s2)) - 0.5 * 0.49 / (var + s2), 1e-9);
}

TEST(Engine, GradientZeroAtSinglePointOptimum) {
    const double var = 1.3, s2 = 0.16;
    Dataset d{{0.0}, {std::sqrt(var + s2)}};
    auto g = mll_gradient(d, KernelSpec::matern12(), {var, 1.7}, NoiseModel{s2});
    EXPECT_NEAR(g[0], 0.0, 1e-9);
}

TEST(Engine, AssemblySinglePointIsPinfInverse) {
    auto spec = KernelSpec::matern32(1.3, 0.9);
    auto P = assemble_prior_precision({0.0}, spec, {1.3, 0.9});
    auto ssm = state_space_of(spec, {1.3, 0.9});
    Matrix prod = P.diag[0] * ssm.Pinf;
    EXPECT_LT((prod - Matrix::Identity(2)).maxAbs(), 1e-8);
}

TEST(Engine, DuplicateTimestampRejected) {
    Dataset d{{0.0, 1.0, 1.0}, {0.0, 0.0, 0.0}};
    EXPECT_THROW(log_marginal_likelihood(d, KernelSpec::matern32(), {1.0, 1.0}, NoiseModel{0.1}), DuplicateTimestamp);
}

TEST(Engine, PredictVariancesNonNegativeAndNoiseFlag) {
    std::mt19937_64 rng(3);
    Dataset d;
    double t = 0;
    for (int i = 0; i < 300; ++i) {
        t += 0.05 + 0.1 * std::uniform_real_distribution<double>(0, 1)(rng);
        d.times.push_back(t);
        d.values.push_back(std::sin(t));
    }
    auto a = predict(d, KernelSpec::matern32(1.0, 2.0), {1.0, 2.0}, NoiseModel{0.09}, false);
    auto b = predict(d, KernelSpec::matern32(1.0, 2.0), {1.0, 2.0}, NoiseModel{0.09}, true);
    for (size_t i = 0; i < d.times.size(); ++i) {
        EXPECT_GE(a.variance[i], 0.0);
        EXPECT_NEAR(b.variance[i] - a.variance[i], 0.09, 1e-12);
    }
}

// SPEC.md:302 example: test time = train time, sigma_n -> 1e-8: the predictive mean
// approaches y there (1e-4) and the latent variance ~0; far test points revert to the prior.
TEST(Engine, PredictAtTestTimesInterpolatesAndReverts) {
    Dataset d;
    for (int i = 0; i < 50; ++i) {
        d.times.push_back(0.2 * i);
        d.values.push_back(std::sin(0.2 * i));
    }
    const std::vector<double> tt = {d.times[10], 1000.0, d.times[33]};
    auto p = predict(d, KernelSpec::matern32(1.0, 2.0), {1.0, 2.0}, NoiseModel{1e-16}, tt, false);
    EXPECT_NEAR(p.mean[0], d.values[10], 1e-4);
    EXPECT_NEAR(p.mean[2], d.values[33], 1e-4);
    EXPECT_NEAR(p.variance[0], 0.0, 1e-4);
    EXPECT_NEAR(p.mean[1], 0.0, 1e-6);
    EXPECT_NEAR(p.variance[1], 1.0, 1e-6);  // k(0) = var
    EXPECT_EQ(p.times.size(), tt.size());
    EXPECT_EQ(p.mll_grad.size(), 3u);
}

TEST(Engine, MultiDeviceOneGpuEqualsSingle) {  // spingp_eval_partitioned, P = 1
    std::mt19937_64 g(42);
    std::uniform_real_distribution<double> u(0.05, 0.15);
    std::normal_distribution<double> z;
    Dataset d;
    double tt = 0.0;
    for (int i = 0; i < 5000; ++i) {
        tt += u(g);
        d.times.push_back(tt);
        d.values.push_back(std::sin(0.5 * tt) + 0.3 * z(g));
    }
    const auto spec = KernelSpec::matern52(2.0, 1.5);
    const HyperparameterSet th{2.0, 1.5};
    MultiDevice md({0});
    EXPECT_TRUE(md.size() == 1);
    const double a = log_marginal_likelihood(d, spec, th, NoiseModel{0.09}, md);
    const double b = log_marginal_likelihood(d, spec, th, NoiseModel{0.09});
    EXPECT_NEAR(a, b, 1e-10 * std::abs(b));
    const auto ga = mll_gradient(d, spec, th, NoiseModel{0.09}, md);
    const auto gb = mll_gradient(d, spec, th, NoiseModel{0.09});
    for (size_t i = 0; i < ga.size(); ++i) EXPECT_NEAR(ga[i], gb[i], 1e-9 * std::abs(gb[i]) + 1e-12);
}

int main() { return minitest::run_all(); }
