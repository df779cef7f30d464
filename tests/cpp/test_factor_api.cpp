// GPU: the device-resident BTDFactor (include/spingp/btd.hpp over spingp_btd_factorize):
// the SPEC.md:135-140 invariants (positive pivot diagonals, reconstruction of the SymBTD
// from {L_i, M_i} to 1e-8), the SPEC known answers, solve / selective_inverse reusing the
// kept factor against cr_solve and the dense inverse, and the matvec round trip
// (SPEC.md:217).
#include <cmath>
#include <random>

#include "minitest.hpp"
#include "spingp/engine.hpp"

using namespace spingp;

static SymBTD random_spd(Index n, Index b, unsigned seed) {
    std::mt19937_64 g(seed);
    std::normal_distribution<double> z;
    SymBTD m(n, b);
    for (Index i = 0; i < n; ++i) {
        Matrix a(b, b);
        for (Index p = 0; p < b; ++p)
            for (Index q = 0; q < b; ++q) a(p, q) = z(g);
        m.diag[i] = a * a.transpose();
        for (Index p = 0; p < b; ++p) m.diag[i](p, p) += 4.0 * b;
    }
    for (Index i = 0; i + 1 < n; ++i)
        for (Index p = 0; p < b; ++p)
            for (Index q = 0; q < b; ++q) m.upper[i](p, q) = z(g);
    return m;
}

static double relerr(const Matrix& a, const Matrix& b) {
    double num = 0.0, den = 0.0;
    for (Index i = 0; i < a.rows(); ++i)
        for (Index j = 0; j < a.cols(); ++j) {
            num = std::max(num, std::abs(a(i, j) - b(i, j)));
            den = std::max(den, std::abs(b(i, j)));
        }
    return num / std::max(den, 1e-300);
}

TEST(Factor, KnownAnswers) {
    SymBTD one(1, 1);
    one.diag[0](0, 0) = 4.0;
    auto f1 = factorize(one);
    EXPECT_NEAR(f1.L[0](0, 0), 2.0, 1e-15);
    EXPECT_NEAR(logdet(f1), std::log(4.0), 1e-15);
    SymBTD two(2, 1);
    two.diag[0](0, 0) = two.diag[1](0, 0) = 2.0;
    two.upper[0](0, 0) = -1.0;
    auto f2 = factorize(two);  // pivots S = [2, 1.5]
    EXPECT_NEAR(f2.L[0](0, 0), std::sqrt(2.0), 1e-14);
    EXPECT_NEAR(f2.L[1](0, 0), std::sqrt(1.5), 1e-14);
    EXPECT_NEAR(f2.M[0](0, 0), -0.5, 1e-14);  // M_0 = U_0^T S_0^{-1}
    EXPECT_NEAR(logdet(f2), std::log(3.0), 1e-15);
}

TEST(Factor, ReconstructionAndPositivePivots) {
    for (Index b : {1, 2, 3, 4, 6}) {
        const Index n = 30;
        SymBTD m = random_spd(n, b, 7 + static_cast<unsigned>(b));
        auto f = factorize(m);
        double err = 0.0;
        for (Index i = 0; i < n; ++i) {
            for (Index k = 0; k < b; ++k) EXPECT_TRUE(f.L[i](k, k) > 0.0);
            const Matrix S = f.L[i] * f.L[i].transpose();
            Matrix D = S;
            if (i > 0) D = D + f.M[i - 1] * (f.L[i - 1] * f.L[i - 1].transpose()) * f.M[i - 1].transpose();
            err = std::max(err, relerr(D, m.diag[i]));
            if (i + 1 < n) err = std::max(err, relerr(S * f.M[i].transpose(), m.upper[i]));
        }
        EXPECT_TRUE(err < 1e-8);
    }
}

TEST(Factor, SolveAndSelectiveInverseReuseTheFactor) {
    const Index n = 30, b = 3;
    SymBTD m = random_spd(n, b, 99);
    auto f = factorize(m);
    // the dense inverse by cr_solve on the identity (n b right-hand sides)
    const Matrix I = Matrix::Identity(n * b);
    auto inv = cr_solve(m, I);
    EXPECT_NEAR(inv.logdet, logdet(f), 1e-9 * std::abs(logdet(f)));
    Matrix rhs(n * b, 3);
    std::mt19937_64 g(5);
    std::normal_distribution<double> z;
    for (Index i = 0; i < n * b; ++i)
        for (Index c = 0; c < 3; ++c) rhs(i, c) = z(g);
    const Matrix x = solve(f, rhs);
    EXPECT_TRUE(relerr(x, cr_solve(m, rhs).x) < 1e-8);
    for (Index c = 0; c < 3; ++c) {  // residual M x - rhs
        Matrix xc(n * b, 1), rc(n * b, 1);
        for (Index i = 0; i < n * b; ++i) {
            xc(i, 0) = x(i, c);
            rc(i, 0) = rhs(i, c);
        }
        EXPECT_TRUE(relerr(matvec(m, xc), rc) < 1e-8);
    }
    const SymBTD C = selective_inverse(f);
    double err = 0.0;
    for (Index i = 0; i < n; ++i)
        for (Index p = 0; p < b; ++p)
            for (Index q = 0; q < b; ++q) {
                err = std::max(err, std::abs(C.diag[i](p, q) - inv.x(i * b + p, i * b + q)));
                if (i + 1 < n) err = std::max(err, std::abs(C.upper[i](p, q) - inv.x(i * b + p, (i + 1) * b + q)));
            }
    EXPECT_TRUE(err < 1e-8);
}

TEST(Factor, RoundTripUnitVectors) {  // matvec(m, solve(factorize(m), e_j)) = e_j
    const Index n = 50, b = 4;
    SymBTD m = random_spd(n, b, 3);
    auto f = factorize(m);
    std::mt19937_64 g(11);
    for (int r = 0; r < 10; ++r) {
        Matrix e(n * b, 1);
        e(static_cast<Index>(g() % static_cast<uint64_t>(n * b)), 0) = 1.0;
        const Matrix back = matvec(m, solve(f, e));
        EXPECT_TRUE(relerr(back, e) < 1e-7);
    }
}

TEST(Factor, LongSeriesChunkedSubstitution) {  // many substitution chunks (kChunk = 64)
    const Index n = 5000, b = 2;
    SymBTD m = random_spd(n, b, 17);
    auto f = factorize(m);
    Matrix rhs(n * b, 2, 1.0);
    EXPECT_TRUE(relerr(solve(f, rhs), cr_solve(m, rhs).x) < 1e-9);
}

TEST(Factor, IndefiniteRaises) {
    SymBTD m(1, 1);
    m.diag[0](0, 0) = -1.0;
    bool thrown = false;
    try {
        factorize(m);
    } catch (const NotPositiveDefinite&) {
        thrown = true;
    }
    EXPECT_TRUE(thrown);
}

int main() { return minitest::run_all(); }
