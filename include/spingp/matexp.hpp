#pragma once
// Matrix functions of the reference API (proj/include/spingp/matexp.hpp:10-52),
// Eigen-free.  Host-side setup only: the per-step hot loop runs on the B200 with
// closed-form transitions (paper_1610_08035_b200/csrc/model_dev.cuh); these are
// the reference-compatible entry points for API users and tests.

#include <cmath>

#include "spingp/matrix.hpp"

namespace spingp {

namespace detail {
inline double norm1(const Matrix& a) {
    double best = 0;
    for (Index j = 0; j < a.cols(); ++j) {
        double s = 0;
        for (Index i = 0; i < a.rows(); ++i) s += std::abs(a(i, j));
        best = std::max(best, s);
    }
    return best;
}
// Horner-free Padé sums: U = A * sum_{odd} b_k A^{k-1}, V = sum_{even} b_k A^k,
// using the powers A^2, A^4, ... (Higham 2005, Algorithm 2.3).
inline void pade_uv(const Matrix& A, const double* b, int m, Matrix& U, Matrix& V) {
    const Index n = A.rows();
    const Matrix I = Matrix::Identity(n);
    std::vector<Matrix> pw{I, A * A};  // A^0, A^2, A^4, ...
    while (static_cast<int>(pw.size()) * 2 <= m) pw.push_back(pw.back() * pw[1]);
    Matrix u = Matrix::Zero(n, n), v = Matrix::Zero(n, n);
    for (int k = 0; k <= m; ++k) {
        if (k % 2 == 1) u += b[k] * pw[static_cast<size_t>(k / 2)];
        else v += b[k] * pw[static_cast<size_t>(k / 2)];
    }
    U = A * u;
    V = v;
}
}  // namespace detail

// expm(A): scaling and squaring with the Padé degree chosen from ||A||_1
// (Higham 2005; the algorithm Eigen's MatrixFunctions `exp()` implements,
// matexp.hpp:11-13).
inline Matrix expm(const Matrix& a) {
    static const double b3[] = {120.0, 60.0, 12.0, 1.0};
    static const double b5[] = {30240.0, 15120.0, 3360.0, 420.0, 30.0, 1.0};
    static const double b7[] = {17297280.0, 8648640.0, 1995840.0, 277200.0, 25200.0, 1512.0, 56.0, 1.0};
    static const double b9[] = {17643225600.0, 8821612800.0, 2075673600.0, 302702400.0, 30270240.0,
                                2162160.0,     110880.0,     3960.0,       90.0,        1.0};
    static const double b13[] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                                 1187353796428800.0,  129060195264000.0,   10559470521600.0,
                                 670442572800.0,      33522128640.0,       1323241920.0,
                                 40840800.0,          960960.0,            16380.0,
                                 182.0,               1.0};
    const double l1 = detail::norm1(a);
    Matrix U, V;
    int squarings = 0;
    if (l1 < 1.495585217958292e-2) detail::pade_uv(a, b3, 3, U, V);
    else if (l1 < 2.539398330063230e-1) detail::pade_uv(a, b5, 5, U, V);
    else if (l1 < 9.504178996162932e-1) detail::pade_uv(a, b7, 7, U, V);
    else if (l1 < 2.097847961257068e+0) detail::pade_uv(a, b9, 9, U, V);
    else {
        int e = 0;
        std::frexp(l1 / 5.371920351148152, &e);
        squarings = std::max(0, e);
        detail::pade_uv(a * std::ldexp(1.0, -squarings), b13, 13, U, V);
    }
    Matrix r = lu_solve(V - U, U + V);
    for (int i = 0; i < squarings; ++i) r = r * r;
    return r;
}

// Fréchet derivative of expm along dF over a step dt, from the Van Loan block
// exponential expm([[F, dF], [0, F]] dt) (matexp.hpp:15-32).
inline Matrix expm_frechet(const Matrix& f, const Matrix& df, double dt) {
    const Index b = f.rows();
    Matrix aug = Matrix::Zero(2 * b, 2 * b);
    aug.setBlock(0, 0, f * dt);
    aug.setBlock(0, b, df * dt);
    aug.setBlock(b, b, f * dt);
    return expm(aug).block(0, b, b, b);
}

// F P + P F^T + W = 0 via (I (x) F + F (x) I) vec(P) = -vec(W) (matexp.hpp:34-52).
inline Matrix solve_continuous_lyapunov(const Matrix& f, const Matrix& w) {
    const Index b = f.rows();
    Matrix big = Matrix::Zero(b * b, b * b);
    for (Index j = 0; j < b; ++j)
        for (Index r = 0; r < b; ++r)
            for (Index c = 0; c < b; ++c) big(j * b + r, j * b + c) += f(r, c);
    for (Index j = 0; j < b; ++j)
        for (Index i = 0; i < b; ++i)
            for (Index k = 0; k < b; ++k) big(j * b + k, i * b + k) += f(j, i);
    Matrix rhs(b * b, 1);
    for (Index j = 0; j < b; ++j)
        for (Index i = 0; i < b; ++i) rhs(j * b + i, 0) = -w(i, j);
    const Matrix p = lu_solve(big, rhs);
    Matrix out(b, b);
    for (Index j = 0; j < b; ++j)
        for (Index i = 0; i < b; ++i) out(i, j) = p(j * b + i, 0);
    return symmetrize(out);
}

}  // namespace spingp
