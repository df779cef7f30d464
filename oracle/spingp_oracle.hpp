// spingp_oracle.hpp — CPU ORACLE for the SpInGP sparse-precision inference path.
//
// TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1610_08035_b200/,
// include/) includes, links or calls this file.  Only tests/, __graft_entry__.smoke()
// and bench.py's CPU baseline leg (`cpu_baseline`, `--impl reference`) use it, as
// the checker / the timed reference-CPU arm.
//
// What it is: a plain, sequential restatement of the reference algorithm,
// templated on the scalar type so it can also run in `long double` as an
// extended-precision arbiter:
//   * kernel -> state-space model      kernels.hpp:17-381 (restated literally:
//     leaf builders :137-200, EQ modal realisation :205-321, Sum :357-379)
//   * per-step discretisation          kernels.hpp:392-443 (Padé scaling-and-squaring
//     expm as in Eigen MatrixFunctions, matexp.hpp:11-13; Van Loan Fréchet
//     derivative matexp.hpp:22-32; Kronecker Lyapunov matexp.hpp:37-52)
//   * assembly + jitter + anchoring
//   * block Thomas factor/solve/logdet SPEC.md:143-169 (pivot symmetrisation :219)
//   * Takahashi selected inverse       SPEC.md:170-178 (formula: SURVEY.md App. B)
//   * MLL (stationary form) + gradient SPEC.md:280-297 (formulas: SURVEY.md App. B)
//   * posterior mean / variance
// The reference itself cannot be compiled here (Eigen and GTest are absent,
// SURVEY.md §0.4), so this restatement is pinned against the reference's own
// known-answer tests (proj/tests/test_kernels.cpp, ported in tests/) and the
// SPEC's exact examples, plus a dense-GP and a Kalman-filter oracle at small N.
//
// The quasi-periodic (QP) leaf is NOT in the reference (SPEC.md:117 lists it as a
// non-goal); BASELINE cfg5 needs it.  It is defined here following Solin &
// Särkkä (2014) and documented in DESIGN.md.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------- status ------
enum Status : int {
    OK = 0, NOT_PD = 1, SINGULAR_Q = 2, BAD_ARG = 3, DUPLICATE_TIME = 6, UNSUPPORTED = 7,
    NEG_VARIANCE = 8
};

struct Failure {
    int status;
    int64_t block;
    std::string what;
};

// ---------------------------------------------------------------- matrix ------
template <class R>
struct Mat {
    int r = 0, c = 0;
    std::vector<R> a;
    Mat() = default;
    Mat(int rows, int cols) : r(rows), c(cols), a(static_cast<size_t>(rows) * cols, R(0)) {}
    R& operator()(int i, int j) { return a[static_cast<size_t>(i) * c + j]; }
    const R& operator()(int i, int j) const { return a[static_cast<size_t>(i) * c + j]; }
    static Mat identity(int n) {
        Mat m(n, n);
        for (int i = 0; i < n; ++i) m(i, i) = R(1);
        return m;
    }
};

template <class R>
Mat<R> operator*(const Mat<R>& x, const Mat<R>& y) {
    Mat<R> z(x.r, y.c);
    for (int i = 0; i < x.r; ++i)
        for (int k = 0; k < x.c; ++k) {
            const R v = x(i, k);
            if (v == R(0)) continue;
            for (int j = 0; j < y.c; ++j) z(i, j) += v * y(k, j);
        }
    return z;
}
template <class R>
Mat<R> operator+(Mat<R> x, const Mat<R>& y) {
    for (size_t i = 0; i < x.a.size(); ++i) x.a[i] += y.a[i];
    return x;
}
template <class R>
Mat<R> operator-(Mat<R> x, const Mat<R>& y) {
    for (size_t i = 0; i < x.a.size(); ++i) x.a[i] -= y.a[i];
    return x;
}
template <class R>
Mat<R> operator*(R s, Mat<R> x) {
    for (auto& v : x.a) v *= s;
    return x;
}
template <class R>
Mat<R> tr(const Mat<R>& x) {
    Mat<R> z(x.c, x.r);
    for (int i = 0; i < x.r; ++i)
        for (int j = 0; j < x.c; ++j) z(j, i) = x(i, j);
    return z;
}
template <class R>
Mat<R> sym(const Mat<R>& x) {  // 0.5 (x + x^T)
    Mat<R> z(x.r, x.c);
    for (int i = 0; i < x.r; ++i)
        for (int j = 0; j < x.c; ++j) z(i, j) = R(0.5) * (x(i, j) + x(j, i));
    return z;
}
template <class R>
R trace(const Mat<R>& x) {
    R s = 0;
    for (int i = 0; i < x.r; ++i) s += x(i, i);
    return s;
}
template <class R>
R trace_prod(const Mat<R>& x, const Mat<R>& y) {  // Tr(x y)
    R s = 0;
    for (int i = 0; i < x.r; ++i)
        for (int k = 0; k < x.c; ++k) s += x(i, k) * y(k, i);
    return s;
}
template <class R>
R l1norm(const Mat<R>& x) {  // max column sum
    R best = 0;
    for (int j = 0; j < x.c; ++j) {
        R s = 0;
        for (int i = 0; i < x.r; ++i) s += std::abs(x(i, j));
        best = std::max(best, s);
    }
    return best;
}

// LU with partial pivoting; solves A X = B in place of B.  Returns false if singular.
template <class R>
bool lu_solve(Mat<R> A, Mat<R>& B) {
    const int n = A.r;
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) {
        int p = k;
        R best = std::abs(A(k, k));
        for (int i = k + 1; i < n; ++i)
            if (std::abs(A(i, k)) > best) { best = std::abs(A(i, k)); p = i; }
        if (best == R(0)) return false;
        if (p != k) {
            for (int j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
            for (int j = 0; j < B.c; ++j) std::swap(B(k, j), B(p, j));
        }
        for (int i = k + 1; i < n; ++i) {
            const R f = A(i, k) / A(k, k);
            if (f == R(0)) continue;
            for (int j = k + 1; j < n; ++j) A(i, j) -= f * A(k, j);
            for (int j = 0; j < B.c; ++j) B(i, j) -= f * B(k, j);
        }
    }
    for (int k = n - 1; k >= 0; --k)
        for (int j = 0; j < B.c; ++j) {
            R s = B(k, j);
            for (int m = k + 1; m < n; ++m) s -= A(k, m) * B(m, j);
            B(k, j) = s / A(k, k);
        }
    return true;
}

// Cholesky A = L L^T (lower).  Returns false on a non-positive pivot.
template <class R>
bool cholesky(const Mat<R>& A, Mat<R>& L) {
    const int n = A.r;
    L = Mat<R>(n, n);
    for (int j = 0; j < n; ++j) {
        R d = A(j, j);
        for (int k = 0; k < j; ++k) d -= L(j, k) * L(j, k);
        if (!(d > R(0)) || !std::isfinite(static_cast<double>(d))) return false;
        const R ljj = std::sqrt(d);
        L(j, j) = ljj;
        for (int i = j + 1; i < n; ++i) {
            R s = A(i, j);
            for (int k = 0; k < j; ++k) s -= L(i, k) * L(j, k);
            L(i, j) = s / ljj;
        }
    }
    return true;
}
// X = A^{-1} B given the Cholesky factor L of A.
template <class R>
Mat<R> chol_solve(const Mat<R>& L, Mat<R> B) {
    const int n = L.r;
    for (int j = 0; j < B.c; ++j) {
        for (int i = 0; i < n; ++i) {
            R s = B(i, j);
            for (int k = 0; k < i; ++k) s -= L(i, k) * B(k, j);
            B(i, j) = s / L(i, i);
        }
        for (int i = n - 1; i >= 0; --i) {
            R s = B(i, j);
            for (int k = i + 1; k < n; ++k) s -= L(k, i) * B(k, j);
            B(i, j) = s / L(i, i);
        }
    }
    return B;
}
template <class R>
R chol_logdet(const Mat<R>& L) {
    R s = 0;
    for (int i = 0; i < L.r; ++i) s += std::log(L(i, i));
    return R(2) * s;
}

// ---------------------------------------------------------------- expm --------
// expm(A): scaling-and-squaring Padé (Higham 2005), degree selection and the
// 2^s scaling as Eigen's MatrixFunctions module does for double
// (matexp.hpp:11-13 calls `a.exp()`).  For extended precision the arbiter uses
// a scaled 30-term Taylor series (the reference's test oracle, test_support.hpp:15-32).
template <class R>
Mat<R> expm_taylor(const Mat<R>& A) {
    const int n = A.r;
    R norm = l1norm(A);
    int sq = 0;
    while (norm > R(0.25) && sq < 60) { norm *= R(0.5); ++sq; }
    Mat<R> s = std::ldexp(R(1), -sq) * A;
    Mat<R> term = Mat<R>::identity(n), sum = term;
    for (int k = 1; k <= 30; ++k) {
        term = (R(1) / R(k)) * (term * s);
        sum = sum + term;
    }
    for (int i = 0; i < sq; ++i) sum = sum * sum;
    return sum;
}

inline Mat<double> expm_pade(const Mat<double>& A) {
    using M = Mat<double>;
    const int n = A.r;
    const M I = M::identity(n);
    const double l1 = l1norm(A);
    M U, V;
    int squarings = 0;
    const M A2 = A * A;
    if (l1 < 1.495585217958292e-002) {
        const double b[] = {120.0, 60.0, 12.0, 1.0};
        U = A * (b[3] * A2 + b[1] * I);
        V = b[2] * A2 + b[0] * I;
    } else if (l1 < 2.539398330063230e-001) {
        const double b[] = {30240.0, 15120.0, 3360.0, 420.0, 30.0, 1.0};
        const M A4 = A2 * A2;
        U = A * (b[5] * A4 + b[3] * A2 + b[1] * I);
        V = b[4] * A4 + b[2] * A2 + b[0] * I;
    } else if (l1 < 9.504178996162932e-001) {
        const double b[] = {17297280.0, 8648640.0, 1995840.0, 277200.0,
                            25200.0,    1512.0,    56.0,      1.0};
        const M A4 = A2 * A2, A6 = A4 * A2;
        U = A * (b[7] * A6 + b[5] * A4 + b[3] * A2 + b[1] * I);
        V = b[6] * A6 + b[4] * A4 + b[2] * A2 + b[0] * I;
    } else if (l1 < 2.097847961257068e+000) {
        const double b[] = {17643225600.0, 8821612800.0, 2075673600.0, 302702400.0, 30270240.0,
                            2162160.0,     110880.0,     3960.0,       90.0,        1.0};
        const M A4 = A2 * A2, A6 = A4 * A2, A8 = A6 * A2;
        U = A * (b[9] * A8 + b[7] * A6 + b[5] * A4 + b[3] * A2 + b[1] * I);
        V = b[8] * A8 + b[6] * A6 + b[4] * A4 + b[2] * A2 + b[0] * I;
    } else {
        const double maxnorm = 5.371920351148152;
        int e = 0;
        std::frexp(l1 / maxnorm, &e);
        squarings = std::max(0, e);
        const M As = std::ldexp(1.0, -squarings) * A;
        const double b[] = {64764752532480000.0, 32382376266240000.0, 7771770303897600.0,
                            1187353796428800.0,  129060195264000.0,   10559470521600.0,
                            670442572800.0,      33522128640.0,       1323241920.0,
                            40840800.0,          960960.0,            16380.0,
                            182.0,               1.0};
        const M B2 = As * As, B4 = B2 * B2, B6 = B4 * B2;
        const M tmpU = b[13] * B6 + b[11] * B4 + b[9] * B2;
        U = As * (B6 * tmpU + b[7] * B6 + b[5] * B4 + b[3] * B2 + b[1] * I);
        const M tmpV = b[12] * B6 + b[10] * B4 + b[8] * B2;
        V = B6 * tmpV + b[6] * B6 + b[4] * B4 + b[2] * B2 + b[0] * I;
    }
    M num = U + V;      // (V - U)^{-1} (V + U)
    const M den = V - U;
    if (!lu_solve(den, num)) throw std::runtime_error("expm: singular Pade denominator");
    for (int i = 0; i < squarings; ++i) num = num * num;
    return num;
}

template <class R>
Mat<R> expm(const Mat<R>& A) {
    if constexpr (std::is_same_v<R, double>) return expm_pade(A);
    else return expm_taylor(A);
}

// Van Loan: expm([[F, dF], [0, F]] dt) top-right block (matexp.hpp:22-32).
template <class R>
Mat<R> expm_frechet(const Mat<R>& F, const Mat<R>& dF, R dt) {
    const int b = F.r;
    Mat<R> aug(2 * b, 2 * b);
    for (int i = 0; i < b; ++i)
        for (int j = 0; j < b; ++j) {
            aug(i, j) = F(i, j) * dt;
            aug(i, b + j) = dF(i, j) * dt;
            aug(b + i, b + j) = F(i, j) * dt;
        }
    const Mat<R> e = expm(aug);
    Mat<R> out(b, b);
    for (int i = 0; i < b; ++i)
        for (int j = 0; j < b; ++j) out(i, j) = e(i, b + j);
    return out;
}

// F P + P F^T + W = 0 by Kronecker vectorisation + partial-pivot LU (matexp.hpp:37-52).
template <class R>
Mat<R> solve_continuous_lyapunov(const Mat<R>& f, const Mat<R>& w) {
    const int b = f.r;
    Mat<R> big(b * b, b * b);
    for (int j = 0; j < b; ++j)
        for (int r0 = 0; r0 < b; ++r0)
            for (int c0 = 0; c0 < b; ++c0) big(j * b + r0, j * b + c0) += f(r0, c0);
    for (int j = 0; j < b; ++j)
        for (int i = 0; i < b; ++i)
            for (int k = 0; k < b; ++k) big(j * b + k, i * b + k) += f(j, i);
    Mat<R> rhs(b * b, 1);
    for (int j = 0; j < b; ++j)
        for (int i = 0; i < b; ++i) rhs(j * b + i, 0) = -w(i, j);
    if (!lu_solve(big, rhs)) throw std::runtime_error("lyapunov: singular system");
    Mat<R> out(b, b);
    for (int j = 0; j < b; ++j)
        for (int i = 0; i < b; ++i) out(i, j) = rhs(j * b + i, 0);
    return sym(out);
}

// ---------------------------------------------------------------- kernels -----
enum LeafType { MATERN12 = 0, MATERN32 = 1, MATERN52 = 2, EQ = 3, QP = 4 };

struct Leaf {
    int type;
    int order;
};

inline int leaf_nparams(int type) { return type == QP ? 4 : 2; }
inline int leaf_dim(const Leaf& l) {
    switch (l.type) {
        case MATERN12: return 1;
        case MATERN32: return 2;
        case MATERN52: return 3;
        case EQ: return l.order;
        case QP: return 2 * (l.order + 1);
    }
    return 0;
}

template <class R>
struct Model {
    int b = 0;
    Mat<R> F, Pinf;
    std::vector<R> H;
    std::vector<Mat<R>> dF, dPinf;
    std::vector<int> fconst;
    int ntheta() const { return static_cast<int>(dF.size()); }
};

template <class R>
struct LeafModel {
    Mat<R> F, Pinf;
    std::vector<R> H;
    std::vector<Mat<R>> dF, dPinf;
    std::vector<int> fconst;
};

template <class R>
void check_positive(R v, const char* what) {
    if (!(v > R(0)) || !std::isfinite(static_cast<double>(v)))
        throw std::invalid_argument(std::string("hyperparameter must be positive: ") + what);
}

template <class R>
LeafModel<R> matern12_ss(R var, R len) {  // kernels.hpp:137-147
    LeafModel<R> m;
    m.F = Mat<R>(1, 1); m.F(0, 0) = R(-1) / len;
    m.H = {R(1)};
    m.Pinf = Mat<R>(1, 1); m.Pinf(0, 0) = var;
    Mat<R> dPv(1, 1); dPv(0, 0) = R(1);
    Mat<R> dFl(1, 1); dFl(0, 0) = R(1) / (len * len);
    m.dF = {Mat<R>(1, 1), dFl};
    m.dPinf = {dPv, Mat<R>(1, 1)};
    m.fconst = {1, 0};
    return m;
}

template <class R>
LeafModel<R> matern32_ss(R var, R len) {  // kernels.hpp:149-170
    const R lam = std::sqrt(R(3)) / len;
    LeafModel<R> m;
    m.F = Mat<R>(2, 2);
    m.F(0, 1) = R(1); m.F(1, 0) = -lam * lam; m.F(1, 1) = R(-2) * lam;
    m.H = {R(1), R(0)};
    m.Pinf = Mat<R>(2, 2);
    m.Pinf(0, 0) = var; m.Pinf(1, 1) = var * lam * lam;
    Mat<R> dF(2, 2);
    dF(1, 0) = R(2) * lam * lam / len; dF(1, 1) = R(2) * lam / len;
    Mat<R> dP(2, 2);
    dP(1, 1) = R(-2) * var * lam * lam / len;
    m.dF = {Mat<R>(2, 2), dF};
    m.dPinf = {(R(1) / var) * m.Pinf, dP};
    m.fconst = {1, 0};
    return m;
}

template <class R>
LeafModel<R> matern52_ss(R var, R len) {  // kernels.hpp:172-200
    const R lam = std::sqrt(R(5)) / len;
    const R kap = lam * lam / R(3);
    LeafModel<R> m;
    m.F = Mat<R>(3, 3);
    m.F(0, 1) = R(1); m.F(1, 2) = R(1);
    m.F(2, 0) = -lam * lam * lam; m.F(2, 1) = R(-3) * lam * lam; m.F(2, 2) = R(-3) * lam;
    m.H = {R(1), R(0), R(0)};
    m.Pinf = Mat<R>(3, 3);
    m.Pinf(0, 0) = var; m.Pinf(1, 1) = var * kap; m.Pinf(2, 2) = var * lam * lam * lam * lam;
    m.Pinf(0, 2) = m.Pinf(2, 0) = -var * kap;
    Mat<R> dF(3, 3);
    for (int k = 0; k < 3; ++k) dF(2, k) = -(R(3) - R(k)) / len * m.F(2, k);
    Mat<R> dP(3, 3);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) dP(i, j) = -R(i + j) / len * m.Pinf(i, j);
    m.dF = {Mat<R>(3, 3), dF};
    m.dPinf = {(R(1) / var) * m.Pinf, dP};
    m.fconst = {1, 0};
    return m;
}

// Roots of the monic polynomial z^J + sum_{k<J} c_k z^k by Aberth–Ehrlich
// iteration (stands in for the companion-matrix EigenSolver of kernels.hpp:218;
// the 4 Newton steps of :225-235 that follow make the result independent of it).
template <class R>
std::vector<std::complex<R>> poly_roots(const std::vector<R>& c) {
    using C = std::complex<R>;
    const int J = static_cast<int>(c.size());
    auto eval = [&](C z, C& dp) {
        C p = 1, d = 0;
        for (int k = J - 1; k >= 0; --k) {  // Horner on z^J + ... : p = z*p + c_k
            d = d * z + p;
            p = p * z + c[k];
        }
        dp = d;
        return p;
    };
    R rad = 0;
    for (R v : c) rad = std::max(rad, std::abs(v));
    rad = R(1) + rad;
    std::vector<C> z(J);
    for (int k = 0; k < J; ++k) {
        const R ang = R(2) * R(3.14159265358979323846264338327950288L) * (R(k) + R(0.25)) / R(J);
        z[k] = C(R(0.5) * rad * std::cos(ang), R(0.5) * rad * std::sin(ang));
    }
    for (int it = 0; it < 500; ++it) {
        R maxstep = 0;
        for (int k = 0; k < J; ++k) {
            C dp;
            const C p = eval(z[k], dp);
            if (p == C(0)) continue;
            const C ratio = p / dp;
            C s = 0;
            for (int m = 0; m < J; ++m)
                if (m != k) s += C(1) / (z[k] - z[m]);
            const C w = ratio / (C(1) - ratio * s);
            z[k] -= w;
            maxstep = std::max(maxstep, std::abs(w) / std::max(R(1e-300), std::abs(z[k])));
        }
        if (maxstep < R(16) * std::numeric_limits<R>::epsilon()) break;
    }
    return z;
}

template <class R>
std::vector<std::complex<R>> truncated_exp_roots(int j) {  // kernels.hpp:205-239
    using C = std::complex<R>;
    std::vector<R> c(j);
    for (int k = 0; k < j; ++k) {
        R v = 1;
        for (int i = k + 1; i <= j; ++i) v *= R(i);
        v /= std::pow(R(j), R(j - k));
        c[k] = v;
    }
    std::vector<C> z = poly_roots(c);
    std::vector<C> roots(j);
    for (int k = 0; k < j; ++k) {
        C y = z[k] * R(j);
        for (int it = 0; it < 4; ++it) {
            C t = 1, tp = 0, term = 1;
            for (int i = 1; i <= j; ++i) {
                tp += term;
                term *= y / R(i);
                t += term;
            }
            if (std::abs(tp) == R(0)) break;
            y -= t / tp;
        }
        roots[k] = y;
    }
    return roots;
}

template <class R>
LeafModel<R> eq_approx_ss(R sigma2, R lengthscale, int order) {  // kernels.hpp:255-321
    using C = std::complex<R>;
    check_positive(sigma2, "eq var");
    check_positive(lengthscale, "eq len");
    if (order < 2 || order % 2 != 0)
        throw std::invalid_argument("eq approximation order must be even and >= 2");
    if (order > 16)
        throw std::invalid_argument("eq approximation order above 16 is numerically unusable");
    const int j = order;
    const auto yroots = truncated_exp_roots<R>(j);
    std::vector<C> roots;
    for (C y : yroots) {
        C r = std::sqrt(R(-2) * y);
        if (r.real() > R(0)) r = -r;
        if (!(r.real() < R(0))) throw std::runtime_error("eq kernel: root on the imaginary axis");
        roots.push_back(r);
    }
    std::vector<C> upper;
    for (C r : roots)
        if (r.imag() > R(0)) upper.push_back(r);
    if (2 * upper.size() != roots.size())
        throw std::runtime_error("eq kernel: roots did not split into conjugate pairs");
    std::sort(upper.begin(), upper.end(), [](C a, C b) {
        return a.real() != b.real() ? a.real() < b.real() : a.imag() < b.imag();
    });
    LeafModel<R> m;
    m.F = Mat<R>(j, j);
    m.H.assign(j, R(0));
    Mat<R> g(j, 1);
    for (size_t p = 0; p < upper.size(); ++p) {
        const C r = upper[p];
        C denom(1, 0);
        for (C other : roots)
            if (other != r) denom *= (r - other);
        const C res = C(1) / denom;
        const int k = static_cast<int>(2 * p);
        m.F(k, k) = r.real() / lengthscale;
        m.F(k, k + 1) = r.imag() / lengthscale;
        m.F(k + 1, k) = -r.imag() / lengthscale;
        m.F(k + 1, k + 1) = r.real() / lengthscale;
        m.H[k] = R(2) * res.real();
        m.H[k + 1] = R(2) * res.imag();
        g(k, 0) = R(1);
    }
    const Mat<R> mm = lengthscale * m.F;
    const Mat<R> p1 = solve_continuous_lyapunov(mm, g * tr(g));
    R k0 = 0;
    for (int a = 0; a < j; ++a)
        for (int bb = 0; bb < j; ++bb) k0 += m.H[a] * p1(a, bb) * m.H[bb];
    if (!(k0 > R(0))) throw std::runtime_error("eq kernel: non-positive variance");
    m.Pinf = (sigma2 / k0) * p1;
    m.dF = {Mat<R>(j, j), (R(-1) / lengthscale) * m.F};
    m.dPinf = {(R(1) / sigma2) * m.Pinf, Mat<R>(j, j)};
    m.fconst = {1, 0};
    return m;
}

// Quasi-periodic leaf: sigma^2 * k_per(tau; period, len) * exp(-|tau|/env), with
// k_per(tau) = exp(-2 sin^2(pi tau / period) / len^2) expanded in cosines and
// truncated at J harmonics (Solin & Särkkä 2014):  k_per ≈ sum_j q_j^2 cos(j w0 tau),
// q_0^2 = I_0(len^-2) e^{-len^-2},  q_j^2 = 2 I_j(len^-2) e^{-len^-2},  w0 = 2 pi / period.
// Harmonic j is a 2x2 block F_j = [[-1/env, -j w0], [j w0, -1/env]],
// Pinf_j = sigma^2 q_j^2 I_2, H_j = [1, 0].  State dimension 2(J+1).
// Hyperparameters (var, len, period, env).  NOT in the reference.
template <class R>
R bessel_i(int nu, R x) {
    if constexpr (std::is_same_v<R, long double>) return std::cyl_bessel_il(R(nu), x);
    else return std::cyl_bessel_i(R(nu), x);
}

template <class R>
LeafModel<R> qp_ss(R var, R len, R period, R env, int J) {
    if (J < 0 || J > 15) throw std::invalid_argument("qp harmonics must be in [0, 15]");
    const int b = 2 * (J + 1);
    const R pi = R(3.14159265358979323846264338327950288L);
    const R w0 = R(2) * pi / period;
    const R x = R(1) / (len * len);
    const R ex = std::exp(-x);
    LeafModel<R> m;
    m.F = Mat<R>(b, b);
    m.Pinf = Mat<R>(b, b);
    m.H.assign(b, R(0));
    Mat<R> dP_len(b, b), dF_per(b, b), dF_env(b, b);
    for (int j = 0; j <= J; ++j) {
        const int k = 2 * j;
        const R cj = j == 0 ? R(1) : R(2);
        const R q2 = cj * bessel_i<R>(j, x) * ex;
        // d q2 / dx = cj e^{-x} (I_j'(x) - I_j(x)),  I_j' = (I_{j-1} + I_{j+1}) / 2
        const R ip = j == 0 ? bessel_i<R>(1, x)
                            : R(0.5) * (bessel_i<R>(j - 1, x) + bessel_i<R>(j + 1, x));
        const R dq2dx = cj * ex * (ip - bessel_i<R>(j, x));
        const R dq2dlen = dq2dx * (R(-2) / (len * len * len));
        m.F(k, k) = R(-1) / env;
        m.F(k + 1, k + 1) = R(-1) / env;
        m.F(k, k + 1) = -R(j) * w0;
        m.F(k + 1, k) = R(j) * w0;
        m.Pinf(k, k) = var * q2;
        m.Pinf(k + 1, k + 1) = var * q2;
        m.H[k] = R(1);
        dP_len(k, k) = var * dq2dlen;
        dP_len(k + 1, k + 1) = var * dq2dlen;
        const R dw = -w0 / period;  // d w0 / d period
        dF_per(k, k + 1) = -R(j) * dw;
        dF_per(k + 1, k) = R(j) * dw;
        dF_env(k, k) = R(1) / (env * env);
        dF_env(k + 1, k + 1) = R(1) / (env * env);
    }
    m.dF = {Mat<R>(b, b), Mat<R>(b, b), dF_per, dF_env};
    m.dPinf = {(R(1) / var) * m.Pinf, dP_len, Mat<R>(b, b), Mat<R>(b, b)};
    m.fconst = {1, 1, 0, 0};
    return m;
}

// state_space_of (kernels.hpp:326-381): Sum = block-diagonal concatenation.
template <class R>
Model<R> state_space_of(const std::vector<Leaf>& leaves, const std::vector<R>& theta) {
    int nt = 0;
    for (const Leaf& l : leaves) nt += leaf_nparams(l.type);
    if (leaves.empty()) throw std::invalid_argument("kernel has no leaves");
    if (static_cast<int>(theta.size()) != nt)
        throw std::invalid_argument("theta size does not match kernel parameter count");
    std::vector<LeafModel<R>> parts;
    int off = 0, total = 0;
    for (const Leaf& l : leaves) {
        const R var = theta[off], len = theta[off + 1];
        check_positive(var, "var");
        check_positive(len, "len");
        switch (l.type) {
            case MATERN12: parts.push_back(matern12_ss(var, len)); break;
            case MATERN32: parts.push_back(matern32_ss(var, len)); break;
            case MATERN52: parts.push_back(matern52_ss(var, len)); break;
            case EQ: parts.push_back(eq_approx_ss(var, len, l.order)); break;
            case QP:
                check_positive(theta[off + 2], "period");
                check_positive(theta[off + 3], "env");
                parts.push_back(qp_ss(var, len, theta[off + 2], theta[off + 3], l.order));
                break;
            default: throw std::invalid_argument("unknown kernel variant");
        }
        total += parts.back().F.r;
        off += leaf_nparams(l.type);
    }
    Model<R> m;
    m.b = total;
    m.F = Mat<R>(total, total);
    m.Pinf = Mat<R>(total, total);
    m.H.assign(total, R(0));
    int o = 0;
    for (const auto& p : parts) {
        const int d = p.F.r;
        for (int i = 0; i < d; ++i) {
            m.H[o + i] = p.H[i];
            for (int j = 0; j < d; ++j) {
                m.F(o + i, o + j) = p.F(i, j);
                m.Pinf(o + i, o + j) = p.Pinf(i, j);
            }
        }
        for (size_t q = 0; q < p.dF.size(); ++q) {
            Mat<R> dF(total, total), dP(total, total);
            for (int i = 0; i < d; ++i)
                for (int j = 0; j < d; ++j) {
                    dF(o + i, o + j) = p.dF[q](i, j);
                    dP(o + i, o + j) = p.dPinf[q](i, j);
                }
            m.dF.push_back(dF);
            m.dPinf.push_back(dP);
            m.fconst.push_back(p.fconst[q]);
        }
        o += d;
    }
    return m;
}

// ---------------------------------------------------------------- discretise --
template <class R>
struct Step {
    Mat<R> Phi, Q;
    std::vector<Mat<R>> dPhi, dQ;
};

template <class R>
Step<R> discretize(const Model<R>& m, R dt, bool grad) {  // kernels.hpp:392-443
    const int b = m.b;
    Step<R> st;
    if (dt < R(0) || !std::isfinite(static_cast<double>(dt)))
        throw std::invalid_argument("dt must be >= 0");
    if (dt == R(0)) {
        st.Phi = Mat<R>::identity(b);
        st.Q = Mat<R>(b, b);
        if (grad)
            for (int p = 0; p < m.ntheta(); ++p) {
                st.dPhi.emplace_back(b, b);
                st.dQ.emplace_back(b, b);
            }
        return st;
    }
    st.Phi = expm(dt * m.F);
    st.Q = sym(m.Pinf - st.Phi * m.Pinf * tr(st.Phi));
    if (grad) {
        const Mat<R> PhiT = tr(st.Phi);
        for (int p = 0; p < m.ntheta(); ++p) {
            Mat<R> dphi = m.fconst[p] ? Mat<R>(b, b) : expm_frechet(m.F, m.dF[p], dt);
            Mat<R> dq = m.dPinf[p] - dphi * m.Pinf * PhiT - st.Phi * m.dPinf[p] * PhiT -
                        st.Phi * m.Pinf * tr(dphi);
            st.dPhi.push_back(dphi);
            st.dQ.push_back(sym(dq));
        }
    }
    return st;
}

template <class R>
R implied_covariance(const Model<R>& m, R tau) {  // kernels.hpp:446-450
    const R t = std::abs(tau);
    Mat<R> P = t == R(0) ? m.Pinf : expm(t * m.F) * m.Pinf;
    R s = 0;
    for (int i = 0; i < m.b; ++i)
        for (int j = 0; j < m.b; ++j) s += m.H[i] * P(i, j) * m.H[j];
    return s;
}

// ---------------------------------------------------------------- parallel for
template <class F>
void parallel_for(int64_t n, int threads, F&& body) {
    if (threads <= 1 || n < 2 * threads) {
        body(int64_t(0), n);
        return;
    }
    std::vector<std::thread> pool;
    const int64_t chunk = (n + threads - 1) / threads;
    for (int k = 0; k < threads; ++k) {
        const int64_t lo = k * chunk, hi = std::min(n, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back([&, lo, hi] { body(lo, hi); });
    }
    for (auto& th : pool) th.join();
}

// ---------------------------------------------------------------- BTD core ----
// Symmetric block-tridiagonal matrix.
template <class R>
struct SymBTD {
    int64_t n = 0;
    int b = 0;
    std::vector<Mat<R>> diag, upper;
};

// Block Thomas / LDL^T with Cholesky pivots.
template <class R>
struct Factor {
    std::vector<Mat<R>> L;     // chol(S_i)
    std::vector<Mat<R>> G;     // S_i^{-1} U_i
    R logdet = 0;
};

template <class R>
Factor<R> thomas_factor(const SymBTD<R>& m) {
    Factor<R> f;
    f.L.resize(m.n);
    f.G.resize(m.n > 0 ? m.n - 1 : 0);
    Mat<R> S = m.diag[0];
    for (int64_t i = 0; i < m.n; ++i) {
        if (i > 0) S = sym(m.diag[i] - tr(m.upper[i - 1]) * f.G[i - 1]);  // pivot symmetrisation :219
        if (!cholesky(S, f.L[i]))
            throw Failure{NOT_PD, i, "factorize: pivot block is not positive definite"};
        f.logdet += chol_logdet(f.L[i]);
        if (i + 1 < m.n) f.G[i] = chol_solve(f.L[i], m.upper[i]);
    }
    return f;
}

// rhs as n blocks of b x k.
template <class R>
std::vector<Mat<R>> thomas_solve(const SymBTD<R>& m, const Factor<R>& f,
                                 std::vector<Mat<R>> z) {
    for (int64_t i = 1; i < m.n; ++i) z[i] = z[i] - tr(f.G[i - 1]) * z[i - 1];
    z[m.n - 1] = chol_solve(f.L[m.n - 1], z[m.n - 1]);
    for (int64_t i = m.n - 2; i >= 0; --i) z[i] = chol_solve(f.L[i], z[i]) - f.G[i] * z[i + 1];
    return z;
}

// Takahashi selected inverse: C_{n-1} = S^{-1}; C_{i,i+1} = -G_i C_{i+1,i+1};
// C_ii = S_i^{-1} - C_{i,i+1} G_i^T.
template <class R>
void takahashi(const SymBTD<R>& m, const Factor<R>& f, std::vector<Mat<R>>& Cd,
               std::vector<Mat<R>>& Cu) {
    const int b = m.b;
    Cd.assign(m.n, Mat<R>());
    Cu.assign(m.n > 0 ? m.n - 1 : 0, Mat<R>());
    Cd[m.n - 1] = sym(chol_solve(f.L[m.n - 1], Mat<R>::identity(b)));
    for (int64_t i = m.n - 2; i >= 0; --i) {
        Cu[i] = R(-1) * (f.G[i] * Cd[i + 1]);
        Cd[i] = sym(chol_solve(f.L[i], Mat<R>::identity(b)) - Cu[i] * tr(f.G[i]));
    }
}

// ---------------------------------------------------------------- engine ------
constexpr double kJitter = 1e-10;  // + 1e-10 * tr(Pinf) / b * I on every Q_i

template <class R>
struct EvalOut {
    R loglik = 0;
    std::vector<R> grad;   // n_theta + 1 (sigma last)
    std::vector<R> mean, var;
    // diagnostics
    R logdetP = 0, logdetQ = 0, fit_y = 0, fit_e = 0;
};

struct EvalFlags {
    bool grad = false, mean = false, var = false, include_noise = false;
};

template <class R>
void check_times(const double* t, int64_t n) {
    for (int64_t i = 1; i < n; ++i) {
        if (!(t[i] >= t[i - 1]) || !std::isfinite(t[i]))
            throw Failure{BAD_ARG, i, "times must be strictly increasing"};
        if (t[i] == t[i - 1]) throw Failure{DUPLICATE_TIME, i, "duplicate training timestamp"};
    }
}

// Per-step discretisation with jitter: Qt_i = Q_i + jit I (Q_0 := Pinf), Qt_i^{-1}.
template <class R>
struct Discretised {
    std::vector<Mat<R>> Phi, Qinv;              // Phi[0] unused
    std::vector<R> logdetQ;
    std::vector<std::vector<Mat<R>>> dPhi, dQt;  // per step, per theta
};

template <class R>
Discretised<R> discretise_all(const Model<R>& m, const double* t, int64_t n, bool grad,
                              int threads) {
    const int b = m.b, nt = m.ntheta();
    const R jit = R(kJitter) * trace(m.Pinf) / R(b);
    std::vector<R> djit(nt);
    for (int p = 0; p < nt; ++p) djit[p] = R(kJitter) * trace(m.dPinf[p]) / R(b);
    Discretised<R> d;
    d.Phi.resize(n);
    d.Qinv.resize(n);
    d.logdetQ.resize(n);
    if (grad) { d.dPhi.resize(n); d.dQt.resize(n); }
    std::vector<int64_t> fail(threads > 0 ? threads : 1, -1);
    parallel_for(n, threads, [&](int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            Mat<R> Qt;
            if (i == 0) {
                d.Phi[0] = Mat<R>::identity(b);
                Qt = m.Pinf;
                if (grad) {
                    d.dPhi[0].assign(nt, Mat<R>(b, b));
                    d.dQt[0] = m.dPinf;
                }
            } else {
                const R dt = R(t[i]) - R(t[i - 1]);
                Step<R> st = discretize(m, dt, grad);
                d.Phi[i] = st.Phi;
                Qt = st.Q;
                if (grad) {
                    d.dPhi[i] = st.dPhi;
                    d.dQt[i] = st.dQ;
                }
            }
            for (int k = 0; k < b; ++k) Qt(k, k) += jit;
            if (grad)
                for (int p = 0; p < nt; ++p)
                    for (int k = 0; k < b; ++k) d.dQt[i][p](k, k) += djit[p];
            Mat<R> L;
            if (!cholesky(Qt, L)) {
                d.logdetQ[i] = std::numeric_limits<R>::quiet_NaN();
                continue;
            }
            d.logdetQ[i] = chol_logdet(L);
            d.Qinv[i] = sym(chol_solve(L, Mat<R>::identity(b)));
        }
    });
    for (int64_t i = 0; i < n; ++i)
        if (std::isnan(static_cast<double>(d.logdetQ[i])))
            throw Failure{SINGULAR_Q, i, "process noise block singular after jitter"};
    return d;
}

// assemble_prior_precision + add_observation_term.
template <class R>
SymBTD<R> assemble(const Model<R>& m, const Discretised<R>& d, int64_t n, R sigma,
                   const unsigned char* observed, int threads) {
    const int b = m.b;
    SymBTD<R> P;
    P.n = n;
    P.b = b;
    P.diag.resize(n);
    P.upper.resize(n > 0 ? n - 1 : 0);
    const R s2 = sigma * sigma;
    parallel_for(n, threads, [&](int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            Mat<R> D = d.Qinv[i];
            if (i + 1 < n) {
                const Mat<R> PtQ = tr(d.Phi[i + 1]) * d.Qinv[i + 1];
                D = D + PtQ * d.Phi[i + 1];
                P.upper[i] = R(-1) * PtQ;
            }
            if (!observed || observed[i])
                for (int a = 0; a < b; ++a)
                    for (int c = 0; c < b; ++c) D(a, c) += m.H[a] * m.H[c] / s2;
            P.diag[i] = sym(D);
        }
    });
    return P;
}

// loglik (+ gradient, mean, var): SPEC.md:280-306 via SURVEY.md Appendix B.
template <class R>
EvalOut<R> evaluate(const Model<R>& m, const double* t, const double* y, int64_t n, R sigma,
                    EvalFlags fl, int threads) {
    if (n < 1) throw Failure{BAD_ARG, 0, "need at least one observation"};
    if (!(sigma > R(0))) throw Failure{BAD_ARG, 0, "sigma must be positive"};
    check_times<R>(t, n);
    const int b = m.b, nt = m.ntheta();
    const Discretised<R> d = discretise_all(m, t, n, fl.grad, threads);
    const SymBTD<R> P = assemble(m, d, n, sigma, nullptr, threads);
    const Factor<R> f = thomas_factor(P);
    const R s2 = sigma * sigma;
    std::vector<Mat<R>> rhs(n, Mat<R>(b, 1));
    for (int64_t i = 0; i < n; ++i)
        for (int a = 0; a < b; ++a) rhs[i](a, 0) = m.H[a] * R(y[i]) / s2;
    const std::vector<Mat<R>> mu = thomas_solve(P, f, rhs);
    std::vector<Mat<R>> Cd, Cu;
    const bool need_C = fl.grad || fl.var;
    if (need_C) takahashi(P, f, Cd, Cu);

    EvalOut<R> out;
    auto Hx = [&](const Mat<R>& v) {
        R s = 0;
        for (int a = 0; a < b; ++a) s += m.H[a] * v(a, 0);
        return s;
    };
    auto HCH = [&](const Mat<R>& C) {
        R s = 0;
        for (int a = 0; a < b; ++a)
            for (int c = 0; c < b; ++c) s += m.H[a] * C(a, c) * m.H[c];
        return s;
    };
    // per-step terms, summed afterwards in index order (deterministic for any thread count)
    std::vector<R> fit_y(n), fit_e(n), noise_t(n);
    std::vector<R> gterm(fl.grad ? static_cast<size_t>(n) * nt : 0);
    parallel_for(n, threads, [&](int64_t lo, int64_t hi) {
        for (int64_t i = lo; i < hi; ++i) {
            const R r = R(y[i]) - Hx(mu[i]);
            fit_y[i] = r * r / s2;
            Mat<R> e = mu[i];
            if (i > 0) e = e - d.Phi[i] * mu[i - 1];
            fit_e[i] = (tr(e) * d.Qinv[i] * e)(0, 0);
            if (fl.grad) {
                noise_t[i] = r * r + HCH(Cd[i]);
                Mat<R> E, Z;
                if (i == 0) {
                    E = Cd[0] + mu[0] * tr(mu[0]);
                } else {
                    const Mat<R>& Ph = d.Phi[i];
                    const Mat<R> PC = Ph * Cu[i - 1];  // Phi C_{i-1,i}
                    E = Cd[i] - PC - tr(PC) + Ph * Cd[i - 1] * tr(Ph) + e * tr(e);
                    Z = Cu[i - 1] - Cd[i - 1] * tr(Ph) + mu[i - 1] * tr(e);
                }
                const Mat<R> A = d.Qinv[i] * E * d.Qinv[i];
                const Mat<R> B = i > 0 ? Z * d.Qinv[i] : Mat<R>();
                for (int p = 0; p < nt; ++p) {
                    R g = R(-0.5) * trace_prod(d.Qinv[i], d.dQt[i][p]) +
                          R(0.5) * trace_prod(A, d.dQt[i][p]);
                    if (i > 0) g += trace_prod(d.dPhi[i][p], B);  // Tr(Qinv dPhi Z)
                    gterm[static_cast<size_t>(i) * nt + p] = g;
                }
            }
        }
    });
    R sy = 0, se = 0, ldq = 0;
    for (int64_t i = 0; i < n; ++i) {
        sy += fit_y[i];
        se += fit_e[i];
        ldq += d.logdetQ[i];
    }
    const R pi = R(3.14159265358979323846264338327950288L);
    out.fit_y = sy;
    out.fit_e = se;
    out.logdetP = f.logdet;
    out.logdetQ = ldq;
    out.loglik = R(-0.5) * (sy + se) - R(0.5) * (f.logdet + ldq + R(n) * std::log(s2)) -
                 R(0.5) * R(n) * std::log(R(2) * pi);
    if (fl.grad) {
        out.grad.assign(nt + 1, R(0));
        for (int64_t i = 0; i < n; ++i)
            for (int p = 0; p < nt; ++p) out.grad[p] += gterm[static_cast<size_t>(i) * nt + p];
        R sn = 0;
        for (int64_t i = 0; i < n; ++i) sn += noise_t[i];
        out.grad[nt] = R(2) * sigma * (R(-0.5) * R(n) / s2 + sn / (R(2) * s2 * s2));
    }
    if (fl.mean) {
        out.mean.resize(n);
        for (int64_t i = 0; i < n; ++i) out.mean[i] = Hx(mu[i]);
    }
    if (fl.var) {
        out.var.resize(n);
        for (int64_t i = 0; i < n; ++i) {
            R v = HCH(Cd[i]);
            if (v < R(-1e-10)) throw Failure{NEG_VARIANCE, i, "negative posterior variance"};
            if (v < R(0)) v = 0;  // clamp [-1e-10, 0) -> 0
            out.var[i] = fl.include_noise ? v + s2 : v;
        }
    }
    return out;
}


// ------------------------------------------------------------- Kalman / RTS ----
// The sequential state-space oracle of SPEC.md:379-396 (kf_mll, kf_rts_predict): a
// Kalman filter over the (merged) time grid, observations masked by `observed` (a test
// time is a missing observation: the update is skipped, SPEC.md DESIGN DECISIONS), MLL by
// the prediction-error decomposition Σ ln N(y_i; H m_i^-, H P_i^- H^T + σ²), then a
// Rauch-Tung-Striebel backward pass.  The transition is the same jittered discretisation
// the precision uses (Q̃_i = Q_i + jit I, Q̃_0 = P∞ + jit I), so the
// three oracles (dense, KF/RTS, sparse precision) describe one model.  Covariances are
// symmetrised after every update (SPEC.md DESIGN DECISIONS).
template <class R>
struct KfOut {
    R loglik = 0;
    std::vector<R> mean, var, fvar;  // smoothed H m^s, H P^s H^T; filtered H P H^T
};

template <class R>
KfOut<R> kf_rts(const Model<R>& m, const double* t, const double* y, const unsigned char* observed,
                int64_t n, R sigma) {
    const int b = m.b;
    const R s2 = sigma * sigma;
    const R jit = R(kJitter) * trace(m.Pinf) / R(b);
    std::vector<Mat<R>> Phi(n), mf(n), Pf(n), mp(n), Pp(n);
    auto HPH = [&](const Mat<R>& P) {
        R v = 0;
        for (int i = 0; i < b; ++i)
            for (int j = 0; j < b; ++j) v += m.H[i] * P(i, j) * m.H[j];
        return v;
    };
    KfOut<R> out;
    const R kLog2Pi = R(1.8378770664093454835606594728112L);
    for (int64_t i = 0; i < n; ++i) {
        Mat<R> Qt;
        if (i == 0) {
            Phi[0] = Mat<R>::identity(b);
            Qt = m.Pinf;
            mp[0] = Mat<R>(b, 1);
        } else {
            const R dt = R(t[i]) - R(t[i - 1]);
            if (!(dt > R(0))) throw Failure{DUPLICATE_TIME, i, "duplicate training timestamp"};
            const Step<R> st = discretize(m, dt, false);
            Phi[i] = st.Phi;
            Qt = st.Q;
            mp[i] = Phi[i] * mf[i - 1];
        }
        for (int k = 0; k < b; ++k) Qt(k, k) += jit;
        Pp[i] = i == 0 ? Qt : sym(Phi[i] * Pf[i - 1] * tr(Phi[i]) + Qt);
        if (observed && !observed[i]) {
            mf[i] = mp[i];
            Pf[i] = Pp[i];
            continue;
        }
        Mat<R> PH(b, 1);
        for (int a = 0; a < b; ++a)
            for (int c = 0; c < b; ++c) PH(a, 0) += Pp[i](a, c) * m.H[c];
        R hm = 0, S = s2;
        for (int a = 0; a < b; ++a) {
            hm += m.H[a] * mp[i](a, 0);
            S += m.H[a] * PH(a, 0);
        }
        if (!(S > R(0))) throw Failure{NOT_PD, i, "innovation variance <= 0"};
        const R v = R(y[i]) - hm;
        out.loglik += R(-0.5) * (kLog2Pi + std::log(S) + v * v / S);
        mf[i] = mp[i];
        Pf[i] = Pp[i];
        for (int a = 0; a < b; ++a) {
            mf[i](a, 0) += PH(a, 0) * v / S;
            for (int c = 0; c < b; ++c) Pf[i](a, c) -= PH(a, 0) * PH(c, 0) / S;
        }
        Pf[i] = sym(Pf[i]);
    }
    out.mean.resize(n);
    out.var.resize(n);
    out.fvar.resize(n);
    Mat<R> ms = mf[n - 1], Ps = Pf[n - 1];
    for (int64_t i = n - 1; i >= 0; --i) {
        if (i < n - 1) {
            // G = P_i Φ_{i+1}^T (P^-_{i+1})^{-1}:  G^T = (P^-_{i+1})^{-1} Φ_{i+1} P_i
            Mat<R> Lp;
            if (!cholesky(Pp[i + 1], Lp)) throw Failure{NOT_PD, i + 1, "predictive covariance not PD"};
            const Mat<R> G = tr(chol_solve(Lp, Phi[i + 1] * Pf[i]));
            ms = mf[i] + G * (ms - mp[i + 1]);
            Ps = sym(Pf[i] + G * (Ps - Pp[i + 1]) * tr(G));
        }
        R hm = 0;
        for (int a = 0; a < b; ++a) hm += m.H[a] * ms(a, 0);
        out.mean[i] = hm;
        out.var[i] = HPH(Ps);
        out.fvar[i] = HPH(Pf[i]);
    }
    return out;
}

}  // namespace oracle
