#pragma once
// Small Eigen-free dense matrix used by the drop-in C++ API.
//
// The reference stores model and step matrices as Eigen::MatrixXd /
// Eigen::RowVectorXd (kernels.hpp:111-128,385-390).  Eigen is not available in
// this image, so the API exposes this row-major type instead; it keeps the
// accessors the reference code and tests use: (i, j), rows(), cols(), data(),
// size(), Zero/Identity/Constant, transpose(), block arithmetic.  This is the one
// deliberate API deviation.

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <initializer_list>
#include <stdexcept>
#include <vector>

namespace spingp {

using Index = std::ptrdiff_t;

class Matrix {
public:
    Matrix() = default;
    Matrix(Index r, Index c, double v = 0.0) : r_(r), c_(c), a_(static_cast<size_t>(r * c), v) {}

    static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
    static Matrix Constant(Index r, Index c, double v) { return Matrix(r, c, v); }
    static Matrix Identity(Index n, Index = -1) {
        Matrix m(n, n);
        for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
    static Matrix RowOnes(Index n) { return Matrix(1, n, 1.0); }

    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double* data() { return a_.data(); }
    const double* data() const { return a_.data(); }

    double& operator()(Index i, Index j) { return a_[static_cast<size_t>(i * c_ + j)]; }
    double operator()(Index i, Index j) const { return a_[static_cast<size_t>(i * c_ + j)]; }
    // vector-style access for 1 x n / n x 1 matrices (RowVectorXd in the reference)
    double& operator()(Index k) { return a_[static_cast<size_t>(k)]; }
    double operator()(Index k) const { return a_[static_cast<size_t>(k)]; }

    void setZero(Index r, Index c) { *this = Matrix(r, c); }
    void setZero(Index n) { *this = Matrix(1, n); }  // RowVectorXd::setZero(n)
    void setZero() { std::fill(a_.begin(), a_.end(), 0.0); }

    Matrix transpose() const {
        Matrix t(c_, r_);
        for (Index i = 0; i < r_; ++i)
            for (Index j = 0; j < c_; ++j) t(j, i) = (*this)(i, j);
        return t;
    }
    double trace() const {
        double s = 0;
        for (Index i = 0; i < std::min(r_, c_); ++i) s += (*this)(i, i);
        return s;
    }
    double norm() const {  // Frobenius
        double s = 0;
        for (double v : a_) s += v * v;
        return std::sqrt(s);
    }
    double maxAbs() const {
        double s = 0;
        for (double v : a_) s = std::max(s, std::abs(v));
        return s;
    }
    double value() const { return a_.at(0); }  // 1x1 -> scalar
    bool isZero(double tol = 0.0) const {
        for (double v : a_)
            if (std::abs(v) > tol) return false;
        return true;
    }
    bool isIdentity(double tol = 0.0) const {
        for (Index i = 0; i < r_; ++i)
            for (Index j = 0; j < c_; ++j)
                if (std::abs((*this)(i, j) - (i == j ? 1.0 : 0.0)) > tol) return false;
        return true;
    }
    Matrix block(Index i0, Index j0, Index nr, Index nc) const {
        Matrix b(nr, nc);
        for (Index i = 0; i < nr; ++i)
            for (Index j = 0; j < nc; ++j) b(i, j) = (*this)(i0 + i, j0 + j);
        return b;
    }
    void setBlock(Index i0, Index j0, const Matrix& b) {
        for (Index i = 0; i < b.rows(); ++i)
            for (Index j = 0; j < b.cols(); ++j) (*this)(i0 + i, j0 + j) = b(i, j);
    }

    Matrix& operator+=(const Matrix& o) {
        check_same(o);
        for (size_t i = 0; i < a_.size(); ++i) a_[i] += o.a_[i];
        return *this;
    }
    Matrix& operator-=(const Matrix& o) {
        check_same(o);
        for (size_t i = 0; i < a_.size(); ++i) a_[i] -= o.a_[i];
        return *this;
    }
    Matrix& operator*=(double s) {
        for (double& v : a_) v *= s;
        return *this;
    }
    Matrix& operator/=(double s) {
        for (double& v : a_) v /= s;
        return *this;
    }
    friend Matrix operator+(Matrix a, const Matrix& b) { return a += b; }
    friend Matrix operator-(Matrix a, const Matrix& b) { return a -= b; }
    friend Matrix operator-(Matrix a) { return a *= -1.0; }
    friend Matrix operator*(Matrix a, double s) { return a *= s; }
    friend Matrix operator*(double s, Matrix a) { return a *= s; }
    friend Matrix operator/(Matrix a, double s) { return a /= s; }
    friend Matrix operator*(const Matrix& a, const Matrix& b) {
        if (a.c_ != b.r_) throw std::invalid_argument("matrix product: dimension mismatch");
        Matrix z(a.r_, b.c_);
        for (Index i = 0; i < a.r_; ++i)
            for (Index k = 0; k < a.c_; ++k) {
                const double v = a(i, k);
                if (v == 0.0) continue;
                for (Index j = 0; j < b.c_; ++j) z(i, j) += v * b(k, j);
            }
        return z;
    }
    bool operator==(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_ && a_ == o.a_; }

private:
    void check_same(const Matrix& o) const {
        if (r_ != o.r_ || c_ != o.c_) throw std::invalid_argument("matrix sum: dimension mismatch");
    }
    Index r_ = 0, c_ = 0;
    std::vector<double> a_;
};

using RowVector = Matrix;  // 1 x n, stands in for Eigen::RowVectorXd

// 0.5 (A + A^T)
inline Matrix symmetrize(const Matrix& a) { return 0.5 * (a + a.transpose()); }

// Solve A X = B by LU with partial pivoting.  Throws on exact singularity.
inline Matrix lu_solve(Matrix A, Matrix B) {
    const Index n = A.rows();
    if (A.cols() != n || B.rows() != n) throw std::invalid_argument("lu_solve: dimension mismatch");
    for (Index k = 0; k < n; ++k) {
        Index p = k;
        for (Index i = k + 1; i < n; ++i)
            if (std::abs(A(i, k)) > std::abs(A(p, k))) p = i;
        if (A(p, k) == 0.0) throw std::runtime_error("lu_solve: singular matrix");
        if (p != k) {
            for (Index j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
            for (Index j = 0; j < B.cols(); ++j) std::swap(B(k, j), B(p, j));
        }
        const double piv = A(k, k);
        for (Index i = k + 1; i < n; ++i) {
            const double f = A(i, k) / piv;
            if (f == 0.0) continue;
            for (Index j = k + 1; j < n; ++j) A(i, j) -= f * A(k, j);
            for (Index j = 0; j < B.cols(); ++j) B(i, j) -= f * B(k, j);
        }
    }
    for (Index k = n - 1; k >= 0; --k)
        for (Index j = 0; j < B.cols(); ++j) {
            double s = B(k, j);
            for (Index m = k + 1; m < n; ++m) s -= A(k, m) * B(m, j);
            B(k, j) = s / A(k, k);
        }
    return B;
}

}  // namespace spingp
