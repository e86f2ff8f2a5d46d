// ORACLE support (test infrastructure only; never part of the product). A small, eager, column-major stand-in for
// the subset of the Eigen 3 API that the reference's hot-path sources use (R/src/{scene,linalg,estimators,
// spectrum}.cpp), so those files compile and run HERE, unmodified and in place, into oracle/_ref (Eigen 3 itself is
// absent from this image: SURVEY.md §0 F3). Dense decompositions call LAPACK (scipy's bundled OpenBLAS):
//   SelfAdjointEigenSolver -> zheevd, JacobiSVD -> zgesvd, BDCSVD -> zgesdd, HouseholderQR -> zgeqrf + zungqr,
//   ColPivHouseholderQR -> zgeqp3 + zungqr with Eigen's rank() rule (maxpivot, nonzero-pivot cut, p * eps).
// The reference's control flow, thresholds, redraws, RNG and peak rules therefore run as written; only the
// decomposition internals are LAPACK's instead of Eigen's (outputs agree up to rounding and unitary freedom, to
// which every quantity the path consumes is invariant: projectors, spectra, peaks).
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <limits>
#include <stdexcept>
#include <type_traits>
#include <vector>

// ILP64 LAPACKE of numpy's bundled OpenBLAS (the same library instance numpy itself uses, so one OpenBLAS per
// process when the oracle is driven from Python)
extern "C" {
using fm_lapack_int = long long;
fm_lapack_int scipy_LAPACKE_zheevd64_(int layout, char jobz, char uplo, fm_lapack_int n, void* a, fm_lapack_int lda,
                                      double* w);
fm_lapack_int scipy_LAPACKE_zgesvd64_(int layout, char jobu, char jobvt, fm_lapack_int m, fm_lapack_int n, void* a,
                                      fm_lapack_int lda, double* s, void* u, fm_lapack_int ldu, void* vt,
                                      fm_lapack_int ldvt, double* superb);
fm_lapack_int scipy_LAPACKE_zgesdd64_(int layout, char jobz, fm_lapack_int m, fm_lapack_int n, void* a,
                                      fm_lapack_int lda, double* s, void* u, fm_lapack_int ldu, void* vt,
                                      fm_lapack_int ldvt);
fm_lapack_int scipy_LAPACKE_zgeqrf64_(int layout, fm_lapack_int m, fm_lapack_int n, void* a, fm_lapack_int lda,
                                      void* tau);
fm_lapack_int scipy_LAPACKE_zungqr64_(int layout, fm_lapack_int m, fm_lapack_int n, fm_lapack_int k, void* a,
                                      fm_lapack_int lda, const void* tau);
fm_lapack_int scipy_LAPACKE_zgeqp364_(int layout, fm_lapack_int m, fm_lapack_int n, void* a, fm_lapack_int lda,
                                      fm_lapack_int* jpvt, void* tau);
// CBLAS of the same library: dense products and the Hermitian rank update run where Eigen would run its own
// blocked, vectorised kernels (the eager loops over std::complex would time libgcc's __muldc3 instead)
void scipy_cblas_zgemm64_(int layout, int ta, int tb, fm_lapack_int m, fm_lapack_int n, fm_lapack_int k,
                          const void* alpha, const void* a, fm_lapack_int lda, const void* b, fm_lapack_int ldb,
                          const void* beta, void* c, fm_lapack_int ldc);
void scipy_cblas_dgemm64_(int layout, int ta, int tb, fm_lapack_int m, fm_lapack_int n, fm_lapack_int k, double alpha,
                          const double* a, fm_lapack_int lda, const double* b, fm_lapack_int ldb, double beta,
                          double* c, fm_lapack_int ldc);
void scipy_cblas_zherk64_(int layout, int uplo, int trans, fm_lapack_int n, fm_lapack_int k, double alpha,
                          const void* a, fm_lapack_int lda, double beta, void* c, fm_lapack_int ldc);
}

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum UpLo { Lower = 1, Upper = 2 };
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum DecompositionOptions { ComputeFullU = 4, ComputeThinU = 8, ComputeFullV = 16, ComputeThinV = 32 };
struct NoChange_t {};
static constexpr NoChange_t NoChange{};

template <typename T>
struct NumTraits {
    using Real = T;
    static constexpr T epsilon() { return std::numeric_limits<T>::epsilon(); }
};
template <typename T>
struct NumTraits<std::complex<T>> {
    using Real = T;
    static constexpr T epsilon() { return std::numeric_limits<T>::epsilon(); }
};

namespace internal {
template <typename A, typename B>
using promote_t = decltype(std::declval<A>() * std::declval<B>());
inline double conj_(double x) { return x; }
inline std::complex<double> conj_(std::complex<double> x) { return std::conj(x); }
inline double abs2_(double x) { return x * x; }
inline double abs2_(std::complex<double> x) { return std::norm(x); }
inline double re_(double x) { return x; }
inline double re_(std::complex<double> x) { return x.real(); }
inline double im_(double) { return 0.0; }
inline double im_(std::complex<double> x) { return x.imag(); }
}  // namespace internal

template <typename S, int R = Dynamic, int C = Dynamic>
class Matrix;
template <typename S>
class DiagonalWrapper;
template <typename M>
class Block;

// ------------------------------------------------------------------ dense matrix (column-major, eager)
template <typename S, int R, int C>
class Matrix {
public:
    using Scalar = S;
    using RealScalar = typename NumTraits<S>::Real;

    Matrix() : r_(R == 1 ? 1 : 0), c_(C == 1 ? 1 : 0) {}
    Matrix(Index r, Index c) : r_(r), c_(c), d_(static_cast<size_t>(r * c)) {}
    explicit Matrix(Index n) : r_(C == 1 ? n : 1), c_(C == 1 ? 1 : n), d_(static_cast<size_t>(n)) {}
    template <int R2, int C2>
    Matrix(const Matrix<S, R2, C2>& o) : r_(o.rows()), c_(o.cols()), d_(o.raw()) {
        if (C == 1 && c_ != 1 && r_ == 1) std::swap(r_, c_);  // row -> column vector
    }
    template <int R2, int C2>
    Matrix& operator=(const Matrix<S, R2, C2>& o) {
        r_ = o.rows();
        c_ = o.cols();
        d_ = o.raw();
        return *this;
    }

    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    S& operator()(Index i, Index j) { return d_[static_cast<size_t>(j * r_ + i)]; }
    const S& operator()(Index i, Index j) const { return d_[static_cast<size_t>(j * r_ + i)]; }
    S& operator()(Index i) { return d_[static_cast<size_t>(i)]; }
    const S& operator()(Index i) const { return d_[static_cast<size_t>(i)]; }
    S* data() { return d_.data(); }
    const S* data() const { return d_.data(); }
    const std::vector<S>& raw() const { return d_; }
    std::vector<S>& raw() { return d_; }

    static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
    static Matrix Zero(Index n) { return Matrix(n); }
    static Matrix Identity(Index r, Index c) {
        Matrix m(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = S(1);
        return m;
    }
    void setZero() { std::fill(d_.begin(), d_.end(), S(0)); }
    void resize(Index r, Index c) {
        r_ = r;
        c_ = c;
        d_.assign(static_cast<size_t>(r * c), S(0));
    }
    void conservativeResize(Index r, Index c) {
        Matrix n(r, c);
        for (Index j = 0; j < std::min(c, c_); ++j)
            for (Index i = 0; i < std::min(r, r_); ++i) n(i, j) = (*this)(i, j);
        *this = n;
    }
    void conservativeResize(NoChange_t, Index c) { conservativeResize(r_, c); }
    Matrix& noalias() { return *this; }

    Matrix<S> adjoint() const {
        Matrix<S> o(c_, r_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) o(j, i) = internal::conj_((*this)(i, j));
        return o;
    }
    Matrix<S> transpose() const {
        Matrix<S> o(c_, r_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i) o(j, i) = (*this)(i, j);
        return o;
    }
    template <typename T>
    Matrix<T, R, C> cast() const {
        Matrix<T, R, C> o(r_, c_);
        for (Index e = 0; e < size(); ++e) o(e) = T(d_[static_cast<size_t>(e)]);
        return o;
    }
    Matrix<RealScalar, R, C> cwiseAbs() const {
        Matrix<RealScalar, R, C> o(r_, c_);
        for (Index e = 0; e < size(); ++e) o(e) = std::abs(d_[static_cast<size_t>(e)]);
        return o;
    }
    Matrix<RealScalar, R, C> real() const {
        Matrix<RealScalar, R, C> o(r_, c_);
        for (Index e = 0; e < size(); ++e) o(e) = internal::re_(d_[static_cast<size_t>(e)]);
        return o;
    }
    Matrix<RealScalar, R, C> imag() const {
        Matrix<RealScalar, R, C> o(r_, c_);
        for (Index e = 0; e < size(); ++e) o(e) = internal::im_(d_[static_cast<size_t>(e)]);
        return o;
    }
    // lvalue views of the real / imaginary parts (c.real() = ..., R/src/estimators.cpp:124-125)
    struct PartRef {
        Matrix* m;
        bool imag;
        template <typename Rhs>
        PartRef& operator=(const Rhs& rhs) {
            const Matrix<RealScalar> v = rhs;
            for (Index e = 0; e < m->size(); ++e) {
                S& x = (*m)(e);
                if constexpr (std::is_same_v<S, std::complex<double>>) x = imag ? S(x.real(), v(e)) : S(v(e), x.imag());
                else if (!imag) x = v(e);
            }
            return *this;
        }
    };
    PartRef real() { return PartRef{this, false}; }
    PartRef imag() { return PartRef{this, true}; }

    RealScalar squaredNorm() const {
        RealScalar s = 0;
        for (const S& x : d_) s += internal::abs2_(x);
        return s;
    }
    RealScalar norm() const { return std::sqrt(squaredNorm()); }
    S sum() const {
        S s = S(0);
        for (const S& x : d_) s += x;
        return s;
    }
    S trace() const {
        S s = S(0);
        for (Index i = 0; i < std::min(r_, c_); ++i) s += (*this)(i, i);
        return s;
    }
    S maxCoeff() const { return *std::max_element(d_.begin(), d_.end()); }
    S minCoeff() const { return *std::min_element(d_.begin(), d_.end()); }
    bool allFinite() const {
        for (const S& x : d_)
            if (!std::isfinite(internal::re_(x)) || !std::isfinite(internal::im_(x))) return false;
        return true;
    }
    Matrix<S, R, C> reverse() const {
        Matrix<S, R, C> o(r_, c_);
        for (Index e = 0; e < size(); ++e) o(e) = d_[static_cast<size_t>(size() - 1 - e)];
        return o;
    }
    struct Rowwise {
        const Matrix* m;
        Matrix<S> reverse() const {  // reverse every row = reverse the column order
            Matrix<S> o(m->rows(), m->cols());
            for (Index j = 0; j < m->cols(); ++j)
                for (Index i = 0; i < m->rows(); ++i) o(i, j) = (*m)(i, m->cols() - 1 - j);
            return o;
        }
    };
    Rowwise rowwise() const { return Rowwise{this}; }
    DiagonalWrapper<S> asDiagonal() const { return DiagonalWrapper<S>(*this); }
    struct Array {
        Matrix<S> v;
        Array operator-(S s) const {
            Array a{v};
            for (auto& x : a.v.raw()) x -= s;
            return a;
        }
        Array operator/(S s) const {
            Array a{v};
            for (auto& x : a.v.raw()) x /= s;
            return a;
        }
        operator Matrix<S, R, C>() const { return v; }
    };
    Array array() const { return Array{*this}; }
    template <int UpLo>
    Matrix<S> triangularView() const {
        Matrix<S> o(r_, c_);
        for (Index j = 0; j < c_; ++j)
            for (Index i = 0; i < r_; ++i)
                if ((UpLo == Upper && i <= j) || (UpLo == Lower && i >= j)) o(i, j) = (*this)(i, j);
        return o;
    }
    // selfadjointView<Lower>(): rankUpdate on the lower triangle; dense conversion mirrors it
    template <int UpLo>
    struct SelfAdjoint {
        Matrix* m;
        const Matrix* cm;
        template <typename Y>
        void rankUpdate(const Y& yy, RealScalar alpha) {
            const Matrix<S> y = yy;
            if constexpr (std::is_same_v<S, std::complex<double>>) {  // lower triangle += alpha y y^H (zherk)
                if (m->rows() > 0 && y.cols() > 0)
                    scipy_cblas_zherk64_(102 /*ColMajor*/, 122 /*Lower*/, 111 /*NoTrans*/, m->rows(), y.cols(), alpha,
                                         y.data(), y.rows(), 1.0, m->data(), m->rows());
                return;
            }
            for (Index j = 0; j < m->cols(); ++j)
                for (Index i = j; i < m->rows(); ++i) {
                    S acc = S(0);
                    for (Index q = 0; q < y.cols(); ++q) acc += y(i, q) * internal::conj_(y(j, q));
                    (*m)(i, j) += alpha * acc;
                }
        }
        operator Matrix<S>() const {
            const Matrix& a = *cm;
            Matrix<S> o(a.rows(), a.cols());
            for (Index j = 0; j < a.cols(); ++j)
                for (Index i = j; i < a.rows(); ++i) {
                    o(i, j) = a(i, j);
                    if (i != j) o(j, i) = internal::conj_(a(i, j));
                }
            return o;
        }
    };
    template <int UpLo>
    SelfAdjoint<UpLo> selfadjointView() {
        return SelfAdjoint<UpLo>{this, this};
    }
    template <int UpLo>
    SelfAdjoint<UpLo> selfadjointView() const {
        return SelfAdjoint<UpLo>{nullptr, this};
    }

    // blocks (eager copies that write back into the root matrix when assigned)
    Block<Matrix> block(Index i, Index j, Index r, Index c) const;
    Block<Matrix> topRows(Index n) const { return block(0, 0, n, c_); }
    Block<Matrix> bottomRows(Index n) const { return block(r_ - n, 0, n, c_); }
    Block<Matrix> leftCols(Index n) const { return block(0, 0, r_, n); }
    Block<Matrix> rightCols(Index n) const { return block(0, c_ - n, r_, n); }
    Block<Matrix> col(Index j) const { return block(0, j, r_, 1); }
    Block<Matrix> row(Index i) const { return block(i, 0, 1, c_); }
    Block<Matrix> head(Index n) const { return block(0, 0, n, 1); }
    Block<Matrix> bottomRightCorner(Index r, Index c) const { return block(r_ - r, c_ - c, r, c); }

    template <typename Rhs>
    Matrix& operator+=(const Rhs& o) {
        const Matrix<S> b = o;
        for (Index e = 0; e < size(); ++e) d_[static_cast<size_t>(e)] += b(e);
        return *this;
    }
    template <typename Rhs>
    Matrix& operator-=(const Rhs& o) {
        const Matrix<S> b = o;
        for (Index e = 0; e < size(); ++e) d_[static_cast<size_t>(e)] -= b(e);
        return *this;
    }
    Matrix& operator/=(S s) {
        for (auto& x : d_) x /= s;
        return *this;
    }

protected:
    Index r_ = 0, c_ = 0;
    std::vector<S> d_;
};

// Block: a copy of a region of its root matrix; assignment writes through to the root (also for blocks of blocks).
template <typename M>
class Block : public Matrix<typename M::Scalar> {
public:
    using S = typename M::Scalar;
    using Base = Matrix<S>;
    Block(const M* root, Index i, Index j, Index r, Index c) : Base(r, c), root_(const_cast<M*>(root)), i0_(i), j0_(j) {
        for (Index b = 0; b < c; ++b)
            for (Index a = 0; a < r; ++a) (*this)(a, b) = (*root)(i + a, j + b);
    }
    Block(const Block&) = default;
    template <typename Rhs>
    Block& operator=(const Rhs& rhs) {
        const Base v = rhs;
        for (Index b = 0; b < this->cols(); ++b)
            for (Index a = 0; a < this->rows(); ++a) {
                (*this)(a, b) = v(a, b);
                (*root_)(i0_ + a, j0_ + b) = v(a, b);
            }
        return *this;
    }
    Block& operator=(const Block& rhs) { return operator=<Base>(static_cast<const Base&>(rhs)); }
    Block block(Index i, Index j, Index r, Index c) const { return Block(root_, i0_ + i, j0_ + j, r, c); }
    Block topRows(Index n) const { return block(0, 0, n, this->cols()); }
    Block bottomRows(Index n) const { return block(this->rows() - n, 0, n, this->cols()); }
    Block leftCols(Index n) const { return block(0, 0, this->rows(), n); }
    Block rightCols(Index n) const { return block(0, this->cols() - n, this->rows(), n); }
    Block head(Index n) const { return block(0, 0, n, 1); }

private:
    M* root_;
    Index i0_, j0_;
};

template <typename S, int R, int C>
Block<Matrix<S, R, C>> Matrix<S, R, C>::block(Index i, Index j, Index r, Index c) const {
    return Block<Matrix<S, R, C>>(this, i, j, r, c);
}

template <typename S>
class DiagonalWrapper {
public:
    template <int R, int C>
    explicit DiagonalWrapper(const Matrix<S, R, C>& v) : v_(v) {}
    const Matrix<S>& diag() const { return v_; }

private:
    Matrix<S> v_;
};

using MatrixXcd = Matrix<std::complex<double>>;
using MatrixXd = Matrix<double>;
using VectorXcd = Matrix<std::complex<double>, Dynamic, 1>;
using VectorXd = Matrix<double, Dynamic, 1>;
using VectorXi = Matrix<Index, Dynamic, 1>;

// ------------------------------------------------------------------ arithmetic (eager)
template <typename A, int R1, int C1, typename B, int R2, int C2>
Matrix<internal::promote_t<A, B>> operator*(const Matrix<A, R1, C1>& a, const Matrix<B, R2, C2>& b) {
    using S = internal::promote_t<A, B>;
    if (a.cols() != b.rows()) throw std::logic_error("eigen_lite: product size mismatch");
    Matrix<S> o(a.rows(), b.cols());
    if (a.rows() > 0 && b.cols() > 0 && a.cols() > 0) {
        if constexpr (std::is_same_v<S, std::complex<double>>) {
            auto promote = [](const auto& x) {  // real operands to complex
                Matrix<S> o2(x.rows(), x.cols());
                for (Index i = 0; i < x.size(); ++i) o2.data()[i] = S(x.data()[i]);
                return o2;
            };
            const S one(1.0, 0.0), zero(0.0, 0.0);
            const S* pa = nullptr;
            const S* pb = nullptr;
            Matrix<S> ac, bc;
            if constexpr (std::is_same_v<A, S>) pa = a.data();
            else pa = (ac = promote(a)).data();
            if constexpr (std::is_same_v<B, S>) pb = b.data();
            else pb = (bc = promote(b)).data();
            scipy_cblas_zgemm64_(102, 111, 111, a.rows(), b.cols(), a.cols(), &one, pa, a.rows(), pb, b.rows(), &zero,
                                 o.data(), o.rows());
            return o;
        } else if constexpr (std::is_same_v<S, double> && std::is_same_v<A, double> && std::is_same_v<B, double>) {
            scipy_cblas_dgemm64_(102, 111, 111, a.rows(), b.cols(), a.cols(), 1.0, a.data(), a.rows(), b.data(),
                                 b.rows(), 0.0, o.data(), o.rows());
            return o;
        }
    }
    for (Index j = 0; j < b.cols(); ++j)
        for (Index q = 0; q < a.cols(); ++q) {
            const S bq = S(b(q, j));
            for (Index i = 0; i < a.rows(); ++i) o(i, j) += S(a(i, q)) * bq;
        }
    return o;
}
template <typename A, typename B, int R, int C>
Matrix<internal::promote_t<A, B>> operator*(const DiagonalWrapper<A>& d, const Matrix<B, R, C>& m) {
    Matrix<internal::promote_t<A, B>> o(m.rows(), m.cols());
    for (Index j = 0; j < m.cols(); ++j)
        for (Index i = 0; i < m.rows(); ++i) o(i, j) = d.diag()(i) * m(i, j);
    return o;
}
template <typename A, int R, int C, typename B>
Matrix<internal::promote_t<A, B>> operator*(const Matrix<A, R, C>& m, const DiagonalWrapper<B>& d) {
    Matrix<internal::promote_t<A, B>> o(m.rows(), m.cols());
    for (Index j = 0; j < m.cols(); ++j)
        for (Index i = 0; i < m.rows(); ++i) o(i, j) = m(i, j) * d.diag()(j);
    return o;
}
template <typename A, int R, int C, typename T, typename = std::enable_if_t<std::is_arithmetic_v<T> ||
                                                                        std::is_same_v<T, std::complex<double>>>>
Matrix<internal::promote_t<A, T>> operator*(const T& s, const Matrix<A, R, C>& m) {
    Matrix<internal::promote_t<A, T>> o(m.rows(), m.cols());
    for (Index e = 0; e < m.size(); ++e) o(e) = s * m(e);
    return o;
}
template <typename A, int R1, int C1, int R2, int C2>
Matrix<A> operator+(const Matrix<A, R1, C1>& a, const Matrix<A, R2, C2>& b) {
    Matrix<A> o(a.rows(), a.cols());
    for (Index e = 0; e < a.size(); ++e) o(e) = a(e) + b(e);
    return o;
}
template <typename A, int R1, int C1, int R2, int C2>
Matrix<A> operator-(const Matrix<A, R1, C1>& a, const Matrix<A, R2, C2>& b) {
    Matrix<A> o(a.rows(), a.cols());
    for (Index e = 0; e < a.size(); ++e) o(e) = a(e) - b(e);
    return o;
}

// ------------------------------------------------------------------ decompositions (LAPACK)
namespace internal {
inline void lapack_check(long long info, const char* what) {
    if (info < 0) throw std::logic_error(std::string("eigen_lite: bad argument to ") + what);
}
constexpr int kColMajor = 102;
}  // namespace internal

template <typename M>
class SelfAdjointEigenSolver {
public:
    explicit SelfAdjointEigenSolver(const M& a) : vec_(a), val_(a.rows()) {
        const int n = static_cast<int>(a.rows());
        const long long info = scipy_LAPACKE_zheevd64_(internal::kColMajor, 'V', 'L', n, vec_.data(), n, val_.data());
        internal::lapack_check(info, "zheevd");
        info_ = info == 0 ? Success : NoConvergence;
    }
    const VectorXd& eigenvalues() const { return val_; }  // ascending
    const M& eigenvectors() const { return vec_; }
    ComputationInfo info() const { return info_; }

private:
    M vec_;
    VectorXd val_;
    ComputationInfo info_ = Success;
};

template <typename M>
class JacobiSVD {
public:
    JacobiSVD(const M& a, int) {
        const int m = static_cast<int>(a.rows()), n = static_cast<int>(a.cols()), k = std::min(m, n);
        M w = a;
        u_ = M(m, k);
        M vt(k, n);
        s_ = VectorXd(k);
        std::vector<double> superb(static_cast<size_t>(std::max(1, k)));
        if (k > 0) {
            const long long info = scipy_LAPACKE_zgesvd64_(internal::kColMajor, 'S', 'S', m, n, w.data(), m, s_.data(), u_.data(),
                                                  m, vt.data(), k, superb.data());
            internal::lapack_check(info, "zgesvd");
            info_ = info == 0 ? Success : NoConvergence;
        }
        v_ = vt.adjoint();
    }
    const VectorXd& singularValues() const { return s_; }
    const M& matrixU() const { return u_; }
    const M& matrixV() const { return v_; }
    ComputationInfo info() const { return info_; }

protected:
    M u_, v_;
    VectorXd s_;
    ComputationInfo info_ = Success;
};

template <typename M>
class BDCSVD {
public:
    BDCSVD(const M& a, int) {
        const int m = static_cast<int>(a.rows()), n = static_cast<int>(a.cols()), k = std::min(m, n);
        M w = a;
        u_ = M(m, k);
        M vt(k, n);
        s_ = VectorXd(k);
        if (k > 0) {
            const long long info = scipy_LAPACKE_zgesdd64_(internal::kColMajor, 'S', m, n, w.data(), m, s_.data(), u_.data(), m,
                                                  vt.data(), k);
            internal::lapack_check(info, "zgesdd");
            info_ = info == 0 ? Success : NoConvergence;
        }
        v_ = vt.adjoint();
    }
    const VectorXd& singularValues() const { return s_; }
    const M& matrixU() const { return u_; }
    const M& matrixV() const { return v_; }
    ComputationInfo info() const { return info_; }

private:
    M u_, v_;
    VectorXd s_;
    ComputationInfo info_ = Success;
};

namespace internal {
// full m x m Q from the Householder reflectors of zgeqrf / zgeqp3
inline MatrixXcd householder_q(const MatrixXcd& qr, const MatrixXcd& tau) {
    const int m = static_cast<int>(qr.rows()), n = static_cast<int>(qr.cols()), k = std::min(m, n);
    MatrixXcd q(m, m);
    for (Index j = 0; j < std::min<Index>(n, m); ++j)
        for (Index i = 0; i < m; ++i) q(i, j) = qr(i, j);
    if (m > 0) {
        const long long info = scipy_LAPACKE_zungqr64_(kColMajor, m, m, k, q.data(), m, tau.data());
        lapack_check(info, "zungqr");
    }
    return q;
}
}  // namespace internal

template <typename M>
class HouseholderQR {
public:
    explicit HouseholderQR(const M& a) : qr_(a), tau_(std::min(a.rows(), a.cols()), 1) {
        const int m = static_cast<int>(a.rows()), n = static_cast<int>(a.cols());
        if (m > 0 && n > 0) internal::lapack_check(scipy_LAPACKE_zgeqrf64_(internal::kColMajor, m, n, qr_.data(), m,
                                                                         tau_.data()), "zgeqrf");
    }
    const M& matrixQR() const { return qr_; }
    M householderQ() const { return internal::householder_q(qr_, tau_); }

private:
    M qr_, tau_;
};

struct PermutationIndices {
    VectorXi idx;
    const VectorXi& indices() const { return idx; }
};

template <typename M>
class ColPivHouseholderQR {
public:
    explicit ColPivHouseholderQR(const M& a) : qr_(a), tau_(std::min(a.rows(), a.cols()), 1) {
        const int m = static_cast<int>(a.rows()), n = static_cast<int>(a.cols());
        std::vector<fm_lapack_int> jpvt(static_cast<size_t>(n), 0);
        // Eigen's nonzero-pivot cut uses the initial largest column norm
        double max_col_sq = 0.0;
        for (Index j = 0; j < n; ++j) max_col_sq = std::max(max_col_sq, a.col(j).squaredNorm());
        if (m > 0 && n > 0)
            internal::lapack_check(scipy_LAPACKE_zgeqp364_(internal::kColMajor, m, n, qr_.data(), m, jpvt.data(),
                                                        tau_.data()), "zgeqp3");
        perm_.idx = VectorXi(n);
        for (Index j = 0; j < n; ++j) perm_.idx(j) = jpvt[static_cast<size_t>(j)] - 1;
        const Index size = std::min(a.rows(), a.cols());
        const double eps = NumTraits<double>::epsilon();
        const double threshold_helper = max_col_sq * eps * eps / static_cast<double>(std::max<Index>(m, 1));
        nonzero_ = size;
        maxpivot_ = 0.0;
        for (Index k = 0; k < size; ++k) {
            const double piv = std::abs(qr_(k, k));
            if (nonzero_ == size && piv * piv < threshold_helper * static_cast<double>(m - k)) nonzero_ = k;
            maxpivot_ = std::max(maxpivot_, piv);
        }
    }
    Index rank() const {  // Eigen ColPivHouseholderQR::rank(): |R_kk| > maxpivot * diagonalSize * eps
        const double thr = maxpivot_ * static_cast<double>(std::min(qr_.rows(), qr_.cols())) *
                           NumTraits<double>::epsilon();
        Index r = 0;
        for (Index k = 0; k < nonzero_; ++k) r += std::abs(qr_(k, k)) > thr ? 1 : 0;
        return r;
    }
    const PermutationIndices& colsPermutation() const { return perm_; }
    const M& matrixQR() const { return qr_; }
    M householderQ() const { return internal::householder_q(qr_, tau_); }

private:
    M qr_, tau_;
    PermutationIndices perm_;
    Index nonzero_ = 0;
    double maxpivot_ = 0.0;
};

// LDLT (no pivoting; the reference's matrix-inverse baseline only, which is out of this build's scope)
template <typename M>
class LDLT {
public:
    explicit LDLT(const M& a) : l_(M::Identity(a.rows(), a.rows())), d_(a.rows()) {
        const Index n = a.rows();
        for (Index j = 0; j < n; ++j) {
            std::complex<double> dj = a(j, j);
            for (Index q = 0; q < j; ++q) dj -= l_(j, q) * std::conj(l_(j, q)) * d_(q);
            d_(j) = dj;
            if (std::abs(dj) == 0.0) info_ = NumericalIssue;
            for (Index i = j + 1; i < n; ++i) {
                std::complex<double> v = a(i, j);
                for (Index q = 0; q < j; ++q) v -= l_(i, q) * std::conj(l_(j, q)) * d_(q);
                l_(i, j) = dj != 0.0 ? v / dj : 0.0;
            }
        }
    }
    ComputationInfo info() const { return info_; }
    const VectorXcd& vectorD() const { return d_; }
    M solve(const M& b) const {
        M x = b;
        const Index n = l_.rows();
        for (Index c = 0; c < x.cols(); ++c) {
            for (Index i = 0; i < n; ++i)
                for (Index q = 0; q < i; ++q) x(i, c) -= l_(i, q) * x(q, c);
            for (Index i = 0; i < n; ++i) x(i, c) /= d_(i);
            for (Index i = n - 1; i >= 0; --i)
                for (Index q = i + 1; q < n; ++q) x(i, c) -= std::conj(l_(q, i)) * x(q, c);
        }
        return x;
    }

private:
    M l_;
    VectorXcd d_;
    ComputationInfo info_ = Success;
};

// unsupported/Eigen/FFT: forward DFT, unscaled, exp(-2 pi i k n / N) (the reference's FFT baseline only)
template <typename T>
class FFT {
public:
    void fwd(std::vector<std::complex<T>>& out, const std::vector<std::complex<T>>& in) const {
        const size_t n = in.size();
        out.assign(n, std::complex<T>(0, 0));
        for (size_t k = 0; k < n; ++k) {
            std::complex<T> acc(0, 0);
            for (size_t t = 0; t < n; ++t) {
                const T ang = T(-2) * T(3.14159265358979323846) * T((k * t) % n) / T(n);
                acc += in[t] * std::complex<T>(std::cos(ang), std::sin(ang));
            }
            out[k] = acc;
        }
    }
};

}  // namespace Eigen
