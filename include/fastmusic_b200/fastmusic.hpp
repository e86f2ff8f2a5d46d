// Reference-named C++ facade over the fastmusic_b200 C ABI.
//
// Drop-in for the hot-path part of the reference API (R/include/fastmusic/):
//   types.hpp:11-90      Complex/CxMat/CxVec/RealVec/Index, error classes, Method, HermitianMatrix
//   estimators.hpp:13-44 SubspaceEstimate, Fast1Params, Fast2Params, exact_signal_subspace,
//                        fast_music_1, fast_music_2
//   spectrum.hpp:12-62   AngleGrid, PseudoSpectrum, PeakSet, music_spectrum, extract_peaks
//   scene.hpp:60,72      steering_vector, spatial_covariance
// Eigen is replaced by a minimal column-major dense type with the same element layout
// (Eigen::MatrixXcd::data()). All numeric work runs on the GPU through fm_z_* (fp64);
// BatchEstimator exposes the batched complex64 pipeline (fm_plan) for frame streams.
#pragma once

#include <algorithm>
#include <complex>
#include <type_traits>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../fastmusic_b200.h"

namespace fastmusic {

using Complex = std::complex<double>;
using Index = std::ptrdiff_t;

// Column-major dense matrix (Eigen::MatrixXcd storage order).
template <typename S>
class Dense {
public:
    Dense() = default;
    Dense(Index r, Index c) : r_(r), c_(c), d_(static_cast<std::size_t>(r * c)) {}
    explicit Dense(Index n) : Dense(n, 1) {}  // column vector, as Eigen's VectorX(n)
    static Dense Zero(Index r, Index c) { return Dense(r, c); }
    static Dense Identity(Index r, Index c) {
        Dense m(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = S(1);
        return m;
    }
    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    S& operator()(Index i, Index j) { return d_[static_cast<std::size_t>(j * r_ + i)]; }
    const S& operator()(Index i, Index j) const { return d_[static_cast<std::size_t>(j * r_ + i)]; }
    S& operator()(Index i) { return d_[static_cast<std::size_t>(i)]; }
    const S& operator()(Index i) const { return d_[static_cast<std::size_t>(i)]; }
    S* data() { return d_.data(); }
    const S* data() const { return d_.data(); }
    Dense adjoint() const {
        Dense out(c_, r_);
        for (Index i = 0; i < r_; ++i)
            for (Index j = 0; j < c_; ++j) out(j, i) = conj_(operator()(i, j));
        return out;
    }
    Dense leftCols(Index k) const {
        Dense out(r_, k);
        for (Index j = 0; j < k; ++j)
            for (Index i = 0; i < r_; ++i) out(i, j) = operator()(i, j);
        return out;
    }
    double squaredNorm() const {
        double s = 0.0;
        for (const S& v : d_) s += std::norm(Complex(v));
        return s;
    }

private:
    static S conj_(const S& v) {
        if constexpr (std::is_same_v<S, Complex>) return std::conj(v);
        else return v;
    }
    Index r_ = 0, c_ = 0;
    std::vector<S> d_;
};

using CxMat = Dense<Complex>;
using CxVec = Dense<Complex>;   // M x 1
using RealVec = Dense<double>;  // n x 1

CxMat operator*(const CxMat& a, const CxMat& b);
CxMat operator-(const CxMat& a, const CxMat& b);

// R/include/fastmusic/types.hpp:18-43
class NonConvergenceError : public std::runtime_error {
public:
    NonConvergenceError(const std::string& what, double residual) : std::runtime_error(what), residual_(residual) {}
    double residual() const { return residual_; }

private:
    double residual_;
};
class RankDeficiencyError : public std::runtime_error {
public:
    RankDeficiencyError(const std::string& what, Index column) : std::runtime_error(what), column_(column) {}
    Index column() const { return column_; }

private:
    Index column_;
};
class SingularMatrixError : public std::runtime_error {
public:
    explicit SingularMatrixError(const std::string& what) : std::runtime_error(what) {}
};

enum class Method { Exact, Fast1, Fast2, Lanczos, MatrixInverse, Propagator, Fft };
const char* method_name(Method m);
Method method_from_name(const std::string& name);  // std::invalid_argument("unknown method name: ...")

// R/include/fastmusic/types.hpp:59-62, R/src/linalg.cpp:36-44
bool is_finite(const CxMat& a);
void ensure_finite(const CxMat& a, const char* what);  // std::invalid_argument("<what>: non-finite entries")

// Square complex matrix kept Hermitian by symmetrising on construction (R/src/linalg.cpp:46-52).
class HermitianMatrix {
public:
    explicit HermitianMatrix(const CxMat& a);
    Index dim() const { return m_.rows(); }
    const CxMat& mat() const { return m_; }

private:
    CxMat m_;
};

// R/include/fastmusic/types.hpp:78-90. Eigenvalues descending, column i of `eigenvectors` pairs with eigenvalue i;
// thin SVD with singular values descending.
struct EigResult {
    RealVec eigenvalues;
    CxMat eigenvectors;
};
struct SvdResult {
    CxMat u;
    RealVec sigma;
    CxMat v;
};
// R/include/fastmusic/linalg.hpp:13 (R/src/linalg.cpp:77-89): one-sided Jacobi on the GPU, fp64.
EigResult hermitian_eig(const HermitianMatrix& s);

struct SubspaceEstimate {
    CxMat basis;
    RealVec eigenvalues;
    Method method = Method::Exact;
    double cost_seconds = 0.0;
};
struct Fast1Params {
    Index p = 0;
    std::uint64_t seed = 0;
};
struct Fast2Params {
    Index p = 0;
    int iterations = 1;
    std::uint64_t seed = 0;
};

// L angles spanning [theta0, theta1]; the one-argument form is the reference grid [0, pi].
class AngleGrid {
public:
    explicit AngleGrid(Index l, double theta0 = 0.0, double theta1 = 3.14159265358979323846);
    Index size() const { return l_; }
    double spacing() const { return (t1_ - t0_) / static_cast<double>(l_ - 1); }
    double theta(Index i) const { return t0_ + ((t1_ - t0_) * static_cast<double>(i)) / static_cast<double>(l_ - 1); }
    Index nearest(double theta) const;
    double theta0() const { return t0_; }
    double theta1() const { return t1_; }
    bool operator==(const AngleGrid& o) const { return l_ == o.l_ && t0_ == o.t0_ && t1_ == o.t1_; }

private:
    Index l_;
    double t0_, t1_;
};

struct PseudoSpectrum {
    AngleGrid grid;
    RealVec values;
    Method method = Method::Exact;
    bool degenerate = false;
};

struct PeakSet {
    std::vector<double> angles;
    std::vector<double> heights;
    double baseline = 0.0;
    bool shortfall = false;
    std::vector<Index> cells;  // extension: selected grid cells, ascending
};

CxVec steering_vector(double theta, Index m, double d, double lambda);
HermitianMatrix spatial_covariance(const CxMat& y);
HermitianMatrix temporal_covariance(const CxMat& y);  // scene.hpp:72, T = Y^H Y / M
SubspaceEstimate exact_signal_subspace(const HermitianMatrix& s, Index k);
SubspaceEstimate fast_music_1(const HermitianMatrix& s, Index k, const Fast1Params& params);
SubspaceEstimate fast_music_2(const HermitianMatrix& s, Index k, const Fast2Params& params);
// estimators.hpp:45-50 (the paper's accurate baseline; fp64 on the GPU)
SubspaceEstimate block_lanczos_subspace(const HermitianMatrix& s, Index k, Index block, int max_iterations);
PseudoSpectrum music_spectrum(const SubspaceEstimate& estimate, const AngleGrid& grid, double d, double lambda);
PeakSet extract_peaks(const PseudoSpectrum& p, Index k, Index min_separation_cells);

// io.hpp:17-27 (matrix / spectrum files; scene files belong to the FMCW front end, out of scope)
void write_matrix_binary(const std::string& path, const CxMat& a);
CxMat read_matrix_binary(const std::string& path);
void write_matrix_csv(const std::string& path, const CxMat& a);
void write_spectrum_csv(const std::string& path, const PseudoSpectrum& spectrum);

// Batched complex64 pipeline over device-resident frames (fm_plan); one per host thread.
class BatchEstimator {
public:
    BatchEstimator(const fm_plan_desc& desc, int device = 0);
    ~BatchEstimator();
    BatchEstimator(const BatchEstimator&) = delete;
    BatchEstimator& operator=(const BatchEstimator&) = delete;
    // Device pointers; see fm_batch_io. Throws std::runtime_error on a CUDA failure.
    void run(std::int64_t frames, const fm_batch_io& io, void* stream = nullptr);
    // Host buffers end to end (redraws included). Throws like the single-frame API.
    void estimate_host(std::int64_t frames, const float* x, const std::uint64_t* draw_seeds, fm_host_out& out,
                       void* stream = nullptr);
    fm_plan plan() const { return plan_; }

private:
    fm_plan plan_ = nullptr;
};

}  // namespace fastmusic
