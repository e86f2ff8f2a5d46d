// Reference-named C++ facade (include/fastmusic_b200/fastmusic.hpp) over the C ABI.
// Argument validation and error mapping follow the reference line by line; numeric
// work is delegated to the GPU entry points (fm_z_*).

#include "../../include/fastmusic_b200/fastmusic.hpp"

#include <cmath>
#include <string>

namespace fastmusic {

namespace {

constexpr double kPi = 3.14159265358979323846;

[[noreturn]] void raise(fm_status st, Index column = -1) {
    const std::string msg = fm_last_error();
    switch (st) {
        case FM_EINVAL: throw std::invalid_argument(msg);
        case FM_ERANK: throw RankDeficiencyError(msg, column);
        case FM_ENOCONV: throw NonConvergenceError(msg, std::nan(""));
        case FM_ESINGULAR: throw SingularMatrixError(msg);
        default: throw std::runtime_error(msg);
    }
}

void check(fm_status st) {
    if (st != FM_OK) raise(st);
}

bool finite(const CxMat& a) {
    for (Index i = 0; i < a.size(); ++i)
        if (!std::isfinite(a(i).real()) || !std::isfinite(a(i).imag())) return false;
    return true;
}

const double* raw(const CxMat& a) { return reinterpret_cast<const double*>(a.data()); }
double* raw(CxMat& a) { return reinterpret_cast<double*>(a.data()); }

}  // namespace

CxMat operator*(const CxMat& a, const CxMat& b) {
    if (a.cols() != b.rows()) throw std::invalid_argument("operator*: shape mismatch");
    CxMat out(a.rows(), b.cols());
    for (Index j = 0; j < b.cols(); ++j)
        for (Index q = 0; q < a.cols(); ++q) {
            const Complex bq = b(q, j);
            for (Index i = 0; i < a.rows(); ++i) out(i, j) += a(i, q) * bq;
        }
    return out;
}

CxMat operator-(const CxMat& a, const CxMat& b) {
    CxMat out(a.rows(), a.cols());
    for (Index i = 0; i < a.size(); ++i) out(i) = a(i) - b(i);
    return out;
}

const char* method_name(Method m) {
    switch (m) {
        case Method::Exact: return "exact";
        case Method::Fast1: return "fast1";
        case Method::Fast2: return "fast2";
        case Method::Lanczos: return "lanczos";
        case Method::MatrixInverse: return "matrix_inverse";
        case Method::Propagator: return "propagator";
        case Method::Fft: return "fft";
    }
    return "unknown";
}

Method method_from_name(const std::string& name) {
    for (Method m : {Method::Exact, Method::Fast1, Method::Fast2, Method::Lanczos, Method::MatrixInverse,
                     Method::Propagator, Method::Fft})
        if (name == method_name(m)) return m;
    throw std::invalid_argument("unknown method name: " + name);
}

bool is_finite(const CxMat& a) { return finite(a); }

void ensure_finite(const CxMat& a, const char* what) {
    if (!finite(a)) throw std::invalid_argument(std::string(what) + ": non-finite entries");
}

HermitianMatrix::HermitianMatrix(const CxMat& a) {
    if (a.rows() != a.cols() || a.rows() < 1)
        throw std::invalid_argument("HermitianMatrix: input must be square and non-empty");
    if (!finite(a)) throw std::invalid_argument("HermitianMatrix: non-finite entries");
    const Index n = a.rows();
    m_ = CxMat(n, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) m_(i, j) = 0.5 * (a(i, j) + std::conj(a(j, i)));
}

AngleGrid::AngleGrid(Index l, double theta0, double theta1) : l_(l), t0_(theta0), t1_(theta1) {
    if (l < 2) throw std::invalid_argument("AngleGrid: L >= 2 required");
}

Index AngleGrid::nearest(double theta) const {
    const Index i = static_cast<Index>(std::llround((theta - t0_) / spacing()));
    return std::clamp(i, Index{0}, l_ - 1);
}

CxVec steering_vector(double theta, Index m, double d, double lambda) {
    if (m < 1 || d <= 0.0 || lambda <= 0.0)
        throw std::invalid_argument("steering_vector: need M >= 1, d > 0, lambda > 0");
    const double step = 2.0 * kPi * d * std::sin(theta) / lambda;
    CxVec a(m, 1);
    for (Index i = 0; i < m; ++i) a(i) = std::polar(1.0, step * static_cast<double>(i));
    return a;
}

HermitianMatrix spatial_covariance(const CxMat& y) {
    if (y.rows() < 1 || y.cols() < 1) throw std::invalid_argument("covariance: empty signal matrix");
    CxMat s(y.rows(), y.rows());
    check(fm_z_spatial_covariance(y.rows(), y.cols(), raw(y), raw(s)));
    return HermitianMatrix(s);
}

HermitianMatrix temporal_covariance(const CxMat& y) {
    if (y.rows() < 1 || y.cols() < 1) throw std::invalid_argument("covariance: empty signal matrix");
    CxMat t(y.cols(), y.cols());
    check(fm_z_temporal_covariance(y.rows(), y.cols(), raw(y), raw(t)));
    return HermitianMatrix(t);
}

static SubspaceEstimate make_estimate(Index m, Index k, Method method) {
    SubspaceEstimate out;
    out.basis = CxMat(m, k);
    out.eigenvalues = RealVec(k, 1);
    out.method = method;
    return out;
}

EigResult hermitian_eig(const HermitianMatrix& s) {
    EigResult out;
    out.eigenvalues = RealVec(s.dim(), 1);
    out.eigenvectors = CxMat(s.dim(), s.dim());
    check(fm_z_hermitian_eig(s.dim(), raw(s.mat()), out.eigenvalues.data(), raw(out.eigenvectors)));
    return out;
}

SubspaceEstimate exact_signal_subspace(const HermitianMatrix& s, Index k) {
    if (k < 1 || k >= s.dim()) throw std::invalid_argument("exact_signal_subspace: need 1 <= K < M");
    SubspaceEstimate out = make_estimate(s.dim(), k, Method::Exact);
    check(fm_z_exact_signal_subspace(s.dim(), raw(s.mat()), k, raw(out.basis), out.eigenvalues.data(),
                                     &out.cost_seconds));
    return out;
}

SubspaceEstimate fast_music_1(const HermitianMatrix& s, Index k, const Fast1Params& params) {
    const Index m = s.dim();
    if (k < 1 || k >= m) throw std::invalid_argument("fast_music_1: need 1 <= K < M");
    if (params.p < k || params.p > m) throw std::invalid_argument("fast_music_1: need K <= p <= M");
    SubspaceEstimate out = make_estimate(m, k, Method::Fast1);
    check(fm_z_fast_music_1(m, raw(s.mat()), k, params.p, params.seed, raw(out.basis), out.eigenvalues.data(),
                            &out.cost_seconds));
    return out;
}

SubspaceEstimate fast_music_2(const HermitianMatrix& s, Index k, const Fast2Params& params) {
    const Index m = s.dim();
    if (k < 1 || k >= m) throw std::invalid_argument("fast_music_2: need 1 <= K < M");
    if (params.p < k || params.p > m) throw std::invalid_argument("fast_music_2: need K <= p <= M");
    if (params.iterations < 1 || params.iterations > 20) throw std::invalid_argument("fast_music_2: need 1 <= t <= 20");
    SubspaceEstimate out = make_estimate(m, k, Method::Fast2);
    int64_t col = -1;
    const fm_status st = fm_z_fast_music_2(m, raw(s.mat()), k, params.p, params.iterations, params.seed,
                                           raw(out.basis), out.eigenvalues.data(), &out.cost_seconds, &col);
    if (st != FM_OK) raise(st, col);
    return out;
}

SubspaceEstimate block_lanczos_subspace(const HermitianMatrix& s, Index k, Index block, int max_iterations) {
    const Index m = s.dim();
    if (k < 1 || k >= m) throw std::invalid_argument("block_lanczos_subspace: need 1 <= K < M");
    if (block < k) throw std::invalid_argument("block_lanczos_subspace: need block >= K");
    if (max_iterations < 1) throw std::invalid_argument("block_lanczos_subspace: iters >= 1");
    SubspaceEstimate out = make_estimate(m, k, Method::Lanczos);
    double last = 0.0;
    const fm_status st = fm_z_block_lanczos_subspace(m, raw(s.mat()), k, block, max_iterations, raw(out.basis),
                                                     out.eigenvalues.data(), &out.cost_seconds, &last);
    if (st == FM_ENOCONV) throw NonConvergenceError(fm_last_error(), last);
    check(st);
    return out;
}

PseudoSpectrum music_spectrum(const SubspaceEstimate& estimate, const AngleGrid& grid, double d, double lambda) {
    const Index m = estimate.basis.rows();
    if (m < 1) throw std::invalid_argument("music_spectrum: empty basis");
    PseudoSpectrum out{grid, RealVec(grid.size(), 1), estimate.method, false};
    check(fm_z_music_spectrum(m, estimate.basis.cols(), raw(estimate.basis), grid.size(), grid.theta0(),
                              grid.theta1(), d, lambda, out.values.data()));
    return out;
}

PeakSet extract_peaks(const PseudoSpectrum& p, Index k, Index min_separation_cells) {
    if (k < 1) throw std::invalid_argument("extract_peaks: K >= 1 required");
    std::vector<int64_t> cells(static_cast<std::size_t>(k));
    std::vector<double> heights(static_cast<std::size_t>(k));
    int64_t count = 0;
    double base = 0.0;
    int32_t shortfall = 0;
    check(fm_z_extract_peaks(p.values.data(), p.values.size(), k, min_separation_cells, cells.data(), heights.data(),
                             &count, &base, &shortfall));
    PeakSet out;
    out.baseline = base;
    out.shortfall = shortfall != 0;
    for (int64_t i = 0; i < count; ++i) {
        out.cells.push_back(cells[static_cast<std::size_t>(i)]);
        out.angles.push_back(p.grid.theta(cells[static_cast<std::size_t>(i)]));
        out.heights.push_back(heights[static_cast<std::size_t>(i)]);
    }
    return out;
}

// R/src/io.cpp:71-131 (the file formats themselves live in csrc/io.cpp)
void write_matrix_binary(const std::string& path, const CxMat& a) {
    check(fm_z_fmcx_write(path.c_str(), a.rows(), a.cols(), raw(a)));
}

CxMat read_matrix_binary(const std::string& path) {
    int64_t rows = 0, cols = 0;
    check(fm_fmcx_read_header(path.c_str(), &rows, &cols));
    CxMat a(rows, cols);
    check(fm_z_fmcx_read(path.c_str(), rows, cols, raw(a)));
    return a;
}

void write_matrix_csv(const std::string& path, const CxMat& a) {
    check(fm_z_write_matrix_csv(path.c_str(), a.rows(), a.cols(), raw(a)));
}

void write_spectrum_csv(const std::string& path, const PseudoSpectrum& spectrum) {
    if (spectrum.values.size() != spectrum.grid.size())
        throw std::invalid_argument("write_spectrum_csv: values / grid size mismatch");
    check(fm_write_spectrum_csv(path.c_str(), spectrum.grid.size(), spectrum.grid.theta0(), spectrum.grid.theta1(),
                                spectrum.values.data()));
}

BatchEstimator::BatchEstimator(const fm_plan_desc& desc, int device) { check(fm_plan_create(&desc, device, &plan_)); }

BatchEstimator::~BatchEstimator() {
    if (plan_) fm_plan_destroy(plan_);
}

void BatchEstimator::run(std::int64_t frames, const fm_batch_io& io, void* stream) {
    check(fm_run_batch(plan_, frames, &io, stream));
}

void BatchEstimator::estimate_host(std::int64_t frames, const float* x, const std::uint64_t* draw_seeds,
                                   fm_host_out& out, void* stream) {
    check(fm_estimate_batch_host(plan_, frames, x, draw_seeds, &out, stream));
}

}  // namespace fastmusic
