// ORACLE support (test infrastructure only). C entry points over the REFERENCE's own hot-path functions, compiled
// in place from /root/reference (R/src/{scene,linalg,estimators,spectrum}.cpp, never copied) against the Eigen-API
// shim oracle/eigen_shim (LAPACK decompositions), into oracle/_ref/libref_fastmusic.so. tests/golden/make_ref_golden.py
// turns their outputs into committed golden vectors that pin the oracle restatement and the GPU paths.
// Matrices are column-major interleaved complex128 (Eigen::MatrixXcd::data() layout).
// Status: 0 ok, 1 std::invalid_argument, 2 RankDeficiencyError (column in *aux), 3 NonConvergenceError.
#include <cstdint>
#include <cstring>
#include <stdexcept>

#include "fastmusic/estimators.hpp"
#include "fastmusic/linalg.hpp"
#include "fastmusic/scene.hpp"
#include "fastmusic/spectrum.hpp"

using namespace fastmusic;

namespace {
CxMat load(const double* a, Index r, Index c) {
    CxMat m(r, c);
    std::memcpy(m.data(), a, sizeof(double) * 2 * r * c);
    return m;
}
void store(const CxMat& m, double* out) { std::memcpy(out, m.data(), sizeof(double) * 2 * m.rows() * m.cols()); }

template <typename F>
int guard(F&& f, int64_t* aux) {
    try {
        f();
        return 0;
    } catch (const RankDeficiencyError& e) {
        if (aux) *aux = e.column();
        return 2;
    } catch (const NonConvergenceError&) {
        return 3;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

void store_estimate(const SubspaceEstimate& est, double* basis, double* eig) {
    store(est.basis, basis);
    for (Index i = 0; i < est.eigenvalues.size(); ++i) eig[i] = est.eigenvalues(i);
}
}  // namespace

extern "C" {

int ref_steering_vector(double theta, int64_t m, double d, double lambda, double* out) {
    return guard([&] { store(steering_vector(theta, m, d, lambda), out); }, nullptr);
}

// spatial_covariance (R/src/scene.cpp:138-159): y M x N -> S M x M
int ref_spatial_covariance(const double* y, int64_t m, int64_t n, double* s_out) {
    return guard([&] { store(spatial_covariance(load(y, m, n)).mat(), s_out); }, nullptr);
}

// temporal_covariance (R/src/scene.cpp:161-163): y M x N -> T N x N
int ref_temporal_covariance(const double* y, int64_t m, int64_t n, double* t_out) {
    return guard([&] { store(temporal_covariance(load(y, m, n)).mat(), t_out); }, nullptr);
}

int ref_exact_signal_subspace(const double* s, int64_t m, int64_t k, double* basis, double* eig) {
    return guard([&] { store_estimate(exact_signal_subspace(HermitianMatrix(load(s, m, m)), k), basis, eig); }, nullptr);
}

int ref_fast_music_1(const double* s, int64_t m, int64_t k, int64_t p, uint64_t seed, double* basis, double* eig) {
    return guard([&] { store_estimate(fast_music_1(HermitianMatrix(load(s, m, m)), k, Fast1Params{p, seed}), basis, eig); },
                 nullptr);
}

int ref_fast_music_2(const double* s, int64_t m, int64_t k, int64_t p, int t, uint64_t seed, double* basis, double* eig,
                     int64_t* deficient_column) {
    return guard([&] {
        store_estimate(fast_music_2(HermitianMatrix(load(s, m, m)), k, Fast2Params{p, t, seed}), basis, eig);
    }, deficient_column);
}

// music_spectrum on the reference grid AngleGrid(L) = [0, pi] (R/src/spectrum.cpp:18-33, 50-68)
int ref_music_spectrum(const double* basis, int64_t m, int64_t kb, int64_t L, double d, double lambda, double* out) {
    return guard([&] {
        SubspaceEstimate est;
        est.basis = load(basis, m, kb);
        const PseudoSpectrum p = music_spectrum(est, AngleGrid(L), d, lambda);
        for (Index l = 0; l < L; ++l) out[l] = p.values(l);
    }, nullptr);
}

// extract_peaks (R/src/spectrum.cpp:182-188) on arbitrary values: the grid only labels the cells, which are
// recovered exactly from the returned angles (theta = pi c / (L - 1)).
int ref_extract_peaks(const double* values, int64_t L, int64_t k, int64_t min_sep, int64_t* cells, double* heights,
                      int64_t* count, double* baseline, int32_t* shortfall) {
    return guard([&] {
        RealVec v(L);
        for (Index l = 0; l < L; ++l) v(l) = values[l];
        const AngleGrid grid(std::max<int64_t>(L, 2));
        const PeakSet ps = extract_peaks(PseudoSpectrum{grid, v, Method::Exact, false}, k, min_sep);
        *count = static_cast<int64_t>(ps.angles.size());
        for (size_t i = 0; i < ps.angles.size(); ++i) {
            cells[i] = static_cast<int64_t>(std::llround(ps.angles[i] / grid.spacing()));
            heights[i] = ps.heights[i];
        }
        *baseline = ps.baseline;
        *shortfall = ps.shortfall ? 1 : 0;
    }, nullptr);
}

// The whole reference path for one frame, the CPU arm of bench.py (R/src/bench.cpp:574-591 pattern): covariance
// (spatial, or temporal for the ToA path) -> estimator -> music_spectrum on AngleGrid(L) -> extract_peaks.
// method: 0 exact, 1 fast1, 2 fast2, 3 block-Lanczos (block = p or K, cap t). Returns the status; cells (K) and
// *count receive the peaks, spectrum (L, may be null) the pseudo-spectrum.
int ref_run_frame(const double* y, int64_t m, int64_t n, int temporal, int method, int64_t k, int64_t p, int t,
                  uint64_t seed, int64_t L, int64_t min_sep, int64_t* cells, int64_t* count, double* spectrum) {
    return guard([&] {
        const CxMat x = load(y, m, n);
        const HermitianMatrix s = temporal ? temporal_covariance(x) : spatial_covariance(x);
        SubspaceEstimate est;
        if (method == 0) est = exact_signal_subspace(s, k);
        else if (method == 1) est = fast_music_1(s, k, Fast1Params{p, seed});
        else if (method == 2) est = fast_music_2(s, k, Fast2Params{p, t, seed});
        else est = block_lanczos_subspace(s, k, p > 0 ? p : k, t);
        const PseudoSpectrum ps = music_spectrum(est, AngleGrid(L), 0.5, 1.0);
        const PeakSet pk = extract_peaks(ps, k, min_sep);
        const AngleGrid grid(L);
        *count = static_cast<int64_t>(pk.angles.size());
        for (size_t i = 0; i < pk.angles.size(); ++i) cells[i] = static_cast<int64_t>(std::llround(pk.angles[i] / grid.spacing()));
        if (spectrum)
            for (Index l = 0; l < L; ++l) spectrum[l] = ps.values(l);
    }, nullptr);
}

// Sample a frame with the reference's own FMCW beat-signal synthesis (R/src/scene.cpp:100-134) for fixture inputs.
int ref_synthesize_beat_signal(int64_t m, int64_t n, int64_t k, const double* angles, double noise_var, uint64_t seed,
                               double* y) {
    return guard([&] {
        const FMCWConfig cfg = FMCWConfig::typical_77ghz(m, n);
        TargetScene scene;
        for (int64_t i = 0; i < k; ++i) scene.targets.push_back({angles[i], 1e-8 * static_cast<double>(i + 1), Complex(1, 0)});
        store(synthesize_beat_signal(cfg, scene, noise_var, seed), y);
    }, nullptr);
}

}  // extern "C"
