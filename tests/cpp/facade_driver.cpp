// Drop-in check of the C++ facade (namespace fastmusic, reference-named API) through the shared
// library: a deterministic two-source scene -> spatial_covariance -> exact / fast_music_1 /
// fast_music_2 -> music_spectrum -> extract_peaks, plus the reference's error conventions.
// Prints one "key value..." line per quantity; tests/test_gpu_facade_cpp.py checks them.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <limits>
#include <string>

#include "fastmusic_b200/fastmusic.hpp"

using namespace fastmusic;

static double lcg(std::uint64_t& s) {  // deterministic noise in [-0.5, 0.5)
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return static_cast<double>(s >> 11) * (1.0 / 9007199254740992.0) - 0.5;
}

// "io <dir>": R/tests/test_io.cpp through the facade (host-only, runs without a GPU)
static int io_mode(const std::string& dir) {
    CxMat a(7, 3);
    std::uint64_t st = 5;
    for (Index i = 0; i < 7; ++i)
        for (Index j = 0; j < 3; ++j) a(i, j) = Complex(lcg(st), lcg(st));
    write_matrix_binary(dir + "/mat.bin", a);
    const CxMat back = read_matrix_binary(dir + "/mat.bin");
    double err = 0.0, nrm = 0.0;
    for (Index i = 0; i < a.size(); ++i) {
        err += std::norm(back(i) - a(i));
        nrm += std::norm(a(i));
    }
    std::printf("io_roundtrip %ld %ld %.3g\n", static_cast<long>(back.rows()), static_cast<long>(back.cols()),
                std::sqrt(err / nrm));
    std::FILE* f = std::fopen((dir + "/junk.bin").c_str(), "wb");
    std::fputs("NOPE furthermore", f);
    std::fclose(f);
    try {
        (void)read_matrix_binary(dir + "/junk.bin");
        std::printf("io_badmagic no-throw\n");
    } catch (const std::runtime_error&) {
        std::printf("io_badmagic runtime_error\n");
    }
    CxMat bad(2, 2);
    bad(1, 0) = Complex(std::nan(""), 0.0);
    try {
        write_matrix_binary(dir + "/nan.bin", bad);
        std::printf("io_nonfinite no-throw\n");
    } catch (const std::invalid_argument&) {
        std::printf("io_nonfinite invalid_argument\n");
    }
    CxMat eye(2, 2);
    eye(0, 0) = eye(1, 1) = Complex(1.0, 0.0);
    write_matrix_csv(dir + "/mat.csv", eye);
    PseudoSpectrum p{AngleGrid(3), RealVec(3), Method::Exact, false};
    p.values(0) = 0.5;
    p.values(1) = 1.5;
    p.values(2) = 0.25;
    write_spectrum_csv(dir + "/spec.csv", p);
    std::printf("io_csv written\n");
    return 0;
}

int main(int argc, char** argv) {
    if (argc == 3 && std::string(argv[1]) == "io") return io_mode(argv[2]);
    const Index m = 16, n = 64;
    const double pi = 3.14159265358979323846, d = 0.5, lam = 1.0;
    const double th[2] = {-20.0 * pi / 180.0, 25.0 * pi / 180.0};
    CxMat y(m, n);
    std::uint64_t st = 12345;
    for (int src = 0; src < 2; ++src) {
        const CxVec a = steering_vector(th[src], m, d, lam);
        for (Index t = 0; t < n; ++t) {
            const Complex amp(lcg(st) * 2.0, lcg(st) * 2.0);
            for (Index i = 0; i < m; ++i) y(i, t) += a(i) * amp;
        }
    }
    for (Index t = 0; t < n; ++t)
        for (Index i = 0; i < m; ++i) y(i, t) += Complex(0.05 * lcg(st), 0.05 * lcg(st));
    const HermitianMatrix s = spatial_covariance(y);
    const AngleGrid grid(361, -pi / 2, pi / 2);
    const SubspaceEstimate ex = exact_signal_subspace(s, 2);
    const SubspaceEstimate f1 = fast_music_1(s, 2, Fast1Params{8, 7});
    const SubspaceEstimate f2 = fast_music_2(s, 2, Fast2Params{6, 2, 11});
    for (const auto* e : {&ex, &f1, &f2}) {
        const PseudoSpectrum ps = music_spectrum(*e, grid, d, lam);
        const PeakSet pk = extract_peaks(ps, 2, 3);
        std::printf("%s peaks", method_name(e->method));
        for (Index c : pk.cells) std::printf(" %ld", static_cast<long>(c));
        std::printf(" eig %.9g %.9g\n", e->eigenvalues(0), e->eigenvalues(1));
    }
    std::printf("true_cells %ld %ld\n", static_cast<long>(grid.nearest(th[0])), static_cast<long>(grid.nearest(th[1])));
    // types.hpp:56-62 / linalg.hpp:13: the full decomposition pairs with the exact estimator's leading part
    const EigResult full = hermitian_eig(s);
    std::printf("heig %.9g %.9g n %ld name %s\n", full.eigenvalues(0), full.eigenvalues(1),
                static_cast<long>(full.eigenvectors.cols()), method_name(method_from_name("fast2")));
    try {
        method_from_name("nope");
        std::printf("bad_name no-throw\n");
    } catch (const std::invalid_argument& e) {
        std::printf("bad_name %s\n", std::string(e.what()) == "unknown method name: nope" ? "invalid_argument" : e.what());
    }
    {
        CxMat bad(2, 2);
        bad(1, 0) = Complex(std::numeric_limits<double>::infinity(), 0.0);
        try {
            ensure_finite(bad, "thin_svd");
            std::printf("nonfinite no-throw\n");
        } catch (const std::invalid_argument& e) {
            std::printf("nonfinite %s\n", std::string(e.what()) == "thin_svd: non-finite entries" && !is_finite(bad)
                                               ? "invalid_argument" : e.what());
        }
    }
    try {
        fast_music_2(s, m, Fast2Params{m, 1, 1});
        std::printf("invalid_k no-throw\n");
    } catch (const std::invalid_argument&) {
        std::printf("invalid_k invalid_argument\n");
    }
    try {
        fast_music_2(s, 2, Fast2Params{6, 21, 1});
        std::printf("invalid_t no-throw\n");
    } catch (const std::invalid_argument&) {
        std::printf("invalid_t invalid_argument\n");
    }
    return 0;
}
