// Drop-in check of the C++ facade (namespace fastmusic, reference-named API) through the shared
// library: a deterministic two-source scene -> spatial_covariance -> exact / fast_music_1 /
// fast_music_2 -> music_spectrum -> extract_peaks, plus the reference's error conventions.
// Prints one "key value..." line per quantity; tests/test_gpu_facade_cpp.py checks them.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>

#include "fastmusic_b200/fastmusic.hpp"

using namespace fastmusic;

static double lcg(std::uint64_t& s) {  // deterministic noise in [-0.5, 0.5)
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return static_cast<double>(s >> 11) * (1.0 / 9007199254740992.0) - 0.5;
}

int main() {
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
