// ORACLE — test infrastructure only. Never linked into the product.
//
// CPU restatement (C++, fp64) of the reference's random streams and of the
// BASELINE synthetic frame model. Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference leg of bench.py may load this library.
//
// Restated reference lines (R/ = /root/reference/proj):
//   Rng ctor / next_u64 / uniform01 / normal / below   R/include/fastmusic/rng.hpp:17-49
//   Rng::sample_without_replacement                    R/src/linalg.cpp:54-68
//   Rng::derive (splitmix64 finalizer)                 R/src/linalg.cpp:70-75
//   gaussian_matrix_real (row-major fill)              R/src/linalg.cpp:180-192
//   steering_vector (std::polar per element)           R/src/scene.cpp:72-82
//   noise convention sigma^2 = total power / 10^(snr/10)  R/src/bench.cpp:262-264
// Pinned against the reference's own rng.hpp compiled here (oracle/ref_rng_probe.cpp,
// golden stream in tests/golden/rng_ref.json) and the C++ standard's mt19937_64
// check value (10000th output = 9981545732273789042).
//
// Frame model (BASELINE configs; documented in DESIGN.md §3):
//   s_f = derive(base_seed, f)
//   Rng(derive(s_f,1)): K angles by rejection (uniform in [lo,hi], pairwise
//       |dtheta| >= min_sep), sorted; then snr = lo + (hi-lo)*uniform01().
//   Rng(derive(s_f,2)): sources S[k][n] = (normal, normal)/sqrt(2) row-major
//       (real part drawn first), then noise N[m][n] = sqrt(sigma2/2)*(normal, normal).
//   X[m][n] = sum_k a_k[m] S[k][n] (k ascending) + N[m][n], fp64, rounded to c64.
//   Omega = gaussian_matrix_real(M, p, derive(s_f,4));
//   fast1 indices = Rng(derive(s_f,3)).sample_without_replacement(M, p).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

namespace {

constexpr double kPi = 3.14159265358979323846;

struct OracleRng {
    std::mt19937_64 gen;
    bool have_spare = false;
    double spare = 0.0;
    explicit OracleRng(std::uint64_t seed) : gen(seed) {}
    std::uint64_t next_u64() { return gen(); }
    double uniform01() { return static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53; }
    double normal() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        const double u1 = uniform01();
        const double u2 = uniform01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * M_PI * u2;
        spare = r * std::sin(a);
        have_spare = true;
        return r * std::cos(a);
    }
    std::uint64_t below(std::uint64_t n) {
        const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        std::uint64_t x;
        do {
            x = next_u64();
        } while (x >= limit);
        return x % n;
    }
};

std::uint64_t derive(std::uint64_t seed, std::uint64_t tag) {
    std::uint64_t z = seed ^ (tag * 0x9E3779B97F4A7C15ULL + 0xD1B54A32D192ED03ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

}  // namespace

extern "C" {

std::uint64_t or_derive(std::uint64_t seed, std::uint64_t tag) { return derive(seed, tag); }

void or_u64_stream(std::uint64_t seed, std::int64_t n, std::uint64_t* out) {
    OracleRng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

void or_uniform_stream(std::uint64_t seed, std::int64_t n, double* out) {
    OracleRng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.uniform01();
}

void or_normal_stream(std::uint64_t seed, std::int64_t n, double* out) {
    OracleRng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.normal();
}

void or_below_stream(std::uint64_t seed, std::uint64_t bound, std::int64_t n, std::uint64_t* out) {
    OracleRng r(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = r.below(bound);
}

// R/src/linalg.cpp:54-68. Returns 0 on success, -1 on invalid (p < 1 or p > m).
int or_sample_without_replacement(std::uint64_t seed, std::int64_t m, std::int64_t p,
                                  std::int64_t* out) {
    if (p < 1 || p > m) return -1;
    OracleRng r(seed);
    std::vector<std::int64_t> pool(static_cast<std::size_t>(m));
    std::iota(pool.begin(), pool.end(), std::int64_t{0});
    for (std::int64_t i = 0; i < p; ++i) {
        const std::int64_t j = i + static_cast<std::int64_t>(r.below(static_cast<std::uint64_t>(m - i)));
        std::swap(pool[static_cast<std::size_t>(i)], pool[static_cast<std::size_t>(j)]);
    }
    pool.resize(static_cast<std::size_t>(p));
    std::sort(pool.begin(), pool.end());
    std::copy(pool.begin(), pool.end(), out);
    return 0;
}

// R/src/linalg.cpp:180-192: entry (i, j) is the (i*p + j)-th normal; out is M x p row-major.
void or_gaussian_matrix_real(std::int64_t m, std::int64_t p, std::uint64_t seed, double* out) {
    OracleRng r(seed);
    for (std::int64_t i = 0; i < m; ++i)
        for (std::int64_t j = 0; j < p; ++j) out[i * p + j] = r.normal();
}

// R/src/scene.cpp:72-82 (no theta restriction), out interleaved (re, im) x M.
void or_steering_vector(double theta, std::int64_t m, double d, double lambda, double* out) {
    const double step = 2.0 * kPi * d * std::sin(theta) / lambda;
    for (std::int64_t i = 0; i < m; ++i) {
        const double ph = step * static_cast<double>(i);
        out[2 * i] = std::cos(ph);
        out[2 * i + 1] = std::sin(ph);
    }
}

// One BASELINE frame. x_out: M x N complex64 interleaved, row-major.
// fixed_angles_rad may be null (then K angles are drawn). Returns 0, or -2 if the
// rejection sampler cannot place K angles.
int or_generate_frame(std::uint64_t frame_seed, std::int64_t m, std::int64_t n, std::int64_t k,
                      double theta_lo, double theta_hi, double min_sep, double snr_lo_db,
                      double snr_hi_db, const double* fixed_angles_rad, double d, double lambda,
                      float* x_out, double* angles_out, double* snr_out) {
    std::vector<double> angles;
    OracleRng ra(derive(frame_seed, 1));
    if (fixed_angles_rad != nullptr) {
        angles.assign(fixed_angles_rad, fixed_angles_rad + k);
    } else {
        int attempts = 0;
        while (static_cast<std::int64_t>(angles.size()) < k) {
            if (++attempts > 100000) return -2;
            const double th = theta_lo + ra.uniform01() * (theta_hi - theta_lo);
            bool ok = true;
            for (double a : angles) {
                if (std::abs(th - a) < min_sep) {
                    ok = false;
                    break;
                }
            }
            if (ok) angles.push_back(th);
        }
    }
    std::sort(angles.begin(), angles.end());
    const double snr = snr_lo_db + (snr_hi_db - snr_lo_db) * ra.uniform01();
    const double sigma2 = static_cast<double>(k) / std::pow(10.0, snr / 10.0);

    OracleRng rn(derive(frame_seed, 2));
    const double inv_sqrt2 = 1.0 / std::sqrt(2.0);
    std::vector<double> s(static_cast<std::size_t>(2 * k * n));
    for (std::int64_t i = 0; i < k * n; ++i) {
        const double re = rn.normal();
        const double im = rn.normal();
        s[2 * i] = re * inv_sqrt2;
        s[2 * i + 1] = im * inv_sqrt2;
    }
    std::vector<double> steer(static_cast<std::size_t>(2 * k * m));
    for (std::int64_t q = 0; q < k; ++q) or_steering_vector(angles[q], m, d, lambda, &steer[2 * q * m]);
    const double scale = std::sqrt(sigma2 / 2.0);
    for (std::int64_t i = 0; i < m; ++i) {
        for (std::int64_t j = 0; j < n; ++j) {
            double acc_re = 0.0, acc_im = 0.0;
            for (std::int64_t q = 0; q < k; ++q) {
                const double ar = steer[2 * (q * m + i)], ai = steer[2 * (q * m + i) + 1];
                const double sr = s[2 * (q * n + j)], si = s[2 * (q * n + j) + 1];
                acc_re += ar * sr - ai * si;
                acc_im += ar * si + ai * sr;
            }
            const double nr = rn.normal();
            const double ni = rn.normal();
            acc_re += scale * nr;
            acc_im += scale * ni;
            x_out[2 * (i * n + j)] = static_cast<float>(acc_re);
            x_out[2 * (i * n + j) + 1] = static_cast<float>(acc_im);
        }
    }
    if (angles_out) std::copy(angles.begin(), angles.end(), angles_out);
    if (snr_out) *snr_out = snr;
    return 0;
}

}  // extern "C"
