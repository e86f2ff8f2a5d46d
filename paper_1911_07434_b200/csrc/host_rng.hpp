// Host-side random streams of the reference, bit-exact (product side).
//
//   Rng (mt19937_64; uniform01, Box-Muller normal with cached spare, rejection below)
//                                  R/include/fastmusic/rng.hpp:15-61
//   Rng::derive (splitmix64)       R/src/linalg.cpp:70-75
//   sample_without_replacement     R/src/linalg.cpp:54-68
//   gaussian_matrix_real           R/src/linalg.cpp:180-192
// Omega and the fast1 column indices are drawn here and copied to the device, as the
// BASELINE contract requires. Bit-exactness is tested against the reference's own
// rng.hpp compiled in the dev container (tests/golden/rng_ref.json).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

namespace fmhost {

class Rng {
public:
    explicit Rng(std::uint64_t seed) : gen_(seed) {}
    std::uint64_t next_u64() { return gen_(); }
    double uniform01() { return static_cast<double>((next_u64() >> 11) + 1) * 0x1.0p-53; }
    double normal() {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        const double u1 = uniform01();
        const double u2 = uniform01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * M_PI * u2;
        spare_ = r * std::sin(a);
        have_spare_ = true;
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
    static std::uint64_t derive(std::uint64_t seed, std::uint64_t tag) {
        std::uint64_t z = seed ^ (tag * 0x9E3779B97F4A7C15ULL + 0xD1B54A32D192ED03ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    // p distinct sorted indices from [0, m) (partial Fisher-Yates). Caller validates 1 <= p <= m.
    std::vector<std::int64_t> sample_without_replacement(std::int64_t m, std::int64_t p) {
        std::vector<std::int64_t> pool(static_cast<std::size_t>(m));
        std::iota(pool.begin(), pool.end(), std::int64_t{0});
        for (std::int64_t i = 0; i < p; ++i) {
            const std::int64_t j = i + static_cast<std::int64_t>(below(static_cast<std::uint64_t>(m - i)));
            std::swap(pool[static_cast<std::size_t>(i)], pool[static_cast<std::size_t>(j)]);
        }
        pool.resize(static_cast<std::size_t>(p));
        std::sort(pool.begin(), pool.end());
        return pool;
    }

private:
    std::mt19937_64 gen_;
    bool have_spare_ = false;
    double spare_ = 0.0;
};

// M x p row-major, entry (i, j) = (i*p + j)-th normal of Rng(seed).
template <typename T>
inline void gaussian_matrix_real(std::int64_t m, std::int64_t p, std::uint64_t seed, T* out) {
    Rng rng(seed);
    for (std::int64_t i = 0; i < m * p; ++i) out[i] = static_cast<T>(rng.normal());
}

}  // namespace fmhost
