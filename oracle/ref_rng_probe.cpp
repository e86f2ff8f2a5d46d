// ORACLE support (test infrastructure). Compiles the reference's OWN header
// R/include/fastmusic/rng.hpp (read in place from /root/reference, never copied)
// against oracle/shim and prints its streams, so tests/golden/rng_ref.json pins
// the oracle restatement (oracle/oracle_rng.cpp) and the product's host RNG to
// the reference implementation bit for bit.
// Usage: ref_rng_probe <seed> <n>   -> JSON on stdout
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include "fastmusic/rng.hpp"

int main(int argc, char** argv) {
    const std::uint64_t seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 42;
    const int n = argc > 2 ? std::atoi(argv[2]) : 16;
    fastmusic::Rng a(seed), b(seed), c(seed), d(seed);
    std::printf("{\"seed\": %" PRIu64 ", \"u64\": [", seed);
    for (int i = 0; i < n; ++i) std::printf("%s\"%" PRIu64 "\"", i ? ", " : "", a.next_u64());
    std::printf("], \"uniform01\": [");
    for (int i = 0; i < n; ++i) std::printf("%s%.17g", i ? ", " : "", b.uniform01());
    std::printf("], \"normal\": [");
    for (int i = 0; i < n; ++i) std::printf("%s%.17g", i ? ", " : "", c.normal());
    std::printf("], \"below7\": [");
    for (int i = 0; i < n; ++i) std::printf("%s%" PRIu64, i ? ", " : "", d.below(7));
    std::printf("]}\n");
    return 0;
}
