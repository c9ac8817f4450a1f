// test_util.hpp — helpers for the C++ drop-in API tests: an mt19937_64 bit source that is
// independent of the library's keyed stream, a deliberately naive dense GF(2) product
// (the role of the reference's tests/oracle_gf2.hpp), and a monobit statistic.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>

#include "ssbh/bitstring.hpp"
#include "ssbh/toeplitz.hpp"

namespace tu {

inline ssbh::BitString random_bits(std::mt19937_64& rng, std::uint64_t nbits) {
    ssbh::BitString b(nbits);
    for (std::uint64_t i = 0; i < nbits; ++i)
        if (rng() & 1) b.set(i, true);
    return b;
}

// K[i] = XOR_j seed[n-1+i-j] & x[j], one bit at a time.
inline ssbh::BitString dense_product(const ssbh::ToeplitzSeed& s, const ssbh::BitString& x) {
    ssbh::BitString out(s.m);
    for (std::uint64_t i = 0; i < s.m; ++i) {
        bool acc = false;
        for (std::uint64_t j = 0; j < s.n; ++j) acc ^= s.seed.get(s.n - 1 + i - j) && x.get(j);
        out.set(i, acc);
    }
    return out;
}

inline double monobit_sigma(const ssbh::BitString& b) {
    const double n = static_cast<double>(b.size());
    return std::fabs(static_cast<double>(b.popcount()) - n / 2) / std::sqrt(n / 4);
}

}  // namespace tu
