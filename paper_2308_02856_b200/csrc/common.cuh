// common.cuh — shared device/host helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define SSBH_HD __host__ __device__ __forceinline__

namespace ssbh_dev {


// 64-bit rotate by a compile-time constant (lowered to two SHF.L.W funnel shifts,
// or a register swap for r == 32). Round 2 A/B: the rotation as two IMAD.WIDE.U32 on the FMA
// pipe (a * 2^r = (a >> (32 - r)) : (a << r)) made the count pass slower, 14.9 -> 16.1 ms.
template <int R>
SSBH_HD uint64_t rotl(uint64_t x) {
    return (x << R) | (x >> (64 - R));
}

struct U64x4 {
    uint64_t v[4];
};

// Threefry4x64-20 — restates proj/src/prf.cpp:47-76 (Threefish-256 rotation schedule,
// 20 rounds, key parity 0x1BD11BDAA9FC1A22, injection every 4 rounds, x1<->x3 swap).
// The swap is folded into the unrolled data flow (no moves). Fully unrolled with
// compile-time rotation constants.
SSBH_HD void threefry_ks(const uint64_t key[4], uint64_t ks[5]) {
    ks[0] = key[0];
    ks[1] = key[1];
    ks[2] = key[2];
    ks[3] = key[3];
    ks[4] = 0x1BD11BDAA9FC1A22ull ^ key[0] ^ key[1] ^ key[2] ^ key[3];
}

// 64-bit adds stay IADD3 pairs: moving them to the FMA pipe (IMAD.WIDE.U32 + IMAD, a dev A/B
// build) made the Threefry count pass slower (config 3: 14.9 -> 19.2 ms).
#define SSBH_ADD(a, b) ((a) + (b))

#define SSBH_TF_ROUND(RA, RB)                         \
    do {                                              \
        x0 = SSBH_ADD(x0, x1);                        \
        x1 = rotl<RA>(x1) ^ x0;                       \
        x2 = SSBH_ADD(x2, x3);                        \
        x3 = rotl<RB>(x3) ^ x2;                       \
        const uint64_t t_ = x1;                       \
        x1 = x3;                                      \
        x3 = t_;                                      \
    } while (0)

#define SSBH_TF_INJECT(S)                             \
    do {                                              \
        x0 = SSBH_ADD(x0, ks[(S) % 5]);               \
        x1 = SSBH_ADD(x1, ks[((S) + 1) % 5]);         \
        x2 = SSBH_ADD(x2, ks[((S) + 2) % 5]);         \
        x3 = SSBH_ADD(x3, ks[((S) + 3) % 5] + (uint64_t)(S)); \
    } while (0)

SSBH_HD U64x4 threefry(const uint64_t ks[5], uint64_t c0, uint64_t c1, uint64_t c2,
                       uint64_t c3) {
    uint64_t x0 = c0 + ks[0], x1 = c1 + ks[1], x2 = c2 + ks[2], x3 = c3 + ks[3];
    SSBH_TF_ROUND(14, 16); SSBH_TF_ROUND(52, 57); SSBH_TF_ROUND(23, 40); SSBH_TF_ROUND(5, 37);
    SSBH_TF_INJECT(1);
    SSBH_TF_ROUND(25, 33); SSBH_TF_ROUND(46, 12); SSBH_TF_ROUND(58, 22); SSBH_TF_ROUND(32, 32);
    SSBH_TF_INJECT(2);
    SSBH_TF_ROUND(14, 16); SSBH_TF_ROUND(52, 57); SSBH_TF_ROUND(23, 40); SSBH_TF_ROUND(5, 37);
    SSBH_TF_INJECT(3);
    SSBH_TF_ROUND(25, 33); SSBH_TF_ROUND(46, 12); SSBH_TF_ROUND(58, 22); SSBH_TF_ROUND(32, 32);
    SSBH_TF_INJECT(4);
    SSBH_TF_ROUND(14, 16); SSBH_TF_ROUND(52, 57); SSBH_TF_ROUND(23, 40); SSBH_TF_ROUND(5, 37);
    SSBH_TF_INJECT(5);
    U64x4 r;
    r.v[0] = x0;
    r.v[1] = x1;
    r.v[2] = x2;
    r.v[3] = x3;
    return r;
}

// Word 0 only (what KeyedStream::word / uniform_below consume, prf.cpp:80-88). The last
// injection's other three lanes are dead code, which the compiler removes.
SSBH_HD uint64_t threefry_w0(const uint64_t ks[5], uint64_t c0, uint64_t c1, uint64_t c2,
                             uint64_t c3) {
    return threefry(ks, c0, c1, c2, c3).v[0];
}

// KeyedStream::uniform_below (prf.cpp:84-94): pow-2 bound -> mask; else rejection with
// the attempt counter in ctr[3]. 64-bit modulo only on the (unused by BASELINE) slow path.
SSBH_HD uint64_t uniform_below(const uint64_t ks[5], uint64_t tag, uint64_t sub, uint64_t bound,
                               uint64_t index) {
    if ((bound & (bound - 1)) == 0) return threefry_w0(ks, tag, sub, index, 0) & (bound - 1);
    const uint64_t limit = ~0ull - (~0ull % bound + 1) % bound;
    for (uint64_t attempt = 0;; ++attempt) {
        const uint64_t r = threefry_w0(ks, tag, sub, index, attempt);
        if (r <= limit) return r % bound;
    }
}

// prf::tag (prf.hpp:29-37), FNV-1a-64.
SSBH_HD uint64_t fnv1a(const char* s, size_t len) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (size_t i = 0; i < len; ++i) {
        h ^= (uint8_t)s[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

constexpr uint64_t kTagSampling = 0xc723b18281303050ull;  // fnv1a("sampling")
constexpr uint64_t kTagHashSeed = 0xc1d9934d9f44cf81ull;  // fnv1a("hash-seed")
constexpr uint64_t kTagInput = 0x1ebbae8f5810b65bull;     // fnv1a("input")

}  // namespace ssbh_dev
