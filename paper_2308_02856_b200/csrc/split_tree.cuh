// split_tree.cuh — the 3-for-4 split's tree arithmetic shared by toeplitz_split.cu (leaf
// seeds, combine) and toeplitz_mma.cu (leaf inputs built inside the leaf GEMM).
#pragma once

#include <stdint.h>

namespace ssbh_impl {

constexpr int kMaxL = 9;  // k = 2^21 (config 5) reaches leaves of 2^12 positions at L = 9

// Offsets (bits) whose windows / pieces a leaf XORs. seed: S windows; input: y pieces.
__device__ __forceinline__ int leaf_offsets(uint32_t path, uint32_t L, uint64_t k, uint64_t base,
                                            bool seed, uint64_t* off) {
    int n = 1;
    off[0] = base;
    uint64_t m = k;
    for (uint32_t l = 0; l < L; ++l) {
        m >>= 1;
        // digit l of the path (most significant = level 0)
        uint32_t p = path;
        for (uint32_t q = l + 1; q < L; ++q) p /= 3;
        const uint32_t d = p % 3;  // 0 = P, 1 = Q, 2 = R
        const int n0 = n;
        if (seed) {
            if (d == 0) {
                for (int e = 0; e < n0; ++e) off[e] += m;                       // B1
            } else if (d == 1) {
                for (int e = 0; e < n0; ++e) off[n0 + e] = off[e] + m;          // B0 ^ B1
                n = 2 * n0;
            } else {
                for (int e = 0; e < n0; ++e) { off[n0 + e] = off[e] + m; off[e] += 2 * m; }  // B2 ^ B1
                n = 2 * n0;
            }
        } else {
            if (d == 0) {
                for (int e = 0; e < n0; ++e) off[n0 + e] = off[e] + m;          // x0 ^ x1
                n = 2 * n0;
            } else if (d == 2) {
                for (int e = 0; e < n0; ++e) off[e] += m;                       // x1
            }                                                                   // Q: x0
        }
    }
    return n;
}

}  // namespace ssbh_impl
