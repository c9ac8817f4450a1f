// rounds.cu — the protocol-round front end of run_extraction on the device.
//
//   k_simulate_rounds : simulate_rounds (proj/src/pipeline.cpp:20-55) — five keyed streams
//                       per round, every draw index-addressed, so one thread per 4 rounds
//                       writes one u32 of RoundRecord bytes (pipeline.hpp:15-38).
//   k_rounds_split    : one pass over the RoundRecord bytes producing what the sifted
//                       extraction consumes — the bit-packed hash input (bit_a of every
//                       round, gather_bits pipeline.cpp:59-65), the bit-packed sift mask
//                       (is_key_round, pipeline.cpp:109-110) — and the test-round counters of
//                       the statistics check (pipeline.cpp:91-99). HBM bound: n bytes in,
//                       n/4 bytes out.
#include "common.cuh"
#include "internal.h"

namespace ssbh_impl {
using namespace ssbh_dev;

namespace {

// RoundRecord bits (proj/include/ssbh/pipeline.hpp:18-25)
constexpr uint32_t kBasisAx = 1u << 0, kBasisBx = 1u << 1, kDetected = 1u << 2,
                   kBitA = 1u << 3, kBitB = 1u << 4, kIsTest = 1u << 5;

struct RoundKeys {
    uint64_t ks[5];
    uint64_t tag_a, tag_b, tag_det, tag_bit, tag_noise;
    double p_x, p_det, e_ph, e_bit;
};

// KeyedStream::bernoulli (prf.cpp:96-102): exact in IEEE double on the device too.
__device__ __forceinline__ bool bern(const uint64_t* ks, uint64_t tag, double p, uint64_t i) {
    const uint64_t r = threefry_w0(ks, tag, 0, i, 0);
    return (double)(r >> 11) * 0x1.0p-53 < p;
}

__device__ __forceinline__ uint32_t one_round(const RoundKeys& k, uint64_t i) {
    const bool ax = bern(k.ks, k.tag_a, k.p_x, i);
    const bool bx = bern(k.ks, k.tag_b, k.p_x, i);
    uint32_t r = (ax ? kBasisAx : 0u) | (bx ? kBasisBx : 0u) | (ax && bx ? kIsTest : 0u);
    if (bern(k.ks, k.tag_det, k.p_det, i)) {
        r |= kDetected;
        const uint64_t w = threefry_w0(k.ks, k.tag_bit, 0, i, 0);
        const bool a = (w & 1) != 0;
        bool b;
        if (ax == bx)
            b = a ^ bern(k.ks, k.tag_noise, ax ? k.e_ph : k.e_bit, i);
        else
            b = ((w >> 1) & 1) != 0;  // basis mismatch: uncorrelated outcomes
        r |= (a ? kBitA : 0u) | (b ? kBitB : 0u);
    }
    return r;
}

__global__ void __launch_bounds__(256) k_simulate_rounds(RoundKeys k, uint64_t n, uint8_t* out,
                                                         bool aligned) {
    const uint64_t nq = (n + 3) / 4;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nq;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i0 = q * 4;
        if (aligned && i0 + 4 <= n) {
            uint32_t v = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) v |= one_round(k, i0 + t) << (8 * t);
            reinterpret_cast<uint32_t*>(out)[q] = v;
        } else {
            for (uint64_t i = i0; i < n && i < i0 + 4; ++i) out[i] = (uint8_t)one_round(k, i);
        }
    }
}

// One thread per 32-round word: 32 record bytes -> bit_a word, key-round word, counters.
__global__ void __launch_bounds__(256) k_rounds_split(const uint8_t* __restrict__ rounds,
                                                      uint64_t n, uint32_t* __restrict__ bits32,
                                                      uint32_t* __restrict__ keep32,
                                                      unsigned long long* __restrict__ counts,
                                                      bool aligned) {
    const uint64_t nw = (n + 31) / 32;
    unsigned long long c_test = 0, c_err = 0, c_nodet = 0, c_key = 0;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw;
         w += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t rec[8];
        if (aligned && (w + 1) * 32 <= n) {
            const uint4* p = reinterpret_cast<const uint4*>(rounds + w * 32);
            const uint4 a = __ldg(p), b = __ldg(p + 1);
            rec[0] = a.x; rec[1] = a.y; rec[2] = a.z; rec[3] = a.w;
            rec[4] = b.x; rec[5] = b.y; rec[6] = b.z; rec[7] = b.w;
        } else {
            for (int q = 0; q < 8; ++q) rec[q] = 0;
            for (uint64_t i = w * 32; i < n && i < (w + 1) * 32; ++i)
                rec[(i & 31) >> 2] |= (uint32_t)rounds[i] << (8 * (i & 3));
        }
        uint32_t bw = 0, kw = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint32_t r = (rec[q] >> (8 * t)) & 0xffu;
                const int bit = q * 4 + t;
                bw |= ((r >> 3) & 1u) << bit;
                kw |= ((r & 7u) == kDetected ? 1u : 0u) << bit;  // detected, Z/Z basis
                const bool test = (r & kIsTest) != 0, det = (r & kDetected) != 0;
                c_test += test;
                c_nodet += test && !det;
                c_err += test && det && (((r >> 3) ^ (r >> 4)) & 1u);
            }
        }
        c_key += __popc(kw);
        bits32[w] = bw;
        keep32[w] = kw;
    }
    // zero-filled tail records never count: their IsTest / Detected bits are clear
    for (int o = 16; o > 0; o >>= 1) {
        c_test += __shfl_xor_sync(0xffffffffu, c_test, o);
        c_err += __shfl_xor_sync(0xffffffffu, c_err, o);
        c_nodet += __shfl_xor_sync(0xffffffffu, c_nodet, o);
        c_key += __shfl_xor_sync(0xffffffffu, c_key, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (c_test) atomicAdd(counts + 0, c_test);
        if (c_err) atomicAdd(counts + 1, c_err);
        if (c_nodet) atomicAdd(counts + 2, c_nodet);
        if (c_key) atomicAdd(counts + 3, c_key);
    }
}

int grid_for(uint64_t items) {
    uint64_t b = (items + 255) / 256;
    const uint64_t cap = 148ull * 8;
    return (int)(b == 0 ? 1 : (b > cap ? cap : b));
}

uint64_t tag_of(const char* s) {
    size_t len = 0;
    while (s[len]) ++len;
    return fnv1a(s, len);
}

}  // namespace

void launch_simulate_rounds(const uint64_t key[4], uint64_t n, double p_x, double e_ph,
                            double e_bit, double p_det, uint8_t* d_rounds, cudaStream_t st) {
    RoundKeys k{};
    threefry_ks(key, k.ks);
    k.tag_a = tag_of("basis-a");
    k.tag_b = tag_of("basis-b");
    k.tag_det = tag_of("detect");
    k.tag_bit = tag_of("bit-a");
    k.tag_noise = tag_of("noise");
    k.p_x = p_x;
    k.p_det = p_det;
    k.e_ph = e_ph;
    k.e_bit = e_bit;
    k_simulate_rounds<<<grid_for((n + 3) / 4), 256, 0, st>>>(k, n, d_rounds,
                                                              ((uintptr_t)d_rounds & 3) == 0);
}

void launch_rounds_split(const uint8_t* d_rounds, uint64_t n, uint32_t* d_bits32,
                         uint32_t* d_keep32, unsigned long long* d_counts4, cudaStream_t st) {
    k_rounds_split<<<grid_for((n + 31) / 32), 256, 0, st>>>(d_rounds, n, d_bits32, d_keep32,
                                                            d_counts4,
                                                            ((uintptr_t)d_rounds & 15) == 0);
}

}  // namespace ssbh_impl
