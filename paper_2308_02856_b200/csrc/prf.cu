// prf.cu — KeyedStream on the device (proj/src/prf.cpp:80-115) and the synthetic input
// generator. Every output word is index-addressed (counter-based PRF), so the kernels are
// embarrassingly parallel grid-stride loops; int-ALU bound (Threefry, ~200 ALU-pipe SASS
// per block call), not memory bound.
#include "common.cuh"
#include "internal.h"

namespace ssbh_impl {
using namespace ssbh_dev;

namespace {

struct Key {
    uint64_t ks[5];
};

Key make_key(const uint64_t key[4]) {
    Key k;
    threefry_ks(key, k.ks);
    return k;
}

int grid_for(uint64_t work, int threads) {
    uint64_t b = (work + threads - 1) / threads;
    const uint64_t cap = 148ull * 16;
    if (b > cap) b = cap;
    if (b == 0) b = 1;
    return (int)b;
}

__global__ void k_stream_words(Key key, uint64_t tag, uint64_t sub, uint64_t first,
                               uint64_t count, uint64_t* out) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < count;
         q += (uint64_t)gridDim.x * blockDim.x)
        out[q] = threefry_w0(key.ks, tag, sub, first + q, 0);
}

__global__ void k_stream_uniform(Key key, uint64_t tag, uint64_t sub, uint64_t bound,
                                 uint64_t first, uint64_t count, uint64_t* out) {
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < count;
         q += (uint64_t)gridDim.x * blockDim.x)
        out[q] = uniform_below(key.ks, tag, sub, bound, first + q);
}

// bernoulli (prf.cpp:96-102): (double)(r >> 11) * 2^-53 < p is exact in IEEE double, so
// the device compare is bit-identical to the host. Packed 32 draws per word via ballot.
__global__ void k_stream_bernoulli(Key key, uint64_t tag, uint64_t sub, double p, uint64_t first,
                                   uint64_t count, uint32_t* out32) {
    const uint64_t nw = (count + 31) / 32;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t w = warp; w < nw; w += nwarps) {
        const uint64_t q = w * 32 + lane;
        bool b = false;
        if (q < count) {
            const uint64_t r = threefry_w0(key.ks, tag, sub, first + q, 0);
            b = (double)(r >> 11) * 0x1.0p-53 < p;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, b);
        if (lane == 0) out32[w] = m;
    }
}

// bits (prf.cpp:104-115): u64 word w = block({tag, sub, w/4, 1})[w%4]; as u32 words,
// quad f produces u32 words 8f..8f+7. Tail beyond nbits zeroed.
__global__ void k_stream_bits(Key key, uint64_t tag, uint64_t sub, uint64_t nbits,
                              uint32_t* out32) {
    const uint64_t nw32 = (nbits + 31) / 32;
    const uint64_t nquads = (nw32 + 7) / 8;
    for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f < nquads;
         f += (uint64_t)gridDim.x * blockDim.x) {
        const U64x4 r = threefry(key.ks, tag, sub, f, 1);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint64_t w = f * 8 + e;
            if (w >= nw32) break;
            uint32_t v = (uint32_t)(r.v[e >> 1] >> ((e & 1) * 32));
            const uint64_t lo_bit = w * 32;
            if (lo_bit + 32 > nbits) {
                const uint32_t keep = (uint32_t)(nbits - lo_bit);
                v &= keep >= 32 ? 0xffffffffu : ((1u << keep) - 1u);
            }
            out32[w] = v;
        }
    }
}

}  // namespace

void launch_stream_words(const uint64_t key[4], uint64_t tag, uint64_t sub, uint64_t first,
                         uint64_t count, uint64_t* d_out, cudaStream_t st) {
    if (!count) return;
    k_stream_words<<<grid_for(count, 256), 256, 0, st>>>(make_key(key), tag, sub, first, count,
                                                          d_out);
}

void launch_stream_uniform(const uint64_t key[4], uint64_t tag, uint64_t sub, uint64_t bound,
                           uint64_t first, uint64_t count, uint64_t* d_out, cudaStream_t st) {
    if (!count) return;
    k_stream_uniform<<<grid_for(count, 256), 256, 0, st>>>(make_key(key), tag, sub, bound, first,
                                                            count, d_out);
}

void launch_stream_bernoulli(const uint64_t key[4], uint64_t tag, uint64_t sub, double p,
                             uint64_t first, uint64_t count, uint32_t* d_out32,
                             cudaStream_t st) {
    if (!count) return;
    k_stream_bernoulli<<<grid_for(count, 256), 256, 0, st>>>(make_key(key), tag, sub, p, first,
                                                              count, d_out32);
}

void launch_stream_bits(const uint64_t key[4], uint64_t tag, uint64_t sub, uint64_t nbits,
                        uint32_t* d_out32, cudaStream_t st) {
    if (!nbits) return;
    k_stream_bits<<<grid_for((nbits + 255) / 256, 256), 256, 0, st>>>(make_key(key), tag, sub,
                                                                        nbits, d_out32);
}

void launch_make_input(const uint64_t key[4], double p, uint64_t nbits, uint32_t* d_out32,
                       cudaStream_t st) {
    if (p == 0.5)
        launch_stream_bits(key, kTagInput, 0, nbits, d_out32, st);
    else
        launch_stream_bernoulli(key, kTagInput, 0, p, 0, nbits, d_out32, st);
}

}  // namespace ssbh_impl
