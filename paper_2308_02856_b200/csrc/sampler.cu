// sampler.cu — the seeded sub-block sampler on the device.
//
// Restates assign_subblocks + sift_partition + gather (proj/src/sampling.cpp:10-39,
// proj/tools/ssbh_main.cpp:317-331) as three passes over the rounds, without ever
// materialising the reference's 12 B/round host structures:
//
//  pass 1 (k_sample_count, int-ALU bound): V_i = uniform_below(s, i) from
//      KeyedStream(seed, "sampling") — Threefry is counter based, so every round is
//      independent. Emits a 2-byte payload V | x_i<<15 (4-byte when s > 2^15 or a keep
//      mask is given) and counts rounds per (warp-chunk, owned block) with
//      __match_any_sync-aggregated atomics.
//  pass 2 (k_scan_*, HBM/latency bound, tiny): exclusive scan of the count table along
//      chunks -> per-(chunk, block) start rank; block totals n_j.
//  pass 3 (k_scatter, HBM/latency bound): one warp walks its chunk in round order, ranks
//      rounds inside each block with __match_any_sync + a running per-block counter
//      (stable by construction: rank = chunk start + earlier groups + earlier lanes),
//      and writes the data bit straight into block j's REVERSED packed input
//      y_j[n_j-1-rank] (reversal turns the Toeplitz product into forward seed windows,
//      see toeplitz.cu) with a red.or on a zeroed buffer — OR of distinct bits is order
//      independent, so the result is deterministic.
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace ssbh_impl {
using namespace ssbh_dev;

namespace {

struct Key {
    uint64_t ks[5];
};

template <typename P>
struct PayloadBits;
template <>
struct PayloadBits<uint16_t> {
    static constexpr uint32_t kDataShift = 15;
    static constexpr uint32_t kKeepShift = 32;  // none
    static constexpr uint32_t kVMask = 0x7fffu;
};
template <>
struct PayloadBits<uint32_t> {
    static constexpr uint32_t kDataShift = 31;
    static constexpr uint32_t kKeepShift = 30;
    static constexpr uint32_t kVMask = 0x3fffffffu;
};

template <typename P, bool kPow2>
__global__ void __launch_bounds__(256) k_sample_count(Key key, uint64_t n, uint64_t s,
                                                      const uint32_t* __restrict__ in32,
                                                      const uint8_t* __restrict__ keep,
                                                      uint32_t j_lo, uint32_t nown, int cs,
                                                      P* __restrict__ payload,
                                                      uint32_t* __restrict__ counts,
                                                      uint32_t* __restrict__ assign_out) {
    using B = PayloadBits<P>;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t ngroups = (n + 31) / 32;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t g = warp; g < ngroups; g += nwarps) {
        const uint64_t i = g * 32 + lane;
        const bool valid = i < n;
        uint32_t v = 0;
        if (valid) {
            if (kPow2)
                v = (uint32_t)(threefry_w0(key.ks, kTagSampling, 0, i, 0) & (s - 1));
            else
                v = (uint32_t)uniform_below(key.ks, kTagSampling, 0, s, i);
        }
        uint32_t bit = 0;
        if (in32) bit = (__ldg(in32 + g) >> lane) & 1u;
        bool kept = valid;
        if (keep && valid) kept = keep[i] != 0;
        if (valid) {
            if (payload) {
                uint32_t pv = v | (bit << B::kDataShift);
                if (B::kKeepShift < 32 && !kept) pv |= 1u << (B::kKeepShift & 31);
                payload[i] = (P)pv;
            }
            if (assign_out) assign_out[i] = v + 1;
        }
        const uint32_t jj = v - j_lo;
        const bool in = kept && jj < nown;
        const uint32_t peers = __match_any_sync(0xffffffffu, in ? jj : 0xffffffffu);
        if (in && lane == (uint32_t)(__ffs(peers) - 1))
            atomicAdd(counts + (i >> cs) * nown + jj, (uint32_t)__popc(peers));
    }
}

// counts[c][jj] -> group sums gsum[g][jj] (u64)
__global__ void k_scan_groups(const uint32_t* __restrict__ counts, uint64_t nchunks,
                              uint32_t nown, uint64_t group_chunks,
                              unsigned long long* __restrict__ gsum) {
    const uint32_t jj = blockIdx.x * blockDim.x + threadIdx.x;
    if (jj >= nown) return;
    const uint64_t g = blockIdx.y;
    const uint64_t c0 = g * group_chunks;
    const uint64_t c1 = min(nchunks, c0 + group_chunks);
    unsigned long long t = 0;
    for (uint64_t c = c0; c < c1; ++c) t += counts[c * nown + jj];
    gsum[g * nown + jj] = t;
}

// exclusive scan over groups per block, totals -> nj
__global__ void k_scan_totals(unsigned long long* __restrict__ gsum, uint64_t ngroups,
                              uint32_t nown, unsigned long long* __restrict__ nj) {
    const uint32_t jj = blockIdx.x * blockDim.x + threadIdx.x;
    if (jj >= nown) return;
    unsigned long long run = 0;
    for (uint64_t g = 0; g < ngroups; ++g) {
        const unsigned long long t = gsum[g * nown + jj];
        gsum[g * nown + jj] = run;
        run += t;
    }
    nj[jj] = run;
}

// counts -> per-chunk start ranks (in place, u32: device path limits n_j < 2^32, checked
// by the layout kernel)
__global__ void k_scan_apply(uint32_t* __restrict__ counts, uint64_t nchunks, uint32_t nown,
                             uint64_t group_chunks,
                             const unsigned long long* __restrict__ gsum) {
    const uint32_t jj = blockIdx.x * blockDim.x + threadIdx.x;
    if (jj >= nown) return;
    const uint64_t g = blockIdx.y;
    const uint64_t c0 = g * group_chunks;
    const uint64_t c1 = min(nchunks, c0 + group_chunks);
    unsigned long long base = gsum[g * nown + jj];
    for (uint64_t c = c0; c < c1; ++c) {
        const uint32_t t = counts[c * nown + jj];
        counts[c * nown + jj] = (uint32_t)base;
        base += t;
    }
}

template <typename P, bool kSmemRow>
__global__ void __launch_bounds__(256) k_scatter(const P* __restrict__ payload, uint64_t n,
                                                 uint32_t j_lo, uint32_t nown, int cs,
                                                 uint64_t nchunks, uint32_t* __restrict__ offs,
                                                 const unsigned long long* __restrict__ nj,
                                                 const unsigned long long* __restrict__ yoff,
                                                 uint32_t* __restrict__ ybuf,
                                                 unsigned long long* __restrict__ idx_out,
                                                 const unsigned long long* __restrict__ csr_off) {
    using B = PayloadBits<P>;
    extern __shared__ uint32_t srow_all[];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t wib = threadIdx.x >> 5;
    const uint32_t wpb = blockDim.x >> 5;
    for (uint64_t c = blockIdx.x * (uint64_t)wpb + wib; c < nchunks;
         c += (uint64_t)gridDim.x * wpb) {
        uint32_t* row = offs + c * nown;
        if (kSmemRow) {
            uint32_t* srow = srow_all + (size_t)wib * nown;
            for (uint32_t t = lane; t < nown; t += 32) srow[t] = row[t];
            __syncwarp();
            row = srow;
        }
        const uint64_t i0 = c << cs;
        const uint64_t i1 = min(n, (c + 1) << cs);
        for (uint64_t ib = i0; ib < i1; ib += 32) {
            const uint64_t i = ib + lane;
            const bool valid = i < i1;
            const uint32_t p = valid ? (uint32_t)payload[i] : 0u;
            const uint32_t v = p & B::kVMask;
            const uint32_t bit = (p >> B::kDataShift) & 1u;
            bool kept = valid;
            if (B::kKeepShift < 32) kept = kept && !((p >> (B::kKeepShift & 31)) & 1u);
            const uint32_t jj = v - j_lo;
            const bool in = kept && jj < nown;
            const uint32_t peers = __match_any_sync(0xffffffffu, in ? jj : 0xffffffffu);
            const uint32_t leader = __ffs(peers) - 1;
            uint32_t base = 0;
            if (in && lane == leader) base = atomicAdd(row + jj, (uint32_t)__popc(peers));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (in) {
                const uint64_t pos = (uint64_t)base + __popc(peers & lanemask_lt());
                if (idx_out) {
                    idx_out[csr_off[jj] + pos] = i;
                } else if (bit) {
                    const uint64_t q = nj[jj] - 1 - pos;
                    atomicOr(ybuf + yoff[jj] + (q >> 5), 1u << (q & 31));
                }
            }
            __syncwarp();
        }
        __syncwarp();
    }
}


// sift_partition API path: payload from a caller-given assignment (values 1-based) and keep
// mask; counts as in pass 1; out-of-range values raise *bad.
__global__ void k_payload_from_assignment(const uint32_t* __restrict__ assign,
                                          const uint8_t* __restrict__ keep, uint64_t n,
                                          uint64_t s, int cs, uint32_t* __restrict__ payload,
                                          uint32_t* __restrict__ counts, uint32_t* bad) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t ngroups = (n + 31) / 32;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t g = warp; g < ngroups; g += nwarps) {
        const uint64_t i = g * 32 + lane;
        const bool valid = i < n;
        uint32_t v = 0;
        bool kept = false;
        if (valid) {
            const uint32_t a = assign[i];
            if (a == 0 || a > s) {
                atomicOr(bad, 1u);
            } else {
                v = a - 1;
                kept = keep ? keep[i] != 0 : true;
            }
            payload[i] = v | (kept ? 0u : (1u << 30));
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, kept ? v : 0xffffffffu);
        if (kept && lane == (uint32_t)(__ffs(peers) - 1))
            atomicAdd(counts + (i >> cs) * s + v, (uint32_t)__popc(peers));
    }
}

// CSR offsets = exclusive prefix of n_j (single CTA, sequential per 1024-slice carry).
__global__ void k_csr_offsets(const unsigned long long* __restrict__ nj, uint32_t nown,
                              unsigned long long* __restrict__ off) {
    __shared__ unsigned long long sh[1024];
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t base = 0; base < nown; base += 1024) {
        const uint32_t j = base + threadIdx.x;
        const unsigned long long v = j < nown ? nj[j] : 0ull;
        sh[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const unsigned long long t = threadIdx.x >= (unsigned)o ? sh[threadIdx.x - o] : 0ull;
            __syncthreads();
            sh[threadIdx.x] += t;
            __syncthreads();
        }
        if (j < nown) off[j] = carry + sh[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += sh[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) off[nown] = carry;
}

int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

}  // namespace

SamplerGeom make_sampler_geom(uint64_t n, uint64_t s, uint32_t j_lo, uint32_t nown,
                              bool has_keep) {
    SamplerGeom g{};
    g.n = n;
    g.s = s;
    g.j_lo = j_lo;
    g.nown = nown;
    g.payload_bytes = (!has_keep && s <= 32768) ? 2 : 4;
    // warp-chunk: enough chunks for latency hiding in the scatter pass, bounded count table
    int cs = 10;
    auto table_bytes = [&](int shift) {
        const uint64_t nc = (n + (1ull << shift) - 1) >> shift;
        return nc * (uint64_t)nown * 4ull;
    };
    while (cs < 40 && (((n >> cs) > 16384ull) || table_bytes(cs) > (256ull << 20))) ++cs;
    g.chunk_shift = cs;
    g.nchunks = (n + (1ull << cs) - 1) >> cs;
    if (g.nchunks == 0) g.nchunks = 1;
    g.group_chunks = 64;
    g.ngroups = (g.nchunks + g.group_chunks - 1) / g.group_chunks;
    return g;
}

void launch_sample_count(const SamplerGeom& g, const uint64_t key[4], const uint32_t* d_in32,
                         const uint8_t* d_keep, void* d_payload, uint32_t* d_counts,
                         uint32_t* d_assign_out, cudaStream_t st) {
    if (g.n == 0) return;
    Key k;
    threefry_ks(key, k.ks);
    const uint64_t groups = (g.n + 31) / 32;
    uint64_t blocks = (groups + 7) / 8;
    const uint64_t cap = (uint64_t)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    const bool pow2 = (g.s & (g.s - 1)) == 0;
    if (g.payload_bytes == 2) {
        auto* pl = static_cast<uint16_t*>(d_payload);
        if (pow2)
            k_sample_count<uint16_t, true><<<(unsigned)blocks, 256, 0, st>>>(
                k, g.n, g.s, d_in32, d_keep, g.j_lo, g.nown, g.chunk_shift, pl, d_counts,
                d_assign_out);
        else
            k_sample_count<uint16_t, false><<<(unsigned)blocks, 256, 0, st>>>(
                k, g.n, g.s, d_in32, d_keep, g.j_lo, g.nown, g.chunk_shift, pl, d_counts,
                d_assign_out);
    } else {
        auto* pl = static_cast<uint32_t*>(d_payload);
        if (pow2)
            k_sample_count<uint32_t, true><<<(unsigned)blocks, 256, 0, st>>>(
                k, g.n, g.s, d_in32, d_keep, g.j_lo, g.nown, g.chunk_shift, pl, d_counts,
                d_assign_out);
        else
            k_sample_count<uint32_t, false><<<(unsigned)blocks, 256, 0, st>>>(
                k, g.n, g.s, d_in32, d_keep, g.j_lo, g.nown, g.chunk_shift, pl, d_counts,
                d_assign_out);
    }
}

void launch_scan(const SamplerGeom& g, uint32_t* d_counts, unsigned long long* d_gsum,
                 unsigned long long* d_nj, cudaStream_t st) {
    if (g.nown == 0) return;
    const dim3 grid((g.nown + 255) / 256, (unsigned)g.ngroups);
    k_scan_groups<<<grid, 256, 0, st>>>(d_counts, g.nchunks, g.nown, g.group_chunks, d_gsum);
    k_scan_totals<<<(g.nown + 255) / 256, 256, 0, st>>>(d_gsum, g.ngroups, g.nown, d_nj);
    k_scan_apply<<<grid, 256, 0, st>>>(d_counts, g.nchunks, g.nown, g.group_chunks, d_gsum);
}

void launch_scatter(const SamplerGeom& g, const void* d_payload, uint32_t* d_offsets,
                    const unsigned long long* d_nj, const unsigned long long* d_yoff,
                    uint32_t* d_ybuf, unsigned long long* d_idx_out,
                    const unsigned long long* d_csr_off, cudaStream_t st) {
    if (g.n == 0 || g.nown == 0) return;
    const size_t row_bytes = (size_t)g.nown * 4;
    const bool smem = row_bytes <= 32768;
    int wpb = 8;
    size_t shm = 0;
    if (smem) {
        wpb = (int)std::min<size_t>(8, std::max<size_t>(1, (96 * 1024) / row_bytes));
        shm = row_bytes * wpb;
    }
    uint64_t blocks = (g.nchunks + wpb - 1) / wpb;
    const int threads = wpb * 32;
#define SSBH_SCATTER(P, SM)                                                                   \
    do {                                                                                      \
        auto kern = k_scatter<P, SM>;                                                         \
        if (shm > 48 * 1024)                                                                  \
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm); \
        kern<<<(unsigned)blocks, threads, shm, st>>>(                                         \
            static_cast<const P*>(d_payload), g.n, g.j_lo, g.nown, g.chunk_shift, g.nchunks,  \
            d_offsets, d_nj, d_yoff, d_ybuf, d_idx_out, d_csr_off);                           \
    } while (0)
    if (g.payload_bytes == 2) {
        if (smem)
            SSBH_SCATTER(uint16_t, true);
        else
            SSBH_SCATTER(uint16_t, false);
    } else {
        if (smem)
            SSBH_SCATTER(uint32_t, true);
        else
            SSBH_SCATTER(uint32_t, false);
    }
#undef SSBH_SCATTER
}

void launch_payload_from_assignment(const SamplerGeom& g, const uint32_t* d_assign,
                                    const uint8_t* d_keep, uint32_t* d_payload,
                                    uint32_t* d_counts, uint32_t* d_bad, cudaStream_t st) {
    if (g.n == 0) return;
    const uint64_t groups = (g.n + 31) / 32;
    uint64_t blocks = std::min<uint64_t>((groups + 7) / 8, (uint64_t)sm_count() * 8);
    k_payload_from_assignment<<<(unsigned)std::max<uint64_t>(blocks, 1), 256, 0, st>>>(
        d_assign, d_keep, g.n, g.s, g.chunk_shift, d_payload, d_counts, d_bad);
}

void launch_csr_offsets(const unsigned long long* d_nj, uint32_t nown,
                        unsigned long long* d_off, cudaStream_t st) {
    k_csr_offsets<<<1, 1024, 0, st>>>(d_nj, nown, d_off);
}

}  // namespace ssbh_impl
