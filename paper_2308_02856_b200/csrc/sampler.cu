// sampler.cu — the seeded sub-block sampler on the device.
//
// Restates assign_subblocks + sift_partition + gather (proj/src/sampling.cpp:10-39,
// proj/tools/ssbh_main.cpp:317-331) as three passes over the rounds, without ever
// materialising the reference's 12 B/round host structures:
//
//  pass 1 (count, int-ALU bound): V_i = uniform_below(s, i) from KeyedStream(seed,
//      "sampling") — Threefry is counter based, so every round is independent. Emits a
//      2-byte payload V | x_i<<15 (4-byte when s >= 2^15 or a keep mask is given) and counts
//      rounds per (warp-chunk, key) — key = owned block, or (sharded runs) owning rank.
//  pass 2 (k_scan_*, tiny): exclusive scan of the count table along chunks -> per-(chunk,
//      key) start rank; key totals (n_j).
//  pass 3 (k_scatter): one warp walks its chunk in round order, ranks rounds inside each key
//      with ballot peer masks + a warp-owned running counter (stable by construction: rank =
//      chunk start + earlier groups + earlier lanes) and emits:
//        Bits  — the data bit into block j's REVERSED packed input y_j[n_j-1-rank] with a
//                red.or on a zeroed buffer (OR of distinct bits is order independent);
//        Index — the round index into a CSR list (sift_partition API);
//        Owner — the payload itself into the owning rank's receive buffer at a global rank,
//                by direct stores through NVLink peer memory (multi-GPU sharded sampling:
//                the dispatch half of an all-to-all fused into the partition pass).
//
//  In-memory single-level plans (configs 1-3) take the ranked variant of passes 1 and 3
//  (make_ranked): pass 1 (k_count_ranked) also finds each round's stable rank inside its
//  (chunk, block) cell — it is ALU-bound on Threefry, so the ranking is free there — and
//  stores it with the payload; pass 3 (k_scatter_windowed) then needs no order at all: a CTA
//  takes a chunk, ORs each cell's bits into a shared-memory window and writes whole words.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

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
    static constexpr uint32_t kKeepShift = 32;  // none: V = 0x7fff marks a sifted-out round
    static constexpr uint32_t kVMask = 0x7fffu;
};
template <>
struct PayloadBits<uint32_t> {
    static constexpr uint32_t kDataShift = 31;
    static constexpr uint32_t kKeepShift = 30;
    static constexpr uint32_t kVMask = 0x3fffffffu;
};

// Owning rank of block v when s blocks are split into `owners` contiguous balanced ranges
// [o*s/N, (o+1)*s/N) (multigpu.owned_range): the largest o with floor(o*s/N) <= v, i.e.
// o = floor(((v+1)*N - 1) / s).
__device__ __forceinline__ uint32_t owner_of(uint32_t v, uint32_t owners, uint64_t s) {
    return (uint32_t)(((uint64_t)(v + 1) * owners - 1) / s);
}

// ---- pass-1 sources: produce one group's keys (and payload) ---------------------------
// Threefry source: V_i for rounds base+i, optional payload / assignment write.
template <typename P, bool kPow2>
struct TFSource {
    using Bits = PayloadBits<P>;
    Key key;
    uint64_t n, base, s;
    const uint32_t* in32;    // data bits, bit 0 = local round 0 (may be null)
    const uint32_t* keep32;  // sift mask, same layout (may be null)
    P* payload;              // local index (may be null)
    uint32_t* assign_out;    // V+1 per local round (may be null)
    uint32_t j_lo, nown, owners;
    uint32_t bshift;         // > 0: keys are buckets of 2^bshift owned blocks (two-level split)
    __device__ __forceinline__ uint32_t operator()(uint64_t g, uint32_t lane) const {
        const uint64_t i = g * 32 + lane;
        const bool valid = i < n;
        uint32_t v = 0;
        if (valid) {
            if (kPow2)
                v = (uint32_t)(threefry_w0(key.ks, kTagSampling, 0, base + i, 0) & (s - 1));
            else
                v = (uint32_t)uniform_below(key.ks, kTagSampling, 0, s, base + i);
        }
        uint32_t bit = 0;
        if (in32) bit = (__ldg(in32 + g) >> lane) & 1u;
        bool kept = valid;
        if (keep32 && valid) kept = ((__ldg(keep32 + g) >> lane) & 1u) != 0;
        if (valid) {
            if (payload) {
                uint32_t pv = v | (bit << Bits::kDataShift);
                if (!kept) {
                    if (Bits::kKeepShift < 32)
                        pv |= 1u << (Bits::kKeepShift & 31);
                    else
                        pv |= Bits::kVMask;  // u16 (s < 2^15): V = 0x7fff marks sifted-out
                }
                payload[i] = (P)pv;
            }
            if (assign_out) assign_out[i] = v + 1;
        }
        if (!kept) return 0xffffffffu;
        if (owners) return owner_of(v, owners, s);
        const uint32_t jj = v - j_lo;
        return jj < nown ? jj >> bshift : 0xffffffffu;
    }
};

// Payload source: a pass-1 payload already in memory (an owner's received rounds).
template <typename P>
struct PayloadCountSource {
    using Bits = PayloadBits<P>;
    const P* payload;
    uint64_t n;
    uint32_t j_lo, nown;
    uint32_t bshift;  // > 0: bucket keys (see TFSource)
    __device__ __forceinline__ uint32_t operator()(uint64_t g, uint32_t lane) const {
        const uint64_t i = g * 32 + lane;
        if (i >= n) return 0xffffffffu;
        const uint32_t p = payload[i];
        if (Bits::kKeepShift < 32 && ((p >> (Bits::kKeepShift & 31)) & 1u)) return 0xffffffffu;
        const uint32_t jj = (p & Bits::kVMask) - j_lo;
        return jj < nown ? jj >> bshift : 0xffffffffu;
    }
};

// Pass 1, small key spaces: every warp counts one (chunk, part) range into a warp-private
// smem histogram (match_any-aggregated plain read-modify-writes — the warp owns the row),
// then flushes the non-zero bins to the global (chunk, key) table.
template <typename Src>
__global__ void __launch_bounds__(256) k_count_rows(Src src, uint64_t n, uint32_t nkeys, int cs,
                                                    uint64_t nchunks, uint32_t parts,
                                                    uint32_t* __restrict__ counts) {
    extern __shared__ uint32_t hist_all[];
    const uint32_t lane = threadIdx.x & 31;
    uint32_t* hist = hist_all + (size_t)(threadIdx.x >> 5) * nkeys;
    const uint64_t gpc = (1ull << cs) / 32;  // groups per chunk
    const uint64_t ngroups = (n + 31) / 32;
    const uint64_t total = nchunks * parts;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t w = warp; w < total; w += nwarps) {
        const uint64_t c = w / parts, part = w % parts;
        for (uint32_t t = lane; t < nkeys; t += 32) hist[t] = 0;
        __syncwarp();
        const uint64_t g0 = c * gpc + part * gpc / parts;
        const uint64_t g1 = min(ngroups, c * gpc + (part + 1) * gpc / parts);
        // shared-memory atomics into the warp's own histogram (MATCH.ANY aggregation is
        // throughput-bound on sm_100; lanes rarely collide on a bin)
        auto tally = [&](uint32_t jj) {
            if (jj != 0xffffffffu) atomicAdd(&hist[jj], 1u);
        };
        uint64_t g = g0;
        for (; g + 1 < g1; g += 2) {  // two independent Threefry chains per lane (ILP)
            const uint32_t ja = src(g, lane);
            const uint32_t jb = src(g + 1, lane);
            tally(ja);
            tally(jb);
        }
        if (g < g1) tally(src(g, lane));
        __syncwarp();
        for (uint32_t t = lane; t < nkeys; t += 32)
            if (hist[t]) atomicAdd(counts + c * nkeys + t, hist[t]);
        __syncwarp();
    }
}

// Mask of the lanes whose `in` is set and whose key equals this lane's key (kbits low
// bits compared): one ballot per key bit.
__device__ __forceinline__ uint32_t peers_by_ballot(uint32_t key, bool in, int kbits) {
    uint32_t m = __ballot_sync(0xffffffffu, in);
    for (int b = 0; b < kbits; ++b) {
        const uint32_t kb = (key >> b) & 1u;
        const uint32_t bb = __ballot_sync(0xffffffffu, kb);
        m &= bb ^ (kb - 1u);  // kb ? bb : ~bb
    }
    return m;
}

// Ranked pass 1 (SamplerGeom::ranked): one warp per chunk, in round order. V by Threefry (two
// independent chains per lane), then the stable rank of every round among its block's rounds of
// this chunk (running rank in the warp's shared-memory row), stored with the payload: V | bit << 15 | rank << 16 (0x7fff:
// sifted out). The row is the chunk's count row at the end (plain stores, no atomics).
template <bool kPow2>
__global__ void __launch_bounds__(256) k_count_ranked(Key key, uint64_t n, uint64_t s,
                                                      uint32_t j_lo, uint32_t nown,
                                                      const uint32_t* __restrict__ in32,
                                                      const uint32_t* __restrict__ keep32,
                                                      uint32_t* __restrict__ payload, int cs,
                                                      uint64_t nchunks, int kbits,
                                                      uint32_t* __restrict__ counts) {
    extern __shared__ uint32_t hist_all[];
    const uint32_t lane = threadIdx.x & 31;
    uint32_t* hist = hist_all + (size_t)(threadIdx.x >> 5) * 2 * nown;
    uint32_t* own = hist + nown;  // per block: the lane that ranks next (0xffffffff: none)
    for (uint32_t t = lane; t < nown; t += 32) own[t] = 0xffffffffu;
    const uint64_t gpc = (1ull << cs) / 32;  // groups per chunk
    const uint64_t ngroups = (n + 31) / 32;
    auto draw = [&](uint64_t g) -> uint32_t {
        const uint64_t i = g * 32 + lane;
        if (i >= n) return 0;
        return kPow2 ? (uint32_t)(threefry_w0(key.ks, kTagSampling, 0, i, 0) & (s - 1))
                     : (uint32_t)uniform_below(key.ks, kTagSampling, 0, s, i);
    };
    auto rank_store = [&](uint64_t g, uint32_t v) {
        const uint64_t i = g * 32 + lane;
        const bool valid = i < n;
        const uint32_t bit = in32 ? (__ldg(in32 + g) >> lane) & 1u : 0u;
        const bool kept = valid && (keep32 ? ((__ldg(keep32 + g) >> lane) & 1u) != 0 : true);
        const uint32_t jj = v - j_lo;
        const bool in = kept && jj < nown;
        // Stable rank without a peer mask (one ballot per key bit made pass 1 VOTE-bound: +3.4
        // ms at config 3): the lanes of a block race for its owner word with atomicMin, the
        // lowest lane wins, takes the running rank and frees the word; the others go again.
        // Most groups (62 % at 1024 blocks) have no two rounds of one block: one pass.
        uint32_t rank = 0;
        bool pend = in;
        while (__any_sync(0xffffffffu, pend)) {
            if (pend) atomicMin(&own[jj], lane);
            __syncwarp();
            if (pend && own[jj] == lane) {
                rank = hist[jj];
                hist[jj] = rank + 1;
                own[jj] = 0xffffffffu;
                pend = false;
            }
            __syncwarp();
        }
        if (valid) payload[i] = kept ? (v | (bit << 15) | (rank << 16)) : 0x7fffu;
    };
    // chunks are handed out dynamically (the counter is the word after the count table, zeroed
    // with it): equal work per chunk, but a static split leaves the last CTAs of a 2.7-wave
    // grid running alone
    uint32_t* next_chunk = counts + nchunks * nown;
    for (;;) {
        uint32_t cn = 0;
        if (lane == 0) cn = atomicAdd(next_chunk, 1u);
        const uint64_t c = __shfl_sync(0xffffffffu, cn, 0);
        if (c >= nchunks) break;
        for (uint32_t t = lane; t < nown; t += 32) hist[t] = 0;
        __syncwarp();
        const uint64_t g0 = c * gpc, g1 = min(ngroups, g0 + gpc);
        uint64_t g = g0;
        for (; g + 1 < g1; g += 2) {
            const uint32_t va = draw(g), vb = draw(g + 1);
            rank_store(g, va);
            rank_store(g + 1, vb);
        }
        if (g < g1) rank_store(g, draw(g));
        __syncwarp();
        for (uint32_t t = lane; t < nown; t += 32) counts[c * nown + t] = hist[t];
        __syncwarp();
    }
}

// Ranked pass 3: position = the chunk's scanned offset of the block + the rank stored with the
// round; no order between rounds is needed. One warp per chunk (its offset row in shared
// memory), 8 groups of 32 rounds in flight.
template <bool kLate>
__global__ void __launch_bounds__(256) k_scatter_ranked(const uint32_t* __restrict__ payload,
                                                        const uint32_t* __restrict__ in32_late,
                                                        uint64_t n, int cs, uint64_t nchunks,
                                                        uint32_t j_lo, uint32_t nown,
                                                        const uint32_t* __restrict__ offs,
                                                        const unsigned long long* __restrict__ nj,
                                                        const unsigned long long* __restrict__ yoff,
                                                        uint32_t* __restrict__ ybuf) {
    constexpr int U = 8;
    extern __shared__ __align__(16) uint8_t rk_smem[];
    unsigned long long* s_key = reinterpret_cast<unsigned long long*>(rk_smem);
    uint32_t* row = reinterpret_cast<uint32_t*>(rk_smem + (size_t)nown * 8) +
                    (size_t)(threadIdx.x >> 5) * nown;
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t t = threadIdx.x; t < nown; t += blockDim.x)
        s_key[t] = yoff[t] * 32ull + nj[t] - 1ull;  // the block's last bit: rank r lands on it - r
    __syncthreads();
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t c = warp; c < nchunks; c += nwarps) {
        for (uint32_t t = lane; t < nown; t += 32) row[t] = offs[c * nown + t];
        __syncwarp();
        const uint64_t i0 = c << cs, i1 = min(n, (c + 1) << cs);
        for (uint64_t ib = i0; ib < i1; ib += 32 * U) {
            uint32_t p[U], lw[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const uint64_t i = ib + 32 * q + lane;
                p[q] = i < i1 ? payload[i] : 0x7fffu;
                if (kLate) lw[q] = i < i1 ? __ldg(in32_late + (i >> 5)) : 0u;
            }
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const uint32_t v = p[q] & 0x7fffu, jj = v - j_lo;
                const uint32_t bit = kLate ? (lw[q] >> lane) & 1u : (p[q] >> 15) & 1u;
                if (v != 0x7fffu && jj < nown && bit) {
                    const unsigned long long qb = s_key[jj] - (row[jj] + (p[q] >> 16));
                    atomicOr(ybuf + (qb >> 5), 1u << (qb & 31));
                }
            }
        }
        __syncwarp();
    }
}

// Ranked pass 3, windowed: a CTA takes one chunk at a time. The rounds of one (chunk, block)
// cell land on a run of consecutive bits that ends at top = the block's last bit - the chunk's
// scanned offset, so their bits are first ORed into a window of W words per block in shared
// memory (plane-major; word w of the window is global word (top >> 5) - w) and each non-zero
// window word goes out as ONE global red.or — a cell of ~32 rounds costs ~2 L2 atomics instead
// of one per set bit (the per-bit form is bound by the L2's atomic throughput). Ranks past the
// window fall back to the per-bit global atomic.
// A/B (config 3, ms): one warp per chunk with per-bit global atomics 3.06; this kernel 1.42 —
// insensitive to occupancy (4-7 CTAs per SM) and to prefetching the next group into registers
// (1.46-1.55): issue slots and the shared-memory pipe are both ~2/3 busy.
constexpr int kWinThreads = 256;
template <bool kLate>
__global__ void __launch_bounds__(kWinThreads) k_scatter_windowed(
    const uint32_t* __restrict__ payload, const uint32_t* __restrict__ in32_late, uint64_t n, int cs,
    uint64_t nchunks, uint32_t j_lo, uint32_t nown, uint32_t W, const uint32_t* __restrict__ offs,
    const unsigned long long* __restrict__ nj, const unsigned long long* __restrict__ yoff,
    uint32_t* __restrict__ ybuf) {
    constexpr int U = 8;
    extern __shared__ __align__(16) uint8_t rk_smem[];
    // s_key: the last bit of each block (rank r of a chunk lands on it - (offset + r))
    unsigned long long* s_key = reinterpret_cast<unsigned long long*>(rk_smem);  // [nown]
    unsigned long long* top = s_key + nown;                                       // [nown]
    uint32_t* win = reinterpret_cast<uint32_t*>(top + nown);                      // [W][nown]
    const uint32_t* top_lo = reinterpret_cast<const uint32_t*>(top);
    const uint32_t win_a = smem_u32(win);
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t t = threadIdx.x; t < nown; t += kWinThreads)
        s_key[t] = yoff[t] * 32ull + nj[t] - 1ull;
    for (uint32_t t = threadIdx.x; t < nown * W; t += kWinThreads) win[t] = 0u;
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        __syncthreads();  // s_key / the zeroed window; the previous chunk's flush
        for (uint32_t t = threadIdx.x; t < nown; t += kWinThreads)
            top[t] = s_key[t] - offs[c * nown + t];
        __syncthreads();
        const uint64_t i0 = c << cs;
        const uint32_t len = (uint32_t)(min(n, (c + 1) << cs) - i0);
        const uint32_t* pl = payload + i0 + lane;
        const uint32_t* lt = kLate ? in32_late + (i0 >> 5) : nullptr;
        for (uint32_t ib = (threadIdx.x & ~31u) * U; ib < len; ib += kWinThreads * U) {
            uint32_t p[U], lw[U];
            if (ib + 32 * U <= len) {
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    p[q] = pl[ib + 32 * q];
                    if (kLate) lw[q] = __ldg(lt + (ib >> 5) + q);
                }
            } else {
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const bool in = ib + 32 * q + lane < len;
                    p[q] = in ? pl[ib + 32 * q] : 0x7fffu;
                    if (kLate) lw[q] = in ? __ldg(lt + (ib >> 5) + q) : 0u;
                }
            }
            // straight-line per round: sifted-out rounds carry block 0x7fff (>= j_lo + nown)
            bool past = false;
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const uint32_t jj = (p[q] & 0x7fffu) - j_lo;
                const uint32_t bit = kLate ? (lw[q] >> lane) & 1u : p[q] & 0x8000u;
                const bool ok = jj < nown && bit;
                const uint32_t jc = ok ? jj : 0u;
                const uint32_t o = top_lo[2 * jc] & 31u, r = p[q] >> 16;
                const uint32_t w = (r + 31u - o) >> 5;
                red_or_shared_if(win_a + (w * nown + jc) * 4u, 1u << ((o - r) & 31u), ok && w < W);
                past |= ok && w >= W;
            }
            if (past) {  // a cell longer than the window: per-bit global atomics for its tail
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const uint32_t jj = (p[q] & 0x7fffu) - j_lo;
                    const uint32_t bit = kLate ? (lw[q] >> lane) & 1u : p[q] & 0x8000u;
                    if (jj < nown && bit) {
                        const unsigned long long tp = top[jj];
                        const uint32_t o = (uint32_t)tp & 31u, r = p[q] >> 16;
                        if (((r + 31u - o) >> 5) >= W)
                            atomicOr(ybuf + ((tp - r) >> 5), 1u << ((o - r) & 31u));
                    }
                }
            }
        }
        __syncthreads();
        for (uint32_t w = 0; w < W; ++w)
            for (uint32_t jj = threadIdx.x; jj < nown; jj += kWinThreads) {
                const uint32_t val = win[w * nown + jj];
                if (val) {
                    atomicOr(ybuf + ((top[jj] >> 5) - w), val);
                    win[w * nown + jj] = 0u;
                }
            }
    }
}

// Pass 1, large key spaces: counts go straight to the global (chunk, key) table.
template <typename Src>
__global__ void __launch_bounds__(256) k_count_global(Src src, uint64_t n, uint32_t nkeys, int cs,
                                                      uint32_t* __restrict__ counts) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t ngroups = (n + 31) / 32;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t g = warp; g < ngroups; g += nwarps) {
        const uint32_t jj = src(g, lane);
        const uint32_t peers = __match_any_sync(0xffffffffu, jj);
        if (jj != 0xffffffffu && lane == (uint32_t)(__ffs(peers) - 1))
            atomicAdd(counts + ((g * 32) >> cs) * nkeys + jj, (uint32_t)__popc(peers));
    }
}

// counts[c][jj] -> group sums gsum[g][jj] (u64)
// The count table is scanned along chunks per key in three steps: group sums, an
// exclusive scan of the group sums (one warp per key), and the in-place rewrite of every
// count to its chunk's start rank. Loads are issued in batches of kScanBatch before any
// store: the compiler cannot hoist a load of counts[c+1] above the store to counts[c]
// (same array), which serialised the rewrite on DRAM latency.
constexpr int kScanBatch = 8;

__global__ void k_scan_groups(const uint32_t* __restrict__ counts, uint64_t nchunks,
                              uint32_t nown, uint64_t group_chunks,
                              unsigned long long* __restrict__ gsum) {
    // flat grid: (group, 256-key slice) — a grid's y extent is capped at 65535 groups
    const uint32_t kslices = (nown + blockDim.x - 1) / blockDim.x;
    const uint64_t g = blockIdx.x / kslices;
    const uint32_t jj = (blockIdx.x % kslices) * blockDim.x + threadIdx.x;
    if (jj >= nown) return;
    const uint64_t c0 = g * group_chunks;
    const uint64_t c1 = min(nchunks, c0 + group_chunks);
    unsigned long long t = 0;
    for (uint64_t c = c0; c < c1; c += kScanBatch) {
        uint32_t v[kScanBatch];
#pragma unroll
        for (int e = 0; e < kScanBatch; ++e) v[e] = c + e < c1 ? counts[(c + e) * nown + jj] : 0u;
#pragma unroll
        for (int e = 0; e < kScanBatch; ++e) t += v[e];
    }
    gsum[g * nown + jj] = t;
}

// exclusive scan over groups per key (one warp per key, lane-contiguous group ranges),
// totals -> nj. Segmented (two-level split, pass B): every `gps` consecutive groups form one
// bucket region whose scan restarts at 0; warp (seg, key) writes nj[seg * nown + key].
__global__ void k_scan_totals(unsigned long long* __restrict__ gsum, uint64_t ngroups,
                              uint32_t nown, unsigned long long* __restrict__ nj,
                              uint64_t gps, uint64_t nseg) {
    const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (wid >= nseg * nown) return;  // warp-uniform
    const uint32_t jj = (uint32_t)(wid % nown);
    const uint64_t seg = wid / nown;
    const uint64_t gbeg = seg * gps, gend = min(ngroups, gbeg + gps);
    const uint64_t span = gend > gbeg ? gend - gbeg : 0;
    const uint64_t per = (span + 31) / 32;
    const uint64_t g0 = min(gend, gbeg + lane * per), g1 = min(gend, g0 + per);
    unsigned long long mine = 0;
    for (uint64_t g = g0; g < g1; g += kScanBatch) {
        unsigned long long v[kScanBatch];
#pragma unroll
        for (int e = 0; e < kScanBatch; ++e) v[e] = g + e < g1 ? gsum[(g + e) * nown + jj] : 0ull;
#pragma unroll
        for (int e = 0; e < kScanBatch; ++e) mine += v[e];
    }
    unsigned long long inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (uint32_t)o) inc += y;
    }
    unsigned long long run = inc - mine;
    if (lane == 31) nj[seg * nown + jj] = inc;
    for (uint64_t g = g0; g < g1; g += kScanBatch) {
        unsigned long long v[kScanBatch];
#pragma unroll
        for (int e = 0; e < kScanBatch; ++e) v[e] = g + e < g1 ? gsum[(g + e) * nown + jj] : 0ull;
#pragma unroll
        for (int e = 0; e < kScanBatch; ++e) {
            if (g + e < g1) gsum[(g + e) * nown + jj] = run;
            run += v[e];
        }
    }
}

// counts -> per-chunk start ranks (in place, u32: device path limits n_j < 2^32, checked
// by the layout kernel)
__global__ void k_scan_apply(uint32_t* __restrict__ counts, uint64_t nchunks, uint32_t nown,
                             uint64_t group_chunks,
                             const unsigned long long* __restrict__ gsum) {
    // flat grid: (group, 256-key slice) — a grid's y extent is capped at 65535 groups
    const uint32_t kslices = (nown + blockDim.x - 1) / blockDim.x;
    const uint64_t g = blockIdx.x / kslices;
    const uint32_t jj = (blockIdx.x % kslices) * blockDim.x + threadIdx.x;
    if (jj >= nown) return;
    const uint64_t c0 = g * group_chunks;
    const uint64_t c1 = min(nchunks, c0 + group_chunks);
    unsigned long long base = gsum[g * nown + jj];
    for (uint64_t c = c0; c < c1; c += kScanBatch) {
        uint32_t v[kScanBatch];
#pragma unroll
        for (int e = 0; e < kScanBatch; ++e) v[e] = c + e < c1 ? counts[(c + e) * nown + jj] : 0u;
#pragma unroll
        for (int e = 0; e < kScanBatch; ++e) {
            if (c + e < c1) counts[(c + e) * nown + jj] = (uint32_t)base;
            base += v[e];
        }
    }
}

// ---- pass-3 sources -------------------------------------------------------------------
//  PayloadSrc — the payload written by pass 1 (in-memory plans, sharded owners);
//  StreamSrc  — recomputed: V by Threefry, the bit from the current input chunk (streaming
//               plans: no payload buffer, input fed chunk by chunk).
template <typename P>
struct PayloadSrc {
    using Bits = PayloadBits<P>;
    const P* __restrict__ payload;
    __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return payload[i]; }
};

// The payload carries V only and the data bit comes from the input words (the host path copies
// the input while the count pass runs, which needs only the round indices). A separate type,
// so the default scatter keeps its inner loop free of the extra branch.
template <class P>
struct PayloadInSrc {
    using Bits = PayloadBits<P>;
    const P* __restrict__ payload;
    const uint32_t* __restrict__ in32;
    __device__ __forceinline__ uint32_t operator()(uint64_t i) const {
        return payload[i] | (((__ldg(in32 + (i >> 5)) >> (i & 31)) & 1u) << Bits::kDataShift);
    }
};

struct StreamSrc {
    using Bits = PayloadBits<uint32_t>;
    Key key;
    uint64_t s;
    bool pow2;
    const uint32_t* __restrict__ in32;  // chunk words; bit 0 = round `first`
    uint64_t first;
    __device__ __forceinline__ uint32_t operator()(uint64_t i) const {
        const uint64_t r = i - first;
        const uint32_t v =
            pow2 ? (uint32_t)(threefry_w0(key.ks, kTagSampling, 0, i, 0) & (s - 1))
                 : (uint32_t)uniform_below(key.ks, kTagSampling, 0, s, i);
        return v | (((__ldg(in32 + (r >> 5)) >> (r & 31)) & 1u) << Bits::kDataShift);
    }
};

// Bucket — two-level split, pass A: the round goes to its bucket's staging region (rank =
//          position inside the region) as a u16 (local block index | bit << 15).
enum ScatterMode { kModeBits = 0, kModeIndex = 1, kModeOwner = 2, kModeBucket = 3 };

struct ScatterArgs {
    uint64_t c_begin, c_end;  // warp-chunks processed by this launch
    uint64_t n_end;           // one past the last round of this launch
    uint32_t j_lo, nown;      // key space: blocks [j_lo, j_lo+nown), or owners (kModeOwner),
                              // or buckets (kModeBucket), or local blocks (staged kModeBits)
    int kbits, cs;
    uint64_t s;               // kModeOwner: blocks, for owner_of
    uint32_t* offs;           // per-(chunk, key) running ranks
    const unsigned long long* nj;
    const unsigned long long* yoff;
    uint32_t* ybuf;
    unsigned long long* idx_out;
    const unsigned long long* csr_off;
    void* const* dst;                    // kModeOwner: per-owner receive buffers (peer mapped)
    const unsigned long long* dst_base;  // kModeOwner: this rank's first global rank per owner
    // two-level split
    uint32_t bshift;            // log2 blocks per bucket
    uint32_t nblocks;           // kModeBucket: owned blocks
    uint64_t cap;               // kModeBucket: staged rounds per bucket region
    uint16_t* staging;          // kModeBucket: destination regions
    uint32_t* flags;            // kModeBucket: kFlagBucketOverflow on a full region
    const unsigned long long* tot;  // kModeBucket: rounds per bucket (end of the last chunk)
    uint64_t cpb;               // staged kModeBits: chunks per bucket region (0: not staged)
    const uint32_t* rank_base;  // staged kModeBits: per-block rank offset (streaming) or null
    uint64_t fwd_cap;           // staged kModeBits, forward streaming: block jf's bit r goes to
                                // jf * fwd_cap + r of ybuf (n_j unknown yet); 0: reversed blocks
};

template <typename Src, bool kSmemRow, int kMode>
__global__ void __launch_bounds__(256) k_scatter(Src src, ScatterArgs a) {
    using B = typename Src::Bits;
    using P = typename std::conditional<B::kDataShift == 15, uint16_t, uint32_t>::type;
    constexpr int U = 4;  // groups of 32 rounds whose payloads are in flight per warp
    extern __shared__ __align__(16) uint8_t scatter_smem[];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t wib = threadIdx.x >> 5;
    const uint32_t wpb = blockDim.x >> 5;
    const uint32_t nown = a.nown, j_lo = a.j_lo;
    // per-key u64 table: Bits — the end bit yend[jj] (rank pos lands on yend - pos);
    // Owner — this rank's first global rank in owner jj's receive buffer
    unsigned long long* s_key = reinterpret_cast<unsigned long long*>(scatter_smem);
    uint32_t* srow_all = reinterpret_cast<uint32_t*>(scatter_smem + (size_t)nown * 8);
    // kModeBucket: per-warp write combining — a region's staged stream is contiguous per
    // chunk, so every completed 32-B sector leaves as two 16-B stores. Each bucket has a ring
    // of 64 u16 slots (4 sectors, slot = position & 63): one group gives a bucket <= 32
    // consecutive positions, i.e. <= 3 sectors including the one still filling from earlier
    // groups, so no two live elements share a slot; a sector is flushed (after the group's
    // writes) in the group that completes it, before any later group can reuse its slots.
    uint16_t* wb = reinterpret_cast<uint16_t*>(
        scatter_smem + (((size_t)nown * 8 + (size_t)wpb * nown * 4 + 15) & ~(size_t)15) +
        (size_t)wib * nown * 128);
    if (kSmemRow) {
        if (kMode == kModeBits && !a.cpb)
            for (uint32_t t = threadIdx.x; t < nown; t += blockDim.x)
                s_key[t] = a.yoff[t] * 32ull + a.nj[t] - 1ull;
        else if (kMode == kModeOwner)
            for (uint32_t t = threadIdx.x; t < nown; t += blockDim.x) s_key[t] = a.dst_base[t];
        __syncthreads();
    }
    for (uint64_t c = a.c_begin + blockIdx.x * (uint64_t)wpb + wib; c < a.c_end;
         c += (uint64_t)gridDim.x * wpb) {
        uint32_t* row = a.offs + c * nown;
        if (kSmemRow) {
            uint32_t* srow = srow_all + (size_t)wib * nown;
            for (uint32_t t = lane; t < nown; t += 32) srow[t] = row[t];
            __syncwarp();
            row = srow;
        }
        const uint64_t i0 = c << a.cs;
        const uint64_t i1 = min(a.n_end, (c + 1) << a.cs);
        uint32_t cur[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const uint64_t i = i0 + 32 * q + lane;
            cur[q] = i < i1 ? src(i) : 0u;
        }
        for (uint64_t ib = i0; ib < i1; ib += 32 * U) {
            // software pipeline: the next batch's payloads are in flight while this batch is
            // ranked (the ranking itself must stay in round order)
            uint32_t nxt[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const uint64_t i = ib + 32 * (U + q) + lane;
                nxt[q] = i < i1 ? src(i) : 0u;
            }
            // (1) peer masks of the U groups: independent of the running ranks
            //     (ballots per key bit; MATCH.ANY is throughput-bound on sm_100)
            uint32_t jjv[U], peers[U];
            bool inv[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const uint64_t i = ib + 32 * q + lane;
                const uint32_t p = cur[q];
                bool kept = i < i1;
                if (B::kKeepShift < 32) kept = kept && !((p >> (B::kKeepShift & 31)) & 1u);
                if (kMode == kModeOwner) {
                    // shard payloads carry no sift marker (no keep mask on that path), so a
                    // u16 V may be 0x7fff (s = 2^15)
                    jjv[q] = owner_of(p & B::kVMask, nown, a.s);
                    inv[q] = kept;
                } else if (kMode == kModeBucket) {
                    // pass-A payloads carry no u16 marker (a keep mask forces u32 payloads)
                    const uint32_t jb = (p & B::kVMask) - j_lo;
                    jjv[q] = jb >> a.bshift;
                    inv[q] = kept && jb < a.nblocks;
                } else {
                    jjv[q] = (p & B::kVMask) - j_lo;
                    inv[q] = kept && jjv[q] < nown;
                }
                // one __ballot_sync per key bit (MATCH.ANY is throughput-bound on sm_100:
                // round 1, config 3 scatter 8.6 -> 6.3 ms)
                peers[q] = peers_by_ballot(jjv[q], inv[q], a.kbits);
            }
            // (2) in round order: all peers read the running rank (same address: broadcast),
            //     the highest peer writes it back. The warp owns `row` (no atomics); groups
            //     are ordered by __syncwarp.
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const uint64_t i = ib + 32 * q + lane;
                const uint32_t jj = jjv[q];
                const uint32_t pm = peers[q];
                uint64_t pos = 0;
                if (inv[q]) {
                    const uint32_t base = row[jj];
                    if ((pm >> lane) == 1u) row[jj] = base + (uint32_t)__popc(pm);
                    pos = (uint64_t)base + __popc(pm & lanemask_lt());
                    if constexpr (kMode == kModeIndex) {
                        a.idx_out[a.csr_off[jj] + pos] = i;
                    } else if constexpr (kMode == kModeOwner) {
                        const unsigned long long gb = kSmemRow ? s_key[jj] : a.dst_base[jj];
                        static_cast<P*>(a.dst[jj])[gb + pos] = (P)cur[q];
                    } else if constexpr (kMode == kModeBucket) {
                        const uint32_t p = cur[q];
                        const uint32_t local = ((p & B::kVMask) - j_lo) & ((1u << a.bshift) - 1u);
                        const uint16_t v = (uint16_t)(local | (((p >> B::kDataShift) & 1u) << 15));
                        if (pos >= a.cap)
                            atomicOr(a.flags, kFlagBucketOverflow);
                        else if (kSmemRow)
                            wb[jj * 64 + (uint32_t)(pos & 63)] = v;
                        else
                            a.staging[jj * a.cap + pos] = v;
                    } else if ((cur[q] >> B::kDataShift) & 1u) {
                        if (a.cpb) {  // staged rounds: chunk c lies in bucket c / cpb
                            const uint32_t jf = (uint32_t)((c / a.cpb) << a.bshift) + jj;
                            const uint64_t r = pos + (a.rank_base ? __ldg(a.rank_base + jf) : 0u);
                            if (a.fwd_cap) {
                                const uint64_t qb = (uint64_t)jf * a.fwd_cap + r;
                                if (r < a.fwd_cap) atomicOr(a.ybuf + (qb >> 5), 1u << (qb & 31));
                            } else {
                                const uint64_t qb =
                                    __ldg(a.yoff + jf) * 32ull + __ldg(a.nj + jf) - 1ull - r;
                                atomicOr(a.ybuf + (qb >> 5), 1u << (qb & 31));
                            }
                        } else {
                            const unsigned long long e =
                                kSmemRow ? s_key[jj]
                                         : __ldg(a.yoff + jj) * 32ull + __ldg(a.nj + jj) - 1ull;
                            const uint64_t qb = e - pos;
                            atomicOr(a.ybuf + (qb >> 5), 1u << (qb & 31));
                        }
                    }
                }
                __syncwarp();
                if constexpr (kMode == kModeBucket && kSmemRow) {
                    // flush a sector when this round completes it, or ends the chunk's range
                    // in the bucket; sectors shared with a neighbouring chunk go element-wise
                    if (inv[q] && pos < a.cap) {
                        const uint32_t slot = (uint32_t)(pos & 15);
                        bool flush = slot == 15;
                        if (!flush) {
                            const uint64_t end = c + 1 < a.c_end ? a.offs[(c + 1) * nown + jj]
                                                                 : a.tot[jj];
                            flush = pos + 1 == end;
                        }
                        if (flush) {
                            const uint64_t start = a.offs[c * nown + jj];  // global row: unchanged
                            const uint64_t s0 = pos & ~15ull;
                            uint16_t* dst = a.staging + jj * a.cap;
                            const uint16_t* w = wb + jj * 64;
                            if (slot == 15 && s0 >= start) {
                                uint4* d4 = reinterpret_cast<uint4*>(dst + s0);
                                const uint4* w4 = reinterpret_cast<const uint4*>(w + (s0 & 63));
                                d4[0] = w4[0];
                                d4[1] = w4[1];
                            } else {
                                for (uint64_t t = s0 > start ? s0 : start; t <= pos; ++t)
                                    dst[t] = w[t & 63];
                            }
                        }
                    }
                    __syncwarp();
                }
            }
#pragma unroll
            for (int q = 0; q < U; ++q) cur[q] = nxt[q];
        }
        __syncwarp();
    }
    if (kMode == kModeOwner) __threadfence_system();  // peer stores visible to the owners
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

// Pass-1 launcher for any source over n local rounds and nkeys count columns.
template <typename Src>
void count_launch(const Src& src, uint64_t n, uint32_t nkeys, int cs, uint64_t nchunks,
                  uint32_t* d_counts, cudaStream_t st) {
    if (n == 0) return;
    const uint64_t groups = (n + 31) / 32;
    const size_t row_bytes = (size_t)nkeys * 4;
    if (row_bytes * 8 <= 96 * 1024) {
        // enough (chunk, part) work units for ~2 waves of 64 warps per SM, but every unit
        // keeps >= max(8, nkeys/8) 32-round groups so that zeroing and flushing its
        // nkeys-bin histogram stays small against the Threefry work
        const uint64_t gpc = (1ull << cs) / 32;
        const uint64_t want = (uint64_t)sm_count() * 128;
        const uint64_t gmin = std::max<uint64_t>(8, nkeys / 8);
        const uint32_t parts = (uint32_t)std::min<uint64_t>(
            std::max<uint64_t>(1, gpc / gmin), std::max<uint64_t>(1, (want + nchunks - 1) / nchunks));
        const uint64_t units = nchunks * parts;
        const uint64_t blocks = std::min<uint64_t>((units + 7) / 8, (uint64_t)sm_count() * 8);
        const size_t shm = row_bytes * 8;
        auto kern = k_count_rows<Src>;
        if (shm > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        kern<<<(unsigned)std::max<uint64_t>(blocks, 1), 256, shm, st>>>(src, n, nkeys, cs,
                                                                         nchunks, parts, d_counts);
        return;
    }
    uint64_t blocks = (groups + 7) / 8;
    const uint64_t cap = (uint64_t)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    k_count_global<Src><<<(unsigned)blocks, 256, 0, st>>>(src, n, nkeys, cs, d_counts);
}

template <typename P, bool kPow2>
void sample_count_t(const SamplerGeom& g, const Key& k, const uint32_t* d_in32,
                    const uint32_t* d_keep, P* pl, uint32_t* d_counts, uint32_t* d_assign_out,
                    uint64_t base, uint32_t owners, uint32_t bshift, cudaStream_t st) {
    TFSource<P, kPow2> src{k,  g.n,          base,   g.s,    d_in32, d_keep,
                           pl, d_assign_out, g.j_lo, g.nown, owners, bshift};
    const uint32_t nkeys = owners ? owners : (bshift ? ((g.nown - 1) >> bshift) + 1 : g.nown);
    count_launch(src, g.n, nkeys, g.chunk_shift, g.nchunks, d_counts, st);
}

void sample_count_any(const SamplerGeom& g, const uint64_t key[4], const uint32_t* d_in32,
                      const uint32_t* d_keep, void* d_payload, uint32_t* d_counts,
                      uint32_t* d_assign_out, uint64_t base, uint32_t owners, uint32_t bshift,
                      cudaStream_t st) {
    if (g.n == 0) return;
    Key k;
    threefry_ks(key, k.ks);
    const bool pow2 = (g.s & (g.s - 1)) == 0;
    if (g.payload_bytes == 2) {
        auto* pl = static_cast<uint16_t*>(d_payload);
        if (pow2)
            sample_count_t<uint16_t, true>(g, k, d_in32, d_keep, pl, d_counts, d_assign_out, base,
                                           owners, bshift, st);
        else
            sample_count_t<uint16_t, false>(g, k, d_in32, d_keep, pl, d_counts, d_assign_out,
                                            base, owners, bshift, st);
    } else {
        auto* pl = static_cast<uint32_t*>(d_payload);
        if (pow2)
            sample_count_t<uint32_t, true>(g, k, d_in32, d_keep, pl, d_counts, d_assign_out, base,
                                           owners, bshift, st);
        else
            sample_count_t<uint32_t, false>(g, k, d_in32, d_keep, pl, d_counts, d_assign_out,
                                            base, owners, bshift, st);
    }
}

template <int kMode, typename Src>
void scatter_launch(const Src& src, ScatterArgs a, cudaStream_t st) {
    // per-warp bytes: running-rank row (+ write-combining sectors for the bucket split)
    const size_t row_bytes = (size_t)a.nown * 4 + (kMode == kModeBucket ? (size_t)a.nown * 128 : 0);
    const bool smem = row_bytes <= 32768;
    int wpb = 8;
    size_t shm = 0;
    if (smem) {  // per-warp rows (+ sectors) + the per-key u64 table
        wpb = (int)std::min<size_t>(8, std::max<size_t>(1, (96 * 1024) / row_bytes));
        shm = row_bytes * wpb + (size_t)a.nown * 8 + 16;
    }
    const uint64_t nc = a.c_end - a.c_begin;
    const uint64_t blocks = std::max<uint64_t>(1, (nc + wpb - 1) / wpb);
    a.kbits = 1;
    while ((1ull << a.kbits) < a.nown) ++a.kbits;
    auto go = [&](auto kern) {
        if (shm > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        kern<<<(unsigned)blocks, wpb * 32, shm, st>>>(src, a);
    };
    if (smem)
        go(k_scatter<Src, true, kMode>);
    else
        go(k_scatter<Src, false, kMode>);
}

ScatterArgs scatter_args(const SamplerGeom& g, uint32_t* d_offsets,
                         const unsigned long long* d_nj, const unsigned long long* d_yoff,
                         uint32_t* d_ybuf, unsigned long long* d_idx_out,
                         const unsigned long long* d_csr_off) {
    ScatterArgs a{};
    a.c_begin = 0;
    a.c_end = g.nchunks;
    a.n_end = g.n;
    a.j_lo = g.j_lo;
    a.nown = g.nown;
    a.cs = g.chunk_shift;
    a.s = g.s;
    a.offs = d_offsets;
    a.nj = d_nj;
    a.yoff = d_yoff;
    a.ybuf = d_ybuf;
    a.idx_out = d_idx_out;
    a.csr_off = d_csr_off;
    return a;
}

// Count-table geometry (round 1 A/B: a table budget of n >> 7 entries, <= 16384 chunks).
constexpr int kTableBudgetShift = 7;
constexpr uint64_t kMaxTableChunks = 16384;

}  // namespace

SamplerGeom make_sampler_geom(uint64_t n, uint64_t s, uint32_t j_lo, uint32_t nown,
                              bool has_keep, int max_chunk_shift) {
    SamplerGeom g{};
    g.n = n;
    g.s = s;
    g.j_lo = j_lo;
    g.nown = nown;
    // u16 needs V <= 0x7ffe so that 0x7fff can mark sifted-out rounds
    g.payload_bytes = (!has_keep && s < 32768) ? 2 : 4;
    // warp-chunk: enough chunks for latency hiding in the scatter pass, bounded count table
    // (256-round chunks at the low end: small inputs still spread over every SM)
    int cs = std::min(8, max_chunk_shift);
    auto table_bytes = [&](int shift) {
        const uint64_t nc = (n + (1ull << shift) - 1) >> shift;
        return nc * (uint64_t)nown * 4ull;
    };
    // table budget: 256 MiB, or n / 2^budget_shift bytes for very large n (configs 4-5)
    const uint64_t budget = std::max<uint64_t>(256ull << 20, n >> kTableBudgetShift);
    const uint64_t max_chunks = kMaxTableChunks;
    while (cs < max_chunk_shift && (((n >> cs) > max_chunks) || table_bytes(cs) > budget)) ++cs;
    g.chunk_shift = cs;
    g.nchunks = (n + (1ull << cs) - 1) >> cs;
    if (g.nchunks == 0) g.nchunks = 1;
    // scan groups: enough (group, key) threads to fill the GPU, at most 64 chunks deep
    g.group_chunks = std::min<uint64_t>(
        64, std::max<uint64_t>(8, g.nchunks * (uint64_t)std::max<uint32_t>(nown, 1) / (148ull * 2048)));
    g.ngroups = (g.nchunks + g.group_chunks - 1) / g.group_chunks;
    return g;
}

SamplerGeom geom_with_n(const SamplerGeom& g0, uint64_t n) {
    SamplerGeom g = g0;
    g.n = n;
    g.nchunks = std::max<uint64_t>(1, (n + (1ull << g.chunk_shift) - 1) >> g.chunk_shift);
    g.ngroups = (g.nchunks + g.group_chunks - 1) / g.group_chunks;
    return g;
}

SamplerGeom make_ranked(const SamplerGeom& g0) {
    SamplerGeom g = g0;
    // u16-eligible, both rows of a warp in shared memory, payload doubled to <= 8 GiB
    if (g.payload_bytes != 2 || (size_t)g.nown * 8 * 8 > 96 * 1024 || g.n > (1ull << 31)) return g;
    g.ranked = true;
    g.payload_bytes = 4;
    // one warp per chunk in pass 1: twice the chunks of the two-part count kernel when the
    // input is large enough to want them (table <= 256 MiB)
    while (g.chunk_shift > 8 && g.nchunks < 2 * kMaxTableChunks &&
           (g.nchunks * 2) * (uint64_t)g.nown * 4 <= (256ull << 20) && (g.n >> g.chunk_shift) >= kMaxTableChunks) {
        --g.chunk_shift;
        g.nchunks = (g.n + (1ull << g.chunk_shift) - 1) >> g.chunk_shift;
    }
    g.group_chunks = std::min<uint64_t>(
        64, std::max<uint64_t>(8, g.nchunks * (uint64_t)std::max<uint32_t>(g.nown, 1) / (148ull * 2048)));
    g.ngroups = (g.nchunks + g.group_chunks - 1) / g.group_chunks;
    return g;
}

void launch_sample_count(const SamplerGeom& g, const uint64_t key[4], const uint32_t* d_in32,
                         const uint32_t* d_keep, void* d_payload, uint32_t* d_counts,
                         uint32_t* d_assign_out, cudaStream_t st) {
    if (g.ranked && d_payload && !d_assign_out) {
        if (g.n == 0) return;
        Key k;
        threefry_ks(key, k.ks);
        int kbits = 1;
        while ((1ull << kbits) < g.nown) ++kbits;
        const int cwarps = 8;
        const size_t shm = (size_t)g.nown * 8 * cwarps;  // rank row + owner row per warp
        auto go = [&](auto kern) {
            if (shm > 48 * 1024)
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
            int per_sm = 1;  // resident CTAs only: the warps fetch chunks from a counter
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, cwarps * 32, shm);
            const uint64_t blocks = std::min<uint64_t>(
                (g.nchunks + 7) / 8, (uint64_t)sm_count() * std::max(per_sm, 1));
            kern<<<(unsigned)std::max<uint64_t>(blocks, 1), cwarps * 32, shm, st>>>(
                k, g.n, g.s, g.j_lo, g.nown, d_in32, d_keep, static_cast<uint32_t*>(d_payload),
                g.chunk_shift, g.nchunks, kbits, d_counts);
        };
        if ((g.s & (g.s - 1)) == 0)
            go(k_count_ranked<true>);
        else
            go(k_count_ranked<false>);
        return;
    }
    sample_count_any(g, key, d_in32, d_keep, d_payload, d_counts, d_assign_out, 0, 0, 0, st);
}

void launch_sample_slice(const SamplerGeom& g, const uint64_t key[4], uint64_t base,
                         const uint32_t* d_in32, void* d_payload, uint32_t owners,
                         uint32_t* d_counts, cudaStream_t st) {
    sample_count_any(g, key, d_in32, nullptr, d_payload, d_counts, nullptr, base, owners, 0, st);
}

void launch_sample_buckets(const BucketGeom& bg, const SamplerGeom& ga, const uint64_t key[4],
                           uint64_t base, const uint32_t* d_in32, const uint32_t* d_keep,
                           void* d_payload, uint32_t* d_counts, cudaStream_t st) {
    sample_count_any(ga, key, d_in32, d_keep, d_payload, d_counts, nullptr, base, 0, bg.shift,
                     st);
}

void launch_count_payload(const SamplerGeom& g, const void* d_payload, uint32_t* d_counts,
                          cudaStream_t st, uint32_t bshift) {
    const uint32_t nkeys = bshift ? ((g.nown - 1) >> bshift) + 1 : g.nown;
    if (g.payload_bytes == 2)
        count_launch(PayloadCountSource<uint16_t>{static_cast<const uint16_t*>(d_payload), g.n,
                                                  g.j_lo, g.nown, bshift},
                     g.n, nkeys, g.chunk_shift, g.nchunks, d_counts, st);
    else
        count_launch(PayloadCountSource<uint32_t>{static_cast<const uint32_t*>(d_payload), g.n,
                                                  g.j_lo, g.nown, bshift},
                     g.n, nkeys, g.chunk_shift, g.nchunks, d_counts, st);
}

void launch_scan(const SamplerGeom& g, uint32_t* d_counts, unsigned long long* d_gsum,
                 unsigned long long* d_nj, cudaStream_t st, uint64_t seg_groups) {
    if (g.nown == 0) return;
    const uint64_t gps = seg_groups ? seg_groups : g.ngroups;
    const uint64_t nseg = (g.ngroups + gps - 1) / gps;
    const unsigned grid = (unsigned)(((g.nown + 255) / 256) * g.ngroups);
    k_scan_groups<<<grid, 256, 0, st>>>(d_counts, g.nchunks, g.nown, g.group_chunks, d_gsum);
    k_scan_totals<<<(unsigned)((nseg * g.nown + 7) / 8), 256, 0, st>>>(d_gsum, g.ngroups, g.nown,
                                                                       d_nj, gps, nseg);
    k_scan_apply<<<grid, 256, 0, st>>>(d_counts, g.nchunks, g.nown, g.group_chunks, d_gsum);
}

// ---- two-level split for large key spaces ---------------------------------------------
BucketGeom make_bucket_geom(uint64_t n_src, uint64_t s, uint32_t j_lo, uint32_t nown,
                            double mean_per_block, bool has_keep, int max_chunk_shift) {
    BucketGeom bg{};
    // >= 128 blocks per bucket and <= kMaxBuckets buckets (the split's per-warp shared memory
    // grows with the bucket count)
    bg.shift = kBucketShift;
    while (((uint64_t)nown + (1ull << bg.shift) - 1) >> bg.shift > kMaxBuckets) ++bg.shift;
    const uint32_t bb = 1u << bg.shift;
    bg.nbuckets = (nown + bb - 1) / bb;
    // pass A: keys = buckets; u16 payload whenever V fits 15 bits (no keep marker needed)
    bg.a = make_sampler_geom(n_src ? n_src : 1, s, j_lo, bg.nbuckets, has_keep, max_chunk_shift);
    bg.a.n = n_src;
    bg.a.nown = nown;
    bg.a.payload_bytes = (!has_keep && s <= 32768) ? 2 : 4;
    // pass B: one fixed region per bucket = mean + 16 sigma (+ slack), in whole scan groups of
    // 2^cs chunks; count table <= max(64 MiB, n/16 bytes)
    const double mean = mean_per_block * bb;
    const uint64_t cap0 = (uint64_t)(mean + 16.0 * std::sqrt(mean) + 4096.0);
    const uint64_t budget = std::max<uint64_t>(64ull << 20, n_src / 16);
    int cs = 10;
    while (cs < 20 && (uint64_t)bg.nbuckets * (cap0 >> cs) * bb * 4 > budget) ++cs;
    const uint64_t gc = 16;
    const uint64_t span = (1ull << cs) * gc;
    bg.cap = (cap0 + span - 1) / span * span;
    bg.cpb = bg.cap >> cs;
    bg.gps = bg.cpb / gc;
    SamplerGeom& b = bg.b;
    b.n = (uint64_t)bg.nbuckets * bg.cap;
    b.s = s;
    b.j_lo = 0;
    b.nown = bb;
    b.chunk_shift = cs;
    b.nchunks = (uint64_t)bg.nbuckets * bg.cpb;
    b.group_chunks = gc;
    b.ngroups = (uint64_t)bg.nbuckets * bg.gps;
    b.payload_bytes = 2;
    return bg;
}

void launch_bucket_split(const BucketGeom& bg, const SamplerGeom& ga, const void* d_payload,
                         uint32_t* d_offsets_a, const unsigned long long* d_tot_a,
                         uint16_t* d_staging, uint32_t* d_flags, cudaStream_t st,
                         const uint32_t* d_in32_late) {
    if (ga.n == 0) return;
    ScatterArgs a = scatter_args(ga, d_offsets_a, nullptr, nullptr, nullptr, nullptr, nullptr);
    a.nown = bg.nbuckets;
    a.nblocks = ga.nown;
    a.bshift = bg.shift;
    a.cap = bg.cap;
    a.staging = d_staging;
    a.flags = d_flags;
    a.tot = d_tot_a;
    const auto* p16 = static_cast<const uint16_t*>(d_payload);
    const auto* p32 = static_cast<const uint32_t*>(d_payload);
    if (d_in32_late) {
        if (ga.payload_bytes == 2)
            scatter_launch<kModeBucket>(PayloadInSrc<uint16_t>{p16, d_in32_late}, a, st);
        else
            scatter_launch<kModeBucket>(PayloadInSrc<uint32_t>{p32, d_in32_late}, a, st);
    } else if (ga.payload_bytes == 2) {
        scatter_launch<kModeBucket>(PayloadSrc<uint16_t>{p16}, a, st);
    } else {
        scatter_launch<kModeBucket>(PayloadSrc<uint32_t>{p32}, a, st);
    }
}

void launch_bucket_count(const BucketGeom& bg, const uint16_t* d_staging, uint32_t* d_counts_b,
                         cudaStream_t st) {
    const SamplerGeom& b = bg.b;
    count_launch(PayloadCountSource<uint16_t>{d_staging, b.n, 0, b.nown, 0}, b.n, b.nown,
                 b.chunk_shift, b.nchunks, d_counts_b, st);
}

void launch_bucket_scatter(const BucketGeom& bg, const uint16_t* d_staging, uint32_t* d_offsets_b,
                           const unsigned long long* d_nj, const unsigned long long* d_yoff,
                           uint32_t* d_ybuf, const uint32_t* d_rank_base, cudaStream_t st,
                           uint64_t fwd_cap) {
    ScatterArgs a = scatter_args(bg.b, d_offsets_b, d_nj, d_yoff, d_ybuf, nullptr, nullptr);
    a.bshift = bg.shift;
    a.cpb = bg.cpb;
    a.rank_base = d_rank_base;
    a.fwd_cap = fwd_cap;
    scatter_launch<kModeBits>(PayloadSrc<uint16_t>{d_staging}, a, st);
}

// Forward streaming: the blocks' running ranks after an input chunk (+= the chunk's per-block
// totals of pass B; a rank past the block's capacity raises the overflow flag), and the block
// lengths at the end.
__global__ void k_add_ranks(uint32_t* __restrict__ run_rank,
                            const unsigned long long* __restrict__ nj_chunk, uint32_t nown,
                            uint64_t cap, uint32_t* __restrict__ flags) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nown) return;
    const unsigned long long r = run_rank[j] + nj_chunk[j];
    if (r > cap) atomicOr(flags, kFlagBucketOverflow);
    run_rank[j] = (uint32_t)(r > cap ? cap : r);
}
__global__ void k_ranks_to_nj(const uint32_t* __restrict__ run_rank, uint32_t nown,
                              unsigned long long* __restrict__ nj) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < nown) nj[j] = run_rank[j];
}
void launch_add_ranks(uint32_t* d_run_rank, const unsigned long long* d_nj_chunk, uint32_t nown,
                      uint64_t cap, uint32_t* d_flags, cudaStream_t st) {
    if (nown) k_add_ranks<<<(nown + 255) / 256, 256, 0, st>>>(d_run_rank, d_nj_chunk, nown, cap, d_flags);
}
void launch_ranks_to_nj(const uint32_t* d_run_rank, uint32_t nown, unsigned long long* d_nj,
                        cudaStream_t st) {
    if (nown) k_ranks_to_nj<<<(nown + 255) / 256, 256, 0, st>>>(d_run_rank, nown, d_nj);
}

void launch_scatter(const SamplerGeom& g, const void* d_payload, uint32_t* d_offsets,
                    const unsigned long long* d_nj, const unsigned long long* d_yoff,
                    uint32_t* d_ybuf, unsigned long long* d_idx_out,
                    const unsigned long long* d_csr_off, cudaStream_t st,
                    const uint32_t* d_in32_late) {
    if (g.n == 0 || g.nown == 0) return;
    if (g.ranked && !d_idx_out &&
        (g.scatter_window > 0 || (g.scatter_window == 0 && (1ull << g.chunk_shift) >= 8ull * g.s))) {
        // cells of >= 8 rounds: combine a cell's bits in shared memory first. Window = mean
        // cell + 6 sigma + the word alignment, within 48 KB.
        const double mean = (double)(1ull << g.chunk_shift) / (double)g.s;
        uint32_t W = (uint32_t)((mean + 6.0 * std::sqrt(mean) + 31.0) / 32.0) + 1;
        W = std::max<uint32_t>(2, std::min<uint32_t>(W, (48u * 1024u) / (4u * g.nown)));
        if (g.scatter_window > 0)
            W = std::min<uint32_t>((uint32_t)g.scatter_window, (160u * 1024u) / (4u * g.nown));
        const size_t shm = (size_t)g.nown * (16 + 4 * (size_t)W);
        auto go = [&](auto kern) {
            if (shm > 48 * 1024)
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
            int per_sm = 1;  // one wave of resident CTAs: the chunks are equal work
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWinThreads, shm);
            const uint64_t blocks =
                std::min<uint64_t>(g.nchunks, (uint64_t)sm_count() * std::max(per_sm, 1));
            kern<<<(unsigned)std::max<uint64_t>(blocks, 1), kWinThreads, shm, st>>>(
                static_cast<const uint32_t*>(d_payload), d_in32_late, g.n, g.chunk_shift, g.nchunks,
                g.j_lo, g.nown, W, d_offsets, d_nj, d_yoff, d_ybuf);
        };
        if (d_in32_late)
            go(k_scatter_windowed<true>);
        else
            go(k_scatter_windowed<false>);
        return;
    }
    if (g.ranked && !d_idx_out) {
        const size_t shm = (size_t)g.nown * 8 + (size_t)g.nown * 4 * 8 + 16;
        const uint64_t blocks = std::min<uint64_t>((g.nchunks + 7) / 8, (uint64_t)sm_count() * 16);
        auto go = [&](auto kern) {
            if (shm > 48 * 1024)
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
            kern<<<(unsigned)std::max<uint64_t>(blocks, 1), 256, shm, st>>>(
                static_cast<const uint32_t*>(d_payload), d_in32_late, g.n, g.chunk_shift, g.nchunks,
                g.j_lo, g.nown, d_offsets, d_nj, d_yoff, d_ybuf);
        };
        if (d_in32_late)
            go(k_scatter_ranked<true>);
        else
            go(k_scatter_ranked<false>);
        return;
    }
    const ScatterArgs a = scatter_args(g, d_offsets, d_nj, d_yoff, d_ybuf, d_idx_out, d_csr_off);
    if (d_in32_late) {  // host runs: data bits from the input (no index mode there)
        if (g.payload_bytes == 2)
            scatter_launch<kModeBits>(
                PayloadInSrc<uint16_t>{static_cast<const uint16_t*>(d_payload), d_in32_late}, a, st);
        else
            scatter_launch<kModeBits>(
                PayloadInSrc<uint32_t>{static_cast<const uint32_t*>(d_payload), d_in32_late}, a, st);
        return;
    }
    if (g.payload_bytes == 2) {
        const PayloadSrc<uint16_t> src{static_cast<const uint16_t*>(d_payload)};
        d_idx_out ? scatter_launch<kModeIndex>(src, a, st) : scatter_launch<kModeBits>(src, a, st);
    } else {
        const PayloadSrc<uint32_t> src{static_cast<const uint32_t*>(d_payload)};
        d_idx_out ? scatter_launch<kModeIndex>(src, a, st) : scatter_launch<kModeBits>(src, a, st);
    }
}

void launch_scatter_stream(const SamplerGeom& g, const uint64_t key[4], const uint32_t* d_chunk32,
                           uint64_t first, uint64_t count, uint32_t* d_offsets,
                           const unsigned long long* d_nj, const unsigned long long* d_yoff,
                           uint32_t* d_ybuf, cudaStream_t st) {
    if (count == 0 || g.nown == 0) return;
    ScatterArgs a = scatter_args(g, d_offsets, d_nj, d_yoff, d_ybuf, nullptr, nullptr);
    a.c_begin = first >> g.chunk_shift;
    a.c_end = (first + count + (1ull << g.chunk_shift) - 1) >> g.chunk_shift;
    a.n_end = first + count;
    StreamSrc src{};
    threefry_ks(key, src.key.ks);
    src.s = g.s;
    src.pow2 = (g.s & (g.s - 1)) == 0;
    src.in32 = d_chunk32;
    src.first = first;
    scatter_launch<kModeBits>(src, a, st);
}

void launch_owner_split(const SamplerGeom& g, const void* d_payload, uint32_t owners,
                        uint32_t* d_offsets, void* const* d_dst,
                        const unsigned long long* d_dst_base, cudaStream_t st) {
    if (g.n == 0) return;
    ScatterArgs a = scatter_args(g, d_offsets, nullptr, nullptr, nullptr, nullptr, nullptr);
    a.j_lo = 0;
    a.nown = owners;
    a.dst = d_dst;
    a.dst_base = d_dst_base;
    if (g.payload_bytes == 2)
        scatter_launch<kModeOwner>(PayloadSrc<uint16_t>{static_cast<const uint16_t*>(d_payload)},
                                   a, st);
    else
        scatter_launch<kModeOwner>(PayloadSrc<uint32_t>{static_cast<const uint32_t*>(d_payload)},
                                   a, st);
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
