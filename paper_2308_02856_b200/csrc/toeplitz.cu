// toeplitz.cu — GF(2) Toeplitz hash of every sub-block (proj/src/toeplitz.cpp:34-52),
// plus the per-block layout, seed generation, input reversal and concatenation kernels.
//
// Math. For block j (n = n_j input bits, k output bits) the reference computes
// K[i] = XOR_j T[i][j] x[j] with T[i][j] = seed[(n-1)+i-j] (toeplitz.hpp:9-17). With the
// input reversed, y[c] = x[n-1-c], this is K[i] = XOR_c seed[i+c] y[c]: row i is the
// FORWARD seed window starting at bit i, independent of n — so one shared seed serves
// every block unchanged, and 32 consecutive rows are 32 lanes reading the same two seed
// words shifted by their lane index.
//
// Kernel (int-ALU bound, no FP, no tensor cores). Lane l of a warp owns rows
// 32*(b+r)+l for r = 0..R-1 (R = kHashR output words per warp). For y word u the row word
// b+r needs the 32-bit seed window W_{r+u} = funnelshift(S[b+r+u], S[b+r+u+1], l), so a
// warp keeps a sliding ring of R windows in registers: per y word it issues ONE
// SHF (new window) and R LOP3 `acc_r ^= W_{u+r} & y_u` (LUT 0x78). After the k-tile the
// row parities are POPC(acc_r)&1, packed with __ballot_sync, and XOR-accumulated into
// the output with red.global.xor (split-K over k-tiles is exact: XOR is associative).
// Seed and y tiles are staged into shared memory by 1-D bulk copies (cp.async.bulk,
// UBLKCP) issued by a producer warp into a 2-stage mbarrier ring; y words are warp-
// uniform broadcast LDS.128 reads. Work items (block, row tile, k tile) are laid out on
// the device (k_layout) and walked by a persistent grid, so no host sync is needed
// between sampling and hashing.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace ssbh_impl {
using namespace ssbh_dev;

namespace {

struct Key {
    uint64_t ks[5];
};

constexpr int R = kHashR;
constexpr int NW = kHashWarps;

__host__ __device__ inline uint64_t round_up(uint64_t v, uint64_t m) { return (v + m - 1) / m * m; }

// ------------------------------------------------------------------------------------
// Layout: one CTA scans the owned blocks. Per block: ypad = round_up(ceil(n_j/32), R);
// k-tiles of <= kt_target words (balanced, multiple of R); items = rowtiles * tiles;
// per-block seed region = rowtiles*NW*R + ypad + 8 words (rounded to 8, covers every
// seed word a tile can read: the bits past k+n_j-1 only ever meet zero y bits).
// ------------------------------------------------------------------------------------
constexpr int kLayoutThreads = 1024;

__device__ inline void block_scan3(unsigned long long v[3], unsigned long long tot[3]) {
    // inclusive->exclusive block scan of 3 u64 lanes with 1024 threads
    __shared__ unsigned long long sh[3][kLayoutThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long inc[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        unsigned long long x = v[q];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        inc[q] = x;
        if (lane == 31) sh[q][wid] = x;
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            unsigned long long x = sh[q][lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            sh[q][lane] = x;  // inclusive warp totals
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const unsigned long long before = wid ? sh[q][wid - 1] : 0ull;
        tot[q] = sh[q][kLayoutThreads / 32 - 1];
        v[q] = before + inc[q] - v[q];
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kLayoutThreads) k_layout(Layout lay, uint32_t nown, uint64_t k,
                                                           uint32_t rowtiles, uint32_t kt_target,
                                                           int per_block, uint64_t limit) {
    __shared__ unsigned long long carry[3];
    __shared__ unsigned long long s_max, s_min, s_ops, s_sum;
    __shared__ uint32_t s_flags;
    if (threadIdx.x == 0) {
        carry[0] = carry[1] = carry[2] = 0;
        s_max = 0;
        s_min = ~0ull;
        s_ops = 0;
        s_sum = 0;
        s_flags = 0;
    }
    __syncthreads();
    const uint64_t seed_fixed = (uint64_t)rowtiles * NW * R + 8;
    unsigned long long my_max = 0, my_min = ~0ull, my_ops = 0, my_sum = 0;
    uint32_t my_flags = 0;
    for (uint32_t base = 0; base < nown; base += kLayoutThreads) {
        const uint32_t jj = base + threadIdx.x;
        unsigned long long v[3] = {0, 0, 0};
        if (jj < nown) {
            const unsigned long long nj = lay.nj[jj];
            const uint64_t yw = (nj + 31) / 32;
            const uint64_t yp = round_up(yw, R);
            uint64_t tiles = 0, L = 0;
            if (yp) {
                const uint64_t want = (yp + kt_target - 1) / kt_target;
                L = round_up((yp + want - 1) / want, R);
                tiles = (yp + L - 1) / L;
            }
            lay.ypad[jj] = (uint32_t)yp;
            lay.ktl[jj] = (uint32_t)L;
            v[0] = yp;
            v[1] = (unsigned long long)rowtiles * tiles;
            v[2] = per_block ? round_up(seed_fixed + yp, 8) : 0;
            my_max = max(my_max, nj);
            my_min = min(my_min, nj);
            my_ops += nj * k;
            my_sum += nj;
            if (nj == 0) my_flags |= kFlagEmpty;
            if (limit && nj > limit) my_flags |= kFlagOversize;
            if (nj >= (1ull << 32)) my_flags |= kFlagTooLong;
        }
        unsigned long long tot[3];
        block_scan3(v, tot);
        if (jj < nown) {
            lay.yoff[jj] = carry[0] + v[0];
            lay.items[jj] = carry[1] + v[1];
            lay.soff[jj] = carry[2] + v[2];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            carry[0] += tot[0];
            carry[1] += tot[1];
            carry[2] += tot[2];
        }
        __syncthreads();
    }
    // warp reductions first: 64-bit shared atomicMax/Min are CAS loops, 1024-way contended
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
        my_min = min(my_min, __shfl_xor_sync(0xffffffffu, my_min, o));
        my_ops += __shfl_xor_sync(0xffffffffu, my_ops, o);
        my_sum += __shfl_xor_sync(0xffffffffu, my_sum, o);
        my_flags |= __shfl_xor_sync(0xffffffffu, my_flags, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&s_max, my_max);
        atomicMin(&s_min, my_min);
        atomicAdd(&s_ops, my_ops);
        atomicAdd(&s_sum, my_sum);
        atomicOr(&s_flags, my_flags);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        lay.yoff[nown] = carry[0];
        lay.items[nown] = carry[1];
        lay.soff[nown] = carry[2];
        DevStats* st = lay.stats;
        st->max_nj = s_max;
        st->min_nj = nown ? s_min : 0;
        st->total_items = carry[1];
        st->seed_words = round_up(seed_fixed + round_up((s_max + 31) / 32, R), 8);
        st->hash_word_ops = s_ops / 32;
        st->sum_nj = s_sum;
        st->flags = s_flags;
    }
}

// ------------------------------------------------------------------------------------
// Seeds: KeyedStream(hash, "hash-seed", sub).bits(...) (prf.cpp:104-115), u64 word w =
// block({tag, sub, w/4, 1})[w%4]. Whole regions are filled with stream bits (prefix-
// stable: the first k+n_j-1 bits equal what the reference builds; the rest only meet zero
// y bits). The buffer holds the seed PRE-SHIFTED by one bit, S'[b] = S[b-1] (S'[0] = 0):
// the hash kernel then forms lane l's window with shift amount l+1 in [1, 32], i.e. with
// the multiplier 2^(31-l) on the FMA pipe (see hash_tile).
// Quad f (u32 words 8f..8f+7 of S') needs the top bit of stream block f-1: taken from the
// neighbour lane by shuffle, recomputed by lane 0.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void write_shifted_quad(uint32_t* dst, const U64x4& r,
                                                   uint32_t carry_in) {
    uint32_t w[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) w[e] = (uint32_t)(r.v[e >> 1] >> ((e & 1) * 32));
    uint32_t o[8];
    o[0] = (w[0] << 1) | carry_in;
#pragma unroll
    for (int e = 1; e < 8; ++e) o[e] = (w[e] << 1) | (w[e - 1] >> 31);
    uint4* d = reinterpret_cast<uint4*>(dst);
    d[0] = make_uint4(o[0], o[1], o[2], o[3]);
    d[1] = make_uint4(o[4], o[5], o[6], o[7]);
}

__device__ __forceinline__ void seed_region(const Key& key, uint64_t sub, uint64_t nquads,
                                            uint32_t* dst, uint64_t f0, uint64_t stride) {
    const uint32_t lane = threadIdx.x & 31;
    // all lanes of a warp walk the same trip count so the shuffle stays converged
    for (uint64_t fb = f0 - lane; fb < nquads; fb += stride) {
        const uint64_t f = fb + lane;
        U64x4 r = {};
        if (f < nquads) r = threefry(key.ks, kTagHashSeed, sub, f, 1);
        uint32_t carry = __shfl_up_sync(0xffffffffu, (uint32_t)(r.v[3] >> 63), 1);
        if (lane == 0) carry = f > 0 ? (uint32_t)(threefry(key.ks, kTagHashSeed, sub, f - 1, 1).v[3] >> 63) : 0u;
        if (f < nquads) write_shifted_quad(dst + f * 8, r, carry);
    }
}

__global__ void k_seeds_shared(Key key, const DevStats* __restrict__ st, uint32_t* sbuf) {
    const uint64_t nquads = st->seed_words / 8;
    seed_region(key, 0, nquads, sbuf, blockIdx.x * (uint64_t)blockDim.x + threadIdx.x,
                (uint64_t)gridDim.x * blockDim.x);
}

__global__ void k_seeds_per_block(Key key, const unsigned long long* __restrict__ soff,
                                  uint32_t j_lo, uint32_t jj0, uint32_t* sbuf) {
    const uint32_t jj = jj0 + blockIdx.y;
    const uint64_t w0 = soff[jj];
    seed_region(key, (uint64_t)j_lo + jj, (soff[jj + 1] - w0) / 8, sbuf + w0,
                blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, (uint64_t)gridDim.x * blockDim.x);
}

// ------------------------------------------------------------------------------------
// y[c] = x[n-1-c]: y word u holds x bits [n-32u-32, n-32u-1] bit-reversed.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t reversed_word(const uint32_t* __restrict__ x, uint64_t n,
                                                  uint64_t u) {
    if (32 * u >= n) return 0u;
    const uint64_t xw = (n + 31) / 32;
    const int64_t hi = (int64_t)n - 1 - 32 * (int64_t)u;  // x index of y bit 32u
    const int64_t lo = hi - 31;
    uint32_t v;
    if (lo >= 0) {
        const uint64_t q = (uint64_t)lo >> 5;
        const uint32_t a = x[q];
        const uint32_t b = q + 1 < xw ? x[q + 1] : 0u;
        v = __funnelshift_r(a, b, (uint32_t)(lo & 31));
    } else {
        v = x[0] << (uint32_t)(-lo);  // bits below x[0] do not exist
    }
    return __brev(v);  // y bit e = x bit hi-e = v bit 31-e
}

__global__ void k_reverse(const uint32_t* __restrict__ x, uint64_t n, uint32_t* __restrict__ y,
                          uint64_t ywords) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < ywords;
         u += (uint64_t)gridDim.x * blockDim.x)
        y[u] = reversed_word(x, n, u);
}

// Forward streaming: block jj's bits sit in order at fwd + jj * cap_words (capacity cap_words
// words); its reversed, padded form goes to ybuf + yoff[jj] (ypad[jj] words).
__global__ void k_reverse_blocks(const uint32_t* __restrict__ fwd, uint64_t cap_words, Layout lay,
                                 uint32_t nown, uint32_t* __restrict__ ybuf) {
    for (uint32_t jj = blockIdx.y; jj < nown; jj += gridDim.y) {
        const uint32_t* x = fwd + (uint64_t)jj * cap_words;
        const uint64_t n = lay.nj[jj];
        uint32_t* y = ybuf + lay.yoff[jj];
        const uint64_t yp = lay.ypad[jj];
        for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < yp;
             u += (uint64_t)gridDim.x * blockDim.x)
            y[u] = reversed_word(x, n, u);
    }
}

// Batched API path: CTA row blockIdx.y = block; the blockIdx.x slices of a row copy its seed
// (m+n-1 bits, tail masked, pre-shifted one bit) into the per-block seed region and write the
// reversed input into its y region, gridDim.x * blockDim.x words per sweep.
__global__ void k_pack_blocks(const uint64_t* __restrict__ seeds,
                              const unsigned long long* __restrict__ seed_off,
                              const uint64_t* __restrict__ inputs,
                              const unsigned long long* __restrict__ in_off, Layout lay,
                              uint64_t m, uint32_t count, uint32_t* __restrict__ sbuf,
                              uint32_t* __restrict__ ybuf) {
  for (uint32_t jj = blockIdx.y; jj < count; jj += gridDim.y) {
    const uint64_t n = lay.nj[jj];
    const uint64_t sbits = m + n - 1;
    const uint32_t* s32 = reinterpret_cast<const uint32_t*>(seeds + seed_off[jj]);
    uint32_t* dst = sbuf + lay.soff[jj];
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    // pre-shifted by one bit (S'[b] = S[b-1]), see the seed kernels
    const uint64_t sw = (sbits + 31) / 32;
    auto seed_word = [&](uint64_t w) {
        uint32_t v = s32[w];
        const uint64_t lo = w * 32;
        if (lo + 32 > sbits) v &= (1u << (uint32_t)(sbits - lo)) - 1u;
        return v;
    };
    for (uint64_t w = t0; w <= sw; w += step) {
        const uint32_t cur = w < sw ? seed_word(w) : 0u;
        const uint32_t prev = w ? seed_word(w - 1) : 0u;
        dst[w] = (cur << 1) | (prev >> 31);
    }
    const uint32_t* x32 = reinterpret_cast<const uint32_t*>(inputs + in_off[jj]);
    uint32_t* y = ybuf + lay.yoff[jj];
    const uint64_t yp = lay.ypad[jj];
    for (uint64_t u = t0; u < yp; u += step) y[u] = reversed_word(x32, n, u);
  }
}

// ------------------------------------------------------------------------------------
// The hash kernel.
// ------------------------------------------------------------------------------------
struct ItemDesc {
    uint32_t jj;   // owned block, 0xffffffff = stop
    uint32_t b0;   // first output word of the row tile
    uint32_t L;    // y words of this k tile (multiple of R)
    uint32_t pad;
};

constexpr int kSTileWords = NW * R + kHashKTMax + 8;
constexpr int kStageWords = kHashKTMax + kSTileWords;
constexpr size_t kHashSmem =
    (size_t)kHashStages * kStageWords * 4 + kHashStages * (sizeof(ItemDesc) + 16) + 64;

// Lane l's 32-bit seed window starting at bit 32t + l, from the pre-shifted seed S':
// funnelshift(S'[t], S'[t+1], l+1), one SHF on the ALU pipe. (Round 1 also tried the window
// as two FMA-pipe IMADs, umulhi(S'[t], 2^(31-l)) + S'[t+1] * 2^(31-l), to leave the ALU pipe
// to the LOP3s alone; it measured no faster and is not built.)
__device__ __forceinline__ uint32_t window(uint32_t a, uint32_t b, uint32_t m) {
    return __funnelshift_rc(a, b, m);
}

__device__ __forceinline__ void hash_tile(const uint32_t* __restrict__ Ys,
                                          const uint32_t* __restrict__ Sw, int L,
                                          uint32_t m, uint32_t (&acc)[R]) {
    uint32_t win[R];
#pragma unroll
    for (int t = 0; t < R; ++t) win[t] = window(Sw[t], Sw[t + 1], m);
#pragma unroll 1
    for (int T = 0; T < L; T += R) {
        const uint32_t* sb = Sw + T + R;
        const uint32_t* yb = Ys + T;
#pragma unroll
        for (int g = 0; g < R / 4; ++g) {
            const uint4 y4 = *reinterpret_cast<const uint4*>(yb + 4 * g);
            const uint4 s4 = *reinterpret_cast<const uint4*>(sb + 4 * g);
            const uint32_t s5 = sb[4 * g + 4];
            const uint32_t yv[4] = {y4.x, y4.y, y4.z, y4.w};
            const uint32_t sv[5] = {s4.x, s4.y, s4.z, s4.w, s5};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int q = 4 * g + e;
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] ^= win[(q + r) % R] & yv[e];
                win[q] = window(sv[e], sv[e + 1], m);
            }
        }
    }
}

__device__ __forceinline__ bool decode_item(const HashArgs& a, unsigned long long item,
                                            uint32_t& jj_hint, ItemDesc& d,
                                            unsigned long long& src_y,
                                            unsigned long long& src_s) {
    const unsigned long long total = a.lay.items[a.nown];
    if (item >= total) return false;
    uint32_t jj = jj_hint;
    while (a.lay.items[jj + 1] <= item) ++jj;  // items are walked in increasing order
    jj_hint = jj;
    const unsigned long long local = item - a.lay.items[jj];
    const uint32_t rt = (uint32_t)(local % a.rowtiles);
    const uint32_t kt = (uint32_t)(local / a.rowtiles);
    const uint32_t Lfull = a.lay.ktl[jj];
    const uint32_t yp = a.lay.ypad[jj];
    const uint32_t u0 = kt * Lfull;
    d.jj = jj;
    d.b0 = rt * (uint32_t)(NW * R);
    d.L = min(Lfull, yp - u0);
    src_y = a.lay.yoff[jj] + u0;
    src_s = (a.per_block_seed ? a.lay.soff[jj] : 0ull) + d.b0 + u0;
    return true;
}

__global__ void __launch_bounds__((NW + 1) * 32, 1) k_toeplitz_hash(HashArgs a) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint32_t* stage_base = reinterpret_cast<uint32_t*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)kHashStages * kStageWords * 4);
    uint64_t* empty = full + kHashStages;
    ItemDesc* desc = reinterpret_cast<ItemDesc*>(empty + kHashStages);

    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kHashStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == NW) {
        // ---------------- producer warp: decode items, stage tiles by bulk copy ------------
        if (lane == 0) {
            uint32_t jj_hint = 0;
            uint32_t it = 0;
            for (unsigned long long item = blockIdx.x;; item += gridDim.x, ++it) {
                const int s = it % kHashStages;
                if (it >= (uint32_t)kHashStages) mbar_wait_sleep(&empty[s], ((it / kHashStages) - 1) & 1);
                ItemDesc d;
                unsigned long long sy, ss;
                const bool ok = decode_item(a, item, jj_hint, d, sy, ss);
                if (!ok) {
                    d.jj = 0xffffffffu;
                    desc[s] = d;
                    mbar_arrive(&full[s]);
                    break;
                }
                desc[s] = d;
                uint32_t* Ys = stage_base + (size_t)s * kStageWords;
                uint32_t* Ss = Ys + kHashKTMax;
                const uint32_t ybytes = d.L * 4;
                const uint32_t sbytes = (uint32_t)round_up((uint64_t)NW * R + d.L + 4, 4) * 4;
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&full[s], ybytes + sbytes);
                bulk_g2s(Ys, a.ybuf + sy, ybytes, &full[s]);
                bulk_g2s(Ss, a.sbuf + ss, sbytes, &full[s]);
            }
        }
        return;
    }

    // -------------------- compute warps --------------------------------------------------
    const uint32_t lane_mult = lane + 1;  // per-lane window shift l+1
    for (uint32_t it = 0;; ++it) {
        const int s = it % kHashStages;
        mbar_wait(&full[s], (it / kHashStages) & 1);
        const ItemDesc d = desc[s];
        if (d.jj == 0xffffffffu) break;
        const uint32_t* Ys = stage_base + (size_t)s * kStageWords;
        const uint32_t* Ss = Ys + kHashKTMax;
        uint32_t acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0;
        hash_tile(Ys, Ss + warp * R, (int)d.L, lane_mult, acc);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // stage may be refilled
        // lane r%32 collects output word r (R/32 words per lane, R a multiple of 32)
        static_assert(R % 32 == 0, "R must be a multiple of 32");
        uint32_t mine[R / 32];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t b = __ballot_sync(0xffffffffu, __popc(acc[r]) & 1u);
            if (lane == (uint32_t)(r % 32)) mine[r / 32] = b;
        }
#pragma unroll
        for (int q = 0; q < R / 32; ++q) {
            const uint32_t word = d.b0 + warp * R + q * 32 + lane;
            if (word < a.kw)
                atomicXor(a.out + (unsigned long long)d.jj * a.out_stride + word, mine[q]);
        }
    }
}

// ------------------------------------------------------------------------------------
// Concatenation with bit offsets (bitstring.cpp:42-47), only needed when k % 32 != 0.
// ------------------------------------------------------------------------------------
__device__ inline uint32_t extract_bits(const uint32_t* w, uint64_t bit, uint32_t take) {
    const uint64_t q = bit >> 5;
    const uint32_t r = (uint32_t)(bit & 31);
    uint32_t v = w[q] >> r;
    if (r && take > 32 - r) v |= w[q + 1] << (32 - r);
    return take >= 32 ? v : (v & ((1u << take) - 1u));
}

__global__ void k_concat(const uint32_t* __restrict__ blocks, uint32_t kw, uint32_t nown,
                         uint64_t k, uint32_t* __restrict__ key) {
    const uint64_t total = (uint64_t)nown * k;
    const uint64_t words = (total + 31) / 32;
    for (uint64_t W = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; W < words;
         W += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t bit = W * 32;
        uint64_t jj = bit / k;
        uint64_t i = bit - jj * k;
        uint32_t out = 0, pos = 0;
        while (pos < 32 && bit < total) {
            uint64_t take = (uint64_t)(32 - pos) < k - i ? (uint64_t)(32 - pos) : k - i;
            out |= extract_bits(blocks + jj * kw, i, (uint32_t)take) << pos;
            pos += (uint32_t)take;
            bit += take;
            ++jj;
            i = 0;
        }
        key[W] = out;
    }
}

}  // namespace

void launch_layout(const Layout& lay, uint32_t nown, uint64_t k, uint32_t rowtiles,
                   uint32_t kt_target, int per_block_seed, uint64_t block_limit,
                   cudaStream_t st) {
    k_layout<<<1, kLayoutThreads, 0, st>>>(lay, nown, k, rowtiles,
                                           std::max<uint32_t>(R, std::min<uint32_t>(kt_target, kHashKTMax) / R * R), per_block_seed,
                                           block_limit);
}

void launch_seeds(const uint64_t key[4], const Layout& lay, uint32_t nown, uint32_t j_lo,
                  int per_block_seed, uint64_t max_words_hint, uint32_t* d_sbuf,
                  cudaStream_t st) {
    Key kk;
    threefry_ks(key, kk.ks);
    if (!per_block_seed) {
        uint64_t quads = max_words_hint / 8 + 1;
        uint64_t blocks = std::min<uint64_t>((quads + 255) / 256, 148ull * 8);
        k_seeds_shared<<<(unsigned)std::max<uint64_t>(blocks, 1), 256, 0, st>>>(kk, lay.stats,
                                                                                d_sbuf);
    } else if (nown) {
        const uint64_t per = max_words_hint / 8 + 1;  // quads per block (upper bound)
        unsigned gx = (unsigned)std::min<uint64_t>((per + 255) / 256, 8);
        for (uint32_t jj0 = 0; jj0 < nown; jj0 += 65535u) {  // grid y extent <= 65535
            const uint32_t cnt = std::min<uint32_t>(65535u, nown - jj0);
            k_seeds_per_block<<<dim3(std::max(gx, 1u), cnt), 256, 0, st>>>(kk, lay.soff, j_lo,
                                                                           jj0, d_sbuf);
        }
    }
}

void launch_reverse(const uint32_t* d_x32, uint64_t nbits, uint32_t* d_y, uint64_t ywords,
                    cudaStream_t st) {
    if (!ywords) return;
    const uint64_t blocks = std::min<uint64_t>((ywords + 255) / 256, 148ull * 16);
    k_reverse<<<(unsigned)blocks, 256, 0, st>>>(d_x32, nbits, d_y, ywords);
}

void launch_reverse_blocks(const uint32_t* d_fwd, uint64_t cap_words, const Layout& lay,
                           uint32_t nown, uint64_t mean_words, uint32_t* d_ybuf, cudaStream_t st) {
    if (!nown) return;
    const unsigned gx = (unsigned)std::min<uint64_t>(std::max<uint64_t>(1, (mean_words + 255) / 256), 64);
    const unsigned gy = std::min<unsigned>(nown, 65535u);
    k_reverse_blocks<<<dim3(gx, gy), 256, 0, st>>>(d_fwd, cap_words, lay, nown, d_ybuf);
}

int hash_grid_size(int device) {
    static int cached[64] = {};
    if (device >= 0 && device < 64 && cached[device]) return cached[device];
    cudaFuncSetAttribute(k_toeplitz_hash, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kHashSmem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_toeplitz_hash, (NW + 1) * 32,
                                                  kHashSmem);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int g = std::max(1, per_sm) * sms;
    if (device >= 0 && device < 64) cached[device] = g;
    return g;
}

void launch_hash(const HashArgs& a, int grid, cudaStream_t st) {
    cudaFuncSetAttribute(k_toeplitz_hash, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kHashSmem);
    k_toeplitz_hash<<<grid, (NW + 1) * 32, kHashSmem, st>>>(a);
}

void launch_concat(const uint32_t* d_blocks, uint32_t kw, uint32_t nown, uint64_t k,
                   uint32_t* d_key, cudaStream_t st) {
    const uint64_t words = ((uint64_t)nown * k + 31) / 32;
    if (!words) return;
    const uint64_t blocks = std::min<uint64_t>((words + 255) / 256, 148ull * 16);
    k_concat<<<(unsigned)blocks, 256, 0, st>>>(d_blocks, kw, nown, k, d_key);
}

void launch_pack_blocks(const uint64_t* d_seeds, const unsigned long long* d_seed_off,
                        const uint64_t* d_inputs, const unsigned long long* d_in_off,
                        const Layout& lay, uint32_t count, uint64_t m, uint32_t* d_sbuf,
                        uint32_t* d_ybuf, cudaStream_t st, uint64_t max_words) {
    if (!count) return;
    // ~8 words per thread per sweep; at least one CTA per block, <= 2 waves in total
    uint64_t gx = (max_words + 2047) / 2048;
    gx = std::max<uint64_t>(1, std::min<uint64_t>(gx, std::max<uint64_t>(1, 2048 / count)));
    k_pack_blocks<<<dim3((unsigned)gx, std::min<uint32_t>(count, 65535)), 256, 0, st>>>(
        d_seeds, d_seed_off, d_inputs, d_in_off, lay, m, count, d_sbuf, d_ybuf);
}

}  // namespace ssbh_impl
