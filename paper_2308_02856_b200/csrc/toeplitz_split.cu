// toeplitz_split.cu — fewer MACs than n·k: the 3-for-4 split of a Toeplitz/Hankel
// matrix-vector product, on top of the tensor-core hash kernels (toeplitz_mma.cu). A B200-side
// algorithmic change with no reference counterpart: the keys equal toeplitz_hash's
// (proj/src/toeplitz.cpp:34-52) bit for bit; only the number of bit products drops.
//
// A shared-seed block computes K[i] = XOR_c S[i+c] y[c] for i < k (toeplitz.cu). Cut the input
// into T segments of k positions (t k .. t k + k) plus a remainder: each segment is a square
// k x k Hankel product H_t y_t with H_t[i][c] = S[t k + i + c]. Split a square of size 2m into
// m x m blocks: the Hankel structure gives blocks B_d = window of S at offset d m (d = a + b),
//     K_lo = B0 x0 + B1 x1,  K_hi = B1 x0 + B2 x1,
// and over GF(2)
//     P = B1 (x0 ^ x1),  Q = (B0 ^ B1) x0,  R = (B2 ^ B1) x1,  K_lo = P ^ Q,  K_hi = P ^ R:
// three half-size Hankel products instead of four, with seeds that are XORs of windows of S.
// Applied L times, every square becomes 3^L leaves of size k / 2^L: (3/4)^L of the MACs. The
// leaves are "virtual blocks" of the hash kernels — each with its own seed region (an XOR of up
// to 2^L windows of the seed) and its own input (an XOR of up to 2^L pieces of the block's
// reversed input). Shared seed: the leaves of one (segment, path) share their matrix across
// blocks, so each such group is one all-blocks GEMM (k_toeplitz_f4, seed offset per M tile).
// Per-block seeds: every leaf is a matrix-vector product on the tiled kernel
// (k_toeplitz_mma_pb). The remainder (positions >= T k) runs as one more launch on the original
// input; the combine goes up the tree level by level (node = [P ^ Q | P ^ R]) and XORs the
// segments and the remainder into the key. Leaf buffers are batched over blocks (memory budget).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "split_tree.cuh"

namespace ssbh_impl {

namespace {

// Leaf seed regions (pre-shifted seed S': an XOR of word-aligned windows stays pre-shifted).
// Shared seed: one region per (segment, path), r = blockIdx.y, source sbuf[0, sbuf_words).
// Per-block seeds: one per leaf of the batch, v = blockIdx.y + 65535 blockIdx.z, source the
// block's region sbuf[soff[jj], soff[jj + 1]) (zero past it: those positions meet zero input).
__global__ void k_split_seeds(const uint32_t* __restrict__ sbuf, uint64_t sbuf_words, Layout lay,
                              SplitGeom g, uint32_t jj0, uint32_t nown,
                              uint32_t* __restrict__ vs) {
    const uint64_t v = blockIdx.y + (uint64_t)blockIdx.z * 65535u;
    const uint32_t rs = g.T * g.leaves;
    if (v >= (g.per_block ? g.nvirt : (uint64_t)rs)) return;
    const uint32_t r = g.per_block ? (uint32_t)(v / g.gpad) : (uint32_t)v;  // t * leaves + path
    const uint32_t t = r / g.leaves, path = r % g.leaves;
    const uint32_t* src = sbuf;
    uint64_t bound = sbuf_words;
    if (g.per_block) {
        const uint32_t jl = (uint32_t)(v % g.gpad), jj = jj0 + jl;
        if (jl < g.batch && jj < nown) {
            src = sbuf + lay.soff[jj];
            bound = lay.soff[jj + 1] - lay.soff[jj];
        } else {
            bound = 0;  // past the last block of a partial batch
        }
    }
    __shared__ uint64_t s_off[1 << kMaxL];
    __shared__ int s_n;
    if (threadIdx.x == 0) {
        uint64_t off[1 << kMaxL];
        s_n = leaf_offsets(path, g.L, g.k, (uint64_t)t * g.k, true, off);
        for (int e = 0; e < s_n; ++e) s_off[e] = off[e] / 32;
    }
    __syncthreads();
    const int n = s_n;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < g.seed_words;
         w += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t x = 0;
#pragma unroll 4
        for (int e = 0; e < n; ++e) {
            const uint64_t q = s_off[e] + w;
            if (q < bound) x ^= __ldg(src + q);
        }
        vs[v * g.seed_words + w] = x;
    }
}

// Leaf inputs: block j's reversed input pieces, zero past its padded length. One CTA per leaf:
// its (up to 2^L) piece offsets are computed once into shared memory, then the CTA streams the
// leaf's words (coalesced reads of every piece, one coalesced write).
__global__ void __launch_bounds__(256) k_split_inputs(const uint32_t* __restrict__ ybuf,
                                                      Layout lay, SplitGeom g, uint32_t jj0,
                                                      uint32_t nown, uint32_t* __restrict__ vy) {
    __shared__ uint64_t s_off[1 << kMaxL];
    __shared__ int s_n;
    const uint64_t lw = g.sL / 32;
    // grid index -> (block, leaf) with the leaf fastest, so that the leaves of one block (which
    // all read its input) run together and re-read it from L2
    const uint64_t idx = blockIdx.x + (uint64_t)blockIdx.y * 65535u;
    if (idx >= g.nvirt) return;
    const uint32_t rs = g.T * g.leaves;
    const uint32_t jl = (uint32_t)(idx / rs), jj = jj0 + jl;
    const uint32_t r = (uint32_t)(idx % rs);
    if (jl >= g.batch) return;  // group padding: ypad 0, never read
    const uint64_t v = (uint64_t)r * g.gpad + jl;  // virtual block
    const uint32_t t = r / g.leaves, path = r % g.leaves;
    if (threadIdx.x == 0) {
        uint64_t off[1 << kMaxL];
        s_n = leaf_offsets(path, g.L, g.k, (uint64_t)t * g.k, false, off);
        for (int e = 0; e < s_n; ++e) s_off[e] = off[e] / 32;
    }
    __syncthreads();
    const int n = s_n;
    const bool live = jj < nown;  // the last batch may be partial
    const uint32_t* y = live ? ybuf + lay.yoff[jj] : ybuf;
    const uint64_t yp = live ? lay.ypad[jj] : 0;
    uint32_t* dst = vy + v * g.vlw;
    for (uint64_t w = threadIdx.x; w < g.vlw; w += blockDim.x) {
        uint32_t x = 0;
        if (w < lw) {
#pragma unroll 4
            for (int e = 0; e < n; ++e) {
                const uint64_t q = s_off[e] + w;
                if (q < yp) x ^= __ldg(y + q);
            }
        }
        dst[w] = x;  // zero past the leaf: padding to the GEMM's 512-bit stages
    }
}

// Virtual layouts: leaves (inputs in vy, seeds in vs) and the remainder (original input from
// position T k, seed window at T k).
__global__ void k_split_layout(Layout lay, uint32_t nown, SplitGeom g, Layout vlay, Layout rlay) {
    const uint64_t lw = g.sL / 32;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < g.nvirt;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = (uint32_t)(v / g.gpad);
        vlay.yoff[v] = v * g.vlw;
        vlay.ypad[v] = v % g.gpad < g.batch ? (uint32_t)g.vlw : 0u;
        vlay.soff[v] = (g.per_block ? v : (uint64_t)r) * g.seed_words;
    }
    const uint64_t tw = (uint64_t)g.T * g.k / 32;
    for (uint64_t jj = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; jj < nown;
         jj += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t yp = lay.ypad[jj];
        const uint32_t rp = yp > tw ? (uint32_t)(yp - tw) : 0u;
        // Shared seed: the remainder GEMM's rows in order of remainder length (rank by
        // counting), so that an M tile's K extent — its longest row — follows the tile's own
        // blocks: the tiles of blocks no longer than T k are empty, the others stop at their
        // quantile instead of the longest remainder of all blocks. rlay.ktl[jj] = the row.
        uint32_t row = (uint32_t)jj;
        if (g.gemm) {
            row = 0;
            for (uint32_t i = 0; i < nown; ++i) {
                const uint64_t q = lay.ypad[i];
                const uint32_t rq = q > tw ? (uint32_t)(q - tw) : 0u;
                row += (rq < rp || (rq == rp && i < jj)) ? 1u : 0u;
            }
        }
        rlay.yoff[row] = lay.yoff[jj] + tw;
        rlay.ypad[row] = rp;
        rlay.soff[row] = (g.per_block ? lay.soff[jj] : 0ull) + tw;
        rlay.ktl[jj] = row;
    }
}

// Single-pass combine: leaves -> key. CTA (block jl, chunk c of W words of every leaf) handles,
// per square t, the chunk of all 3^L leaves: each thread reduces depth-D subtrees (3^D leaves at
// one word position, loaded straight into registers: 3^D independent loads in flight) to their
// 2^D-word root, the subtree roots go to shared memory and the remaining L - D levels are
// reduced there (node = [P ^ Q | P ^ R], ping-pong buffers). The squares' level-0 chunks and the
// remainder are XORed and the 2^L key segments the chunk maps to are written (key word
// s * cw + c W + j for segment s, j < W). Every leaf word is read once; no intermediate level
// goes through HBM.
template <int D>
__global__ void __launch_bounds__(256) k_split_tree(const uint32_t* __restrict__ vout,
                                                    const uint32_t* __restrict__ rem,
                                                    const uint32_t* __restrict__ rrow,
                                                    uint32_t jj0, uint32_t jl0, uint32_t count,
                                                    uint32_t kw,
                                                    SplitGeom g, uint32_t W,
                                                    uint32_t* __restrict__ out,
                                                    unsigned long long out_stride) {
    constexpr int kSub = D == 1 ? 3 : D == 2 ? 9 : 27;  // 3^D leaves per subtree
    constexpr int kOut = 1 << D;                         // its root's words per position
    extern __shared__ __align__(16) uint32_t tsm[];
    const uint64_t cw = g.sL / 32;  // leaf words
    const uint32_t nchunks = (uint32_t)(cw / W);
    const uint32_t jl = jl0 + blockIdx.x / nchunks, c = blockIdx.x % nchunks;  // batch-local block
    if (jl >= count) return;
    const uint32_t nsub = g.leaves / kSub;       // subtree roots (level L - D nodes)
    uint32_t* buf0 = tsm;                        // nsub nodes x kOut W words
    uint32_t* buf1 = tsm + (size_t)nsub * kOut * W;  // next level: (nsub / 3) x 2 kOut W
    uint32_t* acc = buf1 + (size_t)(nsub / 3) * 2 * kOut * W;  // 2^L W words
    const uint32_t outw = (1u << g.L) * W;
    for (uint32_t i = threadIdx.x; i < outw; i += blockDim.x) acc[i] = 0;
    const uint64_t lstride = (uint64_t)g.gpad * cw;  // next path, same block
    for (uint32_t t = 0; t < g.T; ++t) {
        const uint32_t* base = vout + ((uint64_t)t * g.leaves * g.gpad + jl) * cw + (uint64_t)c * W;
        for (uint32_t it = threadIdx.x; it < nsub * W; it += blockDim.x) {
            const uint32_t q = it / W, j = it % W;
            uint32_t v[kSub];
            const uint32_t* src = base + (uint64_t)q * kSub * lstride + j;
#pragma unroll
            for (int e = 0; e < kSub; ++e) v[e] = __ldg(src + e * lstride);
            // levels L .. L - D + 1 in registers: n nodes of width w -> n / 3 of width 2 w
#pragma unroll
            for (int n = kSub, w = 1; n > 1; n /= 3, w *= 2) {
#pragma unroll
                for (int p = 0; p < n / 3; ++p) {
                    uint32_t o[64];
#pragma unroll
                    for (int e = 0; e < w; ++e) {
                        o[e] = v[3 * p * w + e] ^ v[(3 * p + 1) * w + e];
                        o[w + e] = v[3 * p * w + e] ^ v[(3 * p + 2) * w + e];
                    }
#pragma unroll
                    for (int e = 0; e < 2 * w; ++e) v[2 * p * w + e] = o[e];
                }
            }
            uint32_t* dst = buf0 + (size_t)q * kOut * W + j;
#pragma unroll
            for (int e = 0; e < kOut; ++e) dst[e * W] = v[e];
        }
        __syncthreads();
        uint32_t* src = buf0;
        uint32_t* dst = buf1;
        uint32_t n = nsub, w = kOut * W;  // nodes and chunk width at the current level
        while (n > 1) {
            const uint32_t np = n / 3, pw = 2 * w;
            for (uint32_t i = threadIdx.x; i < np * pw; i += blockDim.x) {
                const uint32_t pnode = i / pw, e = i % pw;
                const bool hi = e >= w;
                const uint32_t el = hi ? e - w : e;
                const uint32_t* ch = src + (size_t)pnode * 3 * w;
                dst[i] = ch[el] ^ ch[(hi ? 2 : 1) * w + el];
            }
            __syncthreads();
            n = np;
            w = pw;
            uint32_t* tmp = src;
            src = dst;
            dst = tmp;
        }
        // src: the square's level-0 chunk (2^L W words)
        for (uint32_t i = threadIdx.x; i < outw; i += blockDim.x) acc[i] ^= src[i];
        __syncthreads();
    }
    // key segments: acc[s W + j] -> key word s cw + c W + j, XOR the remainder's word
    const uint64_t jj = (uint64_t)jj0 + jl;
    const uint64_t rr = rrow[jj];  // the block's row of the remainder product (k_split_layout)
    for (uint32_t i = threadIdx.x; i < outw; i += blockDim.x) {
        const uint32_t sgm = i / W, j = i % W;
        const uint64_t wk = (uint64_t)sgm * cw + (uint64_t)c * W + j;
        if (wk < kw) out[jj * out_stride + wk] = acc[i] ^ rem[rr * kw + wk];
    }
}

}  // namespace

// Levels. Tiled-kernel leaves (per-block seeds): the leaf work (3/4)^L grows by the window ramp
// (255 D steps per 256-tile window over the leaf's k / 2^L / 128 chunks); L minimises the
// product, a deeper level only when it gains > 8 % (its prep and combine passes grow as 2^L;
// config 4: modelled L = 4 6 % better than L = 3, measured 2.80 vs 2.56 s).
// GEMM leaves (shared seed): no ramp — the deepest level whose leaves keep >= 2^14 positions
// (32 FP4 stages per work item; the per-item epilogue and the 2^L prep / combine passes make
// shorter leaves slower: config 3 hash L = 3 / 4 / 5 / 6 = 69.2 / 55.5 / 48.0 / 48.7 ms).
uint32_t split_levels(uint64_t k, bool gemm) {
    uint32_t best = 0;
    double best_cost = 1.0;
    double f = 1.0;
    for (uint32_t L = 1; L <= (uint32_t)kMaxL; ++L) {
        f *= 0.75;
        if (k % (256ull << L) != 0) break;
        const double nc = (double)(k >> L) / 128.0;
        if (nc < (gemm ? 32 : 64)) break;
        if (gemm) {
            // config 2 (k = 2^15, L = 1) measured no gain: short keys keep the direct GEMM.
            // Leaves >= 2^12 positions: leaves of 2^13 run as leaf-mode items of 16 FP4 stages;
            // leaves of 2^12 run in the leaf GEMM's parent mode (a CTA builds the parent's 2^13
            // positions once for its three children), which is what makes the seventh level pay
            // (config 3 hash L = 6 / 7 = 31.2 / 27.6 ms); config 5 (k = 2^21) takes L = 9: hash of
            // 1024 of its blocks L = 7 / 8 / 9 = 404 / 308 / 240 ms
            if (k < (1ull << 18) || (k >> L) < (1ull << 12)) break;
            best = L;
            continue;
        }
        const double cost = f * (255.0 + nc) / nc;
        if (cost < best_cost * 0.92) {
            best_cost = cost;
            best = L;
        }
    }
    return best;
}

SplitGeom make_split_geom(uint32_t nown, uint64_t k, uint64_t mean_nj, uint32_t L,
                          bool per_block, bool gemm_leaves, uint64_t budget_bytes) {
    SplitGeom g{};
    g.L = L;
    g.per_block = per_block;
    g.k = k;
    g.T = (uint32_t)(mean_nj / k);
    g.leaves = 1;
    for (uint32_t l = 0; l < L; ++l) g.leaves *= 3;
    g.sL = k >> L;
    g.seed_words = 2 * g.sL / 32 + 64;
    // shared seed: the leaves of one (segment, path) share a seed across blocks -> one GEMM of
    // them against that leaf matrix (k_toeplitz_f4, no window ramp); groups padded to 128-block
    // M tiles, leaf inputs to the GEMM's 512-bit stages. Per-block seeds: every leaf is its own
    // matrix-vector product (tiled kernel).
    g.gemm = !per_block && gemm_leaves;
    g.vlw = g.gemm ? (g.sL / 32 + 15) / 16 * 16 : g.sL / 32;
    // blocks per batch within the budget, counted on what the plan allocates: leaf outputs (and
    // tiled leaves' inputs) for gpad (not batch) blocks per (t, path) group, plus the leaf seeds
    // (per leaf for per-block seeds, per (t, path) for a shared seed)
    // (GEMM leaves build their inputs in shared memory: no leaf-input buffer)
    const uint64_t per_blk = (uint64_t)g.T * g.leaves *
                             ((g.gemm ? 0 : g.vlw * 4) + g.sL / 8 +
                              (per_block ? g.seed_words * 4 : 0));
    // + for GEMM leaves the Hankel unit tables (16 B per unit, leaf_unit_stride units per seed)
    g.unit_stride = g.gemm ? leaf_unit_stride(g.sL, g.vlw) : 0;
    const uint64_t fixed =
        per_block ? 0 : (uint64_t)g.T * g.leaves * (g.seed_words * 4 + g.unit_stride * 16);
    const uint64_t avail = budget_bytes > fixed ? budget_bytes - fixed : 0;
    uint64_t b = std::max<uint64_t>(1, std::min<uint64_t>(nown, avail / per_blk));
    if (g.gemm && b < nown) b = std::max<uint64_t>(128, b / 128 * 128);
    g.batch = (uint32_t)std::min<uint64_t>(b, nown);
    g.gpad = g.gemm ? (g.batch + 127) / 128 * 128 : g.batch;
    g.nvirt = (uint64_t)g.gpad * g.T * g.leaves;
    g.bytes = g.gpad * per_blk + fixed;
    return g;
}

bool split_applicable(uint64_t k, uint64_t mean_nj, uint32_t L) {
    if (L == 0 || L > (uint32_t)kMaxL) return false;
    // leaves: whole 128-row tiles and word-aligned offsets; at least one full square
    return k % (256ull << L) == 0 && mean_nj >= k;
}

static void split_seeds(const uint32_t* d_sbuf, uint64_t sbuf_words, const Layout& lay,
                        uint32_t nown, const SplitGeom& g, uint32_t jj0, uint32_t* d_vs,
                        cudaStream_t st) {
    const uint64_t rows = g.per_block ? g.nvirt : (uint64_t)g.T * g.leaves;
    const unsigned gz = (unsigned)((rows + 65534) / 65535);
    const unsigned gy = (unsigned)std::min<uint64_t>(rows, 65535);
    const unsigned gx =
        (unsigned)std::min<uint64_t>((g.seed_words + 255) / 256, g.per_block ? 8 : 64);
    k_split_seeds<<<dim3(gx, gy, gz), 256, 0, st>>>(d_sbuf, sbuf_words, lay, g, jj0, nown, d_vs);
}

void launch_split_setup(const uint32_t* d_sbuf, uint64_t sbuf_words, const SplitGeom& g,
                        uint32_t* d_vs, const Layout& lay, uint32_t nown, const Layout& vlay,
                        const Layout& rlay, cudaStream_t st) {
    if (!g.per_block) split_seeds(d_sbuf, sbuf_words, lay, nown, g, 0, d_vs, st);
    k_split_layout<<<(unsigned)std::min<uint64_t>((std::max<uint64_t>(g.nvirt, nown) + 255) / 256,
                                                  1184),
                     256, 0, st>>>(lay, nown, g, vlay, rlay);
}

void launch_split_batch(const uint32_t* d_ybuf, const uint32_t* d_sbuf, uint64_t sbuf_words,
                        const Layout& lay, uint32_t nown, const SplitGeom& g, uint32_t jj0,
                        uint32_t* d_vy, uint32_t* d_vs, cudaStream_t st) {
    const unsigned gy = (unsigned)((g.nvirt + 65534) / 65535);
    const unsigned gx = (unsigned)std::min<uint64_t>(g.nvirt, 65535);
    k_split_inputs<<<dim3(gx, gy), 256, 0, st>>>(d_ybuf, lay, g, jj0, nown, d_vy);
    if (g.per_block) split_seeds(d_sbuf, sbuf_words, lay, nown, g, jj0, d_vs, st);
}

constexpr size_t kTreeSmemCap = 112 * 1024;

uint32_t launch_split_combine(uint32_t* d_vout, uint32_t* d_tmp, const uint32_t* d_rem,
                              const uint32_t* d_rrow, uint32_t jj0, uint32_t count, uint32_t kw,
                              const SplitGeom& g, uint32_t* d_out, uint64_t out_stride,
                              cudaStream_t st, uint32_t jl0, uint32_t jl1) {
    (void)d_tmp;
    jl1 = std::min(jl1, count);  // batch-local blocks [jl0, jl1): one launch per slice
    if (jl0 >= jl1 || !kw) return 0;
    // one pass from the leaves (round 1: level by level, L launches through HBM, config 3
    // 3.0 ms): depth-D register subtrees, chunk width W words (the largest power of two <= 32
    // and <= the leaf whose buffers fit kTreeSmemCap of shared memory: two CTAs per SM)
    const uint32_t D = g.L >= 3 ? 3 : g.L;
    const uint32_t sub = D == 1 ? 3 : D == 2 ? 9 : 27, outd = 1u << D;
    const uint64_t cw = g.sL / 32;
    const uint32_t nsub = g.leaves / sub;
    auto smem_of = [&](uint32_t w) {
        return ((size_t)nsub * outd * w + (size_t)(nsub / 3) * 2 * outd * w + ((size_t)w << g.L)) * 4;
    };
    // (deep trees — config 5 combines 8 levels of 3^8 nodes — need the wider chunks: at 48 KB W
    // was 2 words, 8-byte reads of 32-byte sectors, 3.2 ms per 1.7 GB batch)
    uint32_t W = 32;
    while (W > 1 && (W > cw || smem_of(W) > 48 * 1024)) W /= 2;
    if (W < 8) {  // deep tree: two CTAs per SM instead
        W = 8;
        while (W > 1 && (W > cw || smem_of(W) > kTreeSmemCap)) W /= 2;
    }
    const size_t smem = smem_of(W);
    const uint64_t grid = (uint64_t)(jl1 - jl0) * (cw / W);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<(unsigned)grid, 256, smem, st>>>(d_vout, d_rem, d_rrow, jj0, jl0, jl1, kw, g, W,
                                                d_out, out_stride);
    };
    if (D == 3)
        go(k_split_tree<3>);
    else if (D == 2)
        go(k_split_tree<2>);
    else
        go(k_split_tree<1>);
    return 1;
}

}  // namespace ssbh_impl
