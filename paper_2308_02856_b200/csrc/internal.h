// internal.h — device-side data structures and kernel launchers shared by the .cu files.
// Not part of the public ABI (include/ssbh_cuda.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ssbh_impl {

// Hash-kernel tile geometry (see toeplitz.cu): each warp owns R consecutive 32-row output
// words, a CTA has kHashWarps compute warps + 1 producer warp, a k-tile covers <= KT_MAX
// words of the reversed input.
constexpr int kHashR = 32;  // R = 64 measured slower (160 regs, 2 CTA/SM, 67 KB loop body)
constexpr int kHashWarps = 4;
constexpr int kHashRowWords = kHashR * kHashWarps;  // output words per row tile
constexpr int kHashKTMax = 2048;                    // max y words per item
constexpr int kHashStages = 2;

// Device-side run statistics / error flags written by the layout kernel.
struct DevStats {
    unsigned long long max_nj;
    unsigned long long min_nj;
    unsigned long long total_items;
    unsigned long long seed_words;     // shared mode: words of the shared seed region
    unsigned long long hash_word_ops;  // sum n_j * k / 32
    unsigned long long sum_nj;
    uint32_t flags;                    // kFlag*
    uint32_t pad;
};
constexpr uint32_t kFlagEmpty = 1u;     // some owned n_j == 0
constexpr uint32_t kFlagOversize = 2u;  // some owned n_j > block_limit
constexpr uint32_t kFlagTooLong = 4u;   // some owned n_j >= 2^32 (device path limit)
constexpr uint32_t kFlagBucketOverflow = 8u;  // a two-level staging region overflowed

// Per-owned-block layout arrays (device).
struct Layout {
    unsigned long long* nj;    // [nown]   block lengths (bits)
    unsigned long long* yoff;  // [nown+1] u32-word offsets of reversed inputs in ybuf
    uint32_t* ypad;            // [nown]   padded y words (multiple of kHashR)
    uint32_t* ktl;             // [nown]   k-tile length (words, multiple of kHashR)
    unsigned long long* items; // [nown+1] hash work-item prefix
    unsigned long long* soff;  // [nown+1] u32-word offsets of per-block seeds (0 if shared)
    DevStats* stats;
};

struct HashArgs {
    const uint32_t* ybuf;
    const uint32_t* sbuf;
    uint32_t* out;           // out[jj * out_stride + word]
    unsigned long long out_stride;
    Layout lay;
    uint32_t nown;
    uint32_t kw;             // output words per block (ceil(k/32))
    uint32_t rowtiles;       // ceil(kw / kHashRowWords)
    uint32_t per_block_seed;
};

// ---- prf / input -------------------------------------------------------------------
void launch_stream_words(const uint64_t key[4], uint64_t tag, uint64_t sub, uint64_t first,
                         uint64_t count, uint64_t* d_out, cudaStream_t st);
void launch_stream_uniform(const uint64_t key[4], uint64_t tag, uint64_t sub, uint64_t bound,
                           uint64_t first, uint64_t count, uint64_t* d_out, cudaStream_t st);
void launch_stream_bernoulli(const uint64_t key[4], uint64_t tag, uint64_t sub, double p,
                             uint64_t first, uint64_t count, uint32_t* d_out32, cudaStream_t st);
// bits(nbits) of (key, tag, sub) as u32 words; tail masked.
void launch_stream_bits(const uint64_t key[4], uint64_t tag, uint64_t sub, uint64_t nbits,
                        uint32_t* d_out32, cudaStream_t st);
void launch_make_input(const uint64_t key[4], double p, uint64_t nbits, uint32_t* d_out32,
                       cudaStream_t st);

// ---- protocol rounds (run_extraction front end, rounds.cu) ----------------------------
void launch_simulate_rounds(const uint64_t key[4], uint64_t n, double p_x, double e_ph,
                            double e_bit, double p_det, uint8_t* d_rounds, cudaStream_t st);
// bits32 = bit_a, keep32 = is_key_round (ceil(n/32) words each); d_counts4 (pre-zeroed):
// test rounds, test rounds with bit_a != bit_b, undetected test rounds, key rounds.
void launch_rounds_split(const uint8_t* d_rounds, uint64_t n, uint32_t* d_bits32,
                         uint32_t* d_keep32, unsigned long long* d_counts4, cudaStream_t st);

// ---- sampler -----------------------------------------------------------------------
struct SamplerGeom {
    uint64_t n;
    uint64_t s;
    uint32_t j_lo, nown;
    int chunk_shift;       // warp-chunk = 2^chunk_shift rounds
    uint64_t nchunks;
    uint64_t group_chunks; // chunks per scan group
    uint64_t ngroups;
    int payload_bytes;     // 2 (u16: V | bit<<15) or 4 (u32: V | keep<<30 | bit<<31)
    bool ranked;           // 4-byte payload V | bit<<15 | rank<<16 (rank = the round's rank in its
                           // block within the warp-chunk, found in pass 1; 0x7fff: sifted out):
                           // pass 3 then needs no ordering at all (make_ranked)
    int scatter_window = 0;  // ranked pass 3: 0 model, W > 0 forced window words, -1 per-bit
};
// Ranked variant of a single-level u16 geometry (in-memory plans): pass 1 is ALU-bound on
// Threefry, so the stable ranking (ballot peer masks + the warp's running-rank row) costs it
// < 1 %, and pass 3 drops from 157 to ~30 SASS per 32 rounds.
SamplerGeom make_ranked(const SamplerGeom& g);
// max_chunk_shift bounds the warp-chunk (streaming: input chunks must be a whole number of
// warp-chunks).
SamplerGeom make_sampler_geom(uint64_t n, uint64_t s, uint32_t j_lo, uint32_t nown,
                              bool has_keep, int max_chunk_shift = 40);
// Pass 1: V_i (Threefry), payload, per-(chunk, owned block) counts (counts pre-zeroed).
// d_keep: optional bit-packed sift mask (bit i = keep round i), like the reference's keep[i].
void launch_sample_count(const SamplerGeom& g, const uint64_t key[4], const uint32_t* d_in32,
                         const uint32_t* d_keep, void* d_payload, uint32_t* d_counts,
                         uint32_t* d_assign_out, cudaStream_t st);
// Pass 2: exclusive scan of counts along chunks (in place -> offsets), nj totals.
// seg_groups > 0: the scan restarts every seg_groups groups (two-level pass B); nj gets one
// row of g.nown totals per segment.
void launch_scan(const SamplerGeom& g, uint32_t* d_counts, unsigned long long* d_gsum,
                 unsigned long long* d_nj, cudaStream_t st, uint64_t seg_groups = 0);
// Pass 3: stable scatter. ybuf mode: reversed bit pack into ybuf (pre-zeroed);
// index mode (d_idx_out != null): CSR indices at csr_off[jj] + rank.
// d_in32_late: the payload holds V only; the data bits are read from these input words.
void launch_scatter(const SamplerGeom& g, const void* d_payload, uint32_t* d_offsets,
                    const unsigned long long* d_nj, const unsigned long long* d_yoff,
                    uint32_t* d_ybuf, unsigned long long* d_idx_out,
                    const unsigned long long* d_csr_off, cudaStream_t st,
                    const uint32_t* d_in32_late = nullptr);
// Pass 3 for streaming plans: rounds [first, first+count) whose data bits are d_chunk32
// (bit 0 = round `first`); V recomputed by Threefry (no payload). `first` and the chunk end
// (unless it is n) must be multiples of the warp-chunk.
void launch_scatter_stream(const SamplerGeom& g, const uint64_t key[4], const uint32_t* d_chunk32,
                           uint64_t first, uint64_t count, uint32_t* d_offsets,
                           const unsigned long long* d_nj, const unsigned long long* d_yoff,
                           uint32_t* d_ybuf, cudaStream_t st);

// ---- multi-GPU sharded sampling ---------------------------------------------------------
// Same geometry with another round count (chunk shift kept; counts table sized for the max).
SamplerGeom geom_with_n(const SamplerGeom& g, uint64_t n);
// Pass 1 over a slice of rounds [base, base + g.n): payload (local index) + counts per
// (chunk, owning rank) for `owners` ranks (block ranges multigpu.owned_range).
void launch_sample_slice(const SamplerGeom& g, const uint64_t key[4], uint64_t base,
                         const uint32_t* d_in32, void* d_payload, uint32_t owners,
                         uint32_t* d_counts, cudaStream_t st);
// Stable split of the slice payload by owner, stored straight into every owner's receive
// buffer (d_dst[o], peer-mapped) at d_dst_base[o] + rank (d_offsets: scanned counts).
void launch_owner_split(const SamplerGeom& g, const void* d_payload, uint32_t owners,
                        uint32_t* d_offsets, void* const* d_dst,
                        const unsigned long long* d_dst_base, cudaStream_t st);
// Pass 1 of an owner: counts per (chunk, owned block) from a received payload (g.n rounds).
// bshift > 0: keys are buckets of 2^bshift owned blocks (two-level pass A).
void launch_count_payload(const SamplerGeom& g, const void* d_payload, uint32_t* d_counts,
                          cudaStream_t st, uint32_t bshift = 0);

// ---- two-level split for large key spaces ---------------------------------------------
// With thousands of owned blocks one warp-chunk touches every block, so the running-rank rows
// no longer fit shared memory and the data bits land on random words of a y buffer far larger
// than L2. Pass A splits the rounds stably by bucket (2^shift consecutive blocks) into a
// staging buffer with one fixed-capacity region per bucket (mean + 16 sigma); pass B counts,
// scans (restarting per region) and scatters the staged rounds with 2^shift keys, so each
// warp's rank row lives in shared memory and its y writes stay within one bucket's blocks.
constexpr uint32_t kBucketShift = 7;           // >= 128 blocks per bucket
constexpr uint32_t kMaxBuckets = 64;           // <= 64 buckets (8 KB of split sectors per warp)
constexpr uint32_t kBucketMinBlocks = 4096;    // below: single-level scatter
struct BucketGeom {
    uint32_t shift;       // log2 blocks per bucket
    uint32_t nbuckets;
    uint64_t cap;         // staged rounds per bucket region
    uint64_t cpb;         // pass-B chunks per region
    uint64_t gps;         // pass-B scan groups per region
    SamplerGeom a;        // pass A over the source rounds (nown = owned blocks)
    SamplerGeom b;        // pass B over nbuckets * cap staged rounds (nown = 2^shift), u16
};
inline SamplerGeom with_keys(SamplerGeom g, uint32_t nkeys) {
    g.nown = nkeys;
    return g;
}
// mean_per_block: expected rounds per owned block among the n_src source rounds.
BucketGeom make_bucket_geom(uint64_t n_src, uint64_t s, uint32_t j_lo, uint32_t nown,
                            double mean_per_block, bool has_keep, int max_chunk_shift = 40);
// Pass A from Threefry (rounds base + [0, ga.n)): payload + per-(chunk, bucket) counts.
void launch_sample_buckets(const BucketGeom& bg, const SamplerGeom& ga, const uint64_t key[4],
                           uint64_t base, const uint32_t* d_in32, const uint32_t* d_keep,
                           void* d_payload, uint32_t* d_counts, cudaStream_t st);
// Pass A split: payload -> staging regions (u16 local block | bit << 15), using the scanned
// pass-A table; a full region raises kFlagBucketOverflow in *d_flags.
void launch_bucket_split(const BucketGeom& bg, const SamplerGeom& ga, const void* d_payload,
                         uint32_t* d_offsets_a, const unsigned long long* d_tot_a,
                         uint16_t* d_staging, uint32_t* d_flags, cudaStream_t st,
                         const uint32_t* d_in32_late = nullptr);
// Pass B counts over the staging regions (empty slots hold 0xffff).
void launch_bucket_count(const BucketGeom& bg, const uint16_t* d_staging, uint32_t* d_counts_b,
                         cudaStream_t st);
// Pass B scatter into the reversed blocks; d_rank_base (per owned block, may be null) is
// added to every rank (streaming: the block's rounds in earlier input chunks).
// fwd_cap > 0 (forward streaming): bit r of block jf goes to jf * fwd_cap + r of d_ybuf.
void launch_bucket_scatter(const BucketGeom& bg, const uint16_t* d_staging, uint32_t* d_offsets_b,
                           const unsigned long long* d_nj, const unsigned long long* d_yoff,
                           uint32_t* d_ybuf, const uint32_t* d_rank_base, cudaStream_t st,
                           uint64_t fwd_cap = 0);
// Forward streaming (two-level streaming plans): no count pass over the whole input — every
// block gets a fixed-capacity region filled in round order chunk by chunk; run_rank holds the
// blocks' lengths so far, and at the end the regions are reversed into the compact layout.
void launch_add_ranks(uint32_t* d_run_rank, const unsigned long long* d_nj_chunk, uint32_t nown,
                      uint64_t cap, uint32_t* d_flags, cudaStream_t st);
void launch_ranks_to_nj(const uint32_t* d_run_rank, uint32_t nown, unsigned long long* d_nj,
                        cudaStream_t st);
void launch_reverse_blocks(const uint32_t* d_fwd, uint64_t cap_words, const Layout& lay,
                           uint32_t nown, uint64_t mean_words, uint32_t* d_ybuf, cudaStream_t st);

// ---- layout / seeds / hash -----------------------------------------------------------
// Computes ypad/ktl/yoff/items/soff/stats from lay.nj for nown blocks.
void launch_layout(const Layout& lay, uint32_t nown, uint64_t k, uint32_t rowtiles,
                   uint32_t kt_target, int per_block_seed, uint64_t block_limit,
                   cudaStream_t st);
// Seeds: shared -> stats.seed_words words of stream (hash,"hash-seed",0);
// per-block -> each region soff[jj].. of stream sub = j_lo + jj.
void launch_seeds(const uint64_t key[4], const Layout& lay, uint32_t nown, uint32_t j_lo,
                  int per_block_seed, uint64_t max_words_hint, uint32_t* d_sbuf,
                  cudaStream_t st);
// y[c] = x[n-1-c] for one block: writes ypad words at d_y (zero padded).
void launch_reverse(const uint32_t* d_x32, uint64_t nbits, uint32_t* d_y, uint64_t ywords,
                    cudaStream_t st);
int hash_grid_size(int device);
void launch_hash(const HashArgs& a, int grid, cudaStream_t st);
// Tensor-core engine for shared-seed plans (toeplitz_mma.cu): the hash of all owned blocks
// as one FP4 GEMM mod 2 (tcgen05.mma kind::mxf4). Same inputs/outputs as launch_hash.
enum HashEngine : int { kEngineAuto = 0, kEngineLop3 = 1, kEngineMma = 2 };
struct MmaGeom {
    uint32_t mtiles;   // ceil(nown / 128)
    uint32_t ntiles;   // ceil(kw / 8): 256 output rows per tile
    uint32_t ksplit;   // K parts per (M, N) tile (red.xor when > 1)
    uint32_t grid;     // persistent CTAs (one per SM)
    uint64_t items;    // mtiles * ntiles * ksplit
};
// Leaf mode of k_toeplitz_f4 (the 3-for-4 split's shared-seed leaves): a CTA keeps one M tile's
// leaf inputs (128 virtual blocks x kpw words) in shared memory for all N tiles, building them
// from the original reversed blocks as XORs of the leaf's input pieces (no materialised leaf
// inputs). Virtual block v = group * gpad + jl (group = segment t * 3^L + path).
struct LeafSrc {
    const uint32_t* ybuf;    // original reversed blocks
    Layout lay;              // their layout (yoff, ypad)
    unsigned long long k;    // square size (bits)
    uint32_t L, leaves, gpad, batch, jj0, nown;
    uint32_t kpw;            // leaf input words per K part (held in shared memory); parent
                             // mode: the parent's input words (2 leaves)
    unsigned long long seed_words;  // u32 words per leaf seed region (SplitGeom::seed_words)
};

struct MmaHashArgs {
    const uint32_t* ybuf;
    const uint32_t* sbuf;    // shared seed, pre-shifted by one bit (see launch_seeds)
    uint32_t* out;           // out[jj * out_stride + word], zeroed when ksplit > 1
    unsigned long long out_stride;
    Layout lay;
    uint32_t nown;
    uint32_t kw;
    uint32_t ntiles, ksplit;
    uint64_t items;
    uint32_t* mt_words;      // [mtiles] device scratch: max ypad per M tile
    uint32_t stage_bits;     // input positions per pipeline stage (set by launch_hash_mma)
    const uint32_t* units;   // leaf modes: Hankel unit tables (launch_hankel_units), 4 words
                             // per unit, unit_stride units per leaf seed
    unsigned long long unit_stride;
    uint32_t leaf;           // 1: leaf mode (src below; items walked N tile innermost per
                             // (M tile, K part); ksplit = K parts); 2: parent mode — a CTA
                             // keeps one M tile of a level L-1 node's input and runs its three
                             // children (P = lo ^ hi, Q = lo, R = hi) N tile by N tile, writing
                             // the parent node's rows [P ^ Q | P ^ R] (out: one row of 2 kw
                             // words per parent virtual block = super-item * 128 + row)
    LeafSrc src;
};
// Per-block seeds on the tensor cores: work item = (owned block, window of 256 row tiles of
// 128 rows); see toeplitz_mma.cu.
struct PbGeom {
    uint32_t ntiles;   // ceil(kw / 4): 128-row tiles per block
    uint32_t nwin;     // ceil(ntiles / 256)
    uint32_t grid;
    uint32_t nparts;   // D-step parts per (block, window): split-K when windows are few
    uint32_t part_steps;  // D steps per part (multiple of 256; the last part takes the rest)
    uint64_t items;    // nown * nwin * nparts
};
struct PbHashArgs {
    const uint32_t* ybuf;
    const uint32_t* sbuf;    // per-block seed regions at lay.soff[jj], pre-shifted by one bit
    uint32_t* out;           // out[jj * out_stride + word]: stored (1 part) or XORed (parts)
    unsigned long long out_stride;
    Layout lay;
    uint32_t nown, kw;
    uint32_t ntiles, nwin;
    uint64_t items;
    uint32_t nparts, part_steps;  // set from PbGeom by launch_hash_mma_pb
};
// mean_bits: expected input bits per block; with few (block, window) items the D steps are
// split into parts (XOR-accumulated into the pre-zeroed output) to fill the grid.
PbGeom make_pb_geom(uint32_t nown, uint32_t kw, int device, uint64_t mean_bits = 0);
void launch_hash_mma_pb(const PbHashArgs& a, const PbGeom& g, cudaStream_t st);
// 3-for-4 split of long shared-seed squares (toeplitz_split.cu): T squares of k x k per block,
// each split L times into 3^L Hankel leaves of size k / 2^L run by the tiled kernel.
struct SplitGeom {
    uint32_t L, T, leaves;   // levels, squares per block, 3^L
    uint64_t k, sL;          // square size (= rows), leaf size
    uint32_t batch;          // owned blocks per leaf batch (memory budget)
    uint64_t nvirt;          // leaves of one batch: batch * T * 3^L
    uint64_t seed_words;     // u32 words per leaf seed region
    bool per_block;          // per-block seeds: leaf seeds per batch leaf (else per (t, path))
    bool gemm;               // leaves hashed by the all-blocks GEMM (shared seed) or tiled kernel
    uint32_t gpad;           // virtual blocks per (t, path) group: batch, 128-aligned for gemm;
                             // virtual block v = (t * leaves + path) * gpad + jl
    uint64_t vlw;            // u32 words per leaf input (sL / 32, 16-aligned for gemm)
    uint64_t bytes;          // leaf inputs + outputs + seeds one batch allocates
    uint64_t unit_stride;    // GEMM leaves: Hankel units per leaf seed (leaf_unit_stride)
};
uint32_t split_levels(uint64_t k, bool gemm);  // 0 = not worth it
SplitGeom make_split_geom(uint32_t nown, uint64_t k, uint64_t mean_nj, uint32_t L,
                          bool per_block, bool gemm_leaves, uint64_t budget_bytes);
bool split_applicable(uint64_t k, uint64_t mean_nj, uint32_t L);
// the batch-relative leaf layout (vlay: yoff/ypad/soff), the remainder layout (rlay: the
// original input from position T k, seed offset T k; shared seed: rows sorted by remainder
// length, rlay.ktl[block] = its row) and, for a shared seed, the leaf seeds
void launch_split_setup(const uint32_t* d_sbuf, uint64_t sbuf_words, const SplitGeom& g,
                        uint32_t* d_vs, const Layout& lay, uint32_t nown, const Layout& vlay,
                        const Layout& rlay, cudaStream_t st);
// leaf inputs (and per-block leaf seeds) of blocks [jj0, jj0 + batch)
void launch_split_batch(const uint32_t* d_ybuf, const uint32_t* d_sbuf, uint64_t sbuf_words,
                        const Layout& lay, uint32_t nown, const SplitGeom& g, uint32_t jj0,
                        uint32_t* d_vy, uint32_t* d_vs, cudaStream_t st);
// out[jj * out_stride + w] = rem[jj * kw + w] ^ the leaves reaching word w, blocks jj0 + [0, count)
// returns the launches made; d_tmp (>= the leaf outputs) holds intermediate levels
uint32_t launch_split_combine(uint32_t* d_vout, uint32_t* d_tmp, const uint32_t* d_rem,
                              const uint32_t* d_rrow, uint32_t jj0, uint32_t count, uint32_t kw,
                              const SplitGeom& g, uint32_t* d_out, uint64_t out_stride,
                              cudaStream_t st, uint32_t jl0 = 0, uint32_t jl1 = 0xffffffffu);
uint32_t mma_mtiles(uint32_t nown);
// Leaf mode (the split's shared-seed leaf GEMM): K parts of <= 8192 positions, N tiles innermost.
// parent: the parent-node variant (leaves of <= 4096 positions: 2 leaves fit the buffer)
MmaGeom make_leaf_geom(uint32_t nvirt, uint32_t lw, int device, bool parent);
MmaGeom make_mma_geom(uint32_t nown, uint32_t kw, uint64_t mean_nj, int device);
void launch_hash_mma(const MmaHashArgs& a, const MmaGeom& g, cudaStream_t st);
// Hankel unit tables of `regions` leaf seeds (seed_words pre-shifted words each at d_vs): unit G
// word j = (S' >> (G + 32 j)) & 0x22222222, unit_stride units (16 B) per region.
void launch_hankel_units(const uint32_t* d_vs, uint64_t seed_words, uint64_t regions,
                         uint64_t unit_stride, uint32_t* d_units, cudaStream_t st);
// units per leaf seed region the leaf GEMM reads (N tiles of 256 rows x stages of 512 positions)
inline uint64_t leaf_unit_stride(uint64_t sL, uint64_t vlw) {
    return ((sL + 255) / 256 * 256 + vlw * 32 + 131 + 7) / 8 * 8;
}

// Concatenate nown blocks of k bits (block stride kw words) into key (bit offset jj*k).
void launch_concat(const uint32_t* d_blocks, uint32_t kw, uint32_t nown, uint64_t k,
                   uint32_t* d_key, cudaStream_t st);

}  // namespace ssbh_impl
