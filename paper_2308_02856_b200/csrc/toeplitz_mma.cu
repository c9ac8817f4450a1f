// toeplitz_mma.cu — the GF(2) Toeplitz hash on the 5th-generation tensor cores (tcgen05.mma,
// accumulators in TMEM). Same product as k_toeplitz_hash (proj/src/toeplitz.cpp:34-52),
// different engine; selected per plan (ssbh_plan_set_engine, ssbh_plan_hash_kernel names it).
//
// Why a tensor-core engine exists. With the input reversed (y_j[c] = x_j[n_j-1-c]) block j's
// output is K_j[i] = XOR_c S[i+c] y_j[c] (toeplitz.cu). With ONE shared seed every block
// multiplies the SAME Hankel matrix H[i][c] = S[i+c], so the whole hash is a GF(2) matrix
// product D = Y * H^T (blocks x input positions times input positions x output rows), and a
// GF(2) product is an integer product mod 2: D[j][i] = (sum_c y_j[c] * S[i+c]) mod 2. The
// tensor cores compute the integer sums exactly on block-scaled FP4 operands (kind::mxf4:
// every element 0 or 1.0 as E2M1, every UE8M0 scale 1.0, f32 accumulator holding exact
// integer counts below 2^24) and the epilogue keeps the parity. Per-block seeds (and long
// shared blocks) tile each block's matrix-vector product into 128 x 128 Hankel blocks
// instead. Kernels in this file:
//   k_toeplitz_f4        shared seeds, direct mode: all owned blocks x one Hankel matrix as a GEMM
//   k_leaf_gemm          the 3-for-4 split's shared-seed leaves (toeplitz_split.cu) as GEMMs
//                        (+ k_hankel_units: its Hankel operand tables)
//   k_toeplitz_mma_pb    tiled matrix-vector products: per-block seeds, long shared blocks
//
// The Hankel operand. With the K order used inside a pipeline stage (chunk q, word w, nibble
// i = position 128g + kc + 4i + 32w), row r of chunk (g, kc) holds seed bits
// base + (r + kc + 128g) + 4i + 32w — a function of the UNIT index u = r + kc + 128g alone. So
// the operand is a table of 16-byte units, unit u word w = the seed window starting at bit
// base + u + 32w (one funnel shift, masked to the E2M1 1.0 nibble bit), and the descriptor
// walks it with LBO = 16 B (next K chunk = next unit) and SBO = 128 B (8 rows = 8 units):
// rows overlap in memory exactly as Hankel rows overlap in the seed.
// Operand nibbles are masked to clean 0 / 1.0: toggling don't-care bits in the multipliers
// drew the 1000 W power cap (SM clock 1.61 GHz instead of 1.965; round 1).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "ptx.cuh"
#include "split_tree.cuh"

namespace ssbh_impl {
using namespace ssbh_dev;

namespace {

constexpr int kM = 128;                      // blocks per M tile (= TMEM lanes)
constexpr int kN = 256;                      // output rows per N tile (= accumulator columns)
constexpr int kFullArrivals = 8;             // 4 A warps + 4 B warps per stage
constexpr int kSetsC = 2;                     // producer sets (kSets below)
constexpr uint32_t kF4StageWords = 16;       // y words per 512-position pipeline stage

// ------------------------------------------------------------------ tcgen05 / cp.async
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Shared-memory matrix descriptor, SWIZZLE_NONE, version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

#define SSBH_TMEM_LD32(taddr, v)                                                                 \
    asm volatile(                                                                                \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"       \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),    \
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),             \
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),          \
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),          \
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),          \
          "=r"(v[31])                                                                            \
        : "r"(taddr))

// Compiler-level fence on 32 registers: later uses of v cannot be scheduled above this point.
#define SSBH_REG_FENCE32(v)                                                                      \
    asm volatile(""                                                                              \
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),       \
                   "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),     \
                   "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), \
                   "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]), \
                   "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), \
                   "+r"(v[30]), "+r"(v[31])::"memory")

#define SSBH_TMEM_ST32(taddr, v)                                                                 \
    asm volatile(                                                                                \
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"   \
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"      \
        ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),          \
        "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]),          \
        "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]),      \
        "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),      \
        "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])                               \
        : "memory")

// 16 accumulator columns v[o .. o + 15] (exact f32 counts < 2^23) -> their parities, column e
// in bit e: bit 0 of count + 2^23 is shifted in from the top (one SHF per column), in two
// independent chains.
__device__ __forceinline__ uint32_t parity16(const uint32_t (&v)[32], int o) {
    uint32_t c0 = 0, c1 = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        c0 = __funnelshift_r(c0, __float_as_uint(__uint_as_float(v[o + e]) + 8388608.0f), 1);
        c1 = __funnelshift_r(c1, __float_as_uint(__uint_as_float(v[o + 8 + e]) + 8388608.0f), 1);
    }
    return __byte_perm(c0, c1, 0x4473);  // c0 bits 24..31 -> 0..7, c1 bits 24..31 -> 8..15
}

// Dev A/B hooks (tools/build_exp.sh): which waits poll instead of suspending.
#if defined(SSBH_EXP_SPIN_ALL)
#define F4_WAIT_T mbar_wait
#define F4_WAIT_S mbar_wait
#elif defined(SSBH_EXP_SPIN_T)
#define F4_WAIT_T mbar_wait
#define F4_WAIT_S mbar_wait_sleep
#else
#define F4_WAIT_T mbar_wait_sleep
#define F4_WAIT_S mbar_wait_sleep
#endif

// ------------------------------------------------------------------ work items
struct Item {
    uint32_t mt, nt;     // M tile (128 owned blocks), N tile (256 output rows)
    uint32_t child;      // parent mode: 0 = P (lo ^ hi), 1 = Q (lo), 2 = R (hi)
    uint32_t ph;         // parent mode: phase of the super-item, 0 = Q, 1 = P, 2 = R
    uint32_t st0, nst;   // stage range [st0, st0 + nst) of this K part
    uint64_t soff;       // seed offset (u32 words) of the M tile's first block: 0 for a plan's
                         // shared seed; the split's leaf groups (128-aligned) each have their own
    uint64_t uoff;       // leaf modes: first unit of the M tile's leaf group in the Hankel unit
                         // tables (k_hankel_units)
};

__device__ __forceinline__ bool decode(const MmaHashArgs& a, uint32_t item, Item& d) {
    if (item >= a.items) return false;
    d.nt = item % a.ntiles;
    d.child = 0;
    d.ph = 0;
    d.uoff = 0;
    if (a.leaf == 2) {
        // item = ((parent group * mpg + M tile in group) * 3 + child) * ntiles + nt
        const uint32_t c3 = item / a.ntiles;
        d.child = c3 % 3;
        const uint32_t sup = c3 / 3;
        const uint32_t mpg = a.src.gpad / kM;
        const uint32_t pg = sup / mpg, mtl = sup % mpg;
        const uint32_t pleaves = a.src.leaves / 3;
        const uint32_t t = pg / pleaves, pp = pg % pleaves;
        const uint32_t grp = t * a.src.leaves + 3 * pp + d.child;  // the child's group
        d.mt = grp * mpg + mtl;
        d.soff = a.lay.soff[(uint64_t)d.mt * kM];
        d.st0 = 0;
        d.nst = a.mt_words[d.mt] / (a.stage_bits / 32);
        return true;
    }
    const uint32_t r = item / a.ntiles;
    const uint32_t kp = r % a.ksplit;
    d.mt = r / a.ksplit;
    d.soff = a.lay.soff[(uint64_t)d.mt * kM];
    const uint32_t ns = a.mt_words[d.mt] / (a.stage_bits / 32);
    const uint32_t lo = (uint32_t)((uint64_t)ns * kp / a.ksplit);
    d.st0 = lo;
    d.nst = (uint32_t)((uint64_t)ns * (kp + 1) / a.ksplit) - lo;
    return true;
}

// A CTA's item sequence. Direct mode: items blockIdx.x, +grid, ..., each decoded on its own.
// Leaf modes: super-items (leaf: M tile x K part; parent mode: the parent's M tile with its
// three children, one child after the other) blockIdx.x, +grid, ..., whose N tiles follow each
// other while the M tile's leaf inputs stay in shared memory. Everything but the N tile (and the child) is decoded once
// per super-item: the per-item decode (five divisions and two layout loads, in every warp) was
// ~1100 clocks of tensor-pipe bubble per item (skeleton A/B, profiles/r02_ab_leaf_gemm.md).
__device__ __forceinline__ uint32_t super_items(const MmaHashArgs& a) {
    return a.leaf == 2 ? 3 * a.ntiles : a.ntiles;
}
struct ItemWalk {
    Item d;
    bool valid;
    uint32_t sup;  // leaf modes: super-item index; direct mode: item index
    __device__ __forceinline__ void load(const MmaHashArgs& a) {
        if (!a.leaf) {
            valid = decode(a, sup, d);
            return;
        }
        valid = sup < (uint32_t)(a.items / super_items(a));
        if (!valid) return;
        d.nt = 0;
        d.child = 0;
        d.ph = 0;
        if (a.leaf == 2) {
            // super-item = parent group * mpg + M tile in the group; child c is leaf group
            // t * leaves + 3 * pp + c, whose M tiles lie c * mpg further and whose seed region /
            // unit table follow the previous child's. The phases run Q, P, R (see next()).
            const uint32_t mpg = a.src.gpad / kM;
            const uint32_t pg = sup / mpg, mtl = sup % mpg;
            const uint32_t pleaves = a.src.leaves / 3;
            const uint32_t t = pg / pleaves, pp = pg % pleaves;
            d.child = 1;
            d.mt = (t * a.src.leaves + 3 * pp + 1) * mpg + mtl;
            d.st0 = 0;
            d.nst = a.mt_words[d.mt] / (kF4StageWords);  // the same rows in all three children
        } else {
            const uint32_t kp = sup % a.ksplit;
            d.mt = sup / a.ksplit;
            const uint32_t ns = a.mt_words[d.mt] / (kF4StageWords);
            d.st0 = (uint32_t)((uint64_t)ns * kp / a.ksplit);
            d.nst = (uint32_t)((uint64_t)ns * (kp + 1) / a.ksplit) - d.st0;
        }
        d.soff = a.lay.soff[(uint64_t)d.mt * kM];
        d.uoff = (uint64_t)(d.mt / (a.src.gpad / kM)) * a.unit_stride;
    }
    __device__ __forceinline__ void start(const MmaHashArgs& a) {
        sup = blockIdx.x;
        load(a);
    }
    __device__ __forceinline__ void next(const MmaHashArgs& a) {
        if (a.leaf == 2) {
            // child by child in the order Q (reads the lo half of the parent's input), P (lo ^
            // hi), R (hi): while R runs the lo half is free for the next parent's input, and
            // while the next Q runs so is the hi half — the epilogue warps build them in the
            // background (k_leaf_gemm)
            if (++d.nt < a.ntiles) return;
            d.nt = 0;
            const uint32_t mpg = a.src.gpad / kM;
            if (d.ph == 0) {  // Q -> P
                d.ph = 1;
                d.child = 0;
                d.mt -= mpg;
                d.soff -= a.src.seed_words;
                d.uoff -= a.unit_stride;
                return;
            }
            if (d.ph == 1) {  // P -> R
                d.ph = 2;
                d.child = 2;
                d.mt += 2 * mpg;
                d.soff += 2 * a.src.seed_words;
                d.uoff += 2 * a.unit_stride;
                return;
            }
        } else if (a.leaf) {
            if (++d.nt < a.ntiles) return;
        }
        sup += gridDim.x;
        load(a);
    }
};

// Walks (item, stage) pairs of this CTA in order; used by the producers twice (consume and
// prefetch kPre stages ahead).
struct StageIt {
    ItemWalk w;
    uint32_t s;      // stage within the item
    __device__ __forceinline__ void start(const MmaHashArgs& a) {
        w.start(a);
        s = 0;
        skip_empty(a);
    }
    __device__ __forceinline__ void skip_empty(const MmaHashArgs& a) {
        while (w.valid && s >= w.d.nst) {
            w.next(a);
            s = 0;
        }
    }
    __device__ __forceinline__ void next(const MmaHashArgs& a) {
        ++s;
        skip_empty(a);
    }
    // skip over the stages other producer sets fill
    __device__ __forceinline__ void advance(const MmaHashArgs& a, int count) {
        for (int i = 0; i < count && w.valid; ++i) next(a);
    }
};

// B producer warp: stage 32 seed words (pre-shifted seed S', S'[b] = S[b-1]) covering the
// stage's windows; lanes 0-7 copy 16 B each.
__device__ __forceinline__ void s_prefetch(const MmaHashArgs& a, const StageIt& p, uint32_t lane,
                                           uint32_t* raw) {
    if (lane < 8) {
        uint64_t q0a = 0;
        if (p.w.valid) {
            const uint64_t b1 =
                (uint64_t)p.w.d.nt * kN + (uint64_t)(p.w.d.st0 + p.s) * a.stage_bits + 1;
            q0a = (b1 >> 5) & ~3ull;
        }
        cp_async16(raw + 4 * lane, a.sbuf + (p.w.valid ? p.w.d.soff : 0ull) + q0a + 4 * lane,
                   p.w.valid ? 16u : 0u);
    }
}

// =========================================================================================
// Shared seeds on FP4 operands (tcgen05.mma kind::mxf4, block-scaled E2M1, every UE8M0 scale
// 1.0): the same Y * H^T product at twice the kind::i8 MAC rate (measured 4.46 vs 2.10 P MAC/s,
// tools/f4_probe.py). Every operand element is 0 or 1.0 (nibble 0b0010), so every product is
// 0 or 1 and the f32 accumulator holds the exact integer count while it stays below 2^24
// (verified by the probe); items longer than kF4MaxStages stages are accumulated in several
// rounds whose parities are XORed (parity of a sum = XOR of the parities of its parts).
// K order inside a 512-position stage: chunk q = 4g + kc (16 B = 32 nibbles), word w,
// nibble i <-> position 128g + kc + 4i + 32w, so
//   A (y, M = 128 blocks, shared memory): chunk (g, kc) word w = ((y word 4g + w) >> kc << 1)
//     & 0x22222222 — one shift and one mask per 8 elements, as in the i8 engine;
//   B (Hankel, N = 256 rows): row r chunk (g, kc) = unit r + kc + 128g, unit u word w =
//     (seed window at bit base + u + 32w << 1) & 0x22222222; 643 units per stage,
//     LBO 16 B, SBO 128 B.
// Block-scaled kinds take A from shared memory only, so both operands are staged in shared
// memory (4 stages x 42 KB); TMEM = one 128 x 256 f32 accumulator + the constant scale
// factors. Warp roles: kE epilogue warps (default 8, two per TMEM sub-partition), one MMA warp,
// then two producer sets alternating stages as in k_toeplitz_mma.
constexpr int kF4StageK = 512;                    // input positions per stage (8 MMAs, K = 64)
constexpr int kF4GUnits = kN + 3 + 384 + 1;       // 643 Hankel units per stage
// A operand (the blocks' y bits as E2M1 nibbles) in TMEM: 64 columns per stage (128 lanes = block
// rows, column 4q + w = chunk q word w; nibble i of a column = K element 8c + i, probed by
// k_f4_tmem_a_probe), a ring of kF4Stages next to the accumulator (columns 0..255) and the scale
// factors (256..287). B (Hankel units) stays in shared memory.
constexpr uint32_t kF4ACol0 = 320;                // A ring: columns 320..511
constexpr int kF4GBytes = ((kF4GUnits * 16 + 127) / 128) * 128;  // 10368
constexpr int kF4Slot = kF4GBytes;                // shared memory per stage: B only
constexpr int kF4Stages = 3;                      // = TMEM A stages (3 x 64 columns)
constexpr int kF4Pre = 2;                         // cp.async prefetch depth per set
constexpr int kF4RawY = kF4Pre * kM * 64;         // per set
constexpr int kF4RawS = 4 * kF4Pre * 128;         // per set
__host__ __device__ constexpr size_t f4_bar(int sets) { return (size_t)kF4Stages * kF4Slot + sets * (kF4RawY + kF4RawS); }
__host__ __device__ constexpr size_t f4_smem(int sets) { return f4_bar(sets) + (2 * kF4Stages + 4) * 8 + 16; }
static_assert(f4_smem(2) <= 232448, "f4 smem budget");
// exact f32 counts per round, < 2^23 so that the epilogue's parity read (count + 2^23: the
// integer lands in the low mantissa bits, FADD instead of the slower F2I) stays exact
constexpr uint32_t kF4MaxStages = (1u << 23) / kF4StageK;
constexpr uint32_t kF4SfCol = kN;                            // scale factors: columns 256..287
// kind::mxf4 instruction descriptor: E2M1 x E2M1, UE8M0 scales, K-major, M = 128, N = 256
constexpr uint32_t kF4Idesc = (1u << 7) | (1u << 10) | ((uint32_t)(kN >> 3) << 17) | (1u << 23) |
                              ((uint32_t)(kM >> 4) << 24);

// kind::mxf4 instruction descriptor with a runtime N (multiple of 16, 16..256; M = 128)
__host__ __device__ constexpr uint32_t f4_idesc(uint32_t n) {
    return (kF4Idesc & ~(0x3Fu << 17)) | ((n >> 3) << 17);
}
__device__ __forceinline__ void mma_f4n(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t sf, uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accum), "r"(sf)
        : "memory");
}

// A operand from TMEM (a_tmem: lane = row, 8 columns per K = 64).
__device__ __forceinline__ void mma_f4_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                          uint32_t sf, uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%5], p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(kF4Idesc), "r"(accum), "r"(sf)
        : "memory");
}

__device__ __forceinline__ void mma_f4(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t sf,
                                       uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(kF4Idesc), "r"(accum), "r"(sf)
        : "memory");
}

__device__ __forceinline__ void y_prefetch_f4(const MmaHashArgs& a, const StageIt& p,
                                              uint32_t jl, uint32_t* raw) {
    const uint32_t* src = a.ybuf;
    uint32_t bytes = 0;
    if (p.w.valid) {
        const uint32_t jj = p.w.d.mt * kM + jl;
        const uint64_t w0 = (uint64_t)(p.w.d.st0 + p.s) * (kF4StageK / 32);
        if (jj < a.nown && w0 < a.lay.ypad[jj]) {
            src = a.ybuf + a.lay.yoff[jj] + w0;
            bytes = 16;
        }
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) cp_async16(raw + h * kM * 4, src + 4 * h, bytes);
}

__device__ __forceinline__ void red_xor(uint32_t* p, uint32_t v) {
    asm volatile("red.global.xor.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// A operand of one stage: the row's 512 y bits (x: 16 words) as E2M1 nibbles into the 64 TMEM
// columns at ta. ((x >> kc) << 1) & M2 == shift by kc - 1 (one SHF), left by one for kc = 0;
// chunk q = 4 gg + kc, word w -> column 4 q + w of the stage.
__device__ __forceinline__ void expand_a(const uint4 (&x)[4], uint32_t ta) {
    constexpr uint32_t M2 = 0x22222222u;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // columns 32h .. 32h + 31: chunks 8h .. 8h + 7
        uint32_t v[32];
#pragma unroll
        for (int g2 = 0; g2 < 2; ++g2) {
            const uint4 xg = x[2 * h + g2];
#pragma unroll
            for (int kc = 0; kc < 4; ++kc) {
                auto f = [&](uint32_t u) { return (kc ? u >> (kc - 1) : u << 1) & M2; };
                v[16 * g2 + 4 * kc + 0] = f(xg.x);
                v[16 * g2 + 4 * kc + 1] = f(xg.y);
                v[16 * g2 + 4 * kc + 2] = f(xg.z);
                v[16 * g2 + 4 * kc + 3] = f(xg.w);
            }
        }
        SSBH_TMEM_ST32(ta + 32u * h, v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Leaf mode (the split's shared-seed leaves): kLeafKpw words of each of the 128 virtual blocks'
// leaf input per K part live in shared memory for all N tiles of the M tile.
constexpr uint32_t kLeafKpw = 256;                     // 8192 positions per K part
constexpr uint32_t kLeafStride = kLeafKpw + 4;
constexpr uint32_t kLeafPieces = 1u << kMaxL;           // input pieces of a leaf, at most

// Offset (bits) of input piece e of the node `path` at level L (digits base 3, most significant
// = level 0; 0 = P: x0 ^ x1 doubles the pieces, 1 = Q: x0, 2 = R: x1) — leaf_offsets
// (split_tree.cuh) in closed form, so that every piece is computed by its own thread. Returns
// the number of pieces through *n.
__device__ __forceinline__ uint64_t piece_offset(uint32_t path, uint32_t L, uint64_t k,
                                                 uint64_t base, uint32_t e, uint32_t* n) {
    uint32_t pw = 1;
    for (uint32_t l = 1; l < L; ++l) pw *= 3;
    uint64_t off = base, m = k;
    uint32_t np = 0;
    for (uint32_t l = 0; l < L; ++l, pw /= 3) {
        m >>= 1;
        const uint32_t dg = path / pw % 3;
        if (dg == 2) off += m;
        if (dg == 0) {
            if ((e >> np) & 1u) off += m;
            ++np;
        }
    }
    *n = 1u << np;
    return off;
}

// Builds the M tile's leaf inputs for K part d (words [d.st0 * 16, + kpw) of each leaf) into
// lraw: row jl = XOR over the leaf's input pieces of the original block's reversed input
// (the k_split_inputs arithmetic, toeplitz_split.cu), zero past the block's padded length and
// for padding rows. Called by all 16 producer warps together (bw = 0..15, named barrier 1,
// 512 threads): the build is bound by the L2 reads in flight, so the Hankel producers, idle
// while the tensor pipe waits for the new inputs, carry half of them. nb = builds done so far
// (the piece offsets are double-buffered, so one barrier covers "last tile's expansions done"
// and "offsets visible").
template <int kBW>
__device__ __forceinline__ void leaf_build(const MmaHashArgs& a, const Item& d, uint32_t bw,
                                           uint32_t lane, uint32_t* lraw,
                                           unsigned long long* loff2, uint32_t nb) {
    const LeafSrc& q = a.src;
    const uint64_t v0 = (uint64_t)d.mt * kM;  // first virtual block (one group per M tile)
    const uint32_t grp = (uint32_t)(v0 / q.gpad), jl0 = (uint32_t)(v0 % q.gpad);
    const uint32_t t = grp / q.leaves, path = grp % q.leaves;
    unsigned long long* loff = loff2 + (nb & 1u) * kLeafPieces;
    // parent mode: the input of the children's parent (level L - 1, path / 3)
    const uint32_t pL = a.leaf == 2 ? q.L - 1 : q.L, ppath = a.leaf == 2 ? path / 3 : path;
    uint32_t un = 1;
    for (uint32_t e = bw * 32 + lane; e < kLeafPieces; e += kBW * 32) {
        const uint64_t off = piece_offset(ppath, pL, q.k, (uint64_t)t * q.k, e, &un);
        if (e < un) loff[e] = off / 32;
    }
    const int n = (int)un;
    asm volatile("bar.sync 1, %0;" ::"n"(kBW * 32) : "memory");  // last tile's expansions done
    const uint64_t w0 = (uint64_t)d.st0 * 16;  // K part start (words, a multiple of 16)
    // 16-B loads with many L2 reads outstanding (the build is latency-bound otherwise): per
    // lane 2 rows x 2 vectors per piece, pieces unrolled by 2; 16 warps x 8 rows
    const uint32_t nvec = q.kpw / 4;  // uint4 per row (>= 4: kpw is a multiple of 16 words)
    constexpr int RB = 2;
    constexpr uint32_t kRows = kM / kBW;
    for (uint32_t r0 = bw * kRows; r0 < bw * kRows + kRows; r0 += RB) {
        const uint4* y[RB];
        uint64_t yp4[RB];
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) {
            const uint32_t jlg = jl0 + r0 + rr, jj = q.jj0 + jlg;
            const bool live = jlg < q.batch && jj < q.nown;
            y[rr] = reinterpret_cast<const uint4*>(live ? q.ybuf + q.lay.yoff[jj] : q.ybuf);
            yp4[rr] = live ? q.lay.ypad[jj] / 4 : 0;  // ypad is a multiple of 32 words
        }
        uint4 acc[RB][2];
#pragma unroll
        for (int rr = 0; rr < RB; ++rr)
#pragma unroll
            for (int h = 0; h < 2; ++h) acc[rr][h] = make_uint4(0, 0, 0, 0);
#pragma unroll 2
        for (int e = 0; e < n; ++e) {
            const uint64_t base4 = (loff[e] + w0) / 4;
#pragma unroll
            for (int rr = 0; rr < RB; ++rr)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t vl = lane + 32u * h;
                    const uint64_t qv = base4 + vl;
                    if (vl < nvec && qv < yp4[rr]) {
                        const uint4 v = __ldg(y[rr] + qv);
                        acc[rr][h].x ^= v.x;
                        acc[rr][h].y ^= v.y;
                        acc[rr][h].z ^= v.z;
                        acc[rr][h].w ^= v.w;
                    }
                }
        }
#pragma unroll
        for (int rr = 0; rr < RB; ++rr)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t vl = lane + 32u * h;
                if (vl < nvec)
                    *reinterpret_cast<uint4*>(lraw + (size_t)(r0 + rr) * kLeafStride + 4u * vl) =
                        acc[rr][h];
            }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kBW * 32) : "memory");
}

#ifdef SSBH_EXP_TRACE  // dev builds: clock64 timestamps of CTA 0's pipeline events for stages
                       // [kTrG0, kTrG0 + kTrN), printed at kernel end (leaf modes only)
constexpr uint32_t kTrG0 = 4000, kTrN = 128, kTrRoles = 10;
#define F4_TRACE(role, g)                                                               \
    do {                                                                                \
        if (blockIdx.x == 0 && a.leaf && (g) >= kTrG0 && (g) < kTrG0 + kTrN)             \
            trace[(role) * kTrN + ((g) - kTrG0)] = clock64();                           \
    } while (0)
#else
#define F4_TRACE(role, g) do { } while (0)
#endif

// Warp roles: 8 epilogue warps (two per TMEM sub-partition, half of the 256 accumulator
// columns each), 1 MMA warp (one elected thread issues), then two producer sets of 4 A + 4 B
// warps that fill alternate stages (one set's per-stage chain — cp.async wait -> expand ->
// tcgen05.st / STS -> arrive — is latency-bound). Direct mode only: whole blocks against a
// plan's shared seed (configs 1-2) and the split's remainder; the split's leaves run on
// k_leaf_gemm below. Round-1 A/B variants that lost (3 producer sets, register-staged y, 4
// epilogue warps, double-buffered TMEM loads, a polling MMA warp) are not built.
constexpr int kSets = kSetsC, kE = 8;
constexpr int kF4Threads = (kE + 1 + 8 * kSets) * 32;
__global__ void __launch_bounds__(kF4Threads, 1) k_toeplitz_f4(MmaHashArgs a) {
    constexpr int kEpiW = kE, kMmaW = kE, kProd0 = kE + 1;
    constexpr int kQW = (kN / 32) / (kE / 4);  // accumulator column groups per epilogue warp
    constexpr int kS = kF4Stages;
    constexpr uint32_t M2 = 0x22222222u;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* slots = smem;
    uint32_t* raw_y = reinterpret_cast<uint32_t*>(smem + (size_t)kS * kF4Slot);
    uint32_t* raw_s = raw_y + kSets * (kF4RawY / 4);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + f4_bar(kSets));
    uint64_t* empty = full + kS;
    uint64_t* tfull = empty + kS;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kS; ++s) {
            mbar_init(&full[s], kFullArrivals);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&tfull[0], 1);
        mbar_init(&tempty[0], kEpiW);
        fence_barrier_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp < 4) {  // constant scale factors: 0x7f = 2^0 in every byte
        uint32_t v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0x7F7F7F7Fu;
        SSBH_TMEM_ST32(tmem + ((warp * 32u) << 16) + kF4SfCol, v);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp < kEpiW) {
        // ---------------------------------------------------------------- epilogue
        const uint32_t sp = warp & 3, qb = (warp >> 2) * kQW;  // TMEM sub-partition, columns
        uint32_t t = 0;  // accumulation rounds consumed
        ItemWalk wk;
        for (wk.start(a); wk.valid; wk.next(a)) {
            const Item d = wk.d;
            const uint32_t rounds = d.nst ? (d.nst + kF4MaxStages - 1) / kF4MaxStages : 1;
            uint32_t acc_w[kQW];
#pragma unroll
            for (int q = 0; q < kQW; ++q) acc_w[q] = 0;
            for (uint32_t rd = 0; rd < rounds; ++rd, ++t) {
                F4_WAIT_T(&tfull[0], t & 1);
                tc_fence_after();
                if (d.nst) {
                    // The hand-off of the single accumulator is serial with the MMAs, so the
                    // warp releases it as soon as its last TMEM load has landed and only then
                    // reduces that load (parity16: independent funnel-shift chains).
#pragma unroll 1
                    for (int q = 0; q < kQW; ++q) {
                        uint32_t v[32];
                        SSBH_TMEM_LD32(tmem + ((sp * 32u) << 16) + 32u * (qb + q), v);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        if (q == kQW - 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&tempty[0]);
                        }
                        acc_w[q] ^= parity16(v, 0) | (parity16(v, 16) << 16);
                    }
                } else {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[0]);
                }
            }
            const uint32_t jj = d.mt * kM + sp * 32 + lane;
            if (d.nst && jj < a.nown) {
                uint32_t* dst =
                    a.out + (unsigned long long)jj * a.out_stride + d.nt * (kN / 32) + qb;
#pragma unroll
                for (int q = 0; q < kQW; ++q)
                    if (d.nt * (kN / 32) + qb + q < a.kw) {
                        if (a.ksplit == 1)
                            dst[q] = acc_w[q];
                        else
                            atomicXor(dst + q, acc_w[q]);
                    }
            }
        }
    } else if (warp == kMmaW) {
        // ---------------------------------------------------------------- MMA issuer
        uint32_t g = 0, t = 0;
        const uint32_t base_g = smem_u32(slots);
        ItemWalk wk;
        for (wk.start(a); wk.valid; wk.next(a)) {
            const Item d = wk.d;
            if (d.nst == 0) {
                if (t >= 1) F4_WAIT_T(&tempty[0], (t - 1) & 1);
                if (lane == 0) mbar_arrive(&tfull[0]);
                ++t;
                continue;
            }
            for (uint32_t s0 = 0; s0 < d.nst; s0 += kF4MaxStages, ++t) {
                if (t >= 1) F4_WAIT_T(&tempty[0], (t - 1) & 1);
                tc_fence_after();
                const uint32_t s1 = min(d.nst, s0 + kF4MaxStages);
                for (uint32_t s = s0; s < s1; ++s, ++g) {
                    const uint32_t slot = g % kS;
                    // hardware-suspended wait: no try_wait polls on the L1 data pipe the
                    // producers' stores and the MMA operand reads share (round 1: 1.1 % faster)
                    F4_WAIT_S(&full[slot], (g / kS) & 1);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t ga = base_g + slot * kF4Slot;
                        const uint32_t at = tmem + kF4ACol0 + 64u * slot;
#pragma unroll
                        for (int m = 0; m < 8; ++m) {  // MMA m: chunks 2m, 2m+1 = columns 8m..
                            const uint32_t unit = 2u * (m & 1) + 128u * (m >> 1);
                            mma_f4_ts(tmem, at + 8u * m, sdesc(ga + 16u * unit, 16, 128),
                                      tmem + kF4SfCol, ((s - s0) | (uint32_t)m) != 0);
                        }
                        mma_commit(&empty[slot]);
                        if (s + 1 == s1) mma_commit(&tfull[0]);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (((warp - kProd0) & 7) < 4) {
        // ---------------------------------------------------------------- A producers
        const uint32_t set = (warp - kProd0) >> 3;
        // TMEM lane = block row: a warp reaches the 32 lanes of its sub-partition (warp % 4)
        const uint32_t jl = 32u * (warp & 3) + lane;
        const uint32_t lane_addr = (32u * (warp & 3)) << 16;
        StageIt cur, pre;
        cur.start(a);
        cur.advance(a, set);
        pre = cur;
        uint32_t* raw = raw_y + set * (kF4RawY / 4) + jl * 4;  // [slot][quarter][jl][4 words]
        for (int i = 0; i < kF4Pre; ++i) {
            y_prefetch_f4(a, pre, jl, raw + i * kM * 16);
            cp_async_commit();
            pre.advance(a, kSets);
        }
        for (uint32_t g = set, i = 0; cur.w.valid; g += kSets, ++i, cur.advance(a, kSets)) {
            const uint32_t rs = i % kF4Pre;
            cp_async_wait<kF4Pre - 1>();
            uint4 x[4];
#pragma unroll
            for (int h = 0; h < 4; ++h)
                x[h] = *reinterpret_cast<const uint4*>(raw + rs * kM * 16 + h * kM * 4);
            const uint32_t slot = g % kS;
            if (g >= (uint32_t)kS) F4_WAIT_S(&empty[slot], ((g / kS) - 1) & 1);
            expand_a(x, tmem + lane_addr + kF4ACol0 + 64u * slot);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[slot]);
            y_prefetch_f4(a, pre, jl, raw + rs * kM * 16);
            cp_async_commit();
            pre.advance(a, kSets);
        }
        cp_async_wait<0>();
    } else {
        // ---------------------------------------------------------------- B producers
        const uint32_t set = (warp - kProd0) >> 3;
        const uint32_t gw = ((warp - kProd0) & 7) - 4;
        const uint32_t gt = gw * 32 + lane;
        uint32_t* raw = raw_s + set * (kF4RawS / 4) + gw * kF4Pre * 32;
        StageIt cur, pre;
        cur.start(a);
        cur.advance(a, set);
        pre = cur;
        for (int i = 0; i < kF4Pre; ++i) {
            s_prefetch(a, pre, lane, raw + i * 32);
            cp_async_commit();
            pre.advance(a, kSets);
        }
        for (uint32_t g = set, i = 0; cur.w.valid; g += kSets, ++i, cur.advance(a, kSets)) {
            const uint32_t rs = i % kF4Pre;
            cp_async_wait<kF4Pre - 1>();
            __syncwarp();
            const uint32_t* sw = raw + rs * 32;
            const uint64_t b1 =
                (uint64_t)cur.w.d.nt * kN + (uint64_t)(cur.w.d.st0 + cur.s) * kF4StageK + 1;
            const uint32_t rel0 = (uint32_t)(b1 - (((b1 >> 5) & ~3ull) << 5));
            const uint32_t slot = g % kS;
            if (g >= (uint32_t)kS) F4_WAIT_S(&empty[slot], ((g / kS) - 1) & 1);
            uint8_t* gs = slots + (size_t)slot * kF4Slot;
            // the window one bit lower (rel0 >= 1: base is a multiple of 256) has S bit
            // base + u + 32w + 4i at bit 4i + 1 — the E2M1 1.0 position. Unit u + 128 starts 4
            // words later with the same shift, so its first word is this unit's last: 4 shared
            // loads per unit instead of 5
            const uint32_t rel = rel0 + gt - 1;
            const uint32_t q0 = rel >> 5, sh = rel & 31;
            uint32_t w0 = sw[q0];
#pragma unroll
            for (int r = 0; r < 6; ++r) {
                const uint32_t u = gt + 128u * r;
                if (u < (uint32_t)kF4GUnits) {
                    const uint32_t q = q0 + 4u * r;
                    const uint32_t w1 = sw[q + 1], w2 = sw[q + 2], w3 = sw[q + 3], w4 = sw[q + 4];
                    *reinterpret_cast<uint4*>(gs + 16 * u) =
                        make_uint4(__funnelshift_r(w0, w1, sh) & M2, __funnelshift_r(w1, w2, sh) & M2,
                                   __funnelshift_r(w2, w3, sh) & M2, __funnelshift_r(w3, w4, sh) & M2);
                    w0 = w4;
                }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[slot]);
            s_prefetch(a, pre, lane, raw + rs * 32);
            cp_async_commit();
            pre.advance(a, kSets);
        }
        cp_async_wait<0>();
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// =========================================================================================
// The split's shared-seed leaves (leaf / parent mode) as their own kernel, k_leaf_gemm. Same
// product and operand layouts as k_toeplitz_f4, re-plumbed after the pipeline trace of round 2
// (profiles/r02_ab_leaf_gemm.md):
//  * the Hankel operand comes from a precomputed table of units (k_hankel_units: for every leaf
//    seed, unit G word j = the seed window at bit G + 32 j masked to the E2M1 1.0 bit). A stage's
//    643 units are consecutive there, so the B tile is ONE 10 KB bulk copy (cp.async.bulk
//    completing on the stage's mbarrier) issued by one thread — no funnel shifts, no shared
//    loads / stores by eight producer warps, which were the last to arrive at every stage;
//  * B has its own ring (kLfBS slots of shared memory, deep enough for the copy latency), the A
//    operand keeps its 3-stage ring in TMEM, filled by 4 warps (one per TMEM sub-partition);
//  * 16 epilogue warps (four per TMEM sub-partition, 64 accumulator columns each): a shorter
//    hand-off of the single accumulator between items;
//  * parent mode runs a parent's children in the order Q, P, R (ItemWalk) and kLfBW build warps
//    prepare the NEXT inputs in the background: the next parent's lo half while R runs (which
//    reads hi only), its hi half while its Q runs (which reads lo only). (Building from the
//    epilogue warps between hand-offs made them late for the next hand-off: 22.5 -> 36 ms.)
//    The first combine level stays fused: the parent's rows are written as lo = Q, then
//    lo ^= P and hi = P, then hi ^= R by the same thread.
constexpr int kLfBS = 8;                    // B ring (Hankel unit tiles, shared memory)
constexpr int kLfAS = 3;                    // A ring (TMEM, 64 columns per stage)
constexpr int kLfEW = 16;                   // epilogue warps
constexpr int kLfAW = 4;                    // A producer warps: sets of 4 (one per sub-partition)
constexpr int kLfSets = kLfAW / 4;          // a set fills every kLfSets-th stage
constexpr int kLfBW = 6;                    // background-build warps (parent mode): 28 warps in
                                            // all keep 72 registers per thread; 8 build warps
                                            // (30 warps, 64 registers) measured 25.1 ms
constexpr int kLfMmaW = kLfEW, kLfLoadW = kLfEW + 1, kLfProd0 = kLfEW + 2;
constexpr int kLfBuild0 = kLfProd0 + kLfAW;
constexpr int kLfThreads = (kLfEW + 2 + kLfAW + kLfBW) * 32;
constexpr size_t kLfBar =
    (size_t)kLfBS * kF4Slot + (size_t)kM * kLeafStride * 4 + 2 * kLeafPieces * 8;
constexpr size_t kLfSmem = kLfBar + (2 * kLfAS + 2 * kLfBS + 8) * 8 + 16;
static_assert(kLfSmem <= 232448, "leaf GEMM smem budget");
constexpr uint32_t kLfTileBytes = kF4GUnits * 16;  // one stage's Hankel units

// Hankel unit tables: region r (a leaf seed of seed_words pre-shifted words at vs), unit G,
// word j = (S' >> (G + 32 j)) & 0x22222222 — what the B producers of k_toeplitz_f4 form per
// stage (unit u of the stage at N tile nt, stage st is G = 256 nt + 512 st + u).
__global__ void __launch_bounds__(256) k_hankel_units(const uint32_t* __restrict__ vs,
                                                      uint64_t seed_words, uint64_t unit_stride,
                                                      uint4* __restrict__ units) {
    const uint64_t r = blockIdx.y;
    const uint32_t* sw = vs + r * seed_words;
    for (uint64_t G = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; G < unit_stride;
         G += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q = G >> 5;
        const uint32_t sh = (uint32_t)G & 31u;
        uint32_t w[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) w[j] = q + j < seed_words ? __ldg(sw + q + j) : 0u;
        constexpr uint32_t M2 = 0x22222222u;
        units[r * unit_stride + G] =
            make_uint4(__funnelshift_r(w[0], w[1], sh) & M2, __funnelshift_r(w[1], w[2], sh) & M2,
                       __funnelshift_r(w[2], w[3], sh) & M2, __funnelshift_r(w[3], w[4], sh) & M2);
    }
}

// Parent mode, background build: rows [r0, r1) of super-item `sup`'s M tile, half h (0 = lo,
// 1 = hi) of the parent's input -> lraw. Row = XOR over the parent's input pieces of the
// original block's reversed input (piece e: base + the P levels' sizes selected by e's bits),
// zero past the block's padded length and for padding rows; one uint4 per lane per piece,
// kBuildInFlight pieces in flight. Variants measured (profiles/r02_ab_leaf_gemm.md): the
// epilogue warps building between hand-offs (late for the next hand-off), one warp through the
// bulk-copy engine (~300 clocks per 512-byte copy) and warps staging pieces with cp.async (slower
// per piece than register loads) all lose to dedicated warps with plain loads.
constexpr int kBuildInFlight = 8;
constexpr uint32_t kLfBRows = (kM + kLfBW - 1) / kLfBW;  // rows of the M tile per build warp
__device__ __forceinline__ void build_half_rows(const MmaHashArgs& a, uint32_t sup, uint32_t h,
                                                uint32_t r0, uint32_t r1, uint32_t lane,
                                                uint32_t* lraw, uint32_t* woff) {
    const LeafSrc& q = a.src;
    const uint32_t mpg = q.gpad / kM, pleaves = q.leaves / 3;
    const uint32_t pg = sup / mpg, jl0 = (sup % mpg) * kM;
    const uint32_t t = pg / pleaves, pp = pg % pleaves;
    const uint32_t hw = q.kpw / 2;  // words per half (= the leaf size)
    // the pieces' word offsets into a block's reversed input, once per call into the warp's
    // table woff (lane e, e + 32, ...): piece_offset in words, + the half
    uint32_t un = 1;
    for (uint32_t e = lane; e < kLeafPieces / 2; e += 32) {
        const uint64_t off = piece_offset(pp, q.L - 1, q.k, (uint64_t)t * q.k, e, &un);
        if (e < un) woff[e] = (uint32_t)(off / 32) + h * hw;
    }
    __syncwarp();
    const uint32_t n = un;
    const bool lane_on = lane < hw / 4;
    for (uint32_t r = r0; r < r1; ++r) {
        const uint32_t jlg = jl0 + r, jj = q.jj0 + jlg;
        const bool live = lane_on && jlg < q.batch && jj < q.nown;
        const uint4* y = reinterpret_cast<const uint4*>(live ? q.ybuf + q.lay.yoff[jj] : q.ybuf);
        const uint32_t yp4 = live ? q.lay.ypad[jj] / 4 : 0;  // ypad is a multiple of 32 words
        uint4 acc = make_uint4(0, 0, 0, 0);
        for (uint32_t e0 = 0; e0 < n; e0 += kBuildInFlight) {
            uint4 v[kBuildInFlight];
#pragma unroll
            for (int i = 0; i < kBuildInFlight; ++i) {
                const uint32_t e = e0 + i;
                const uint32_t qv = (e < n ? woff[e] : 0u) / 4 + lane;
                v[i] = e < n && qv < yp4 ? __ldg(y + qv) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int i = 0; i < kBuildInFlight; ++i) {
                acc.x ^= v[i].x;
                acc.y ^= v[i].y;
                acc.z ^= v[i].z;
                acc.w ^= v[i].w;
            }
        }
        if (lane_on)
            *reinterpret_cast<uint4*>(lraw + (size_t)r * kLeafStride + h * hw + 4u * lane) = acc;
    }
    __syncwarp();
}

__global__ void __launch_bounds__(kLfThreads, 1) k_leaf_gemm(MmaHashArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* bslots = smem;
    uint32_t* lraw = reinterpret_cast<uint32_t*>(smem + (size_t)kLfBS * kF4Slot);
    unsigned long long* loff =
        reinterpret_cast<unsigned long long*>(lraw + (size_t)kM * kLeafStride);  // [2][pieces]
    uint64_t* afull = reinterpret_cast<uint64_t*>(smem + kLfBar);
    uint64_t* aempty = afull + kLfAS;
    uint64_t* bfull = aempty + kLfAS;
    uint64_t* bempty = bfull + kLfBS;
    uint64_t* tfull = bempty + kLfBS;
    uint64_t* tempty = tfull + 1;
    // parent mode: the halves of the parent's input — free (the A warps have read the last
    // stage that uses it) and ready (the 16 build warps have written the next one)
    uint64_t* lo_free = tempty + 1;
    uint64_t* hi_free = lo_free + 1;
    uint64_t* lo_ready = hi_free + 1;
    uint64_t* hi_ready = lo_ready + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hi_ready + 2);
#ifdef SSBH_EXP_TRACE
    long long* trace = reinterpret_cast<long long*>(smem + kLfSmem);
    for (uint32_t i = threadIdx.x; i < kTrRoles * kTrN; i += blockDim.x) trace[i] = 0;
#endif

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nsupers = (uint32_t)(a.items / super_items(a));
    if (threadIdx.x == 0) {
        for (int s = 0; s < kLfAS; ++s) {
            mbar_init(&afull[s], 4);
            mbar_init(&aempty[s], 1);
        }
        for (int s = 0; s < kLfBS; ++s) {
            mbar_init(&bfull[s], 1);
            mbar_init(&bempty[s], 1);
        }
        mbar_init(&tfull[0], 1);
        mbar_init(&tempty[0], kLfEW);
        mbar_init(lo_free, kLfAW);
        mbar_init(hi_free, kLfAW);
        mbar_init(lo_ready, kLfBW);
        mbar_init(hi_ready, kLfBW);
        fence_barrier_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp < 4) {  // constant scale factors: 0x7f = 2^0 in every byte
        uint32_t v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0x7F7F7F7Fu;
        SSBH_TMEM_ST32(tmem + ((warp * 32u) << 16) + kF4SfCol, v);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp < kLfEW) {
        // ---------------------------------------------------------------- epilogue + builds
        constexpr int kQW = (kN / 32) / (kLfEW / 4);  // 32-column groups per warp (2)
        const uint32_t sp = warp & 3, qb = (warp >> 2) * kQW;
        uint32_t t = 0;
#ifdef SSBH_EXP_TRACE
        uint32_t eg = 0;
#endif
        ItemWalk wk;
        wk.start(a);
        for (; wk.valid; wk.next(a)) {
            const Item d = wk.d;
            F4_WAIT_T(&tfull[0], t & 1);
            ++t;
            tc_fence_after();
            if (warp == 0 && lane == 0) F4_TRACE(7, eg);
            uint32_t acc_w[kQW];
#pragma unroll
            for (int q = 0; q < kQW; ++q) acc_w[q] = 0;
#ifndef SSBH_EXP_NODRAIN
            if (d.nst) {
#else
            if (false) {
#endif
#ifndef SSBH_EXP_DRAIN2  // one load at a time (32 registers)
                const uint32_t tcol = tmem + ((sp * 32u) << 16) + 32u * qb;
#pragma unroll
                for (int q = 0; q < kQW; ++q) {
                    uint32_t v[32];
                    SSBH_TMEM_LD32(tcol + 32u * q, v);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (q == kQW - 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[0]);
                    }
                    acc_w[q] = parity16(v, 0) | (parity16(v, 16) << 16);
                }
#else
                // dev A/B: both loads in flight (64 registers: no gain measured, 20.94 vs 21.00 ms)
                uint32_t v0[32], v1[32];
                const uint32_t tcol = tmem + ((sp * 32u) << 16) + 32u * qb;
                SSBH_TMEM_LD32(tcol, v0);
                SSBH_TMEM_LD32(tcol + 32u, v1);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (warp == 0 && lane == 0) F4_TRACE(8, eg);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[0]);
                if (warp == 0 && lane == 0) F4_TRACE(9, eg);
                // the reduction must not be scheduled ahead of the release
                SSBH_REG_FENCE32(v0);
                SSBH_REG_FENCE32(v1);
                acc_w[0] = parity16(v0, 0) | (parity16(v0, 16) << 16);
                acc_w[1] = parity16(v1, 0) | (parity16(v1, 16) << 16);
#endif
            } else {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[0]);
            }
#ifdef SSBH_EXP_TRACE
            eg += d.nst;
#endif
            const uint32_t jj = d.mt * kM + sp * 32 + lane;
            if (a.leaf == 2) {
                // the first combine level: the parent node's rows [P ^ Q | P ^ R] (row = parent
                // M tile row, a.kw words per half) in three steps by the same thread
                if (d.nst && jj < a.nown) {
                    uint32_t* lo = a.out +
                                   (unsigned long long)(wk.sup * kM + sp * 32 + lane) * a.out_stride +
                                   d.nt * (kN / 32) + qb;
                    uint32_t* hi = lo + a.kw;
#pragma unroll
                    for (int q = 0; q < kQW; ++q)
                        if (d.nt * (kN / 32) + qb + q < a.kw) {
                            // XOR by red.global (fire and forget, ordered after this thread's
                            // earlier store to the word): a load-modify-store here put 1024
                            // scattered L2 reads per item into the L1 miss queue, behind which
                            // the A and MMA warps' shared-memory operations stalled
                            if (d.ph == 0) {
                                lo[q] = acc_w[q];
                            } else if (d.ph == 1) {
                                red_xor(lo + q, acc_w[q]);
                                hi[q] = acc_w[q];
                            } else {
                                red_xor(hi + q, acc_w[q]);
                            }
                        }
                }
            } else if (d.nst && jj < a.nown) {
                uint32_t* dst =
                    a.out + (unsigned long long)jj * a.out_stride + d.nt * (kN / 32) + qb;
#pragma unroll
                for (int q = 0; q < kQW; ++q)
                    if (d.nt * (kN / 32) + qb + q < a.kw) {
                        if (a.ksplit == 1)
                            dst[q] = acc_w[q];
                        else
                            atomicXor(dst + q, acc_w[q]);
                    }
            }
        }
    } else if (warp == kLfMmaW) {
        // ---------------------------------------------------------------- MMA issuer
        uint32_t t = 0;
#ifdef SSBH_EXP_TRACE
        uint32_t g = 0;
#endif
        uint32_t sa = 0, pa = 0, sb = 0, pb = 0;  // ring slots and their phases
        const uint32_t base_b = smem_u32(bslots);
        ItemWalk wk;
        for (wk.start(a); wk.valid; wk.next(a)) {
            const uint32_t nst = wk.d.nst;
            if (nst == 0) {
                if (t >= 1) F4_WAIT_T(&tempty[0], (t - 1) & 1);
                ++t;
                if (lane == 0) mbar_arrive(&tfull[0]);
                continue;
            }
            // the first stage's operands are ready long before the accumulator is handed back:
            // their barrier round trips stay off the hand-off path
            F4_WAIT_S(&afull[sa], pa);
            F4_WAIT_S(&bfull[sb], pb);
#ifndef SSBH_EXP_NOTEMPTY
            if (t >= 1) F4_WAIT_T(&tempty[0], (t - 1) & 1);
#endif
            ++t;
            tc_fence_after();
            if (lane == 0) F4_TRACE(6, g);
            for (uint32_t s = 0; s < nst; ++s) {
                if (s) {
                    F4_WAIT_S(&afull[sa], pa);
                    F4_WAIT_S(&bfull[sb], pb);
                    tc_fence_after();
                }
                if (lane == 0) F4_TRACE(4, g);
                if (elect_one()) {
                    const uint32_t gb = base_b + sb * kF4Slot;
                    const uint32_t at = tmem + kF4ACol0 + 64u * sa;
#pragma unroll
                    for (int m = 0; m < 8; ++m) {  // MMA m: chunks 2m, 2m+1 = columns 8m..
                        const uint32_t unit = 2u * (m & 1) + 128u * (m >> 1);
                        mma_f4_ts(tmem, at + 8u * m, sdesc(gb + 16u * unit, 16, 128),
                                  tmem + kF4SfCol, (s | (uint32_t)m) != 0);
                    }
                    mma_commit(&aempty[sa]);
                    mma_commit(&bempty[sb]);
                    if (s + 1 == nst) mma_commit(&tfull[0]);
                }
                __syncwarp();
                if (lane == 0) F4_TRACE(5, g);
#ifdef SSBH_EXP_TRACE
                ++g;
#endif
                if (++sa == kLfAS) {
                    sa = 0;
                    pa ^= 1;
                }
                if (++sb == kLfBS) {
                    sb = 0;
                    pb ^= 1;
                }
            }
        }
    } else if (warp == kLfLoadW) {
        // ---------------------------------------------------------------- B loader
        uint32_t sb = 0, pb = 1;  // waits for the slot's previous use: phase of (use - 1)
        uint32_t g = 0;
        StageIt cur;
        for (cur.start(a); cur.w.valid; cur.next(a), ++g) {
            if (g >= (uint32_t)kLfBS) F4_WAIT_S(&bempty[sb], pb);
            if (lane == 0) F4_TRACE(2, g);
            if (elect_one()) {
                const uint64_t G0 = (uint64_t)cur.w.d.nt * kN +
                                    (uint64_t)(cur.w.d.st0 + cur.s) * kF4StageK;
                mbar_arrive_expect_tx(&bfull[sb], kLfTileBytes);
                bulk_g2s(bslots + (size_t)sb * kF4Slot, a.units + (cur.w.d.uoff + G0) * 4,
                         kLfTileBytes, &bfull[sb]);
            }
            __syncwarp();
            if (lane == 0) F4_TRACE(3, g);
            if (++sb == kLfBS) {
                sb = 0;
                pb ^= 1;
            }
        }
    } else if (warp >= kLfBuild0) {
        // ---------------------------------------------------------------- background builds
        // Parent mode: the next parent's lo half while R runs (free once the A warps are
        // through P), its hi half while its Q runs (free once they are through the previous R).
        // Driven by the half barriers alone.
#ifndef SSBH_EXP_NOBUILD
        if (a.leaf == 2) {
            const uint32_t row0 = (warp - kLfBuild0) * kLfBRows;
            const uint32_t row1 = row0 + kLfBRows < (uint32_t)kM ? row0 + kLfBRows : (uint32_t)kM;
            // parent mode never runs the foreground build: its offset buffer holds the build
            // warps' piece tables (kLeafPieces / 2 words each)
            uint32_t* woff =
                reinterpret_cast<uint32_t*>(loff) + (warp - kLfBuild0) * (kLeafPieces / 2);
            static_assert(kLfBW * (kLeafPieces / 2) * 4 <= 2 * kLeafPieces * 8, "piece tables");
            uint32_t seq = 0;
#ifdef SSBH_EXP_BSTAT
            long long tb = 0, tw = 0;
#endif
            for (uint32_t sup = blockIdx.x; sup < nsupers; sup += gridDim.x, ++seq) {
#ifdef SSBH_EXP_BSTAT
                long long c0 = clock64();
#endif
                if (seq) F4_WAIT_T(lo_free, (seq - 1) & 1);
#ifdef SSBH_EXP_BSTAT
                long long c1 = clock64();
                tw += c1 - c0;
#endif
                build_half_rows(a, sup, 0, row0, row1, lane, lraw, woff);
                __syncwarp();
                if (lane == 0) mbar_arrive(lo_ready);
#ifdef SSBH_EXP_BSTAT
                c0 = clock64();
                tb += c0 - c1;
#endif
                if (seq) F4_WAIT_T(hi_free, (seq - 1) & 1);
#ifdef SSBH_EXP_BSTAT
                c1 = clock64();
                tw += c1 - c0;
#endif
                build_half_rows(a, sup, 1, row0, row1, lane, lraw, woff);
                __syncwarp();
                if (lane == 0) mbar_arrive(hi_ready);
#ifdef SSBH_EXP_BSTAT
                tb += clock64() - c1;
#endif
            }
#ifdef SSBH_EXP_BSTAT
            if (lane == 0 && blockIdx.x < 2)
                printf("EXPBSTAT cta %u: supers %u build clk %lld wait-free clk %lld\n",
                       blockIdx.x, seq, tb, tw);
#endif
        }
#endif
    } else {
        // ---------------------------------------------------------------- A producers
        const uint32_t aw = warp - kLfProd0, set = aw >> 2;
        // TMEM lane = block row: a warp reaches the 32 lanes of its sub-partition (warp % 4)
        const uint32_t jl = 32u * (warp & 3) + lane;
        const uint32_t lane_addr = (32u * (warp & 3)) << 16;
        StageIt cur;
        cur.start(a);
        cur.advance(a, set);
        uint32_t built = 0xFFFFFFFFu, nbuilt = 0;           // leaf mode: foreground builds
        uint32_t seq = 0, cur_sup = 0xFFFFFFFFu, cur_ph = 0;  // parent mode: phase hand-shakes
#ifdef SSBH_EXP_BSTAT
        long long exp_wr = 0;
#endif
        const uint32_t* lrow = lraw + (size_t)jl * kLeafStride;
        const uint32_t half = a.src.kpw / 2;  // parent mode: words of the lo half
        for (uint32_t g = set; cur.w.valid; g += kLfSets, cur.advance(a, kLfSets)) {
#ifndef SSBH_EXP_NOBUILD
            if (a.leaf == 2) {
                if (cur.w.sup != cur_sup || cur.w.d.ph != cur_ph) {
                    __syncwarp();
                    if (cur_sup != 0xFFFFFFFFu && lane == 0) {
                        if (cur_ph == 1) mbar_arrive(lo_free);  // through P: lo is not read again
                        if (cur_ph == 2) mbar_arrive(hi_free);  // through R
                    }
                    if (cur.w.sup != cur_sup) {
                        if (cur_sup != 0xFFFFFFFFu) ++seq;
                        cur_sup = cur.w.sup;
                    }
                    cur_ph = cur.w.d.ph;
#ifdef SSBH_EXP_BSTAT
                    const long long c0 = clock64();
#endif
                    if (cur_ph == 0) F4_WAIT_T(lo_ready, seq & 1);
                    if (cur_ph == 1) F4_WAIT_T(hi_ready, seq & 1);
#ifdef SSBH_EXP_BSTAT
                    exp_wr += clock64() - c0;
#endif
                }
            } else if (cur.w.sup != built) {
                leaf_build<kLfAW>(a, cur.w.d, aw, lane, lraw, loff, nbuilt);
                built = cur.w.sup;
                ++nbuilt;
            }
#endif
            uint4 x[4];
            const uint32_t* src = lrow + 16u * cur.s;
            if (a.leaf == 2 && cur.w.d.child != 1) {
                // P = lo ^ hi, R = hi (Q = lo reads the lo half as a leaf would)
                const uint32_t* hi = src + half;
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    uint4 u = *reinterpret_cast<const uint4*>(hi + 4 * h);
                    if (cur.w.d.child == 0) {
                        const uint4 l = *reinterpret_cast<const uint4*>(src + 4 * h);
                        u.x ^= l.x;
                        u.y ^= l.y;
                        u.z ^= l.z;
                        u.w ^= l.w;
                    }
                    x[h] = u;
                }
            } else {
#pragma unroll
                for (int h = 0; h < 4; ++h) x[h] = *reinterpret_cast<const uint4*>(src + 4 * h);
            }
            const uint32_t slot = g % kLfAS;
            if (g >= (uint32_t)kLfAS) F4_WAIT_S(&aempty[slot], ((g / kLfAS) - 1) & 1);
            if (lane == 0 && aw == 0) F4_TRACE(0, g);
#ifndef SSBH_EXP_NOAPROD
            expand_a(x, tmem + lane_addr + kF4ACol0 + 64u * slot);
#else
            (void)x;
#endif
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&afull[slot]);
            if (lane == 0 && aw == 0) F4_TRACE(1, g);
        }
#ifdef SSBH_EXP_BSTAT
        if (lane == 0 && aw == 0 && blockIdx.x < 2)
            printf("EXPBSTAT cta %u: A wait-ready clk %lld\n", blockIdx.x, exp_wr);
#endif
    }

    tc_fence_before();
    __syncthreads();
#ifdef SSBH_EXP_TRACE
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const long long t00 = trace[4 * kTrN];
        for (uint32_t i = 0; i < kTrN; ++i) {
            printf("EXPTRACE %u", kTrG0 + i);
            for (uint32_t r = 0; r < kTrRoles; ++r)
                printf(" %lld", trace[r * kTrN + i] ? trace[r * kTrN + i] - t00 : 0);
            printf("\n");
        }
    }
#endif
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// =========================================================================================
// Per-block seeds: one Toeplitz matrix per block, i.e. one matrix-VECTOR product per block —
// no second block shares the matrix. The product still maps onto the tensor cores by tiling
// both the rows and the input into 128-wide pieces, i = 128 I + r, c = 128 C + t:
//     K[128 I + r] = sum_C sum_t S[128 (I + C) + r + t] y[128 C + t] = sum_C (H_{I+C} y_C)[r]
// with the 128 x 128 Hankel block H_D[r][t] = S[128 D + r + t]. For one D, the same H_D
// multiplies every pair (I, C = D - I): a work item owns a window of 256 row tiles
// I = I0 + n and walks D; each D step is one 128 x 256 x 128 u8 MMA
//     acc[r][n] += sum_t H_D[r][t] * Y[n][t],   Y[n] = y chunk D - I0 - n (zero outside)
// accumulated in TMEM over all D, so the work is exactly k * n_j MACs plus the ramp of the
// window (< 3 % at config 4). Operands (K order within a 128-position chunk as in the shared
// kernel: byte (kc, w, b) = position kc + 8b + 32w):
//   A = H_D: 136 Hankel units of 16 B in shared memory (unit u word w = seed window at bit
//       128 D + u + 32 w), LBO 16 B, SBO 128 B — generated per D step.
//   B = Y:   column n's chunk moves by one each D step, so the y chunks are laid out in
//       REVERSE order in a shared buffer of 8 K-chunk planes x 512 units (unit (kc, P) =
//       chunk Ctop - P, word w = (y word (4C + w) >> kc) & 0x01010101): column n of step D is
//       unit P = (D's start) + n, i.e. rows 16 B apart (SBO 128 B), planes 8 KB apart (LBO),
//       and stepping D moves the descriptor's start address back by 16 B. One buffer serves
//       256 D steps (511 chunks); two alternate.
// Epilogue: lane = row r, registers = 32 row tiles n -> one __ballot_sync per tile gives the
// key word of rows 128 (I0 + n) + 32 e .. + 31.
constexpr int kPbWin = 256;                  // row tiles per work item (accumulator columns)
constexpr int kPbL = 256;                    // D steps per y buffer
constexpr int kPbUnits = 512;                // units per K-chunk plane of a y buffer
constexpr int kPbHStages = 8;                // Hankel stages in flight
constexpr int kPbThreads = 13 * 32;          // 4 epilogue, 1 MMA, 4 y, 4 Hankel warps
constexpr int kPbEpiWarps = 4, kPbMmaWarp = 4, kPbProdWarp0 = 5;
// kind::i8, M = 128, N = 256 (same instruction descriptor as the shared kernel)

struct PbItem {
    uint32_t jj, I0, ncols;   // block, first row tile, valid row tiles in the window
    uint32_t nD;              // D steps of this item: [s0, s0 + nD) of the window's ncols + nC - 1
    uint32_t nC;              // y chunks of 128 positions
    uint32_t s0;              // first D step (a multiple of kPbL)
    uint32_t nmma;            // MMA N: ncols rounded up to 16 (FP4), 256 (u8)
};

// item = ((block * nwin) + window) * nparts + part
__device__ __forceinline__ bool pb_decode(const PbHashArgs& a, uint32_t item, PbItem& d) {
    if (item >= a.items) return false;
    const uint32_t part = item % a.nparts;
    const uint32_t bw = item / a.nparts;
    d.jj = bw / a.nwin;
    const uint32_t w = bw - d.jj * a.nwin;
    d.I0 = w * kPbWin;
    d.ncols = min((uint32_t)kPbWin, a.ntiles - d.I0);
    d.nmma = (d.ncols + 15) & ~15u;
    d.nC = a.lay.ypad[d.jj] / 4;
    const uint32_t total = d.nC ? d.ncols + d.nC - 1 : 0;
    d.s0 = part * a.part_steps;
    const uint32_t end = part + 1 == a.nparts ? total : min(total, d.s0 + a.part_steps);
    d.nD = end > d.s0 ? end - d.s0 : 0;
    return true;
}

// FP4 operands (kind::mxf4, E2M1 0 / 1.0, unit scales): a D step is 2 MMAs of K = 64; the y
// buffer has 4 K-chunk planes (position kc + 4i + 32w of the 128-chunk, word w =
// ((y word >> kc) << 1) & 0x22222222) and the Hankel unit u word w = (S' window at bit
// 128 D + u + 32 w) & 0x22222222. TMEM: one f32 accumulator + the constant scale factors; the
// f32 counts are exact below 2^24, so longer rows of D steps accumulate in rounds of 2^17 steps
// whose parities are XORed. A pipeline stage is kSD consecutive D steps: H_{D+1} is H_D shifted
// by 128 units, so 128 kSD + 8 units cover all of them and the per-stage barrier work is
// amortised (round 1: 8 steps per stage 144.6 -> 137.6 ms at config 3 against 4).
struct PbGeo {
    static constexpr int planes = 4;               // K-chunk planes of a y buffer
    static constexpr int mmas = 2;                 // MMAs per D step (K = 128 positions)
    static constexpr int sd = 8;                   // D steps per stage
    static constexpr int hunits = 128 * sd + 8;
    static constexpr int hbytes = hunits * 16;
    static constexpr int ybytes = planes * kPbUnits * 16;
    static constexpr size_t bar = 2 * (size_t)ybytes + (size_t)kPbHStages * hbytes;
    static constexpr size_t smem = bar + (2 * kPbHStages + 8) * 8 + 16;
    static_assert(kPbL % sd == 0, "stages must not straddle y buffers");
};
constexpr uint32_t kPbF4MaxSteps = (1u << 24) / 128;  // D steps per f32-exact round

__global__ void __launch_bounds__(kPbThreads, 1) k_toeplitz_mma_pb(PbHashArgs a) {
    using G = PbGeo;
    constexpr uint32_t kRound = kPbF4MaxSteps;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* ybufs = smem;                                  // 2 y buffers
    uint8_t* hst = smem + 2 * (size_t)G::ybytes;            // kPbHStages x G::hbytes
    uint64_t* hfull = reinterpret_cast<uint64_t*>(smem + G::bar);
    uint64_t* hempty = hfull + kPbHStages;
    uint64_t* yfull = hempty + kPbHStages;
    uint64_t* yempty = yfull + 2;
    uint64_t* tfull = yempty + 2;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    constexpr uint32_t M2 = 0x22222222u;

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kPbHStages; ++s) {
            mbar_init(&hfull[s], 4);
            mbar_init(&hempty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&yfull[b], 4);
            mbar_init(&yempty[b], 1);
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kPbEpiWarps);
        }
        fence_barrier_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp < kPbEpiWarps) {  // constant scale factors 0x7f = 2^0
        uint32_t v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = 0x7F7F7F7Fu;
        SSBH_TMEM_ST32(tmem + ((warp * 32u) << 16) + kF4SfCol, v);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp < kPbEpiWarps) {
        // ------------------------------------------------------------------ epilogue
        uint32_t t = 0;  // accumulation rounds consumed
        for (uint32_t item = blockIdx.x;; item += gridDim.x) {
            PbItem d;
            if (!pb_decode(a, item, d)) break;
            const uint32_t rounds = d.nD ? (d.nD - 1) / kRound + 1 : 1;
            uint32_t acc[kPbWin / 32];
#pragma unroll
            for (int q = 0; q < kPbWin / 32; ++q) acc[q] = 0;
            for (uint32_t rd = 0; rd < rounds; ++rd, ++t) {
                mbar_wait_sleep(&tfull[0], t & 1);
                tc_fence_after();
                if (d.nD) {
#pragma unroll 1
                    for (int q = 0; q < kPbWin / 32; ++q) {
                        if (32u * q >= d.ncols) break;  // columns past the window's tiles
                        uint32_t v[32];
                        SSBH_TMEM_LD32(tmem + ((warp * 32u) << 16) + 32u * q, v);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        uint32_t mine = 0;
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const uint32_t bit = __float2uint_rz(__uint_as_float(v[e])) & 1u;
                            const uint32_t wd = __ballot_sync(0xffffffffu, bit);
                            if (lane == (uint32_t)e) mine = wd;
                        }
                        acc[q] ^= mine;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[0]);
            }
            if (d.nD) {
                uint32_t* dst = a.out + (unsigned long long)d.jj * a.out_stride;
#pragma unroll 1
                for (int q = 0; q < kPbWin / 32; ++q) {
                    const uint32_t n = 32u * q + lane;
                    const uint32_t word = 4u * (d.I0 + n) + warp;  // rows 128 I + 32 warp ..
                    if (n < d.ncols && word < a.kw) {
                        if (a.nparts == 1) dst[word] = acc[q];
                        else if (acc[q]) atomicXor(dst + word, acc[q]);  // D parts: XOR
                    }
                }
            }
        }
    } else if (warp == kPbMmaWarp) {
        // ------------------------------------------------------------------ MMA issuer
        uint32_t hs = 0, yb = 0, t = 0;
        const uint32_t ybase = smem_u32(ybufs), hbase = smem_u32(hst);
        for (uint32_t item = blockIdx.x;; item += gridDim.x) {
            PbItem d;
            if (!pb_decode(a, item, d)) break;
            if (d.nD == 0) {
                if (t >= 1) mbar_wait_sleep(&tempty[0], (t - 1) & 1);
                if (lane == 0) mbar_arrive(&tfull[0]);
                ++t;
                continue;
            }
            uint32_t round_end = 0;
            // D0: D step relative to the item's first step d.s0
            for (uint32_t D0 = 0; D0 < d.nD; D0 += kPbL, ++yb) {
                if (D0 % kRound == 0) {  // a new accumulation round (kRound is a multiple of kPbL)
                    if (t >= 1) mbar_wait_sleep(&tempty[0], (t - 1) & 1);
                    tc_fence_after();
                    round_end = min(d.nD, D0 + kRound);
                }
                const uint32_t b = yb & 1;
                mbar_wait(&yfull[b], (yb >> 1) & 1);
                tc_fence_after();
                const uint32_t steps = min((uint32_t)kPbL, d.nD - D0);
                for (uint32_t sb = 0; sb < steps; sb += G::sd, ++hs) {
                    const uint32_t slot = hs % kPbHStages;
                    mbar_wait(&hfull[slot], (hs / kPbHStages) & 1);
                    tc_fence_after();
                    const uint32_t nst = min((uint32_t)G::sd, steps - sb);
                    if (elect_one()) {
                        const uint32_t ha = hbase + slot * G::hbytes;
                        for (uint32_t j = 0; j < nst; ++j) {
                            const uint32_t s = sb + j;
                            // column n of step D0+s is unit (kPbL - 1 - s) + n of the buffer;
                            // H of step j of the stage starts at unit 128 j
                            const uint32_t first = (D0 % kRound) | s;
                            // Only the columns whose y chunk D - n lies inside the block carry
                            // products: n in [D - nC + 1, D]. The window's ramps (255 of its
                            // ncols + nC - 1 steps each way) run as narrower MMAs on that column
                            // range (16-column granularity; an MMA's time falls with N: 87 clocks
                            // at N = 128 against 128 at N = 256). The round's first step stays
                            // full width: it initialises every accumulator column.
                            uint32_t c_lo = 0, c_hi = d.nmma;
                            if (first != 0) {
                                const uint32_t dabs = d.s0 + D0 + s;
                                c_lo = (dabs + 1 > d.nC ? dabs + 1 - d.nC : 0u) & ~15u;
                                c_hi = (min(d.ncols, dabs + 1) + 15u) & ~15u;
                            }
                            const uint32_t idesc_n = f4_idesc(c_hi - c_lo);
                            const uint32_t ya =
                                ybase + b * G::ybytes + 16u * (kPbL - 1 - s) + 16u * c_lo;
#pragma unroll
                            for (int m = 0; m < G::mmas; ++m) {
                                const uint64_t adesc = sdesc(ha + 2048u * j + 32u * m, 16, 128);
                                const uint64_t bdesc = sdesc(ya + 2u * m * (kPbUnits * 16), kPbUnits * 16, 128);
                                mma_f4n(tmem + c_lo, adesc, bdesc, idesc_n, tmem + kF4SfCol,
                                        (first | (uint32_t)m) != 0);
                            }
                        }
                        mma_commit(&hempty[slot]);
                        if (sb + nst == steps) mma_commit(&yempty[b]);
                        if (D0 + sb + nst == round_end) mma_commit(&tfull[0]);
                    }
                    __syncwarp();
                }
                if (D0 + steps == round_end) ++t;
            }
        }
    } else if (warp < kPbProdWarp0 + 4) {
        // ------------------------------------------------------------------ y buffers
        const uint32_t yt = threadIdx.x - kPbProdWarp0 * 32;  // 0..127
        uint32_t yb = 0;
        for (uint32_t item = blockIdx.x;; item += gridDim.x) {
            PbItem d;
            if (!pb_decode(a, item, d)) break;
            const uint32_t* y = a.ybuf + a.lay.yoff[d.jj];
            const uint32_t nunits = kPbL - 1 + d.nmma;  // units the buffer's MMAs read
            for (uint32_t D0 = d.s0; D0 < d.s0 + d.nD; D0 += kPbL, ++yb) {
                const uint32_t b = yb & 1;
                if (yb >= 2) mbar_wait_sleep(&yempty[b], ((yb >> 1) - 1) & 1);
                uint8_t* buf = ybufs + b * G::ybytes;
                // unit P holds chunk C = D0 + kPbL - 1 - P (the buffer's D steps D0 .. +255
                // read units kPbL - 1 - s + n, n < 256)
#pragma unroll 1
                for (uint32_t P = yt; P < nunits; P += 128) {
                    const int64_t C = (int64_t)D0 + kPbL - 1 - P;
                    uint4 x = make_uint4(0, 0, 0, 0);
                    if (C >= 0 && C < (int64_t)d.nC) x = __ldg(reinterpret_cast<const uint4*>(y) + C);
#pragma unroll
                    for (int kc = 0; kc < G::planes; ++kc) {
                        auto f = [&](uint32_t v) { return (kc ? v >> (kc - 1) : v << 1) & M2; };
                        *reinterpret_cast<uint4*>(buf + (kc * kPbUnits + P) * 16) =
                            make_uint4(f(x.x), f(x.y), f(x.z), f(x.w));
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&yfull[b]);
            }
        }
    } else {
        // ------------------------------------------------------------------ Hankel units
        const uint32_t ht = threadIdx.x - (kPbProdWarp0 + 4) * 32;  // 0..127
        uint32_t hs = 0;
        for (uint32_t item = blockIdx.x;; item += gridDim.x) {
            PbItem d;
            if (!pb_decode(a, item, d)) break;
            const uint32_t* sw = a.sbuf + a.lay.soff[d.jj];  // pre-shifted: S'[b + 1] = S[b]
            // stages never straddle y buffers: kSD steps from every multiple of kSD
            for (uint32_t s = 0; s < d.nD; s += G::sd, ++hs) {
                const uint32_t slot = hs % kPbHStages;
                if (hs >= (uint32_t)kPbHStages)
                    mbar_wait_sleep(&hempty[slot], ((hs / kPbHStages) - 1) & 1);
                // D = I0 + s0 + s (column n reads chunk C = D - I0 - n)
                const uint64_t wbase = 4ull * (d.I0 + d.s0 + s);  // word of S' bit 128 D
                uint8_t* hsm = hst + slot * G::hbytes;
#pragma unroll
                for (int r = 0; r < (G::hunits + 127) / 128; ++r) {
                    const uint32_t u = ht + 128u * r;
                    if (u < (uint32_t)G::hunits) {
                        // S bit 128D + u + 32w + 4i at bit 4i + 1 (the S' window at the bit)
                        const uint32_t rel = u, q = rel >> 5, sh = rel & 31;
                        const uint32_t mk = M2;
                        const uint32_t* p = sw + wbase + q;
                        const uint32_t w0 = __ldg(p), w1 = __ldg(p + 1), w2 = __ldg(p + 2),
                                       w3 = __ldg(p + 3), w4 = __ldg(p + 4);
                        *reinterpret_cast<uint4*>(hsm + 16 * u) = make_uint4(
                            __funnelshift_r(w0, w1, sh) & mk, __funnelshift_r(w1, w2, sh) & mk,
                            __funnelshift_r(w2, w3, sh) & mk, __funnelshift_r(w3, w4, sh) & mk);
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&hfull[slot]);
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// Per M tile: the largest padded y length (u32 words) of its owned blocks.
__global__ void k_mma_tiles(const uint32_t* __restrict__ ypad, uint32_t nown,
                            uint32_t* __restrict__ mt_words) {
    const uint32_t jj = blockIdx.x * kM + threadIdx.x;
    uint32_t v = jj < nown ? ypad[jj] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    __shared__ uint32_t wmax[kM / 32];
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t m = 0;
        for (int w = 0; w < kM / 32; ++w) m = max(m, wmax[w]);
        mt_words[blockIdx.x] = m;
    }
}

}  // namespace

uint32_t mma_mtiles(uint32_t nown) { return (nown + kM - 1) / kM; }

MmaGeom make_mma_geom(uint32_t nown, uint32_t kw, uint64_t mean_nj, int device) {
    MmaGeom g{};
    g.mtiles = mma_mtiles(nown);
    g.ntiles = (kw + kN / 32 - 1) / (kN / 32);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    g.grid = sms;
    // K split: the smallest split whose item count leaves the last wave >= 90 % full (or gives
    // >= 8 waves), keeping >= 8 stages per part (FP4 stages are 512 positions)
    const uint64_t stage_bits = kF4StageK;
    const uint64_t mean_stages = std::max<uint64_t>(1, (mean_nj + stage_bits - 1) / stage_bits);
    const uint64_t base = (uint64_t)g.mtiles * g.ntiles;
    g.ksplit = 1;
    for (uint32_t ks = 1; ks <= 16; ++ks) {
        if (ks > 1 && mean_stages / ks < 8) break;
        g.ksplit = ks;
        const uint64_t items = base * ks, waves = (items + sms - 1) / sms;
        if (waves >= 8 || (double)items / (double)(waves * sms) >= 0.9) break;
    }
    g.items = base * g.ksplit;
    return g;
}

MmaGeom make_leaf_geom(uint32_t nvirt, uint32_t lw, int device, bool parent) {
    MmaGeom g{};
    if (parent) {  // one K part; the parent's 2 lw words per row fit the leaf buffer
        g.mtiles = mma_mtiles(nvirt);
        g.ntiles = (lw + kN / 32 - 1) / (kN / 32);
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        g.grid = sms;
        g.ksplit = 1;
        g.items = (uint64_t)g.mtiles * g.ntiles;  // = supers * 3 * ntiles
        return g;
    }
    g.mtiles = mma_mtiles(nvirt);
    g.ntiles = (lw + kN / 32 - 1) / (kN / 32);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    g.grid = sms;
    g.ksplit = (lw + kLeafKpw - 1) / kLeafKpw;  // K parts held in shared memory one at a time
    g.items = (uint64_t)g.mtiles * g.ksplit * g.ntiles;
    return g;
}

PbGeom make_pb_geom(uint32_t nown, uint32_t kw, int device, uint64_t mean_bits) {
    PbGeom g{};
    g.ntiles = (kw + 3) / 4;  // 128-row tiles
    g.nwin = (g.ntiles + kPbWin - 1) / kPbWin;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    g.grid = sms;
    g.nparts = 1;
    g.part_steps = 0xFFFFFFFFu;
    const uint64_t bw = (uint64_t)nown * g.nwin;
    if (mean_bits && bw < (uint64_t)sms) {
        // few (block, window) items: split each one's D steps into parts of >= 1024 steps
        // (4 y buffers) so that ~one wave of items covers the grid
        const uint64_t steps = std::min<uint64_t>(g.ntiles, kPbWin) + mean_bits / 128;
        const uint64_t want = ((uint64_t)sms + bw - 1) / bw;
        const uint64_t maxp = std::max<uint64_t>(1, steps / 1024);
        g.nparts = (uint32_t)std::min<uint64_t>(want, maxp);
        if (g.nparts > 1) {
            const uint64_t ps = (steps + g.nparts - 1) / g.nparts;
            g.part_steps = (uint32_t)((ps + kPbL - 1) / kPbL * kPbL);
        }
    }
    g.items = bw * g.nparts;
    return g;
}

void launch_hash_mma_pb(const PbHashArgs& a0, const PbGeom& g, cudaStream_t st) {
    if (!a0.nown || !g.items) return;
    PbHashArgs a = a0;
    a.nparts = g.nparts;
    a.part_steps = g.part_steps;
    a.items = g.items;
    if (g.nparts > 1)  // the parts XOR into the output rows
        cudaMemset2DAsync(a.out, a.out_stride * 4, 0, (size_t)a.kw * 4, a.nown, st);
    const unsigned grid = (unsigned)std::min<uint64_t>(g.grid, g.items);
    cudaFuncSetAttribute(k_toeplitz_mma_pb, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)PbGeo::smem);
    k_toeplitz_mma_pb<<<grid, kPbThreads, PbGeo::smem, st>>>(a);
}

void launch_hankel_units(const uint32_t* d_vs, uint64_t seed_words, uint64_t regions,
                         uint64_t unit_stride, uint32_t* d_units, cudaStream_t st) {
    if (!regions) return;
    const unsigned gx = (unsigned)std::min<uint64_t>((unit_stride + 255) / 256, 64);
    for (uint64_t r0 = 0; r0 < regions; r0 += 65535) {
        const unsigned gy = (unsigned)std::min<uint64_t>(regions - r0, 65535);
        k_hankel_units<<<dim3(gx, gy), 256, 0, st>>>(
            d_vs + r0 * seed_words, seed_words, unit_stride,
            reinterpret_cast<uint4*>(d_units) + r0 * unit_stride);
    }
}

void launch_hash_mma(const MmaHashArgs& a0, const MmaGeom& g, cudaStream_t st) {
    if (!a0.nown || !g.items) return;
    k_mma_tiles<<<g.mtiles, kM, 0, st>>>(a0.lay.ypad, a0.nown, a0.mt_words);
    const unsigned grid = (unsigned)std::min<uint64_t>(g.grid, g.items);
    MmaHashArgs a = a0;
    a.stage_bits = kF4StageK;
    if (a.leaf) {  // super-items of N tiles (x3 children in parent mode); one wave of CTAs
        const uint64_t supers = g.items / (a.leaf == 2 ? 3ull * a.ntiles : a.ntiles);
        cudaFuncSetAttribute(k_leaf_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kLfSmem);
#ifdef SSBH_EXP_TRACE
        const size_t lsm = kLfSmem + 8 * kTrRoles * kTrN;
        cudaFuncSetAttribute(k_leaf_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm);
        k_leaf_gemm<<<(unsigned)std::min<uint64_t>(g.grid, supers), kLfThreads, lsm, st>>>(a);
#else
        k_leaf_gemm<<<(unsigned)std::min<uint64_t>(g.grid, supers), kLfThreads, kLfSmem, st>>>(a);
#endif
        return;
    }
    const size_t smem = f4_smem(kSets);
    cudaFuncSetAttribute(k_toeplitz_f4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_toeplitz_f4<<<grid, kF4Threads, smem, st>>>(a);
}

}  // namespace ssbh_impl
