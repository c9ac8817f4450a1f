// diag.cu — roofline denominator: measured LOP3 issue rate of this GPU.
//
// MEASURED_PEAKS.json holds only HBM and bf16 tensor peaks, so the integer-ALU peak the
// hash kernel is judged against is measured live: every SM runs independent
// acc ^= a & b chains (each one LOP3.LUT 0x78, the hash kernel's inner instruction) at
// full occupancy, timed with CUDA events.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ssbh_cuda.h"

namespace {

__global__ void __launch_bounds__(256) k_lop3_peak(uint32_t iters, uint32_t* out) {
    uint32_t a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = (threadIdx.x + 1) * 0x9E3779B9u + j * 0x85EBCA6Bu;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] ^= a[(j + 3) & 15] & a[(j + 7) & 15];
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) x ^= a[j];
    if (x == 0x12345678u) out[blockIdx.x] = x;  // keep the chains live
}

// Block-scaled FP4 probe (kind::mxf4, E2M1 operands, every UE8M0 scale = 1.0): rate of
// 128x256x64 MMAs and exactness of the f32 accumulation of integer sums. mode 0: A and B all
// 1.0 (rate); mode 1: A all 1.0, B one 1.0 per row, so every MMA adds exactly 1 and the
// accumulator must read `iters` (checked per element, mismatches counted into *bad).
__global__ void __launch_bounds__(128, 1) k_f4_probe(uint32_t iters, int mode, uint32_t* bad) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef SSBH_EXP_CLOCK
    const long long exp_c0 = clock64();
    unsigned long long exp_t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(exp_t0));
#endif
    uint32_t* w = reinterpret_cast<uint32_t*>(smem);
    if (mode >= 2)  // hash-kernel layouts / K96 tiles: fill the first 44 KB
        for (uint32_t i = threadIdx.x; i < 45056 / 4; i += blockDim.x) w[i] = 0x22222222u;
    for (uint32_t i = threadIdx.x; i < 4096 / 4; i += blockDim.x) w[i] = 0x22222222u;  // A
    for (uint32_t i = threadIdx.x; mode < 2 && i < 8192 / 4; i += blockDim.x) {
        // B: row n occupies bytes (n%8)*16 + (n/8)*256 + kc*128 (kc = 0, 1); one 1.0 per row
        uint32_t v = 0x22222222u;
        if (mode == 1) {
            const uint32_t byte = i * 4, kc = (byte >> 7) & 1, inrow = byte & 15;
            v = (kc == 0 && inrow == 0) ? 0x00000002u : 0u;
        }
        w[1024 + i] = v;
    }
    const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    {   // scale factors: columns 256..287 of every lane = 0x7f (UE8M0 2^0)
        const uint32_t v = 0x7F7F7F7Fu;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
            "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                tmem + ((32u * warp) << 16) + 256u),
            "r"(v)
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
        // mode 3: the K = 96 form of kind::mxf4 (instruction descriptor bit 31), rate only
        const uint32_t idesc = (1u << 7) | (1u << 10) | (32u << 17) | (1u << 23) | (8u << 24) |
                               (mode == 3 ? (1u << 31) : 0u);
        auto desc = [](uint32_t a, uint32_t lbo, uint32_t sbo) {
            return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
                   ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
        };
        for (uint32_t it = 0; it < iters; ++it) {
            const uint32_t m = it & 7;
            const uint64_t a = mode == 2 ? desc(base + 256u * m, 128, 2048)
                               : mode == 3 ? desc(base, 128, 384) : desc(base, 128, 256);
            const uint64_t b = mode == 2
                ? desc(base + 32768u + 16u * (2u * (m & 1) + 128u * (m >> 1)), 16, 128)
                : mode == 3 ? desc(base + 8192u, 128, 384) : desc(base + 4096u, 128, 256);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n}\n"
                ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(it), "r"(tmem + 256u),
                "r"(tmem + 264u)
                : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         bar_a)
                     : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nW:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(bar_a)
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (mode == 1) {
        uint32_t nbad = 0;
        for (int q = 0; q < 8; ++q) {
            uint32_t v[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
                "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                  "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                  "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
                  "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                  "=r"(v[30]), "=r"(v[31])
                : "r"(tmem + ((32u * warp) << 16) + 32u * q));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int e = 0; e < 32; ++e) nbad += __uint_as_float(v[e]) != (float)iters;
            if (blockIdx.x == 0 && threadIdx.x == 0 && q == 0) bad[1] = v[0];
        }
        if (nbad) atomicAdd(bad, nbad);
    }
    (void)lane;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
#ifdef SSBH_EXP_CLOCK
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        const long long c1 = clock64();
        printf("EXPCLOCK k_f4_probe mode=%d ns=%llu MHz=%.1f\n", mode, t1 - exp_t0,
               (double)(c1 - exp_c0) * 1e3 / (double)(t1 - exp_t0));
    }
#endif
}


// A operand from TMEM for kind::mxf4 (tcgen05.mma ... [d], [a_tmem], b_desc ...): lane = row of
// A, 8 columns of 32 bits per K = 64 (assumed: column c nibble i = K element 8c + i).
// mode 0: exactness — A all 1.0, B one 1.0 per row (smem element 0 of its row), every MMA adds
//         exactly 1, the accumulator must read `iters`; mismatches counted into *bad.
// mode 1: layout — one MMA; A row r one-hot at its assumed element r % 64, B row n one-hot at
//         smem element n % 64; D (128 x 256 f32) copied to dout for the host to decode.
// mode 2: rate — A all 1.0 from TMEM, B with the hash kernel's Hankel layout, back to back.
__global__ void __launch_bounds__(128, 1) k_f4_tmem_a_probe(uint32_t iters, int mode,
                                                            uint32_t* bad, float* dout) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* w = reinterpret_cast<uint32_t*>(smem);
    for (uint32_t i = threadIdx.x; i < 45056 / 4; i += blockDim.x) w[i] = 0u;
    __syncthreads();
    if (mode >= 2) {
        for (uint32_t i = threadIdx.x; i < 45056 / 4; i += blockDim.x) w[i] = 0x22222222u;
    } else if (threadIdx.x < 128) {
        // B rows n = threadIdx.x and n + 128: row n, element e at byte (n%8)*16 + (n/8)*256 +
        // (e/32)*128 + (e%32)/2, low nibble for even e
        for (int h = 0; h < 2; ++h) {
            const uint32_t n = threadIdx.x + 128u * h;
            const uint32_t e = mode == 0 ? 0u : n % 64u;
            const uint32_t byte = (n % 8) * 16 + (n / 8) * 256 + (e / 32) * 128 + (e % 32) / 2;
            smem[byte] = (uint8_t)((e & 1) ? 0x20 : 0x02);
        }
    }
    const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    {
        // scale factors (columns 256..287) and A (columns 320..327) of this warp's 32 lanes
        const uint32_t v = 0x7F7F7F7Fu;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
            "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                tmem + ((32u * warp) << 16) + 256u),
            "r"(v)
            : "memory");
        const uint32_t r = 32u * warp + lane, e = r % 64u;
        uint32_t a[8];
        for (int c = 0; c < 8; ++c)
            a[c] = mode == 1 ? ((uint32_t)c == e / 8 ? (2u << (4 * (e % 8))) : 0u) : 0x22222222u;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                         tmem + ((32u * warp) << 16) + 320u),
                     "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]),
                     "r"(a[7])
                     : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
        const uint32_t idesc = (1u << 7) | (1u << 10) | (32u << 17) | (1u << 23) | (8u << 24);
        auto desc = [](uint32_t a, uint32_t lbo, uint32_t sbo) {
            return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
                   ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
        };
        const uint32_t n_it = mode == 1 ? 1u : iters;
        // mode 3: rate of N = 128 MMAs alternating between the two halves of the accumulator
        // (columns 0..127 / 128..255, Hankel rows 128 units further)
        const uint32_t idesc128 = (idesc & ~(0x3Fu << 17)) | (16u << 17);
        for (uint32_t it = 0; it < n_it; ++it) {
            const uint32_t m = it & 7;
            const uint32_t h = mode == 3 ? (it >> 3) & 1u : 0u;
            const uint64_t b = mode >= 2
                ? desc(base + 16u * (2u * (m & 1) + 128u * (m >> 1) + 128u * h), 16, 128)
                : desc(base, 128, 256);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%6], p;\n}\n"
                ::"r"(tmem + 128u * h), "r"(tmem + 320u), "l"(b), "r"(mode == 3 ? idesc128 : idesc),
                "r"(it), "r"(tmem + 256u), "r"(tmem + 264u)
                : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         bar_a)
                     : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nW:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(bar_a)
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (mode <= 1) {
        uint32_t nbad = 0;
        for (int q = 0; q < 8; ++q) {
            uint32_t v[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
                "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                  "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                  "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
                  "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                  "=r"(v[30]), "=r"(v[31])
                : "r"(tmem + ((32u * warp) << 16) + 32u * q));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const uint32_t r = 32u * warp + lane;
            for (int e = 0; e < 32; ++e) {
                const uint32_t n = 32u * q + e;
                const float want = mode == 0 ? (float)iters : (r % 64u == n % 64u ? 1.0f : 0.0f);
                nbad += __uint_as_float(v[e]) != want;
                if (mode == 1 && blockIdx.x == 0) dout[r * 256u + n] = __uint_as_float(v[e]);
            }
        }
        if (nbad) atomicAdd(bad, nbad);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}


// CTA-pair (cta_group::2) kind::mxf4 with A from TMEM: M = 256 across the pair (each CTA's TMEM
// lanes = its 128 rows of A and of D), N = 256 with each CTA holding 128 rows of B at the same
// shared-memory offset, the leader issuing. mode 1: layout — A row r (global) one-hot at element
// r % 64, B row n (global) one-hot at element n % 64; D copied to dout (256 x 256).
// mode 2: rate — back-to-back MMAs, B in the Hankel-unit layout of the leaf GEMM's half table.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_f4_pair_probe(uint32_t iters, int mode, uint32_t* bad, float* dout) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    uint32_t* w = reinterpret_cast<uint32_t*>(smem);
    for (uint32_t i = threadIdx.x; i < 45056 / 4; i += blockDim.x) w[i] = mode == 2 ? 0x22222222u : 0u;
    __syncthreads();
    if (mode == 1) {  // B: this CTA's 128 rows, row n local at bytes (n%8)*16 + (n/8)*256 + ...
        const uint32_t nl = threadIdx.x, n = 128u * rank + nl, e = n % 64u;
        const uint32_t byte = (nl % 8) * 16 + (nl / 8) * 256 + (e / 32) * 128 + (e % 32) / 2;
        smem[byte] = (uint8_t)((e & 1) ? 0x20 : 0x02);
    }
    const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    {
        const uint32_t v = 0x7F7F7F7Fu;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
            "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                tmem + ((32u * warp) << 16) + 256u),
            "r"(v)
            : "memory");
        const uint32_t r = 128u * rank + 32u * warp + lane, e = r % 64u;
        uint32_t a[8];
        for (int c = 0; c < 8; ++c)
            a[c] = mode == 1 ? ((uint32_t)c == e / 8 ? (2u << (4 * (e % 8))) : 0u) : 0x22222222u;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                         tmem + ((32u * warp) << 16) + 320u),
                     "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]),
                     "r"(a[7])
                     : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
        // M = 256 (pair), N = 256
        const uint32_t idesc = (1u << 7) | (1u << 10) | (32u << 17) | (1u << 23) | (16u << 24);
        auto desc = [](uint32_t a, uint32_t lbo, uint32_t sbo) {
            return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
                   ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
        };
        const uint32_t n_it = mode == 1 ? 1u : iters;
        for (uint32_t it = 0; it < n_it; ++it) {
            const uint32_t m = it & 7;
            const uint64_t b = mode == 2
                ? desc(base + 16u * (2u * (m & 1) + 128u * (m >> 1)), 16, 128)
                : desc(base, 128, 256);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%6], p;\n}\n"
                ::"r"(tmem), "r"(tmem + 320u), "l"(b), "r"(idesc), "r"(it), "r"(tmem + 256u),
                "r"(tmem + 264u)
                : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                bar_a), "h"((uint16_t)3)
            : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nW:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(bar_a)
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (mode == 1) {
        uint32_t nbad = 0;
        for (int q = 0; q < 8; ++q) {
            uint32_t v[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
                "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                  "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                  "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
                  "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                  "=r"(v[30]), "=r"(v[31])
                : "r"(tmem + ((32u * warp) << 16) + 32u * q));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const uint32_t r = 128u * rank + 32u * warp + lane;
            for (int e = 0; e < 32; ++e) {
                const uint32_t n = 32u * q + e;
                const float want = (r % 64u == n % 64u) ? 1.0f : 0.0f;
                nbad += __uint_as_float(v[e]) != want;
                if (blockIdx.x < 2) dout[r * 256u + n] = __uint_as_float(v[e]);
            }
        }
        if (nbad) atomicAdd(bad, nbad);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

}  // namespace

// FP4 probe: rate (MAC/s) and exactness (modes above; mode 2 = rate with the hash kernel's
// operand layouts, the roofline denominator of k_toeplitz_f4).
extern "C" ssbh_status ssbh_probe_mma_f4(uint32_t iters, int mode, double* macs_per_s,
                                         double* ms_out, uint32_t* mismatches,
                                         uint32_t* sample_bits) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SSBH_NO_DEVICE;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int smem = 120 * 1024;
    cudaFuncSetAttribute(k_f4_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    uint32_t* bad = nullptr;
    if (cudaMalloc(&bad, 8) != cudaSuccess) return SSBH_CUDA;
    cudaMemset(bad, 0, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_f4_probe<<<sms, 128, smem>>>(iters, mode, bad);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    uint32_t hb[2] = {0, 0};
    cudaMemcpy(hb, bad, 8, cudaMemcpyDeviceToHost);
    cudaFree(bad);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (cudaGetLastError() != cudaSuccess) return SSBH_CUDA;
    if (macs_per_s)
        *macs_per_s = (double)sms * iters * 128.0 * 256.0 * (mode == 3 ? 96.0 : 64.0) / (ms * 1e-3);
    if (ms_out) *ms_out = ms;
    if (mismatches) *mismatches = hb[0];
    if (sample_bits) *sample_bits = hb[1];
    return SSBH_OK;
}

extern "C" ssbh_status ssbh_probe_mma_f4_tmem_a(uint32_t iters, int mode, double* macs_per_s,
                                                double* ms_out, uint32_t* mismatches,
                                                float* d_out_host) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SSBH_NO_DEVICE;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int smem = 120 * 1024;
    cudaFuncSetAttribute(k_f4_tmem_a_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    uint32_t* bad = nullptr;
    float* dout = nullptr;
    if (cudaMalloc(&bad, 8) != cudaSuccess) return SSBH_CUDA;
    if (cudaMalloc(&dout, 128 * 256 * 4) != cudaSuccess) return SSBH_CUDA;
    cudaMemset(bad, 0, 8);
    cudaMemset(dout, 0, 128 * 256 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_f4_tmem_a_probe<<<sms, 128, smem>>>(iters, mode, bad, dout);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    uint32_t hb[2] = {0, 0};
    cudaMemcpy(hb, bad, 8, cudaMemcpyDeviceToHost);
    if (d_out_host) cudaMemcpy(d_out_host, dout, 128 * 256 * 4, cudaMemcpyDeviceToHost);
    cudaFree(bad);
    cudaFree(dout);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (cudaGetLastError() != cudaSuccess) return SSBH_CUDA;
    if (macs_per_s)
        *macs_per_s = (double)sms * iters * 128.0 * (mode == 3 ? 128.0 : 256.0) * 64.0 / (ms * 1e-3);
    if (ms_out) *ms_out = ms;
    if (mismatches) *mismatches = hb[0];
    return SSBH_OK;
}

extern "C" ssbh_status ssbh_probe_mma_f4_pair(uint32_t iters, int mode, double* macs_per_s,
                                              double* ms_out, uint32_t* mismatches,
                                              float* d_out_host) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SSBH_NO_DEVICE;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int smem = 120 * 1024;
    cudaFuncSetAttribute(k_f4_pair_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    uint32_t* bad = nullptr;
    float* dout = nullptr;
    if (cudaMalloc(&bad, 8) != cudaSuccess) return SSBH_CUDA;
    if (cudaMalloc(&dout, 256 * 256 * 4) != cudaSuccess) return SSBH_CUDA;
    cudaMemset(bad, 0, 8);
    cudaMemset(dout, 0, 256 * 256 * 4);
    const int grid = sms & ~1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_f4_pair_probe<<<grid, 128, smem>>>(iters, mode, bad, dout);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    uint32_t hb[2] = {0, 0};
    cudaMemcpy(hb, bad, 8, cudaMemcpyDeviceToHost);
    if (d_out_host) cudaMemcpy(d_out_host, dout, 256 * 256 * 4, cudaMemcpyDeviceToHost);
    cudaFree(bad);
    cudaFree(dout);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (cudaGetLastError() != cudaSuccess) return SSBH_CUDA;
    // per pair and MMA: 256 x 256 x 64 MACs
    if (macs_per_s) *macs_per_s = (double)(grid / 2) * iters * 256.0 * 256.0 * 64.0 / (ms * 1e-3);
    if (ms_out) *ms_out = ms;
    if (mismatches) *mismatches = hb[0];
    return SSBH_OK;
}

extern "C" ssbh_status ssbh_measure_mma_f4_peak(uint32_t iters, double* macs_per_s,
                                                double* ms_out) {
    return ssbh_probe_mma_f4(iters, 2, macs_per_s, ms_out, nullptr, nullptr);
}

extern "C" ssbh_status ssbh_measure_lop3_peak(uint32_t iters, double* lop3_per_s, double* ms_out) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SSBH_NO_DEVICE;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lop3_peak, 256, 0);
    const int grid = sms * (per_sm > 0 ? per_sm : 1);
    uint32_t* out = nullptr;
    if (cudaMalloc(&out, grid * 4) != cudaSuccess) return SSBH_CUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_lop3_peak<<<grid, 256>>>(iters / 8 + 1, out);  // warm-up / clock ramp
    cudaEventRecord(e0);
    k_lop3_peak<<<grid, 256>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (cudaGetLastError() != cudaSuccess) return SSBH_CUDA;
    const double ops = (double)grid * 256.0 * iters * 8.0 * 16.0;
    if (lop3_per_s) *lop3_per_s = ops / (ms * 1e-3);
    if (ms_out) *ms_out = ms;
    return SSBH_OK;
}
