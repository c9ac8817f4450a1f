// ptx.cuh — thin inline-PTX wrappers for the sm_100a async-copy machinery used by the
// hash kernel: mbarriers (tx-count) and 1-D bulk copies global->shared
// (cp.async.bulk, SASS UBLKCP) completing on an mbarrier.
#pragma once

#include <stdint.h>

namespace ssbh_dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

// Make mbarrier inits visible to the async proxy (TMA / bulk copies).
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Same, but the waiting warp is suspended in hardware (suspend-time hint, in ns) instead of
// spinning: used by the hash kernel's producer warp, which waits ~0.1 ms per work item and
// would otherwise steal issue slots from the compute warps sharing its SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}

// 1-D bulk copy (bytes % 16 == 0, both addresses 16-B aligned), completes tx on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// One thread of the (converged) warp. Unlike `lane == 0`, ptxas knows that an elect.sync region
// has a single active thread and feeds tcgen05.mma / commit their uniform-register operands
// directly; under `if (lane == 0)` it wrapped every MMA in an ELECT / R2UR.BROADCAST / BRA.U.ANY
// loop (17 SASS per MMA, ~115 clocks of issue per 128-clock MMA: the tensor pipe starved).
// Predicated shared-memory OR without a branch around it (reduction form: no return value).
__device__ __forceinline__ void red_or_shared_if(uint32_t addr, uint32_t v, bool p) {
    asm volatile(
        "{\n.reg .pred P;\nsetp.ne.u32 P, %2, 0;\n@P red.shared.or.b32 [%0], %1;\n}\n" ::"r"(addr),
        "r"(v), "r"((uint32_t)p));
}

__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile(
        "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n"
        : "=r"(p));
    return p != 0;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace ssbh_dev

