// TMA (cp.async.bulk.tensor) and mbarrier helpers shared by the staged kernels.
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace csn {

// suspend-time hint of the mbarrier wait: a waiting warp sleeps in the barrier unit
// instead of re-issuing try_wait / branch pairs that take issue slots from the warps
// doing the stencil arithmetic
#ifndef CSN_MBAR_SUSPEND_NS
#define CSN_MBAR_SUSPEND_NS 0x989680
#endif

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "MBW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra MBW_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity), "r"(CSN_MBAR_SUSPEND_NS)
        : "memory");
}
// the same on 32-bit shared-window addresses computed once per CTA (the generic ->
// shared conversion otherwise costs an S2R + LEA per call inside a hot loop)
__device__ __forceinline__ void mbar_expect_tx_s(unsigned b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_s(unsigned b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait_s(unsigned b, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "MBWS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra MBWS_%=;\n"
        "}\n" ::"r"(b),
        "r"(parity), "r"(CSN_MBAR_SUSPEND_NS)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_s(unsigned dst, const CUtensorMap* map, unsigned bar,
                                              int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_mbarrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

}  // namespace csn
