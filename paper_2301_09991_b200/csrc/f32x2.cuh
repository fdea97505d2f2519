// Packed fp32x2 arithmetic (sm_100a FFMA2 / FMUL2 / FADD2).
//
// The PG stencil kernels are issue-bound, not FMA-pipe bound: every tap is one FFMA
// per channel.  Blackwell's packed .f32x2 instructions apply one FMA to two fp32 lanes
// per issue slot with the same per-lane IEEE rounding as scalar fmaf (measured on
// B200: 128 lane-FMA/clk/SM for both forms, so half the issue slots).  A thread that
// owns a channel pair therefore halves the issue cost of the tap arithmetic; constant
// taps broadcast as (t, t) are folded by ptxas into the instruction's immediate.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace csn {

__device__ __forceinline__ uint64_t f2u(float2 v) {
    return (uint64_t)__float_as_uint(v.x) | ((uint64_t)__float_as_uint(v.y) << 32);
}
__device__ __forceinline__ float2 u2f(uint64_t u) {
    return make_float2(__uint_as_float((unsigned)u), __uint_as_float((unsigned)(u >> 32)));
}
__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }

// a * b + c
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(d);
}
// t * b + c with a compile-time tap t (immediate operand)
__device__ __forceinline__ float2 fma2c(float t, float2 b, float2 c) { return fma2(bc2(t), b, c); }

__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}

__device__ __forceinline__ float2 ld2(const float* p) {
    return *reinterpret_cast<const float2*>(p);
}
__device__ __forceinline__ void st2(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }

}  // namespace csn
