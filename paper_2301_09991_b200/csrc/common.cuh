// Shared device helpers: geometry, vacuum-rule loads, deterministic reductions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "convsn_sm100.h"

namespace csn {

struct Geo {
    int nx, ny, nd, ng, C, na;
    int ghost_w, ghost_e;
};

inline Geo make_geo(const csn_geom& g) {
    Geo d;
    d.nx = g.nx; d.ny = g.ny; d.nd = g.nd; d.ng = g.ng; d.C = g.nd * g.ng; d.na = g.na;
    d.ghost_w = g.ghost_w; d.ghost_e = g.ghost_e;
    return d;
}

// Storage offset of (x, y, c) in a field with halo h (R/grid.py:47-59 layout).
__device__ __forceinline__ int64_t fidx(int x, int y, int c, int ny, int h, int C) {
    return ((int64_t)(x + h) * (ny + 2 * h) + (y + h)) * (int64_t)C + c;
}

// Vacuum rule of R/grid.py:165-190 in its stateless form: a position outside the
// domain reads 0 if the direction enters through any side it is out on, else the
// nearest interior value.  Ghost x sides (domain decomposition) keep x as is.
// Returns false for a zero; otherwise (x, y) is rewritten to the storage position.
__device__ __forceinline__ bool resolve_vac(int& x, int& y, const Geo& g, bool mpos, bool npos) {
    if (x < 0) {
        if (!g.ghost_w) { if (mpos) return false; x = 0; }
    } else if (x >= g.nx) {
        if (!g.ghost_e) { if (!mpos) return false; x = g.nx - 1; }
    }
    if (y < 0) {
        if (npos) return false;
        y = 0;
    } else if (y >= g.ny) {
        if (!npos) return false;
        y = g.ny - 1;
    }
    return true;
}

template <class Real>
__device__ __forceinline__ Real ldg(const Real* p) { return __ldg(p); }

// Ampere+ async global->shared copy of one element (LDGSTS); src-size 0 zero-fills,
// which is how the vacuum rule's zero halo is staged without a branch in smem.
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? BYTES : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem),
                 "n"(BYTES), "r"(n)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// NaN-propagating min (numpy.minimum semantics, R/discretisation.py:150-158).
template <class Real>
__device__ __forceinline__ Real nanmin(Real a, Real b) {
    if (a != a) return a;
    if (b != b) return b;
    return a < b ? a : b;
}

template <class Real>
__device__ __forceinline__ bool finite(Real v) { return isfinite(v); }

// Block-wide fp64 sum; result valid in thread 0.  Fixed tree => deterministic.
__device__ __forceinline__ double block_sum(double v, double* sh /* >= 32 */) {
    const int lane = threadIdx.x + blockDim.x * threadIdx.y;
    const int tid = lane;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int nwarps = (blockDim.x * blockDim.y * blockDim.z + 31) / 32;
    if ((tid & 31) == 0) sh[tid >> 5] = v;
    __syncthreads();
    if (tid < 32) {
        v = tid < nwarps ? sh[tid] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    return v;
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace csn

namespace csn {
// kernels launched by this library since load (read by csn_launch_count)
extern unsigned long long g_launches;
}

// after EVERY kernel launch, exactly once: count it and surface launch errors
#define CSN_CHECK_LAUNCH()                                   \
    do {                                                     \
        ++csn::g_launches;                                   \
        cudaError_t e__ = cudaGetLastError();                \
        if (e__ != cudaSuccess) return -(int)e__;            \
    } while (0)
