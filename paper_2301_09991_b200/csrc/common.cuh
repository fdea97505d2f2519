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
// same with an already converted 32-bit shared-space address
template <int BYTES>
__device__ __forceinline__ void cp_async_s(unsigned saddr, const void* gmem, bool valid) {
    const int n = valid ? BYTES : 0;
    if (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
                     "r"(n)
                     : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(saddr), "l"(gmem),
                     "n"(BYTES), "r"(n)
                     : "memory");
}

// Row stager of the y-marching stencil kernels.  A staged row holds up to 4 fields x
// W cells x CC channels (smem layout [field][cell][channel]).  An item is one
// (cell, VEC-channel group) and stages that vector of every field, so the thread
// that owns an item can post-process it (psi - delta, the EMA) right after its own
// copies land.  Everything row independent — shared address, x resolution of the
// vacuum rule, the field pointer at (x, y = 0) — is computed once; per row only the
// y rule, one multiply per field kind and an address add per field remain.
//   kind 0 field (psi-like): vacuum rule (zero on incoming sides, else clamp);
//   kind 1 field (k-like):   stored on the +-band, zero outside it, never clamped.
// KMASK bit f = kind of field f.
struct FieldDesc {
    const void* ptr;   // nullptr: field reads as 0
    int halo;
    int xlo = -(1 << 30), xhi = 1 << 30;   // stage only cells with xlo <= x < xhi
};

template <class Real, int VEC, int NI, int NF, int KMASK, int CC = 32>
struct Stager {
    const Real* base[NI][NF];   // field pointer at (x storage, y = 0), nullptr = zero in x
    unsigned soff[NI];          // shared byte offset of the item (field 0, buffer 0)
    bool npos[NI];
    bool item[NI];
    int ny, C, band;

    __device__ __forceinline__ void init(const Geo& g, const FieldDesc* fd, int x0, int W,
                                         int c0, int band_, const Real* mu, const Real* nu,
                                         int tid, int nthreads) {
        constexpr int G4 = CC / VEC;
        ny = g.ny; C = g.C; band = band_;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int e = tid + i * nthreads;
            const bool has = e < W * G4;
            item[i] = has;
            const int xi = has ? e / G4 : 0, q = has ? e % G4 : 0;
            const int c = c0 + q * VEC;
            const bool cval = has && c < g.C;
            const int n = (cval ? c : 0) / g.ng;
            const bool mp = mu[n] > Real(0);
            npos[i] = nu[n] > Real(0);
            soff[i] = (unsigned)((xi * CC + q * VEC) * sizeof(Real));
            const int xg = x0 + xi;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                bool z = !cval || fd[f].ptr == nullptr || xg < fd[f].xlo || xg >= fd[f].xhi;
                int xr = xg;
                if (!((KMASK >> f) & 1)) {
                    if (xr < 0) { if (!g.ghost_w) { z |= mp; xr = 0; } }
                    else if (xr >= g.nx) { if (!g.ghost_e) { z |= !mp; xr = g.nx - 1; } }
                } else {
                    z |= xg < -band || xg >= g.nx + band;
                }
                const int h = fd[f].halo;
                base[i][f] = z ? nullptr
                               : (const Real*)fd[f].ptr +
                                     ((int64_t)(xr + h) * (g.ny + 2 * h) + h) * (int64_t)g.C + c;
            }
        }
    }

    // stage row yy into the buffer at shared address sbuf (field stride fstride bytes)
    __device__ __forceinline__ void issue(int yy, unsigned sbuf, unsigned fstride,
                                          const Real* dummy) const {
        const bool yz1 = yy < -band || yy >= ny + band;
        const int off1 = yy * C;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            if (!item[i]) continue;
            bool yz0 = false;
            int yr = yy;
            if (yr < 0) { yz0 = npos[i]; yr = 0; }
            else if (yr >= ny) { yz0 = !npos[i]; yr = ny - 1; }
            const int off0 = yr * C;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const bool k1 = (KMASK >> f) & 1;
                const bool z = base[i][f] == nullptr || (k1 ? yz1 : yz0);
                const Real* src = z ? dummy : base[i][f] + (k1 ? off1 : off0);
                cp_async_s<VEC * (int)sizeof(Real)>(sbuf + f * fstride + soff[i], src, !z);
            }
        }
    }
};

}  // namespace csn
namespace csn {
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// iterate average pbar' = (1 - theta) pbar + theta psi (R/multigrid.py:217-225) with a
// fixed contraction, so every kernel that forms it rounds identically
__device__ __forceinline__ float ema_rn(float b, float p, float omt, float th) {
    return __fmaf_rn(b, omt, __fmul_rn(th, p));
}
__device__ __forceinline__ double ema_rn(double b, double p, double omt, double th) {
    return __fma_rn(b, omt, __dmul_rn(th, p));
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
