// Transfers (R/multigrid.py:110-146,342-353), boundary fill (R/grid.py:165-190),
// scalar flux (R/grid.py:193-198), group source / fission (R/eigen.py:117-135),
// generic stencils (R/grid.py:85-162) and small vector utilities.
#pragma once
#include "common.cuh"

namespace csn {

// ------------------------------------------------------------------ restriction
// s_c[I,J,N] = sum_{2x2 cells} sum_{children n of N} r[i,j,n] w_n dxf dyf  (raw),
// divided by w_N dxc dyc when normalise (R/multigrid.py:326).
// explicitly rounded products / sums / quotients (no contraction: the restriction's
// rounding does not depend on the compiler's choices)
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

template <class Real>
struct RestrictArgs {
    Geo gf, gc;
    const Real* fine; int fine_h;
    const Real* wf; const Real* wc;
    Real af, ac;      // cell areas
    int angle_coarsens, normalise;
    Real* coarse; int coarse_h;
};

// One thread per coarse channel (blockIdx.x * 256 + threadIdx.x), striding over coarse
// cells with blockIdx.y: the channel decomposition (children, weights, normaliser) is
// done once per thread, the cell loop is loads + the reference's arithmetic order.  With angle coarsening and
// ng == 1 the two column children (pb = 0, 1) are adjacent channels: one 8-byte load.
// (restrict_cells: coarse channel cc over the coarse cells cell0, cell0 + stride, ...)
// Quotients of the coarse level's index decomposition (by ng, n_a^2, n_a, ny): plain
// division here; the coarse-tail kernel passes precomputed multipliers (FastDivs)
struct PlainDivs {
    int ng_, per_, na_, ny_;
    __device__ __forceinline__ int by_ng(int v) const { return v / ng_; }
    __device__ __forceinline__ int by_per(int v) const { return v / per_; }
    __device__ __forceinline__ int by_na(int v) const { return v / na_; }
    __device__ __forceinline__ int by_ny(int v) const { return v / ny_; }
};

template <class Real, class DV>
__device__ __forceinline__ void restrict_cells(const RestrictArgs<Real>& a, const int cc,
                                               const int cell0, const int stride, const DV dv) {
    const Geo &gf = a.gf, &gc = a.gc;
    const int N = dv.by_ng(cc), g = cc - N * gc.ng;
    int cf[4];          // fine child channels (pa, pb) = (0,0), (0,1), (1,0), (1,1)
    Real wn[4];
    int nch = 1;
    if (a.angle_coarsens) {
        const int naf = gf.na, nac = gc.na;
        const int f = dv.by_per(N), rem = N - f * nac * nac;
        const int R = dv.by_na(rem), Cc = rem - R * nac;
#pragma unroll
        for (int pa = 0; pa < 2; ++pa)
#pragma unroll
            for (int pb = 0; pb < 2; ++pb) {
                const int nf = f * naf * naf + (2 * R + pa) * naf + (2 * Cc + pb);
                cf[pa * 2 + pb] = nf * gf.ng + g;
                wn[pa * 2 + pb] = a.wf[nf];
            }
        nch = 4;
    } else {
        cf[0] = cc;
        wn[0] = a.wf[N];
    }
    const Real norm = a.normalise ? mul_rn(a.wc[N], a.ac) : Real(1);
    const Real af = a.af;
    const bool pair = nch == 4 && gf.ng == 1;      // cf[1] == cf[0] + 1, cf[0] even
    const int64_t fpitch = (int64_t)(gf.ny + 2 * a.fine_h) * gf.C;   // x stride (fine)
    const int ncells = gc.nx * gc.ny;
    for (int cell = cell0; cell < ncells; cell += stride) {
        const int I = dv.by_ny(cell), J = cell - I * gc.ny;
        const Real* f0 = a.fine + fidx(2 * I, 2 * J, 0, gf.ny, a.fine_h, gf.C);
        Real acc = Real(0);
        if (pair) {
#pragma unroll
            for (int pa = 0; pa < 2; ++pa) {
                Real sp0 = Real(0), sp1 = Real(0);
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const Real* q = f0 + i * fpitch + j * gf.C + cf[pa * 2];
                        Real v0, v1;
                        if (sizeof(Real) == 4) {
                            const float2 v = *reinterpret_cast<const float2*>(q);
                            v0 = (Real)v.x; v1 = (Real)v.y;
                        } else {
                            v0 = q[0]; v1 = q[1];
                        }
                        sp0 = add_rn(sp0, mul_rn(mul_rn(v0, wn[pa * 2]), af));
                        sp1 = add_rn(sp1, mul_rn(mul_rn(v1, wn[pa * 2 + 1]), af));
                    }
                acc = add_rn(acc, sp0);
                acc = add_rn(acc, sp1);
            }
        } else {
            for (int k = 0; k < nch; ++k) {
                Real sp = Real(0);
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j)
                        sp = add_rn(sp, mul_rn(mul_rn(f0[i * fpitch + j * gf.C + cf[k]], wn[k]), af));
                acc = add_rn(acc, sp);
            }
        }
        if (a.normalise) acc = div_rn(acc, norm);
        a.coarse[fidx(I, J, cc, gc.ny, a.coarse_h, gc.C)] = acc;
    }
}

template <class Real>
__global__ void __launch_bounds__(256) restrict_kernel(const RestrictArgs<Real> a) {
    const int cc = blockIdx.x * blockDim.x + threadIdx.x;
    if (cc >= a.gc.C) return;
    restrict_cells(a, cc, (int)blockIdx.y, (int)gridDim.y,
                   PlainDivs{a.gc.ng, a.gc.na * a.gc.na, a.gc.na, a.gc.ny});
}

template <class Real>
struct ProlongArgs {
    Geo gc, gf;
    const Real* coarse; int coarse_h;
    int angle_coarsens;
    Real* fine; int fine_h;
};

template <class Real>
__global__ void __launch_bounds__(256) prolong_kernel(const ProlongArgs<Real> a) {
    const Geo &gf = a.gf, &gc = a.gc;
    const int64_t total = (int64_t)gf.nx * gf.ny * gf.C;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % gf.C);
        const int64_t cell = e / gf.C;
        const int y = (int)(cell % gf.ny), x = (int)(cell / gf.ny);
        int pc = c;
        if (a.angle_coarsens) {
            const int n = c / gf.ng, g = c - n * gf.ng;
            const int naf = gf.na, nac = gc.na, per = naf * naf;
            const int f = n / per, rem = n - f * per;
            const int row = rem / naf, col = rem - row * naf;
            pc = (f * nac * nac + (row >> 1) * nac + (col >> 1)) * gf.ng + g;
        }
        a.fine[fidx(x, y, c, gf.ny, a.fine_h, gf.C)] =
            a.coarse[fidx(x >> 1, y >> 1, pc, gc.ny, a.coarse_h, gc.C)];
    }
}

// ------------------------------------------------------------------ boundary fill
// 4 channels per thread (16-byte fp32 accesses): C % 4 == 0 and the 4 channels of a
// thread share one direction's signs whenever a face holds a multiple of 4 channels
__global__ void __launch_bounds__(256)
boundary4_kernel(Geo g, float* f, int h, const float* mu, const float* nu) {
    const int c = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (c >= g.C) return;
    const int NY = g.ny + 2 * h;
    const int n_rowcells = 2 * h * NY;
    const int n_cells = n_rowcells + g.nx * 2 * h;
    const int n = c / g.ng;
    const bool mpos = mu[n] > 0.f, npos = nu[n] > 0.f;
    constexpr int BC = 4;
    for (int k0 = blockIdx.y; k0 < n_cells; k0 += BC * gridDim.y) {
        int64_t dst[BC];
        float4 v[BC];
#pragma unroll
        for (int u = 0; u < BC; ++u) {
            const int k = k0 + u * gridDim.y;
            dst[u] = -1;
            v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (k >= n_cells) continue;
            int xs, ys;
            if (k < n_rowcells) {
                const int r = k / NY;
                // a ghost side's rows hold the neighbour's data (domain decomposition):
                // the halo exchange fills them, the boundary leaves them alone
                if (r < h ? g.ghost_w : g.ghost_e) continue;
                ys = k - r * NY;
                xs = r < h ? r : g.nx + r;
            } else {
                const int kk = k - n_rowcells;
                const int r = kk / (2 * h);
                const int cidx = kk - r * 2 * h;
                xs = h + r;
                ys = cidx < h ? cidx : g.ny + cidx;
            }
            int x = xs - h, y = ys - h;
            if (resolve_vac(x, y, g, mpos, npos))
                v[u] = *reinterpret_cast<const float4*>(f + fidx(x, y, c, g.ny, h, g.C));
            dst[u] = ((int64_t)xs * NY + ys) * g.C + c;
        }
#pragma unroll
        for (int u = 0; u < BC; ++u)
            if (dst[u] >= 0) *reinterpret_cast<float4*>(f + dst[u]) = v[u];
    }
}

template <class Real>
__global__ void __launch_bounds__(256)
boundary_kernel(Geo g, Real* f, int h, const Real* mu, const Real* nu) {
    // halo cells only: storage rows [0, h) and [nx+h, nx+2h) fully, plus the h
    // columns on either side of the interior rows.  blockIdx.y walks the halo cells
    // (32-bit index math, done once per cell), threads walk the contiguous channels.
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= g.C) return;
    const int NY = g.ny + 2 * h;
    const int n_rowcells = 2 * h * NY;
    const int n_cells = n_rowcells + g.nx * 2 * h;
    const int n = c / g.ng;
    const bool mpos = mu[n] > Real(0), npos = nu[n] > Real(0);
    // BC cells per trip: all loads in flight before the stores (latency, not bandwidth,
    // bounds a one-cell-per-trip loop)
    constexpr int BC = 4;
    for (int k0 = blockIdx.y; k0 < n_cells; k0 += BC * gridDim.y) {
        int64_t dst[BC];
        Real v[BC];
#pragma unroll
        for (int u = 0; u < BC; ++u) {
            const int k = k0 + u * gridDim.y;
            dst[u] = -1;
            v[u] = Real(0);
            if (k >= n_cells) continue;
            int xs, ys;   // storage coordinates
            if (k < n_rowcells) {
                const int r = k / NY;
                // a ghost side's rows hold the neighbour's data (domain decomposition):
                // the halo exchange fills them, the boundary leaves them alone
                if (r < h ? g.ghost_w : g.ghost_e) continue;
                ys = k - r * NY;
                xs = r < h ? r : g.nx + r;
            } else {
                const int kk = k - n_rowcells;
                const int r = kk / (2 * h);
                const int cidx = kk - r * 2 * h;
                xs = h + r;
                ys = cidx < h ? cidx : g.ny + cidx;
            }
            int x = xs - h, y = ys - h;
            if (resolve_vac(x, y, g, mpos, npos)) v[u] = f[fidx(x, y, c, g.ny, h, g.C)];
            dst[u] = ((int64_t)xs * NY + ys) * g.C + c;
        }
#pragma unroll
        for (int u = 0; u < BC; ++u)
            if (dst[u] >= 0) f[dst[u]] = v[u];
    }
}

// ------------------------------------------------------------------ scalar flux
// one warp per cell, lanes over directions, NG (<= 8) groups per lane: a warp reads its
// cell's 32 * NG contiguous channels per step (coalesced; the per-(cell, group) warp of
// scalar_flux_kernel strides by ng), fp64 accumulation in a fixed order (4 partial sums
// per group for NG == 1), fixed shuffle tree -> deterministic
template <class Real, int NG>
__global__ void __launch_bounds__(256)
scalar_flux_cell_kernel(Geo g, const Real* psi, int h, const Real* w, double* phi) {
    constexpr int NP = NG == 1 ? 4 : 1;            // partial sums per group
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t ncells = (int64_t)g.nx * g.ny;
    for (int64_t cell = warp; cell < ncells; cell += nwarps) {
        const int y = (int)(cell % g.ny), x = (int)(cell / g.ny);
        const Real* base = psi + fidx(x, y, 0, g.ny, h, g.C);
        double acc[NG][NP];
#pragma unroll
        for (int k = 0; k < NG; ++k)
#pragma unroll
            for (int q = 0; q < NP; ++q) acc[k][q] = 0.0;
        for (int n0 = lane; n0 < g.nd; n0 += 32 * NP) {
#pragma unroll
            for (int qq = 0; qq < NP; ++qq) {
                const int n = n0 + 32 * qq;
                if (n < g.nd) {
                    const double wn = (double)w[n];
                    const Real* pn = base + (int64_t)n * NG;
#pragma unroll
                    for (int k = 0; k < NG; ++k) acc[k][qq] = fma(wn, (double)pn[k], acc[k][qq]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < NG; ++k) {
            double v = acc[k][0];
#pragma unroll
            for (int qq = 1; qq < NP; ++qq) v += acc[k][qq];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
            if (lane == 0) phi[cell * NG + k] = v;
        }
    }
}

// one warp per (cell, group); fp64 accumulation, fixed shuffle tree.
template <class Real>
__global__ void __launch_bounds__(256)
scalar_flux_kernel(Geo g, const Real* psi, int h, const Real* w, double* phi) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t total = (int64_t)g.nx * g.ny * g.ng;
    for (int64_t e = warp; e < total; e += nwarps) {
        const int gg = (int)(e % g.ng);
        const int64_t cell = e / g.ng;
        const int y = (int)(cell % g.ny), x = (int)(cell / g.ny);
        const Real* base = psi + fidx(x, y, 0, g.ny, h, g.C);
        double acc = 0.0;
        for (int n = lane; n < g.nd; n += 32) acc += (double)w[n] * (double)base[n * g.ng + gg];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
        if (lane == 0) phi[e] = acc;
    }
}

// ------------------------------------------------------------------ group source
template <class Real>
__global__ void __launch_bounds__(256)
group_source_kernel(Geo g, const double* phi, const double* ss, const double* src,
                    const double* fis, double lam, const double* chi, const double* nsf,
                    Real* q) {
    const int64_t total = (int64_t)g.nx * g.ny * g.ng;
    const int G = g.ng;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(e % G);
        const int64_t cell = e / G;
        const double* ph = phi + cell * G;
        const double* s = ss + cell * G * G;
        double acc = 0.0;
        for (int aa = 0; aa < G; ++aa) acc += s[aa * G + b] * ph[aa];
        acc -= s[b * G + b] * ph[b];
        acc += src[e];
        if (lam != 0.0) {
            double prod = 0.0;
            for (int aa = 0; aa < G; ++aa) prod += nsf[cell * G + aa] * ph[aa];
            acc += lam * chi[e] * prod;
        }
        if (fis) acc += fis[e];
        q[e] = (Real)acc;
    }
}

__global__ void __launch_bounds__(256)
fission_source_kernel(Geo g, const double* phi, const double* chi, const double* nsf,
                      double inv_k, double* out) {
    const int64_t total = (int64_t)g.nx * g.ny * g.ng;
    const int G = g.ng;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cell = e / G;
        double prod = 0.0;
        for (int aa = 0; aa < G; ++aa) prod += nsf[cell * G + aa] * phi[cell * G + aa];
        out[e] = inv_k * chi[e] * prod;
    }
}

__global__ void __launch_bounds__(256)
dot_partials_kernel(const double* a, const double* b, int64_t n, double* partials) {
    __shared__ double red[32];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        acc += a[i] * b[i];
    const double t = block_sum(acc, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

// single CTA, fixed order: deterministic
__global__ void __launch_bounds__(1024)
sum_f64_kernel(const double* x, int64_t n, double scale, double* out) {
    __shared__ double red[32];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += x[i];
    const double t = block_sum(acc, red);
    if (threadIdx.x == 0) *out = t * scale;
}

template <class Real>
__global__ void __launch_bounds__(256) scale_kernel(Real* x, int64_t n, Real s, int divide) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = divide ? x[i] / s : x[i] * s;
}

template <class Real>
__global__ void __launch_bounds__(256)
sub_interior_kernel(Geo g, Real* psi, int ph, const Real* d, int dh) {
    const int64_t total = (int64_t)g.nx * g.ny * g.C;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % g.C);
        const int64_t cell = e / g.C;
        const int y = (int)(cell % g.ny), x = (int)(cell / g.ny);
        psi[fidx(x, y, c, g.ny, ph, g.C)] -= d[fidx(x, y, c, g.ny, dh, g.C)];
    }
}

template <class Real>
__global__ void __launch_bounds__(256)
ema_kernel(Geo g, Real* avg, int ah, const Real* psi, int ph, Real theta, Real omt, int mode) {
    const int64_t total = (int64_t)g.nx * g.ny * g.C;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % g.C);
        const int64_t cell = e / g.C;
        const int y = (int)(cell % g.ny), x = (int)(cell / g.ny);
        const Real p = psi[fidx(x, y, c, g.ny, ph, g.C)];
        Real* o = avg + fidx(x, y, c, g.ny, ah, g.C);
        *o = mode == 1 ? p : ema_rn(*o, p, omt, theta);
    }
}

// ------------------------------------------------------------------ elementwise (modes)
// out = s (ca A[n] x + cb B[n] y); A/B per-ordinate coefficients or null (= 1)
template <class Real>
__global__ void __launch_bounds__(256)
dir_lincomb_kernel(int64_t n, int C, int ng, const Real* x, const Real* A, Real ca, const Real* y,
                   const Real* B, Real cb, Real scale, Real* out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int d = (int)(e % C) / ng;
        const Real a = A ? A[d] * x[e] : x[e];
        const Real b = y ? (B ? B[d] * y[e] : y[e]) : Real(0);
        out[e] = scale * (ca * a + cb * b);
    }
}

// isotropic PG diffusivity (R/discretisation.py:164-185), elementwise
template <class Real>
__global__ void __launch_bounds__(256)
iso_diffusivity_kernel(int64_t n, int C, int ng, const Real* r, const Real* px, const Real* py,
                       const Real* mu, const Real* nu, Real eps, Real a_abs, Real a_sq, Real hh,
                       Real dx, Real dy, Real* k) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int d = (int)(e % C) / ng;
        const Real m = mu[d], v = nu[d];
        const Real rx = r[e], gx = px[e], gy = py[e];
        const Real k_abs = a_abs * fabs(rx) * hh / (eps + Real(0.5) * (fabs(gx) + fabs(gy)));
        const Real ratio = (m * gx + v * gy) / (eps + gx * gx + gy * gy);
        const Real k_sq = a_sq * (rx * rx) * hh /
                          (eps + Real(0.5) * (fabs(ratio * gx) + fabs(ratio * gy)) * (gx * gx + gy * gy));
        const Real k_max = sqrt((dx * m) * (dx * m) + (dy * v) * (dy * v));
        k[e] = nanmin(k_max, nanmin(k_abs, k_sq));
    }
}

// ------------------------------------------------------------------ generic stencils
// R/grid.py:85-105: out = scale[n] * sum_{a,b} w[a][b] src[i+a-l][j+b-l] on
// interior +- margin; whole padded output written (zeros elsewhere).
struct StencilW { double w[121]; };   // up to 11 x 11 taps, passed by value

template <class Real>
__global__ void __launch_bounds__(256)
convolve_kernel(Geo g, const Real* src, int h, const StencilW sw, int width, int margin,
                const Real* scale, Real* out) {
    const double* w = sw.w;
    const int NX = g.nx + 2 * h, NY = g.ny + 2 * h;
    const int l = (width - 1) / 2;
    const int64_t total = (int64_t)NX * NY * g.C;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % g.C);
        const int64_t cell = e / g.C;
        const int ys = (int)(cell % NY), xs = (int)(cell / NY);
        const int x = xs - h, y = ys - h;
        Real acc = Real(0);
        if (x >= -margin && x < g.nx + margin && y >= -margin && y < g.ny + margin) {
            for (int aa = 0; aa < width; ++aa)
                for (int bb = 0; bb < width; ++bb) {
                    const Real wv = (Real)w[aa * width + bb];
                    if (wv == Real(0)) continue;
                    acc += wv * src[((int64_t)(xs + aa - l) * NY + (ys + bb - l)) * g.C + c];
                }
            if (scale) acc *= scale[c / g.ng];
        }
        out[e] = acc;
    }
}

// R/grid.py:108-125: one 1D pass along `axis`, full extent on the other axis.
template <class Real>
__global__ void __launch_bounds__(256)
pass1d_kernel(Geo g, const Real* src, int h, const StencilW sw, int width, int axis,
              int margin, Real* out) {
    const double* w = sw.w;
    const int NX = g.nx + 2 * h, NY = g.ny + 2 * h;
    const int l = (width - 1) / 2;
    const int64_t total = (int64_t)NX * NY * g.C;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % g.C);
        const int64_t cell = e / g.C;
        const int ys = (int)(cell % NY), xs = (int)(cell / NY);
        const int pos = axis == 0 ? xs - h : ys - h;
        const int next = axis == 0 ? g.nx : g.ny;
        Real acc = Real(0);
        if (pos >= -margin && pos < next + margin) {
            for (int aa = 0; aa < width; ++aa) {
                const Real wv = (Real)w[aa];
                if (wv == Real(0)) continue;
                const int64_t o = axis == 0 ? ((int64_t)(xs + aa - l) * NY + ys)
                                            : ((int64_t)xs * NY + (ys + aa - l));
                acc += wv * src[o * g.C + c];
            }
        }
        out[e] = acc;
    }
}

}  // namespace csn
