// Petrov-Galerkin ConvFEM kernels: fused iterate averaging + diffusivities (K2) and
// the PG residual / fused PG Jacobi sweep (K3 / K5).
//
// Both kernels are "2.5D y-marching" stencil engines.  A CTA owns a strip of x cells
// x a chunk of 32 contiguous channels (ordinate-group pairs, the fastest storage axis,
// so every row load is a coalesced 128 B (fp32) segment per cell) and walks along y.
// Each step stages one new y row (plus the x halo) in shared memory; every thread
// runs the x-pass taps of its own cell from shared memory and pushes the results into
// register ring buffers of depth T = 2l+1 indexed by (row mod T).  The y pass then
// reads T ring entries per output.  The y loop is unrolled by T so every ring index
// is a compile-time constant (no local-memory arrays).
//
// Pass order and tap folding follow the reference exactly (x pass first, then y
// pass, taps pre-divided by dx / dx^2 as in R/discretisation.py:114-122,503-504), so
// the fp64 instantiation reproduces the reference to rounding.
#pragma once
#include "common.cuh"

namespace csn {

constexpr int PG_CC = 32;    // channels per CTA (one warp lane per channel)
constexpr int PG_TX = 8;     // x cells per CTA (residual / sweep kernel)
constexpr int K_TXS = 16;    // stage-1 x cells per CTA (diffusivity kernel)

template <class Real, int L>
struct PGTaps {
    Real m[2 * L + 1];    // mass1
    Real gx[2 * L + 1];   // grad1 / dx
    Real gy[2 * L + 1];   // grad1 / dy
    Real sx[2 * L + 1];   // stiff1 / dx^2
    Real sy[2 * L + 1];   // stiff1 / dy^2
};

// ---------------------------------------------------------------------------------
// K3 / K5: PG residual  r = mu psi_x + nu psi_y + diff_x + diff_y + sigma psi - q
//   psi_x = M_y G_x psi,  psi_y = G_y M_x psi,
//   diff_x = 1/2 [Kx(kx psi) + kx Kx(psi) - psi Kx(kx)],  Kx = M_y S_x,
//   diff_y = 1/2 [Ky(ky psi) + ky Ky(psi) - psi Ky(ky)],  Ky = S_y M_x
// (R/discretisation.py:227-276).  SWEEP: psi' = psi - delta on load, output
// psi' - r / (beta d) (R/multigrid.py:159-172,301-304).
// ---------------------------------------------------------------------------------
template <class Real, int L>
struct PGResidArgs {
    Geo g;
    PGTaps<Real, L> t;
    const Real* psi; int psi_h;
    const Real* delta; int delta_h;
    const Real* kx; const Real* ky; int k_h;
    const Real* sigma; const Real* q; int q_per_dof;
    const Real* mu; const Real* nu; const Real* strm;
    Real* r; int r_h;
    Real* out; int out_h; Real beta;
    double* partials;
    int ly;             // y rows per CTA chunk, multiple of T
};

template <class Real, int L, bool SWEEP>
__global__ void __launch_bounds__(PG_CC * PG_TX, (sizeof(Real) == 4 && L <= 3) ? 2 : 1)
pg_residual_kernel(const PGResidArgs<Real, L> a) {
    constexpr int T = 2 * L + 1;
    constexpr int W = PG_TX + 2 * L;
    __shared__ Real sb[2][3][W][PG_CC];
    __shared__ double red[32];

    const Geo& g = a.g;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int c = blockIdx.y * PG_CC + tx;
    const bool cval = c < g.C;
    const int cs = cval ? c : g.C - 1;
    const int n = cs / g.ng, gg = cs - n * g.ng;
    const Real mu = a.mu[n], nu = a.nu[n];
    const bool mpos = mu > Real(0), npos = nu > Real(0);
    const int x0 = blockIdx.x * PG_TX;
    const int x = x0 + ty;
    const int ya = blockIdx.z * a.ly;
    const int yb = min(g.ny, ya + a.ly);
    const bool xval = x < g.nx;

    // x-pass rings (by row mod T)
    Real rgx[T], rmx[T], rsx[T], rsk[T], rkx[T], rmk[T], rky[T];
    Real cp[T], ckx[T], cky[T];

    auto load_row = [&](int yy, int buf) {
        for (int xi = ty; xi < W; xi += PG_TX) {
            const int xg = x0 - L + xi;
            Real vp = Real(0), v1 = Real(0), v2 = Real(0);
            if (cval) {
                int xr = xg, yr = yy;
                if (resolve_vac(xr, yr, g, mpos, npos)) {
                    vp = a.psi[fidx(xr, yr, c, g.ny, a.psi_h, g.C)];
                    if (SWEEP && a.delta) vp -= a.delta[fidx(xr, yr, c, g.ny, a.delta_h, g.C)];
                }
                if (xg >= -L && xg < g.nx + L && yy >= -L && yy < g.ny + L) {
                    const int64_t o = fidx(xg, yy, c, g.ny, a.k_h, g.C);
                    v1 = a.kx[o];
                    v2 = a.ky[o];
                }
            }
            sb[buf][0][xi][tx] = vp;
            sb[buf][1][xi][tx] = v1;
            sb[buf][2][xi][tx] = v2;
        }
    };

#define PG_XPASS(BUF, SLOT)                                                        \
    {                                                                              \
        Real a_g = 0, a_m = 0, a_s = 0, a_sk = 0, a_k = 0, a_mk = 0, a_ky = 0;       \
        _Pragma("unroll") for (int t_ = 0; t_ < T; ++t_) {                         \
            const Real p_ = sb[BUF][0][ty + t_][tx];                               \
            const Real k1_ = sb[BUF][1][ty + t_][tx];                              \
            const Real k2_ = sb[BUF][2][ty + t_][tx];                              \
            a_g += a.t.gx[t_] * p_;                                                \
            a_m += a.t.m[t_] * p_;                                                 \
            a_s += a.t.sx[t_] * p_;                                                \
            a_sk += a.t.sx[t_] * (p_ * k1_);                                       \
            a_k += a.t.sx[t_] * k1_;                                               \
            a_mk += a.t.m[t_] * (p_ * k2_);                                        \
            a_ky += a.t.m[t_] * k2_;                                               \
        }                                                                          \
        rgx[SLOT] = a_g; rmx[SLOT] = a_m; rsx[SLOT] = a_s; rsk[SLOT] = a_sk;       \
        rkx[SLOT] = a_k; rmk[SLOT] = a_mk; rky[SLOT] = a_ky;                       \
        cp[SLOT] = sb[BUF][0][ty + L][tx];                                         \
        ckx[SLOT] = sb[BUF][1][ty + L][tx];                                        \
        cky[SLOT] = sb[BUF][2][ty + L][tx];                                        \
    }

    int step = 0;
    // prologue: rows ya-L .. ya+L-1 (ya is a multiple of T)
#pragma unroll
    for (int k = 0; k < 2 * L; ++k) {
        load_row(ya - L + k, step & 1);
        __syncthreads();
        PG_XPASS(step & 1, (k - L + T) % T);
        ++step;
    }

    double l1 = 0.0;
    for (int y0 = ya; y0 < yb; y0 += T) {
#pragma unroll
        for (int s = 0; s < T; ++s) {
            const int y = y0 + s;
            load_row(y + L, step & 1);
            __syncthreads();
            PG_XPASS(step & 1, (s + L) % T);
            ++step;
            if (y < yb && xval && cval) {
                Real px = 0, py = 0, kxp = 0, kxkp = 0, kxk = 0, kykp = 0, kyp = 0, kyk = 0;
#pragma unroll
                for (int b = 0; b < T; ++b) {
                    const int sl = (s - L + b + T) % T;
                    px += a.t.m[b] * rgx[sl];
                    py += a.t.gy[b] * rmx[sl];
                    kxp += a.t.m[b] * rsx[sl];
                    kxkp += a.t.m[b] * rsk[sl];
                    kxk += a.t.m[b] * rkx[sl];
                    kykp += a.t.sy[b] * rmk[sl];
                    kyp += a.t.sy[b] * rmx[sl];
                    kyk += a.t.sy[b] * rky[sl];
                }
                const Real pc = cp[s], kxc = ckx[s], kyc = cky[s];
                const Real diffx = Real(0.5) * ((kxkp + kxc * kxp) - pc * kxk);
                const Real diffy = Real(0.5) * ((kykp + kyc * kyp) - pc * kyk);
                const int64_t cell = (int64_t)x * g.ny + y;
                const Real sig = a.sigma[cell * g.ng + gg];
                const Real qq = a.q_per_dof ? a.q[cell * g.C + c] : a.q[cell * g.ng + gg];
                const Real r = (((mu * px + nu * py) + diffx) + diffy) + sig * pc - qq;
                if (SWEEP) {
                    const Real d = a.beta * (a.strm[n] + sig);
                    a.out[fidx(x, y, c, g.ny, a.out_h, g.C)] = pc - r / d;
                } else {
                    if (a.r) a.r[fidx(x, y, c, g.ny, a.r_h, g.C)] = r;
                    l1 += fabs((double)r);
                }
            }
        }
    }
#undef PG_XPASS
    if (!SWEEP && a.partials) {
        const double tot = block_sum(l1, red);
        if (threadIdx.x == 0 && threadIdx.y == 0)
            a.partials[((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = tot;
    }
}

// ---------------------------------------------------------------------------------
// K2: iterate averaging (R/multigrid.py:217-225) fused with the anisotropic
// diffusivities (R/discretisation.py:114-161):
//   psi_x = M_y G_x pbar,  psi_y = G_y M_x pbar             (stage 1, +-2l band)
//   R_x = alpha_r mu (M_y M_x psi_x - psi_x)                  (stage 2, +-l band)
//   k_x = min(dx|mu|, min(a_abs |R_x| dx/(eps+|psi_x|), a_sq R_x^2 dx/(eps+|mu| psi_x^2)))
//   NaN / inf -> 0.   (y symmetric)
// Outputs cover the band x, y in [-l, n+l).  Stage 1 runs on K_TXS x cells, stage 2
// on the inner K_TXS - 2l (its x pass reads stage-1 neighbours through smem).
// ---------------------------------------------------------------------------------
template <class Real, int L>
struct PGKArgs {
    Geo g;
    PGTaps<Real, L> t;
    const Real* psi; int psi_h;
    const Real* avg_in; int avg_in_h;
    Real* avg_out; int avg_out_h;
    int avg_mode; Real theta, omt;
    Real alpha_r, eps, a_abs, a_sq, dx, dy;
    const Real* mu; const Real* nu;
    Real* kx; Real* ky; int k_h;
    int ly;     // output rows per CTA chunk (band coordinates), multiple of T
};

template <class Real, int L>
__global__ void __launch_bounds__(PG_CC * K_TXS)
pg_diffusivity_kernel(const PGKArgs<Real, L> a) {
    constexpr int T = 2 * L + 1;
    constexpr int TXO = K_TXS - 2 * L;
    constexpr int W1 = K_TXS + 2 * L;
    __shared__ Real s1[2][W1][PG_CC];
    __shared__ Real s2[2][2][K_TXS][PG_CC];

    const Geo& g = a.g;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int c = blockIdx.y * PG_CC + tx;
    const bool cval = c < g.C;
    const int cs = cval ? c : g.C - 1;
    const int n = cs / g.ng;
    const Real mu = a.mu[n], nu = a.nu[n];
    const Real amu = fabs(mu), anu = fabs(nu);
    const bool mpos = mu > Real(0), npos = nu > Real(0);
    const int x0o = -L + (int)blockIdx.x * TXO;   // first output x of this CTA
    const int x0s = x0o - L;                       // first stage-1 x
    const int xs = x0s + ty;
    const bool s2thr = ty >= L && ty < K_TXS - L;
    const bool xout = s2thr && xs < g.nx + L;
    const int ua = blockIdx.z * a.ly;                      // band rows u = y + L
    const int ub = min(g.ny + 2 * L, ua + a.ly);
    // psi_avg rows / columns this CTA owns (each interior cell written once)
    const int ox0 = max(x0o, 0), ox1 = min(x0o + TXO, g.nx);
    const int oy0 = max(ua - L, 0), oy1 = min(ub - L, g.ny);
    const Real ar_mu = a.alpha_r * mu, ar_nu = a.alpha_r * nu;

    Real r1g[T], r1m[T];   // stage-1 x pass of pbar (by pbar row)
    Real c1x[T], c1y[T];   // psi_x, psi_y (by row)
    Real r2x[T], r2y[T];   // M_x psi_x, M_x psi_y (by row)

    auto load_row = [&](int yy, int buf) {
        for (int xi = ty; xi < W1; xi += K_TXS) {
            const int xg = x0s - L + xi;
            Real v = Real(0);
            if (cval) {
                int xr = xg, yr = yy;
                if (resolve_vac(xr, yr, g, mpos, npos)) {
                    const Real pv = a.psi[fidx(xr, yr, c, g.ny, a.psi_h, g.C)];
                    if (a.avg_mode == 2) {
                        const Real av = a.avg_in[fidx(xr, yr, c, g.ny, a.avg_in_h, g.C)];
                        v = av * a.omt + a.theta * pv;
                    } else {
                        v = pv;
                    }
                    if (a.avg_mode != 0 && xr == xg && yr == yy && xg >= ox0 && xg < ox1 &&
                        yy >= oy0 && yy < oy1)
                        a.avg_out[fidx(xg, yy, c, g.ny, a.avg_out_h, g.C)] = v;
                }
            }
            s1[buf][xi][tx] = v;
        }
    };

    // steps v (band row of the stage-2 output) from vs to ve, vs = ua - T*ceil(4L/T)
    constexpr int PRE = ((4 * L + T - 1) / T) * T;
    const int vs = ua - PRE;
    int step = 0;
    for (int v0 = vs; v0 < ub; v0 += T) {
#pragma unroll
        for (int s = 0; s < T; ++s) {
            const int v = v0 + s;
            const int buf = step & 1;
            ++step;
            // (1) pbar lead row: band row v + 2L  <=>  y = v + L
            load_row(v + L, buf);
            __syncthreads();
            // (2) stage 1 at band row v + L (y = v): x pass of the lead row, then y pass
            {
                Real ag = 0, am = 0;
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    const Real p = s1[buf][ty + t][tx];
                    ag += a.t.gx[t] * p;
                    am += a.t.m[t] * p;
                }
                r1g[(s + 2 * L) % T] = ag;
                r1m[(s + 2 * L) % T] = am;
                Real px = 0, py = 0;
#pragma unroll
                for (int b = 0; b < T; ++b) {
                    px += a.t.m[b] * r1g[(s + b) % T];
                    py += a.t.gy[b] * r1m[(s + b) % T];
                }
                c1x[(s + L) % T] = px;
                c1y[(s + L) % T] = py;
                s2[buf][0][ty][tx] = px;
                s2[buf][1][ty][tx] = py;
            }
            __syncthreads();
            // (3) stage 2: x pass (mass) at band row v + L, y pass (mass) -> row v
            if (s2thr) {
                Real mx = 0, my = 0;
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    mx += a.t.m[t] * s2[buf][0][ty - L + t][tx];
                    my += a.t.m[t] * s2[buf][1][ty - L + t][tx];
                }
                r2x[(s + L) % T] = mx;
                r2y[(s + L) % T] = my;
                if (xout && cval && v >= ua && v < ub) {
                    Real mmx = 0, mmy = 0;
#pragma unroll
                    for (int b = 0; b < T; ++b) {
                        mmx += a.t.m[b] * r2x[(s - L + b + T) % T];
                        mmy += a.t.m[b] * r2y[(s - L + b + T) % T];
                    }
                    const Real px = c1x[s % T], py = c1y[s % T];
                    const Real rx = ar_mu * (mmx - px);
                    const Real ry = ar_nu * (mmy - py);
                    Real kx = nanmin(a.dx * amu,
                                     nanmin(a.a_abs * fabs(rx) * a.dx / (a.eps + fabs(px)),
                                            a.a_sq * (rx * rx) * a.dx / (a.eps + amu * (px * px))));
                    Real ky = nanmin(a.dy * anu,
                                     nanmin(a.a_abs * fabs(ry) * a.dy / (a.eps + fabs(py)),
                                            a.a_sq * (ry * ry) * a.dy / (a.eps + anu * (py * py))));
                    if (!isfinite(kx)) kx = Real(0);
                    if (!isfinite(ky)) ky = Real(0);
                    const int yo = v - L;
                    const int64_t o = fidx(xs, yo, c, g.ny, a.k_h, g.C);
                    a.kx[o] = kx;
                    a.ky[o] = ky;
                }
            }
        }
    }
}

}  // namespace csn
