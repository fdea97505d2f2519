// Petrov-Galerkin ConvFEM kernels: fused iterate averaging + diffusivities (K2) and
// the PG residual / fused PG Jacobi sweep (K3 / K5).
//
// Both kernels are "2.5D y-marching" stencil engines.  A CTA owns a strip of x cells
// x a chunk of 32 contiguous channels (ordinate-group pairs, the fastest storage
// axis, so every row load is one coalesced 128 B (fp32) segment per cell) and walks
// along y.  Rows are staged into an S-deep shared-memory ring with cp.async (LDGSTS,
// zero-fill for the vacuum halo) S-1 rows ahead of use, so DRAM latency hides behind
// the stencil arithmetic of the rows in flight.  Each thread runs the x-pass taps of
// its own cell from shared memory and pushes the results into register ring buffers
// of depth T = 2l+1 indexed by (row mod T); the y pass reads T ring entries per
// output.  The y loop is unrolled by T so every ring index is a compile-time constant.
//
// Unit-spacing taps are compile-time constants (taps_table.cuh, generated from the
// host filter construction) so every tap is an FFMA immediate; the 1/dx, 1/dx^2
// factors the reference folds into its taps (R/discretisation.py:114-122,503-504)
// are applied once per output instead.  Same pass order as the reference (x pass,
// then y pass); the fp64 instantiation agrees with it to ~1e-15 relative per pass.
#pragma once
#include "common.cuh"
#include "taps_table.cuh"

namespace csn {

constexpr int PG_CC = 32;    // channels per CTA (one warp lane per channel)
constexpr int PG_TX = 8;     // x cells per CTA (residual / sweep kernel)

// stage-1 x cells per CTA of the diffusivity kernel (stage-2 outputs = KTile - 2L)
template <class Real, int L>
struct KTile { static constexpr int value = (sizeof(Real) == 8 || L == 1) ? 16 : 24; };

template <class Real>
struct PGStages { static constexpr int value = sizeof(Real) == 4 ? 4 : 3; };

template <class Real>
__device__ __forceinline__ Real fast_div(Real a, Real b) { return a / b; }
// fp32: MUFU reciprocal + one Newton step (<= 1 ulp, no slow-path call); the divisors
// here are positive and finite except in diverging iterates, where NaN -> 0 downstream
// matches the reference's inf/inf -> NaN -> 0.
__device__ __forceinline__ float rcp_nr(float b) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b));
    return fmaf(fmaf(-b, r, 1.0f), r, r);
}
template <>
__device__ __forceinline__ float fast_div<float>(float a, float b) { return a * rcp_nr(b); }

// ---------------------------------------------------------------------------------
// K3 / K5: PG residual  r = mu psi_x + nu psi_y + diff_x + diff_y + sigma psi - q
//   psi_x = M_y G_x psi / dx,  psi_y = G_y M_x psi / dy,
//   diff_x = 1/(2dx^2) [Kx(kx psi) + kx Kx(psi) - psi Kx(kx)],  Kx = M_y S_x,
//   diff_y = 1/(2dy^2) [Ky(ky psi) + ky Ky(psi) - psi Ky(ky)],  Ky = S_y M_x
// (R/discretisation.py:227-276).  SWEEP: psi' = psi - delta on load, output
// psi' - r / (beta d) (R/multigrid.py:159-172,301-304).
// ---------------------------------------------------------------------------------
template <class Real>
struct PGResidArgs {
    Geo g;
    const Real* psi; int psi_h;
    const Real* delta; int delta_h;
    const Real* kx; const Real* ky; int k_h;
    const Real* sigma; const Real* q; int q_per_dof;
    const Real* mu; const Real* nu; const Real* strm;
    Real inv_dx, inv_dy, hx, hy;        // 1/dx, 1/dy, 1/(2 dx^2), 1/(2 dy^2)
    Real* r; int r_h;
    Real* out; int out_h; Real beta;
    double* partials;
    Real* avg; int avg_h; int avg_mode; Real theta, omt;   // fused EMA (frozen cycles)
    int ly;             // y rows per CTA chunk, multiple of T
    int refine_div;     // fp32 sweep: refine r / (beta d) to the rounded quotient
    // k-only term D = -M_y(hx S_x kx) - S_y(hy M_x ky) of the residual (the coefficient
    // of psi at the output cell), unpadded [nx][ny][C]: written (KD 1) by the residual
    // after a diffusivity refresh, read (KD 2) while k is unchanged (TMA kernel)
    Real* dterm;
};

// residual kernel modes: plain residual, residual + fused iterate EMA, fused sweep
constexpr int PG_RESID = 0, PG_RESID_EMA = 1, PG_SWEEP = 2;
// PG_SWEEPF (TMA kernel only): the fused sweep on an iterate the finest correction
// has already folded into (psi' = psi - delta, csn_upwind_smooth_sub): three staged
// fields, no per-read subtraction
constexpr int PG_SWEEPF = 3;

template <class Real, int L, int MODE>
constexpr size_t pg_residual_smem() {
    return (size_t)PGStages<Real>::value * (MODE == PG_RESID ? 3 : 4) * (PG_TX + 2 * L) * PG_CC *
           sizeof(Real);
}

template <class Real, int L, int MODE, int VEC>
__global__ void __launch_bounds__(PG_CC * PG_TX, (sizeof(Real) == 4 && L <= 3) ? 2 : 1)
pg_residual_kernel(const PGResidArgs<Real> a) {
    constexpr bool SWEEP = MODE == PG_SWEEP;
    constexpr bool EMA = MODE == PG_RESID_EMA;
    using TP = UnitTaps<L>;
    constexpr int T = 2 * L + 1;
    constexpr int W = PG_TX + 2 * L;
    constexpr int NT = PG_CC * PG_TX;
    constexpr int G4 = PG_CC / VEC;
    constexpr int NI = (W * G4 + NT - 1) / NT;     // staged items per thread
    constexpr int NF = MODE == PG_RESID ? 3 : 4;   // psi, kx, ky (, delta | pbar)
    constexpr int S = PGStages<Real>::value;       // rows in flight
    constexpr int FS = W * PG_CC;                  // elements per field row
    // centre values of the output row (staged L steps earlier) ride in register rings:
    // the smem ring only holds the rows in flight
    constexpr bool CSM = false;
    constexpr int TC = T;
    extern __shared__ __align__(16) unsigned char smraw[];
    Real* sm = reinterpret_cast<Real*>(smraw);
    __shared__ double red[32];

    const Geo& g = a.g;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * PG_CC + tx;
    const int c0 = blockIdx.y * PG_CC;
    const int c = c0 + tx;
    const bool cval = c < g.C;
    const int cs = cval ? c : g.C - 1;
    const int n = cs / g.ng, gg = cs - n * g.ng;
    const Real mu_dx = a.mu[n] * a.inv_dx, nu_dy = a.nu[n] * a.inv_dy;
    const Real hx = a.hx, hy = a.hy;
    const int x0 = blockIdx.x * PG_TX;
    const int x = x0 + ty;
    const int ya = blockIdx.z * a.ly;
    const int yb = min(g.ny, ya + a.ly);
    const bool act = x < g.nx && cval;
    const int nsteps = 2 * L + (int)(((yb - ya) + T - 1) / T) * T;   // lead rows ya-L ...

    FieldDesc fd[4] = {{a.psi, a.psi_h, -L, g.nx + L}, {a.kx, a.k_h}, {a.ky, a.k_h},
                       {SWEEP ? a.delta : a.avg, SWEEP ? a.delta_h : a.avg_h, -L, g.nx + L}};
    // psi / delta staged only on [-l, nx+l): the last CTA's overhang (nx % TX != 0)
    // is never read by an output and would run past a ghost side's stored rows
    if (EMA) { fd[3].xlo = x0; fd[3].xhi = min(x0 + PG_TX, g.nx); }   // owned columns only
    Stager<Real, VEC, NI, NF, 0x6> st;
    st.init(g, fd, x0 - L, W, c0, L, a.mu, a.nu, tid, NT);
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);
    constexpr unsigned FSB = FS * sizeof(Real);

    // epilogue pointers at y = 0 (per output only y * stride is added)
    const int xs = act ? x : 0;
    const int64_t cell0 = (int64_t)xs * g.ny;
    const Real* sig_p = a.sigma + cell0 * g.ng + gg;
    const int qst = a.q_per_dof ? g.C : g.ng;
    const Real* q_p = a.q + cell0 * qst + (a.q_per_dof ? c : gg);
    Real* o_p = SWEEP ? a.out + fidx(xs, 0, cs, g.ny, a.out_h, g.C)
                      : (a.r ? a.r + fidx(xs, 0, cs, g.ny, a.r_h, g.C) : nullptr);
    const Real dscale = a.beta, strm = a.strm ? a.strm[n] : Real(0);
    // fused iterate averaging (R/multigrid.py:217-225) on the interior cells this CTA
    // owns: elementwise, so in place; psi and pbar_old arrive through the staging ring
    Real* avg_p[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        const int e = tid + i * NT;
        const int xi = e / G4, cc = c0 + (e % G4) * VEC;
        const int xg = x0 - L + xi;
        avg_p[i] = (EMA && e < W * G4 && cc < g.C && xi >= L && xi < L + PG_TX && xg < g.nx)
                       ? a.avg + fidx(xg, 0, cc, g.ny, a.avg_h, g.C) : nullptr;
    }
    const int oy0 = max(ya, 0), oy1 = yb;

    // x-pass rings (by row mod T): A = mu/dx G psi + hx S(kx psi) (M_y later),
    // S psi, S kx (M_y), M psi (G_y and S_y), M(ky psi), M ky (S_y)
    Real ra[T], rsx[T], rkx[T], rmx[T], rmk[T], rky[T];
    Real cp[TC], ckx[TC], cky[TC];

#define PG_STEP(K, SLOT)                                                             \
    {                                                                                \
        const int k_ = (K);                                                          \
        cp_async_wait<S - 2>();                                                      \
        Real* buf_ = sm + (size_t)(k_ % S) * NF * FS;                                \
        if (SWEEP) {                                                                 \
            _Pragma("unroll") for (int i = 0; i < NI; ++i) {                         \
                const int e = tid + i * NT;                                          \
                if (e < W * G4) {                                                    \
                    Real* p_ = buf_ + (e / G4) * PG_CC + (e % G4) * VEC;             \
                    _Pragma("unroll") for (int v = 0; v < VEC; ++v) p_[v] -= p_[3 * FS + v]; \
                }                                                                    \
            }                                                                        \
        } else if (EMA) {                                                            \
            const int yl_ = ya - L + k_;                                             \
            if (yl_ >= oy0 && yl_ < oy1) {                                           \
                _Pragma("unroll") for (int i = 0; i < NI; ++i) {                     \
                    if (avg_p[i]) {                                                  \
                        const int e = tid + i * NT;                                  \
                        const Real* p_ = buf_ + (e / G4) * PG_CC + (e % G4) * VEC;   \
                        Real* o_ = avg_p[i] + (int64_t)yl_ * g.C;                    \
                        _Pragma("unroll") for (int v = 0; v < VEC; ++v)              \
                            o_[v] = a.avg_mode == 2 ? ema_rn(p_[3 * FS + v], p_[v], a.omt, a.theta) \
                                                    : p_[v];                         \
                    }                                                                \
                }                                                                    \
            }                                                                        \
        }                                                                            \
        __syncthreads();                                                             \
        Real a_g = 0, a_m = 0, a_s = 0, a_sk = 0, a_k = 0, a_mk = 0, a_ky = 0;         \
        _Pragma("unroll") for (int t_ = 0; t_ < T; ++t_) {                           \
            const Real p_ = buf_[(ty + t_) * PG_CC + tx];                            \
            const Real k1_ = buf_[FS + (ty + t_) * PG_CC + tx];                      \
            const Real k2_ = buf_[2 * FS + (ty + t_) * PG_CC + tx];                  \
            a_g += Real(TP::g(t_)) * p_;                                             \
            a_m += Real(TP::m(t_)) * p_;                                             \
            a_s += Real(TP::s(t_)) * p_;                                             \
            a_sk += Real(TP::s(t_)) * (p_ * k1_);                                    \
            a_k += Real(TP::s(t_)) * k1_;                                            \
            a_mk += Real(TP::m(t_)) * (p_ * k2_);                                    \
            a_ky += Real(TP::m(t_)) * k2_;                                           \
        }                                                                            \
        ra[SLOT] = mu_dx * a_g + hx * a_sk;                                          \
        rsx[SLOT] = a_s; rkx[SLOT] = a_k; rmx[SLOT] = a_m;                           \
        rmk[SLOT] = a_mk; rky[SLOT] = a_ky;                                          \
        if (!CSM) {                                                                  \
            cp[(SLOT) % TC] = buf_[(ty + L) * PG_CC + tx];                           \
            ckx[(SLOT) % TC] = buf_[FS + (ty + L) * PG_CC + tx];                     \
            cky[(SLOT) % TC] = buf_[2 * FS + (ty + L) * PG_CC + tx];                 \
        }                                                                            \
        if (k_ + S - 1 < nsteps)                                                     \
            st.issue(ya - L + k_ + S - 1, sbase + ((k_ + S - 1) % S) * NF * FSB, FSB, a.psi); \
        cp_async_commit();                                                           \
    }

#pragma unroll
    for (int k = 0; k < S - 1; ++k) {
        if (k < nsteps) st.issue(ya - L + k, sbase + k * NF * FSB, FSB, a.psi);
        cp_async_commit();
    }
    // prologue: lead rows ya-L .. ya+L-1 (ya is a multiple of T)
#pragma unroll
    for (int k = 0; k < 2 * L; ++k) PG_STEP(k, (k - L + T) % T);

    double l1 = 0.0;
    int kbase = 2 * L;
    for (int y0 = ya; y0 < yb; y0 += T, kbase += T) {
#pragma unroll
        for (int s = 0; s < T; ++s) {
            const int y = y0 + s;
            PG_STEP(kbase + s, (s + L) % T);
            if (act && y < yb) {
                Real pa = 0, kxp = 0, kxk = 0, py = 0, kyp = 0, kykp = 0, kyk = 0;
#pragma unroll
                for (int b = 0; b < T; ++b) {
                    const int sl = (s - L + b + T) % T;
                    pa += Real(TP::m(b)) * ra[sl];
                    kxp += Real(TP::m(b)) * rsx[sl];
                    kxk += Real(TP::m(b)) * rkx[sl];
                    py += Real(TP::g(b)) * rmx[sl];
                    kyp += Real(TP::s(b)) * rmx[sl];
                    kykp += Real(TP::s(b)) * rmk[sl];
                    kyk += Real(TP::s(b)) * rky[sl];
                }
                Real pc, kxc, kyc;
                if (CSM) {   // staged buffer of this output row (lead row L steps ago)
                    const Real* cb = sm + (size_t)((kbase + s - L) % S) * NF * FS + (ty + L) * PG_CC + tx;
                    pc = cb[0]; kxc = cb[FS]; kyc = cb[2 * FS];
                } else {
                    pc = cp[s % TC]; kxc = ckx[s % TC]; kyc = cky[s % TC];
                }
                // r = mu psi_x + nu psi_y + hx[K(kx psi) + kx K psi - psi K kx] + hy[...] + sig psi - q
                const Real sig = sig_p[y * g.ng];
                const Real r = (((pa + hx * (kxc * kxp - pc * kxk)) + nu_dy * py) +
                                hy * ((kykp + kyc * kyp) - pc * kyk)) +
                               sig * pc - q_p[y * qst];
                if (SWEEP) {
                    o_p[(int64_t)y * g.C] = pc - fast_div(r, dscale * (strm + sig));
                } else {
                    if (o_p) o_p[(int64_t)y * g.C] = r;
                    l1 += fabs((double)r);
                }
            }
        }
    }
#undef PG_STEP
    cp_async_wait<0>();
    if (!SWEEP && a.partials) {
        const double tot = block_sum(l1, red);
        if (threadIdx.x == 0 && threadIdx.y == 0)
            a.partials[((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = tot;
    }
}

// ---------------------------------------------------------------------------------
// K2: iterate averaging (R/multigrid.py:217-225) fused with the anisotropic
// diffusivities (R/discretisation.py:114-161):
//   psi_x = M_y G_x pbar / dx,  psi_y = G_y M_x pbar / dy       (stage 1, +-2l band)
//   R_x = alpha_r mu (M_y M_x psi_x - psi_x)                      (stage 2, +-l band)
//   k_x = min(dx|mu|, min(a_abs |R_x| dx/(eps+|psi_x|), a_sq R_x^2 dx/(eps+|mu| psi_x^2)))
//   NaN / inf -> 0.   (y symmetric)
// Outputs cover the band x, y in [-l, n+l).  Stage 1 runs on KTile x cells, stage 2
// on the inner KTile - 2l (its x pass reads stage-1 neighbours through smem).
// The averaged iterate pbar = (1 - theta) pbar_old + theta psi is formed on load
// (both rows staged by cp.async) and written back for the cells this CTA owns.
// ---------------------------------------------------------------------------------
template <class Real>
struct PGKArgs {
    Geo g;
    const Real* psi; int psi_h;
    const Real* avg_in; int avg_in_h;
    Real* avg_out; int avg_out_h;
    int avg_mode; Real theta, omt;
    Real alpha_r, eps, a_abs, a_sq, dx, dy, inv_dx, inv_dy;
    // a_abs dx, a_sq dx, a_abs dy, a_sq dy formed once on the host (the same rounded
    // products the kernels used to recompute for every k: ptxas did not keep them live)
    Real cax, csx, cay, csy;
    const Real* mu; const Real* nu;
    Real* kx; Real* ky; int k_h;
    int ly;     // output rows per CTA chunk (band coordinates), multiple of T
};

template <class Real, int L, bool EMA>
constexpr size_t pg_k_smem() {
    constexpr int KT = KTile<Real, L>::value;
    return ((size_t)PGStages<Real>::value * (EMA ? 2 : 1) * (KT + 2 * L) * PG_CC +
            (size_t)2 * 2 * KT * PG_CC) * sizeof(Real);
}

template <class Real, int L, bool EMA, int VEC>
__global__ void __launch_bounds__(PG_CC * KTile<Real, L>::value)
pg_diffusivity_kernel(const PGKArgs<Real> a) {
    using TP = UnitTaps<L>;
    constexpr int KT = KTile<Real, L>::value;
    constexpr int T = 2 * L + 1;
    constexpr int TXO = KT - 2 * L;
    constexpr int W1 = KT + 2 * L;
    constexpr int NT = PG_CC * KT;
    constexpr int G4 = PG_CC / VEC;
    constexpr int NI = (W1 * G4 + NT - 1) / NT;
    constexpr int NF = EMA ? 2 : 1;               // psi (, pbar_old)
    constexpr int S = PGStages<Real>::value;
    constexpr int FS = W1 * PG_CC;
    extern __shared__ __align__(16) unsigned char smraw[];
    Real* s1 = reinterpret_cast<Real*>(smraw);          // [S][NF][W1][CC]
    Real* s2 = s1 + (size_t)S * NF * FS;                 // [2][2][KT][CC]: psi_x, psi_y

    const Geo& g = a.g;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * PG_CC + tx;
    const int c0 = blockIdx.y * PG_CC;
    const int c = c0 + tx;
    const bool cval = c < g.C;
    const int cs = cval ? c : g.C - 1;
    const int n = cs / g.ng;
    const Real mu = a.mu[n], nu = a.nu[n];
    const Real amu = fabs(mu), anu = fabs(nu);
    const int x0o = -L + (int)blockIdx.x * TXO;   // first output x of this CTA
    const int x0s = x0o - L;                       // first stage-1 x
    const int xs = x0s + ty;
    const bool s2thr = ty >= L && ty < KT - L;
    const bool xout = s2thr && xs < g.nx + L && cval;
    const int ua = blockIdx.z * a.ly;                      // band rows u = y + L
    const int ub = min(g.ny + 2 * L, ua + a.ly);
    const int ox0 = max(x0o, 0), ox1 = min(x0o + TXO, g.nx);
    const int oy0 = max(ua - L, 0), oy1 = min(ub - L, g.ny);
    const Real ar_mu = a.alpha_r * mu, ar_nu = a.alpha_r * nu;
    const Real dx = a.dx, dy = a.dy, inv_dx = a.inv_dx, inv_dy = a.inv_dy;
    const Real kxmax = dx * amu, kymax = dy * anu;
    const Real eps = a.eps, cabs_x = a.a_abs * dx, csq_x = a.a_sq * dx;
    const Real cabs_y = a.a_abs * dy, csq_y = a.a_sq * dy;
    const Real omt = a.omt, theta = a.theta;
    const bool write_avg = a.avg_mode != 0;

    constexpr int PRE = ((4 * L + T - 1) / T) * T;
    const int vs = ua - PRE;
    const int nsteps = PRE + (int)(((ub + 1 - ua) + T - 1) / T) * T;   // +1: stage-2 lag
    const int64_t kbase_o = fidx(xout ? xs : 0, 0, cs, g.ny, a.k_h, g.C);

    // the staged band is [-3l, nx+3l): the last CTA's overhang past it is never loaded
    // (past a ghost side it would run off the field)
    FieldDesc fd[2] = {{a.psi, a.psi_h, -3 * L, g.nx + 3 * L},
                       {a.avg_in, a.avg_in_h, -3 * L, g.nx + 3 * L}};
    Stager<Real, VEC, NI, NF, 0> st;
    st.init(g, fd, x0s - L, W1, c0, 0, a.mu, a.nu, tid, NT);
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(s1);
    constexpr unsigned FSB = FS * sizeof(Real);
    // owned pbar write-back per item: output pointer at y storage 0, or null
    Real* own_ptr[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        const int e = tid + i * NT;
        const int xi = e / G4, q = e % G4;
        const int xg = x0s - L + xi, cc = c0 + q * VEC;
        own_ptr[i] = (write_avg && e < W1 * G4 && cc < g.C && xg >= ox0 && xg < ox1)
                         ? a.avg_out + fidx(xg, 0, cc, g.ny, a.avg_out_h, g.C) : nullptr;
    }

    Real r1g[T], r1m[T];   // stage-1 x pass of pbar (by pbar row)
    Real c1x[T], c1y[T];   // psi_x, psi_y (by row)
    Real r2x[T], r2y[T];   // M_x psi_x, M_x psi_y (by row)

    // Step v stages pbar row y = v + L, runs stage 1 at band row v + L and stage 2 on
    // the stage-1 row of step v - 1 (band row v - 1 + L), emitting k at band row v - 1.
    // The barrier of step v publishes both the staged row and step v-1's stage-1 row.
#pragma unroll
    for (int k = 0; k < S - 1; ++k) {
        if (k < nsteps) st.issue(vs + L + k, sbase + k * NF * FSB, FSB, a.psi);
        cp_async_commit();
    }
    int step = 0;
    for (int v0 = vs; v0 <= ub; v0 += T) {
#pragma unroll
        for (int s = 0; s < T; ++s) {
            const int v = v0 + s;
            const int yl = v + L;                  // pbar lead row (y coords)
            cp_async_wait<S - 2>();
            Real* buf = s1 + (size_t)(step % S) * NF * FS;
            if (EMA || write_avg) {                // form pbar on own items; write back owned
                const bool own_row = yl >= oy0 && yl < oy1;
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int e = tid + i * NT;
                    if (e < W1 * G4) {
                        Real* p = buf + (e / G4) * PG_CC + (e % G4) * VEC;
                        Real pv[VEC];
#pragma unroll
                        for (int vv = 0; vv < VEC; ++vv) {
                            pv[vv] = p[vv];
                            if (EMA) pv[vv] = ema_rn(p[FS + vv], pv[vv], omt, theta);
                            p[vv] = pv[vv];
                        }
                        if (own_ptr[i] && own_row) {
                            Real* o = own_ptr[i] + (int64_t)yl * g.C;
#pragma unroll
                            for (int vv = 0; vv < VEC; ++vv) o[vv] = pv[vv];
                        }
                    }
                }
            }
            __syncthreads();
            Real* s2w = s2 + (size_t)(step & 1) * 2 * KT * PG_CC;         // this step's row
            const Real* s2r = s2 + (size_t)((step + 1) & 1) * 2 * KT * PG_CC;  // previous
            {   // stage 1 at band row v + L (y = v)
                Real ag = 0, am = 0;
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    const Real p = buf[(ty + t) * PG_CC + tx];
                    ag += Real(TP::g(t)) * p;
                    am += Real(TP::m(t)) * p;
                }
                r1g[(s + 2 * L) % T] = ag;
                r1m[(s + 2 * L) % T] = am;
                Real px = 0, py = 0;
#pragma unroll
                for (int b = 0; b < T; ++b) {
                    px += Real(TP::m(b)) * r1g[(s + b) % T];
                    py += Real(TP::g(b)) * r1m[(s + b) % T];
                }
                px *= inv_dx;
                py *= inv_dy;
                c1x[(s + L) % T] = px;
                c1y[(s + L) % T] = py;
                s2w[ty * PG_CC + tx] = px;
                s2w[(KT + ty) * PG_CC + tx] = py;
            }
            // stage 2: x pass (mass) at band row v - 1 + L, y pass (mass) -> row v - 1
            if (s2thr) {
                Real mx = 0, my = 0;
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    mx += Real(TP::m(t)) * s2r[(ty - L + t) * PG_CC + tx];
                    my += Real(TP::m(t)) * s2r[(KT + ty - L + t) * PG_CC + tx];
                }
                r2x[(s - 1 + L + T) % T] = mx;
                r2y[(s - 1 + L + T) % T] = my;
                const int vo = v - 1;
                if (xout && vo >= ua && vo < ub) {
                    Real mmx = 0, mmy = 0;
#pragma unroll
                    for (int b = 0; b < T; ++b) {
                        mmx += Real(TP::m(b)) * r2x[(s - 1 - L + b + 2 * T) % T];
                        mmy += Real(TP::m(b)) * r2y[(s - 1 - L + b + 2 * T) % T];
                    }
                    const Real px = c1x[(s - 1 + T) % T], py = c1y[(s - 1 + T) % T];
                    const Real rx = ar_mu * (mmx - px);
                    const Real ry = ar_nu * (mmy - py);
                    // min(dx|mu|, min(a_abs|R|dx/(eps+|p|), a_sq R^2 dx/(eps+|mu| p^2))), where a
                    // NaN candidate makes the result NaN and then 0 (numpy minimum +
                    // nan_to_num); dx|mu| is finite, so the min itself is never +-inf.
                    const Real bx = fast_div(cabs_x * fabs(rx), eps + fabs(px));
                    const Real sx = fast_div(csq_x * (rx * rx), eps + amu * (px * px));
                    const Real by = fast_div(cabs_y * fabs(ry), eps + fabs(py));
                    const Real sy = fast_div(csq_y * (ry * ry), eps + anu * (py * py));
                    const Real kx = (bx != bx || sx != sx) ? Real(0) : fmin(kxmax, fmin(bx, sx));
                    const Real ky = (by != by || sy != sy) ? Real(0) : fmin(kymax, fmin(by, sy));
                    const int64_t o = kbase_o + (int64_t)(vo - L) * g.C;
                    a.kx[o] = kx;
                    a.ky[o] = ky;
                }
            }
            if (step + S - 1 < nsteps)
                st.issue(vs + L + step + S - 1, sbase + ((step + S - 1) % S) * NF * FSB, FSB, a.psi);
            cp_async_commit();
            ++step;
        }
    }
    cp_async_wait<0>();
}

}  // namespace csn
