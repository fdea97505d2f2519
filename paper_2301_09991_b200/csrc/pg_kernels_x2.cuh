// fp32 PG residual / fused sweep with packed fp32x2 arithmetic (K3 / K5, sm_100a).
//
// Same operator as pg_residual_kernel (R/discretisation.py:227-276, fused sweep
// R/multigrid.py:159-172,301-304) and the same 2.5D y-march, re-shaped for the
// instruction-issue bound the scalar kernel hits:
//   * a lane owns a channel PAIR (CTA = 8 x cells x 64 channels): every tap is one
//     FFMA2 (f32x2.h), every staged read one LDS.64, index math is shared by 2 DOF;
//   * the y pass is a scatter: when lead row j's x pass is done it is added into the
//     T pending output accumulators (rows j-L .. j+L) instead of ringing the 6 x-pass
//     results and gathering them T steps later.  Terms that share a centre factor are
//     merged, so 4 rings of T float2 replace 6 rings + 3 centre rings:
//       A = M_y(mu/dx G_x psi + hx S_x(kx psi)) + G_y(nu/dy M_x psi) + S_y(hy M_x(ky psi))
//       B = M_y S_x psi          (x kx(y) hx)        C = S_y M_x psi   (x ky(y) hy)
//       D = -M_y(hx S_x kx) - S_y(hy M_x ky)         (x psi(y))
//       r = A + hx kx B + hy ky C + psi (D + sigma) - q
//   * centre values psi, kx, ky of the output row come from the staging ring, which is
//     S = L + 1 + P rows deep (P rows prefetched ahead + the L rows the output lags).
// The per-lane arithmetic is IEEE fp32 like the scalar kernel; only the summation
// order of the y pass differs (within the fp32 parity tolerance of the tests).
#pragma once
#include "pg_kernels.cuh"
#include "f32x2.cuh"

namespace csn {

constexpr int X2_CC = 64;        // channels per CTA: 32 lanes x 2
constexpr int X2_PREFETCH = 3;   // staged rows in flight ahead of the lead row

template <int L>
struct X2Stages { static constexpr int value = L + 1 + (L <= 3 ? X2_PREFETCH : 2); };

template <int L, int MODE>
constexpr size_t pg_residual_x2_smem() {
    return (size_t)X2Stages<L>::value * (MODE == PG_RESID ? 3 : 4) * (PG_TX + 2 * L) * X2_CC *
           sizeof(float);
}

template <int L, int MODE, int VEC>
__global__ void __launch_bounds__(32 * PG_TX, L <= 3 ? 2 : 1)
pg_residual_x2_kernel(const PGResidArgs<float> a) {
    constexpr bool SWEEP = MODE == PG_SWEEP;
    constexpr bool EMA = MODE == PG_RESID_EMA;
    using TP = UnitTaps<L>;
    constexpr int T = 2 * L + 1;
    constexpr int CC = X2_CC;
    constexpr int W = PG_TX + 2 * L;
    constexpr int NT = 32 * PG_TX;
    constexpr int G4 = CC / VEC;
    constexpr int NI = (W * G4 + NT - 1) / NT;     // staged items per thread
    constexpr int NF = MODE == PG_RESID ? 3 : 4;   // psi, kx, ky (, delta | pbar)
    constexpr int S = X2Stages<L>::value;
    constexpr int P = S - L - 1;
    constexpr int FS = W * CC;                     // floats per field row
    extern __shared__ __align__(16) unsigned char smraw[];
    float* sm = reinterpret_cast<float*>(smraw);
    __shared__ double red[32];

    const Geo& g = a.g;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * 32 + tx;
    const int c0 = blockIdx.y * CC;
    const int c = c0 + 2 * tx;                     // C = n_dir * n_group is even
    const bool cval = c < g.C;
    const int cs = cval ? c : g.C - 2;
    const int n0 = cs / g.ng, g0 = cs - n0 * g.ng;
    const int n1 = (cs + 1) / g.ng, g1 = cs + 1 - n1 * g.ng;
    const float2 mu_dx = make_float2(a.mu[n0] * a.inv_dx, a.mu[n1] * a.inv_dx);
    const float2 nu_dy = make_float2(a.nu[n0] * a.inv_dy, a.nu[n1] * a.inv_dy);
    const float2 hx = bc2(a.hx), hy = bc2(a.hy), mhx = bc2(-a.hx), mhy = bc2(-a.hy);
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
    Stager<float, VEC, NI, NF, 0x6, CC> st;
    st.init(g, fd, x0 - L, W, c0, L, a.mu, a.nu, tid, NT);
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);
    constexpr unsigned FSB = FS * sizeof(float);
    constexpr unsigned SLOTB = NF * FSB;

    // epilogue pointers at y = 0 (per output only y * stride is added)
    const int xs = act ? x : 0;
    const int64_t cell0 = (int64_t)xs * g.ny;
    const float* sig0 = a.sigma + cell0 * g.ng + g0;
    const float* sig1 = a.sigma + cell0 * g.ng + g1;
    const int qst = a.q_per_dof ? g.C : g.ng;
    const float* q0 = a.q + cell0 * qst + (a.q_per_dof ? cs : g0);
    const float* q1 = a.q + cell0 * qst + (a.q_per_dof ? cs + 1 : g1);
    float* o_p = SWEEP ? a.out + fidx(xs, 0, cs, g.ny, a.out_h, g.C)
                       : (a.r ? a.r + fidx(xs, 0, cs, g.ny, a.r_h, g.C) : nullptr);
    const float2 beta2 = bc2(a.beta);
    const float2 strm2 = a.strm ? make_float2(a.strm[n0], a.strm[n1]) : bc2(0.f);
    // fused iterate averaging (R/multigrid.py:217-225) on the interior cells this CTA
    // owns: elementwise; psi and pbar_old arrive through the staging ring
    float* avg_p[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        const int e = tid + i * NT;
        const int xi = e / G4, cc = c0 + (e % G4) * VEC;
        const int xg = x0 - L + xi;
        avg_p[i] = (EMA && e < W * G4 && cc < g.C && xi >= L && xi < L + PG_TX && xg < g.nx)
                       ? a.avg + fidx(xg, 0, cc, g.ny, a.avg_h, g.C) : nullptr;
    }
    const int oy0 = max(ya, 0), oy1 = yb;
    const int lane_off = ty * CC + 2 * tx;          // this lane's pair in a staged row

    float2 rA[T], rB[T], rC[T], rD[T];              // pending outputs, by (y - ya) mod T
#pragma unroll
    for (int i = 0; i < T; ++i) rA[i] = rB[i] = rC[i] = rD[i] = bc2(0.f);

#pragma unroll
    for (int k = 0; k < P; ++k) {
        if (k < nsteps) st.issue(ya - L + k, sbase + k * SLOTB, FSB, a.psi);
        cp_async_commit();
    }
    double l1 = 0.0;
    int slot = 0;   // staging slot of the current step (k mod S)
    // sigma, q of the next output row, loaded a step ahead of use
    float2 sgN = bc2(0.f), qN = bc2(0.f);
    if (act) {
        sgN = make_float2(sig0[ya * g.ng], sig1[ya * g.ng]);
        qN = make_float2(q0[ya * qst], q1[ya * qst]);
    }

    // One step: stage-ready lead row j = ya - L + K; SK = slot of output row j - L in
    // the pending rings; OUT: output row j - L = Y is complete after this step.
#define X2_STEP(K, SK, OUT, Y, SLOTC)                                                 \
    {                                                                                 \
        const int k_ = (K);                                                           \
        const int ss_ = (SLOTC) >= 0 ? (SLOTC) : slot;                                \
        float2 sg_ = sgN, q_ = qN;                                                    \
        if ((OUT) && act && (Y) + 1 < yb) {                                           \
            sgN = make_float2(sig0[((Y) + 1) * g.ng], sig1[((Y) + 1) * g.ng]);       \
            qN = make_float2(q0[((Y) + 1) * qst], q1[((Y) + 1) * qst]);              \
        }                                                                             \
        cp_async_wait<P - 1>();                                                       \
        float* buf_ = sm + ss_ * (NF * FS);                                          \
        if (SWEEP) {                                                                  \
            _Pragma("unroll") for (int i = 0; i < NI; ++i) {                          \
                const int e = tid + i * NT;                                           \
                if (e < W * G4) {                                                     \
                    float* p_ = buf_ + (e / G4) * CC + (e % G4) * VEC;                \
                    _Pragma("unroll") for (int v = 0; v < VEC; ++v) p_[v] -= p_[3 * FS + v]; \
                }                                                                     \
            }                                                                         \
        } else if (EMA) {                                                             \
            const int yl_ = ya - L + k_;                                              \
            if (yl_ >= oy0 && yl_ < oy1) {                                            \
                _Pragma("unroll") for (int i = 0; i < NI; ++i) {                      \
                    if (avg_p[i]) {                                                   \
                        const int e = tid + i * NT;                                   \
                        const float* p_ = buf_ + (e / G4) * CC + (e % G4) * VEC;      \
                        float* o_ = avg_p[i] + (int64_t)yl_ * g.C;                    \
                        _Pragma("unroll") for (int v = 0; v < VEC; ++v)               \
                            o_[v] = a.avg_mode == 2                                   \
                                        ? __fmaf_rn(p_[3 * FS + v], a.omt, __fmul_rn(a.theta, p_[v])) \
                                        : p_[v];                                      \
                    }                                                                 \
                }                                                                     \
            }                                                                         \
        }                                                                             \
        __syncthreads();                                                              \
        float2 a_g = bc2(0.f), a_m = a_g, a_s = a_g, a_sk = a_g, a_k = a_g, a_mk = a_g, a_ky = a_g; \
        {                                                                             \
            const float* bp_ = buf_ + lane_off;                                       \
            _Pragma("unroll") for (int t_ = 0; t_ < T; ++t_) {                        \
                const float2 p_ = ld2(bp_ + t_ * CC);                                \
                const float2 k1_ = ld2(bp_ + FS + t_ * CC);                          \
                const float2 k2_ = ld2(bp_ + 2 * FS + t_ * CC);                      \
                a_g = fma2c((float)TP::g(t_), p_, a_g);                               \
                a_m = fma2c((float)TP::m(t_), p_, a_m);                               \
                a_s = fma2c((float)TP::s(t_), p_, a_s);                               \
                a_sk = fma2c((float)TP::s(t_), mul2(p_, k1_), a_sk);                  \
                a_k = fma2c((float)TP::s(t_), k1_, a_k);                              \
                a_mk = fma2c((float)TP::m(t_), mul2(p_, k2_), a_mk);                  \
                a_ky = fma2c((float)TP::m(t_), k2_, a_ky);                            \
            }                                                                         \
        }                                                                             \
        const float2 xa_ = fma2(mu_dx, a_g, mul2(hx, a_sk));                          \
        const float2 xg_ = mul2(nu_dy, a_m);                                          \
        const float2 xs_ = mul2(hy, a_mk);                                            \
        const float2 xd1_ = mul2(mhx, a_k);                                           \
        const float2 xd2_ = mul2(mhy, a_ky);                                          \
        _Pragma("unroll") for (int i_ = 0; i_ < T; ++i_) {                            \
            const int sl_ = ((SK) + i_) % T;                                          \
            const int b_ = 2 * L - i_;                                                \
            const float m_ = (float)TP::m(b_), gt_ = (float)TP::g(b_), s_ = (float)TP::s(b_); \
            if (i_ == 2 * L) {                                                        \
                rA[sl_] = fma2c(m_, xa_, fma2c(gt_, xg_, mul2(bc2(s_), xs_)));        \
                rB[sl_] = mul2(bc2(m_), a_s);                                         \
                rC[sl_] = mul2(bc2(s_), a_m);                                         \
                rD[sl_] = fma2c(m_, xd1_, mul2(bc2(s_), xd2_));                       \
            } else {                                                                  \
                rA[sl_] = fma2c(m_, xa_, fma2c(gt_, xg_, fma2c(s_, xs_, rA[sl_])));   \
                rB[sl_] = fma2c(m_, a_s, rB[sl_]);                                    \
                rC[sl_] = fma2c(s_, a_m, rC[sl_]);                                    \
                rD[sl_] = fma2c(m_, xd1_, fma2c(s_, xd2_, rD[sl_]));                  \
            }                                                                         \
        }                                                                             \
        if ((OUT) && act && (Y) < yb) {                                               \
            const int y_ = (Y);                                                       \
            const int cs_ = ss_ >= L ? ss_ - L : ss_ - L + S;                      \
            const float* cb_ = sm + cs_ * (NF * FS) + L * CC + lane_off;              \
            const float2 pc_ = ld2(cb_), kxc_ = ld2(cb_ + FS), kyc_ = ld2(cb_ + 2 * FS); \
            float2 r_ = fma2(hx, mul2(kxc_, rB[SK]), rA[SK]);                         \
            r_ = fma2(hy, mul2(kyc_, rC[SK]), r_);                                    \
            r_ = sub2(fma2(pc_, add2(rD[SK], sg_), r_), q_);                          \
            if (SWEEP) {                                                              \
                const float2 d_ = mul2(beta2, add2(strm2, sg_));                      \
                const float2 inv_ = make_float2(rcp_nr(d_.x), rcp_nr(d_.y));          \
                float2 qt_ = mul2(r_, inv_);                                          \
                if (a.refine_div)                                                     \
                    qt_ = fma2(fma2(make_float2(-d_.x, -d_.y), qt_, r_), inv_, qt_);  \
                st2(o_p + (int64_t)y_ * g.C, sub2(pc_, qt_));                         \
            } else {                                                                  \
                if (o_p) st2(o_p + (int64_t)y_ * g.C, r_);                           \
                l1 += fabs((double)r_.x) + fabs((double)r_.y);                        \
            }                                                                         \
        }                                                                             \
        if (k_ + P < nsteps) {                                                        \
            const int is_ = ss_ + P >= S ? ss_ + P - S : ss_ + P;                  \
            st.issue(ya - L + k_ + P, sbase + is_ * SLOTB, FSB, a.psi);               \
        }                                                                             \
        cp_async_commit();                                                            \
        slot = ss_ + 1 == S ? 0 : ss_ + 1;                                              \
    }

    // prologue: lead rows ya-L .. ya+L-1 (outputs below ya are never emitted)
#pragma unroll
    for (int k = 0; k < 2 * L; ++k) X2_STEP(k, (k + 1) % T, false, 0, k % S);

    // when the staging ring is as deep as the tap count (p = 3: S = T = 7) the slot of
    // every unrolled step is a compile-time constant ((2l + s) mod S): shared addresses
    // fold into immediates instead of per-step select / multiply chains
    int kbase = 2 * L;
    for (int y0 = ya; y0 < yb; y0 += T, kbase += T) {
#pragma unroll
        for (int s = 0; s < T; ++s)
            X2_STEP(kbase + s, s, true, y0 + s, S == T ? (2 * L + s) % S : -1);
    }
#undef X2_STEP
    cp_async_wait<0>();
    if (!SWEEP && a.partials) {
        const double tot = block_sum(l1, red);
        if (threadIdx.x == 0 && threadIdx.y == 0)
            a.partials[((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = tot;
    }
}

// k of one channel (R/discretisation.py:150-158) with explicit rounding, shared by every
// fp32 diffusivity kernel so their k agree bit for bit:
//   b = (a_abs d) |R| / (eps + |p|),  s = (a_sq d) R^2 / (eps + |mu| p^2)   (x * rcp_nr),
//   k = NaN in b or s ? 0 : min(d |mu|, min(b, s))
__device__ __forceinline__ float k_coef(float R, float p, float cabs, float csq, float cap,
                                        float amu, float eps) {
    const float b = __fmul_rn(__fmul_rn(cabs, fabsf(R)), rcp_nr(__fadd_rn(eps, fabsf(p))));
    const float s = __fmul_rn(__fmul_rn(csq, __fmul_rn(R, R)),
                              rcp_nr(__fmaf_rn(amu, __fmul_rn(p, p), eps)));
    return (b != b || s != s) ? 0.f : fminf(cap, fminf(b, s));
}

// ---------------------------------------------------------------------------------
// K2 (fp32, L <= 3): iterate averaging fused with the anisotropic diffusivities
// (R/multigrid.py:217-225, R/discretisation.py:114-161), same two-stage march and
// operation order as pg_diffusivity_kernel with a lane per channel pair:
//   stage 1 (all KT cells): psi_x = M_y G_x pbar / dx, psi_y = G_y M_x pbar / dy;
//   stage 2 (inner KT - 2L cells, one step behind): R = alpha_r mu (M_y M_x psi_x - psi_x),
//   k = min(dx|mu|, min(a_abs |R| dx / (eps + |psi_x|), a_sq R^2 dx / (eps + |mu| psi_x^2)))
// Stage-1 rows live in an (L+2)-row shared ring: stage 2 reads its x neighbours from
// the previous row and the centre psi_x, psi_y of its output row from L+1 rows back,
// so only the four y-pass rings stay in registers.  (A one-stage form through the
// composite filters M*G, M*M removes the stage imbalance but reorders the rounding
// enough to push C2 fp32 past the 1e-5 flux tolerance, so the reference order stays.)
// ---------------------------------------------------------------------------------
constexpr int X2_KT = 16;

// resident CTAs per SM the split diffusivity kernels (K2a, K2b) are compiled for:
// 4 (<= 64 registers) at p = 3 (C4 K2 4.14 -> 4.03 ms), 3 below (C3 p = 1: 0.48 ms at
// 3, 0.50 ms at 4); tools/ab_k2minb.sh
#ifndef CSN_K2_MINB
#define CSN_K2_MINB (L >= 3 ? 4 : 3)
#endif   // stage-1 x cells per CTA

template <int L, bool EMA>
constexpr size_t pg_k_x2_smem() {
    return ((size_t)PGStages<float>::value * (EMA ? 2 : 1) * (X2_KT + 2 * L) * X2_CC +
            (size_t)(L + 2) * 2 * X2_KT * X2_CC) * sizeof(float);
}

// resident CTAs per SM of the fused diffusivity kernel: at p = 1 it fits 64 registers
// (2 CTAs/SM; C3 K2 0.46 -> 0.40 ms, C5-weak 21.9 -> 18.5 ms), above that it keeps 1
#ifndef CSN_K2F_MINB1
#define CSN_K2F_MINB1 2
#endif
template <int L, bool EMA, int VEC>
__global__ void __launch_bounds__(32 * X2_KT, L == 1 ? CSN_K2F_MINB1 : 1)
pg_diffusivity_x2_kernel(const PGKArgs<float> a) {
    using TP = UnitTaps<L>;
    constexpr int KT = X2_KT;
    constexpr int T = 2 * L + 1;
    constexpr int TXO = KT - 2 * L;
    constexpr int W1 = KT + 2 * L;
    constexpr int CC = X2_CC;
    constexpr int NT = 32 * KT;
    constexpr int G4 = CC / VEC;
    constexpr int NI = (W1 * G4 + NT - 1) / NT;
    constexpr int NF = EMA ? 2 : 1;               // psi (, pbar_old)
    constexpr int S = PGStages<float>::value;
    constexpr int FS = W1 * CC;
    constexpr int R2 = L + 2;                     // stage-1 row ring depth
    constexpr int F2 = KT * CC;                   // floats per stage-1 field row
    extern __shared__ __align__(16) unsigned char smraw[];
    float* s1 = reinterpret_cast<float*>(smraw);          // [S][NF][W1][CC]
    float* s2 = s1 + (size_t)S * NF * FS;                  // [R2][2][KT][CC]: psi_x, psi_y

    const Geo& g = a.g;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * 32 + tx;
    const int c0 = blockIdx.y * CC;
    const int c = c0 + 2 * tx;
    const bool cval = c < g.C;
    const int cs = cval ? c : g.C - 2;
    const int n0 = cs / g.ng, n1 = (cs + 1) / g.ng;
    const float mu0 = a.mu[n0], mu1 = a.mu[n1], nu0 = a.nu[n0], nu1 = a.nu[n1];
    const int x0o = -L + (int)blockIdx.x * TXO;   // first output x of this CTA
    const int x0s = x0o - L;                       // first stage-1 x
    const int xs = x0s + ty;
    const bool s2thr = ty >= L && ty < KT - L;
    const bool xout = s2thr && xs < g.nx + L && cval;
    const int ua = blockIdx.z * a.ly;                      // band rows u = y + L
    const int ub = min(g.ny + 2 * L, ua + a.ly);
    const int ox0 = max(x0o, 0), ox1 = min(x0o + TXO, g.nx);
    const int oy0 = max(ua - L, 0), oy1 = min(ub - L, g.ny);
    const float2 inv_dx = bc2(a.inv_dx), inv_dy = bc2(a.inv_dy);
    const float omt = a.omt, theta = a.theta;
    const bool write_avg = a.avg_mode != 0;

    constexpr int PRE = ((4 * L + T - 1) / T) * T;
    const int vs = ua - PRE;
    const int nsteps = PRE + (int)(((ub + 1 - ua) + T - 1) / T) * T;   // +1: stage-2 lag
    const int64_t kbase_o = fidx(xout ? xs : 0, 0, cs, g.ny, a.k_h, g.C);

    // the staged band is [-3l, nx+3l): the last CTA's overhang past it is never loaded
    // (past a ghost side it would run off the field)
    FieldDesc fd[2] = {{a.psi, a.psi_h, -3 * L, g.nx + 3 * L},
                       {a.avg_in, a.avg_in_h, -3 * L, g.nx + 3 * L}};
    Stager<float, VEC, NI, NF, 0, CC> st;
    st.init(g, fd, x0s - L, W1, c0, 0, a.mu, a.nu, tid, NT);
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(s1);
    constexpr unsigned FSB = FS * sizeof(float);
    float* own_ptr[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        const int e = tid + i * NT;
        const int xi = e / G4, q = e % G4;
        const int xg = x0s - L + xi, cc = c0 + q * VEC;
        own_ptr[i] = (write_avg && e < W1 * G4 && cc < g.C && xg >= ox0 && xg < ox1)
                         ? a.avg_out + fidx(xg, 0, cc, g.ny, a.avg_out_h, g.C) : nullptr;
    }
    const int lane1 = ty * CC + 2 * tx;         // this lane's pair in a staged pbar row
    const int lane2 = (ty - L) * CC + 2 * tx;   // stage-2 x pass start in a stage-1 row

    float2 r1g[T], r1m[T];   // stage-1 x pass of pbar (by pbar row)
    float2 r2x[T], r2y[T];   // M_x psi_x, M_x psi_y (by row)

#pragma unroll
    for (int k = 0; k < S - 1; ++k) {
        if (k < nsteps) st.issue(vs + L + k, sbase + k * NF * FSB, FSB, a.psi);
        cp_async_commit();
    }
    int step = 0;
    int q2 = 0;   // s2 slot of this step's stage-1 row (step mod R2)
    for (int v0 = vs; v0 <= ub; v0 += T) {
#pragma unroll
        for (int s = 0; s < T; ++s) {
            const int v = v0 + s;
            const int yl = v + L;                  // pbar lead row (y coords)
            cp_async_wait<S - 2>();
            float* buf = s1 + (size_t)(step % S) * NF * FS;
            if (EMA || write_avg) {                // form pbar on own items; write back owned
                const bool own_row = yl >= oy0 && yl < oy1;
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int e = tid + i * NT;
                    if (e < W1 * G4) {
                        float* p = buf + (e / G4) * CC + (e % G4) * VEC;
                        float pv[VEC];
#pragma unroll
                        for (int vv = 0; vv < VEC; ++vv) {
                            pv[vv] = p[vv];
                            if (EMA) pv[vv] = __fmaf_rn(p[FS + vv], omt, __fmul_rn(theta, pv[vv]));
                            p[vv] = pv[vv];
                        }
                        if (own_ptr[i] && own_row) {
                            float* o = own_ptr[i] + (int64_t)yl * g.C;
#pragma unroll
                            for (int vv = 0; vv < VEC; ++vv) o[vv] = pv[vv];
                        }
                    }
                }
            }
            __syncthreads();
            float* s2w = s2 + q2 * (2 * F2);                         // this step's row
            const int qp = q2 == 0 ? R2 - 1 : q2 - 1;                // previous step
            const int qc = q2 + 1 == R2 ? 0 : q2 + 1;                // L + 1 steps back
            {   // stage 1 at band row v + L (y = v)
                float2 ag = bc2(0.f), am = ag;
                const float* bp = buf + lane1;
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    const float2 p = ld2(bp + t * CC);
                    ag = fma2c((float)TP::g(t), p, ag);
                    am = fma2c((float)TP::m(t), p, am);
                }
                r1g[(s + 2 * L) % T] = ag;
                r1m[(s + 2 * L) % T] = am;
                float2 px = bc2(0.f), py = px;
#pragma unroll
                for (int b = 0; b < T; ++b) {
                    px = fma2c((float)TP::m(b), r1g[(s + b) % T], px);
                    py = fma2c((float)TP::g(b), r1m[(s + b) % T], py);
                }
                st2(s2w + ty * CC + 2 * tx, mul2(px, inv_dx));
                st2(s2w + F2 + ty * CC + 2 * tx, mul2(py, inv_dy));
            }
            // stage 2: x pass (mass) at band row v - 1 + L, y pass (mass) -> row v - 1
            if (s2thr) {
                const float* sr = s2 + qp * (2 * F2) + lane2;
                float2 mx = bc2(0.f), my = mx;
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    mx = fma2c((float)TP::m(t), ld2(sr + t * CC), mx);
                    my = fma2c((float)TP::m(t), ld2(sr + F2 + t * CC), my);
                }
                r2x[(s - 1 + L + T) % T] = mx;
                r2y[(s - 1 + L + T) % T] = my;
                const int vo = v - 1;
                if (xout && vo >= ua && vo < ub) {
                    float2 mmx = bc2(0.f), mmy = mmx;
#pragma unroll
                    for (int b = 0; b < T; ++b) {
                        mmx = fma2c((float)TP::m(b), r2x[(s - 1 - L + b + 2 * T) % T], mmx);
                        mmy = fma2c((float)TP::m(b), r2y[(s - 1 - L + b + 2 * T) % T], mmy);
                    }
                    const float* cb = s2 + qc * (2 * F2) + ty * CC + 2 * tx;
                    const float2 pxc = ld2(cb), pyc = ld2(cb + F2);
                    const float2 rx = mul2(make_float2(a.alpha_r * mu0, a.alpha_r * mu1),
                                           sub2(mmx, pxc));
                    const float2 ry = mul2(make_float2(a.alpha_r * nu0, a.alpha_r * nu1),
                                           sub2(mmy, pyc));
                    const float amu[2] = {fabsf(mu0), fabsf(mu1)}, anu[2] = {fabsf(nu0), fabsf(nu1)};
                    const float pxv[2] = {pxc.x, pxc.y}, pyv[2] = {pyc.x, pyc.y};
                    const float rxv[2] = {rx.x, rx.y}, ryv[2] = {ry.x, ry.y};
                    float kx[2], ky[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        kx[h] = k_coef(rxv[h], pxv[h], a.cax, a.csx,
                                       a.dx * amu[h], amu[h], a.eps);
                        ky[h] = k_coef(ryv[h], pyv[h], a.cay, a.csy,
                                       a.dy * anu[h], anu[h], a.eps);
                    }
                    const int64_t o = kbase_o + (int64_t)(vo - L) * g.C;
                    st2(a.kx + o, make_float2(kx[0], kx[1]));
                    st2(a.ky + o, make_float2(ky[0], ky[1]));
                }
            }
            if (step + S - 1 < nsteps)
                st.issue(vs + L + step + S - 1, sbase + ((step + S - 1) % S) * NF * FSB, FSB, a.psi);
            cp_async_commit();
            ++step;
            q2 = q2 + 1 == R2 ? 0 : q2 + 1;
        }
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------
// K2 split through a workspace (fp32, L <= 3): the two stages of the diffusivity
// kernel as two balanced y-marches (R/discretisation.py:114-161).  The fused
// two-stage CTA recomputes 2l stage-1 columns per 10 outputs and idles its 2l edge
// warps through stage 2 behind a CTA-wide barrier; through HBM each stage runs on
// every lane with no x redundancy, at 8 B/DOF written + read for psi_x, psi_y.
// Operation order is the fused kernel's, so k is bit-identical.
//   K2a pg_grad_x2_kernel:  pbar = (1-theta) pbar_old + theta psi (written back on the
//       owned interior), psi_x = M_y G_x pbar / dx, psi_y = G_y M_x pbar / dy on the
//       +-2l band;
//   K2b pg_kcoef_x2_kernel: R = alpha_r mu (M_y M_x psi_x - psi_x), k on the +-l band.
// ---------------------------------------------------------------------------------
template <int L, bool EMA>
constexpr size_t pg_grad_x2_smem() {
    return (size_t)PGStages<float>::value * (EMA ? 2 : 1) * (PG_TX + 2 * L) * X2_CC * sizeof(float);
}

template <int L, bool EMA, int VEC>
__global__ void __launch_bounds__(32 * PG_TX, CSN_K2_MINB)
pg_grad_x2_kernel(const PGKArgs<float> a, float* __restrict__ gx_out,
                  float* __restrict__ gy_out, int gh) {
    using TP = UnitTaps<L>;
    constexpr int T = 2 * L + 1;
    constexpr int CC = X2_CC;
    constexpr int W = PG_TX + 2 * L;
    constexpr int NT = 32 * PG_TX;
    constexpr int G4 = CC / VEC;
    constexpr int NI = (W * G4 + NT - 1) / NT;
    constexpr int NF = EMA ? 2 : 1;               // psi (, pbar_old)
    constexpr int S = PGStages<float>::value;
    constexpr int FS = W * CC;
    extern __shared__ __align__(16) unsigned char smraw[];
    float* sm = reinterpret_cast<float*>(smraw);

    const Geo& g = a.g;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * 32 + tx;
    const int c0 = blockIdx.y * CC;
    const int c = c0 + 2 * tx;
    const bool cval = c < g.C;
    const int cs = cval ? c : g.C - 2;
    const int x0 = -2 * L + (int)blockIdx.x * PG_TX;         // band x in [-2l, nx+2l)
    const int x = x0 + ty;
    const bool act = x < g.nx + 2 * L && cval;
    const int ya = -2 * L + (int)blockIdx.z * a.ly;          // band y in [-2l, ny+2l)
    const int yb = min(g.ny + 2 * L, ya + a.ly);
    const int ox0 = max(x0, 0), ox1 = min(x0 + PG_TX, g.nx);
    const int oy0 = max(ya, 0), oy1 = min(yb, g.ny);
    const float2 inv_dx = bc2(a.inv_dx), inv_dy = bc2(a.inv_dy);
    const float omt = a.omt, theta = a.theta;
    const bool write_avg = a.avg_mode != 0;
    const int nsteps = 2 * L + (int)(((yb - ya) + T - 1) / T) * T;
    const int64_t ob = fidx(act ? x : 0, 0, cs, g.ny, gh, g.C);

    // the staged band is [-3l, nx+3l): the last CTA's overhang past it is never loaded
    // (past a ghost side it would run off the field)
    FieldDesc fd[2] = {{a.psi, a.psi_h, -3 * L, g.nx + 3 * L},
                       {a.avg_in, a.avg_in_h, -3 * L, g.nx + 3 * L}};
    Stager<float, VEC, NI, NF, 0, CC> st;
    st.init(g, fd, x0 - L, W, c0, 0, a.mu, a.nu, tid, NT);
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);
    constexpr unsigned FSB = FS * sizeof(float);
    float* own_ptr[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        const int e = tid + i * NT;
        const int xi = e / G4, q = e % G4;
        const int xg = x0 - L + xi, cc = c0 + q * VEC;
        own_ptr[i] = (write_avg && e < W * G4 && cc < g.C && xg >= ox0 && xg < ox1)
                         ? a.avg_out + fidx(xg, 0, cc, g.ny, a.avg_out_h, g.C) : nullptr;
    }
    const int lane = ty * CC + 2 * tx;
    float2 rG[T], rM[T];   // x pass G, M of pbar by lead row (step mod T)

#pragma unroll
    for (int k = 0; k < S - 1; ++k) {
        if (k < nsteps) st.issue(ya - L + k, sbase + k * NF * FSB, FSB, a.psi);
        cp_async_commit();
    }
    // K: step (lead row ya - L + K); KR = K mod T (compile time); output row Y = lead - l
#define K2A_STEP(K, KR, OUT, Y)                                                                    \
{                                                                                                  \
    const int k_ = (K);                                                                            \
    const int yl_ = ya - L + k_;                                                                   \
    cp_async_wait<S - 2>();                                                                        \
    float* buf_ = sm + (size_t)(k_ % S) * NF * FS;                                                 \
    if (EMA || write_avg) {                                                                        \
        const bool own_row_ = yl_ >= oy0 && yl_ < oy1;                                             \
        _Pragma("unroll") for (int i = 0; i < NI; ++i) {                                           \
            const int e = tid + i * NT;                                                            \
            if (e < W * G4) {                                                                      \
                float* p_ = buf_ + (e / G4) * CC + (e % G4) * VEC;                                 \
                float pv_[VEC];                                                                    \
                _Pragma("unroll") for (int vv = 0; vv < VEC; ++vv) {                               \
                    pv_[vv] = p_[vv];                                                              \
                    if (EMA) pv_[vv] = __fmaf_rn(p_[FS + vv], omt, __fmul_rn(theta, pv_[vv]));     \
                    p_[vv] = pv_[vv];                                                              \
                }                                                                                  \
                if (own_ptr[i] && own_row_) {                                                      \
                    float* o_ = own_ptr[i] + (int64_t)yl_ * g.C;                                   \
                    _Pragma("unroll") for (int vv = 0; vv < VEC; ++vv) o_[vv] = pv_[vv];           \
                }                                                                                  \
            }                                                                                      \
        }                                                                                          \
    }                                                                                              \
    __syncthreads();                                                                               \
    {                                                                                              \
        float2 ag_ = bc2(0.f), am_ = ag_;                                                          \
        const float* bp_ = buf_ + lane;                                                            \
        _Pragma("unroll") for (int t = 0; t < T; ++t) {                                            \
            const float2 p_ = ld2(bp_ + t * CC);                                                   \
            ag_ = fma2c((float)TP::g(t), p_, ag_);                                                 \
            am_ = fma2c((float)TP::m(t), p_, am_);                                                 \
        }                                                                                          \
        rG[(KR)] = ag_;                                                                            \
        rM[(KR)] = am_;                                                                            \
    }                                                                                              \
    if ((OUT) && act && (Y) < yb) {                                                                \
        float2 px_ = bc2(0.f), py_ = px_;                                                          \
        _Pragma("unroll") for (int b = 0; b < T; ++b) {                                            \
            px_ = fma2c((float)TP::m(b), rG[((KR) + 1 + b) % T], px_);                             \
            py_ = fma2c((float)TP::g(b), rM[((KR) + 1 + b) % T], py_);                             \
        }                                                                                          \
        const int64_t o_ = ob + (int64_t)(Y) * g.C;                                                \
        st2(gx_out + o_, mul2(px_, inv_dx));                                                       \
        st2(gy_out + o_, mul2(py_, inv_dy));                                                       \
    }                                                                                              \
    if (k_ + S - 1 < nsteps) st.issue(ya - L + k_ + S - 1, sbase + ((k_ + S - 1) % S) * NF * FSB, FSB, a.psi); \
    cp_async_commit();                                                                             \
}
#pragma unroll
    for (int k = 0; k < 2 * L; ++k) K2A_STEP(k, k % T, false, 0);
    int kb = 2 * L;
    for (int y0 = ya; y0 < yb; y0 += T, kb += T) {
#pragma unroll
        for (int s = 0; s < T; ++s) K2A_STEP(kb + s, (2 * L + s) % T, true, y0 + s);
    }
#undef K2A_STEP
    cp_async_wait<0>();
}

template <int L>
constexpr size_t pg_kcoef_x2_smem() {
    return (size_t)X2Stages<L>::value * 2 * (PG_TX + 2 * L) * X2_CC * sizeof(float);
}

template <int L, int VEC>
__global__ void __launch_bounds__(32 * PG_TX, CSN_K2_MINB)
pg_kcoef_x2_kernel(const PGKArgs<float> a, const float* __restrict__ gx_in,
                   const float* __restrict__ gy_in, int gh) {
    using TP = UnitTaps<L>;
    constexpr int T = 2 * L + 1;
    constexpr int CC = X2_CC;
    constexpr int W = PG_TX + 2 * L;
    constexpr int NT = 32 * PG_TX;
    constexpr int G4 = CC / VEC;
    constexpr int NI = (W * G4 + NT - 1) / NT;
    constexpr int NF = 2;                          // psi_x, psi_y
    constexpr int S = X2Stages<L>::value;
    constexpr int P = S - L - 1;
    constexpr int FS = W * CC;
    extern __shared__ __align__(16) unsigned char smraw[];
    float* sm = reinterpret_cast<float*>(smraw);

    const Geo& g = a.g;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * 32 + tx;
    const int c0 = blockIdx.y * CC;
    const int c = c0 + 2 * tx;
    const bool cval = c < g.C;
    const int cs = cval ? c : g.C - 2;
    const int n0 = cs / g.ng, n1 = (cs + 1) / g.ng;
    const float mu0 = a.mu[n0], mu1 = a.mu[n1], nu0 = a.nu[n0], nu1 = a.nu[n1];
    const int x0 = -L + (int)blockIdx.x * PG_TX;             // band x in [-l, nx+l)
    const int x = x0 + ty;
    const bool act = x < g.nx + L && cval;
    const int ya = -L + (int)blockIdx.z * a.ly;              // band y in [-l, ny+l)
    const int yb = min(g.ny + L, ya + a.ly);
    const int nsteps = 2 * L + (int)(((yb - ya) + T - 1) / T) * T;
    const int64_t kb0 = fidx(act ? x : 0, 0, cs, g.ny, a.k_h, g.C);

    FieldDesc fd[2] = {{gx_in, gh}, {gy_in, gh}};
    Stager<float, VEC, NI, NF, 0x3, CC> st;        // both band fields, zero outside +-2l
    st.init(g, fd, x0 - L, W, c0, 2 * L, a.mu, a.nu, tid, NT);
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);
    constexpr unsigned FSB = FS * sizeof(float);
    constexpr unsigned SLOTB = NF * FSB;
    const int lane = ty * CC + 2 * tx;
    float2 r2x[T], r2y[T];   // M_x psi_x, M_x psi_y by lead row (step mod T)

#pragma unroll
    for (int k = 0; k < P; ++k) {
        if (k < nsteps) st.issue(ya - L + k, sbase + k * SLOTB, FSB, gx_in);
        cp_async_commit();
    }
    int slot = 0;
#define K2B_STEP(K, KR, OUT, Y, SLOTC)                                                             \
{                                                                                                  \
    const int k_ = (K);                                                                            \
    const int ss_ = (SLOTC) >= 0 ? (SLOTC) : slot;                                                 \
    cp_async_wait<P - 1>();                                                                        \
    __syncthreads();                                                                               \
    const float* buf_ = sm + ss_ * (NF * FS) + lane;                                              \
    float2 mx_ = bc2(0.f), my_ = mx_;                                                              \
    _Pragma("unroll") for (int t = 0; t < T; ++t) {                                                \
        mx_ = fma2c((float)TP::m(t), ld2(buf_ + t * CC), mx_);                                     \
        my_ = fma2c((float)TP::m(t), ld2(buf_ + FS + t * CC), my_);                                \
    }                                                                                              \
    r2x[(KR)] = mx_;                                                                               \
    r2y[(KR)] = my_;                                                                               \
    if ((OUT) && act && (Y) < yb) {                                                                \
        float2 mmx = bc2(0.f), mmy = mmx;                                                          \
        _Pragma("unroll") for (int b = 0; b < T; ++b) {                                            \
            mmx = fma2c((float)TP::m(b), r2x[((KR) + 1 + b) % T], mmx);                            \
            mmy = fma2c((float)TP::m(b), r2y[((KR) + 1 + b) % T], mmy);                            \
        }                                                                                          \
        const int cs_ = ss_ >= L ? ss_ - L : ss_ - L + S;                                       \
        const float* cb = sm + cs_ * (NF * FS) + L * CC + lane;                                    \
        const float2 pxc = ld2(cb), pyc = ld2(cb + FS);                                            \
        const float2 rx = mul2(make_float2(a.alpha_r * mu0, a.alpha_r * mu1), sub2(mmx, pxc));     \
        const float2 ry = mul2(make_float2(a.alpha_r * nu0, a.alpha_r * nu1), sub2(mmy, pyc));     \
        const float amu[2] = {fabsf(mu0), fabsf(mu1)}, anu[2] = {fabsf(nu0), fabsf(nu1)};          \
        const float pxv[2] = {pxc.x, pxc.y}, pyv[2] = {pyc.x, pyc.y};                              \
        const float rxv[2] = {rx.x, rx.y}, ryv[2] = {ry.x, ry.y};                                  \
        float kx[2], ky[2];                                                                        \
        _Pragma("unroll") for (int h = 0; h < 2; ++h) {                                                    \
            kx[h] = k_coef(rxv[h], pxv[h], a.cax, a.csx, a.dx * amu[h],         \
                           amu[h], a.eps);                                                       \
            ky[h] = k_coef(ryv[h], pyv[h], a.cay, a.csy, a.dy * anu[h],         \
                           anu[h], a.eps);                                                       \
        }                                                                                        \
        const int64_t o = kb0 + (int64_t)(Y) * g.C;                                                \
        st2(a.kx + o, make_float2(kx[0], kx[1]));                                                  \
        st2(a.ky + o, make_float2(ky[0], ky[1]));                                                  \
    }                                                                                              \
    if (k_ + P < nsteps) {                                                                         \
        const int is_ = ss_ + P >= S ? ss_ + P - S : ss_ + P;                                   \
        st.issue(ya - L + k_ + P, sbase + is_ * SLOTB, FSB, gx_in);                                \
    }                                                                                              \
    cp_async_commit();                                                                             \
    slot = ss_ + 1 == S ? 0 : ss_ + 1;                                                           \
}
#pragma unroll
    for (int k = 0; k < 2 * L; ++k) K2B_STEP(k, k % T, false, 0, k % S);
    int kb = 2 * L;
    for (int y0 = ya; y0 < yb; y0 += T, kb += T) {
#pragma unroll
        for (int s = 0; s < T; ++s)
            K2B_STEP(kb + s, (2 * L + s) % T, true, y0 + s, S == T ? (2 * L + s) % S : -1);
    }
#undef K2B_STEP
    cp_async_wait<0>();
}

}  // namespace csn
