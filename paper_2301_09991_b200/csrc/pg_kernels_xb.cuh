// fp32 PG residual / fused sweep, register-blocked in x (K3 / K5 variant, sm_100a).
//
// pg_residual_x2_kernel (pg_kernels_x2.cuh) gives every warp one x cell: its x pass
// reads T staged columns of psi, kx, ky per output (3T LDS.64) and forms the products
// psi*kx, psi*ky per tap, so the shared-memory pipe (84 B per DOF) and the FMUL2s sit
// next to the FMA pipe as co-limiters.  Here a lane owns a channel pair at TWO
// adjacent x cells: the x pass reads T + 1 columns for both outputs (24 instead of 42
// LDS.64 for p = 3), computes each product once, and the CTA stages 2 NW cells with
// one 2l halo (less staging per DOF).  The price is a second set of y-scatter rings
// (8 rings of T float2), so the kernel runs at ~190 registers, NW warps per CTA.
// Arithmetic per output (tap order of the x pass, the scatter order of the y pass,
// the epilogue) is the x2 kernel's, so results are bit-identical to it
// (tests/test_gpu_parity.py::test_xblocked_residual_matches_x2).
// Operator: R/discretisation.py:227-276; fused sweep R/multigrid.py:159-172,301-304.
#pragma once
#include "pg_kernels_x2.cuh"

namespace csn {

template <int L, int MODE, int NW>
constexpr size_t pg_residual_xb_smem() {
    return (size_t)X2Stages<L>::value * (MODE == PG_RESID ? 3 : 4) * (2 * NW + 2 * L) * X2_CC *
           sizeof(float);
}

template <int L, int MODE, int VEC, int NW>
__global__ void __launch_bounds__(32 * NW, NW <= 4 ? 2 : 1)
pg_residual_xb_kernel(const PGResidArgs<float> a) {
    constexpr bool SWEEP = MODE == PG_SWEEP;
    constexpr bool EMA = MODE == PG_RESID_EMA;
    using TP = UnitTaps<L>;
    constexpr int T = 2 * L + 1;
    constexpr int CC = X2_CC;
    constexpr int XC = 2 * NW;                     // x cells per CTA
    constexpr int W = XC + 2 * L;
    constexpr int NT = 32 * NW;
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
    const int x0 = blockIdx.x * XC;
    const int xa = x0 + 2 * ty;                    // this lane's cells xa, xa + 1
    bool act[2];
    act[0] = xa < g.nx && cval;
    act[1] = xa + 1 < g.nx && cval;
    const int ya = blockIdx.z * a.ly;
    const int yb = min(g.ny, ya + a.ly);
    const int nsteps = 2 * L + (int)(((yb - ya) + T - 1) / T) * T;   // lead rows ya-L ...

    FieldDesc fd[4] = {{a.psi, a.psi_h, -L, g.nx + L}, {a.kx, a.k_h}, {a.ky, a.k_h},
                       {SWEEP ? a.delta : a.avg, SWEEP ? a.delta_h : a.avg_h, -L, g.nx + L}};
    // psi / delta staged only on [-l, nx+l): the last CTA's overhang (nx % TX != 0)
    // is never read by an output and would run past a ghost side's stored rows
    if (EMA) { fd[3].xlo = x0; fd[3].xhi = min(x0 + XC, g.nx); }   // owned columns only
    Stager<float, VEC, NI, NF, 0x6, CC> st;
    st.init(g, fd, x0 - L, W, c0, L, a.mu, a.nu, tid, NT);
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);
    constexpr unsigned FSB = FS * sizeof(float);
    constexpr unsigned SLOTB = NF * FSB;

    // epilogue pointers at y = 0 of cell xa (cell xa + 1 is one x stride further)
    const int xs = act[0] ? xa : 0;
    const int64_t cell0 = (int64_t)xs * g.ny;
    const int64_t sxs = (int64_t)g.ny * g.ng;      // sigma x stride
    const float* sig0 = a.sigma + cell0 * g.ng + g0;
    const float* sig1 = a.sigma + cell0 * g.ng + g1;
    const int qst = a.q_per_dof ? g.C : g.ng;
    const int64_t sxq = (int64_t)g.ny * qst;
    const float* q0 = a.q + cell0 * qst + (a.q_per_dof ? cs : g0);
    const float* q1 = a.q + cell0 * qst + (a.q_per_dof ? cs + 1 : g1);
    float* o_p = SWEEP ? a.out + fidx(xs, 0, cs, g.ny, a.out_h, g.C)
                       : (a.r ? a.r + fidx(xs, 0, cs, g.ny, a.r_h, g.C) : nullptr);
    const int64_t sxo = SWEEP ? (int64_t)(g.ny + 2 * a.out_h) * g.C
                              : (int64_t)(g.ny + 2 * a.r_h) * g.C;
    const float2 beta2 = bc2(a.beta);
    const float2 strm2 = a.strm ? make_float2(a.strm[n0], a.strm[n1]) : bc2(0.f);
    float* avg_p[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
        const int e = tid + i * NT;
        const int xi = e / G4, cc = c0 + (e % G4) * VEC;
        const int xg = x0 - L + xi;
        avg_p[i] = (EMA && e < W * G4 && cc < g.C && xi >= L && xi < L + XC && xg < g.nx)
                       ? a.avg + fidx(xg, 0, cc, g.ny, a.avg_h, g.C) : nullptr;
    }
    const int oy0 = max(ya, 0), oy1 = yb;
    const int lane_off = 2 * ty * CC + 2 * tx;      // this lane's pair at column xa - L

    float2 rA[2][T], rB[2][T], rC[2][T], rD[2][T];  // pending outputs, by (y - ya) mod T
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < T; ++i) rA[h][i] = rB[h][i] = rC[h][i] = rD[h][i] = bc2(0.f);

#pragma unroll
    for (int k = 0; k < P; ++k) {
        if (k < nsteps) st.issue(ya - L + k, sbase + k * SLOTB, FSB, a.psi);
        cp_async_commit();
    }
    double l1 = 0.0;
    int slot = 0;
    float2 sgN[2], qN[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        sgN[h] = bc2(0.f); qN[h] = bc2(0.f);
        if (act[h]) {
            sgN[h] = make_float2(sig0[h * sxs + ya * g.ng], sig1[h * sxs + ya * g.ng]);
            qN[h] = make_float2(q0[h * sxq + ya * qst], q1[h * sxq + ya * qst]);
        }
    }

#define XB_STEP(K, SK, OUT, Y)                                                                     \
    {                                                                                              \
        const int k_ = (K);                                                                        \
        float2 sg_[2], q_[2];                                                                      \
        _Pragma("unroll") for (int h = 0; h < 2; ++h) {                                            \
            sg_[h] = sgN[h]; q_[h] = qN[h];                                                        \
            if ((OUT) && act[h] && (Y) + 1 < yb) {                                                 \
                sgN[h] = make_float2(sig0[h * sxs + ((Y) + 1) * g.ng], sig1[h * sxs + ((Y) + 1) * g.ng]); \
                qN[h] = make_float2(q0[h * sxq + ((Y) + 1) * qst], q1[h * sxq + ((Y) + 1) * qst]); \
            }                                                                                      \
        }                                                                                          \
        cp_async_wait<P - 1>();                                                                    \
        float* buf_ = sm + slot * (NF * FS);                                                       \
        if (SWEEP) {                                                                               \
            _Pragma("unroll") for (int i = 0; i < NI; ++i) {                                       \
                const int e = tid + i * NT;                                                        \
                if (e < W * G4) {                                                                  \
                    float* p_ = buf_ + (e / G4) * CC + (e % G4) * VEC;                             \
                    _Pragma("unroll") for (int v = 0; v < VEC; ++v) p_[v] -= p_[3 * FS + v];       \
                }                                                                                  \
            }                                                                                      \
        } else if (EMA) {                                                                          \
            const int yl_ = ya - L + k_;                                                           \
            if (yl_ >= oy0 && yl_ < oy1) {                                                         \
                _Pragma("unroll") for (int i = 0; i < NI; ++i) {                                   \
                    if (avg_p[i]) {                                                                \
                        const int e = tid + i * NT;                                                \
                        const float* p_ = buf_ + (e / G4) * CC + (e % G4) * VEC;                   \
                        float* o_ = avg_p[i] + (int64_t)yl_ * g.C;                                 \
                        _Pragma("unroll") for (int v = 0; v < VEC; ++v)                            \
                            o_[v] = a.avg_mode == 2                                                \
                                        ? __fmaf_rn(p_[3 * FS + v], a.omt, __fmul_rn(a.theta, p_[v])) \
                                        : p_[v];                                                   \
                    }                                                                              \
                }                                                                                  \
            }                                                                                      \
        }                                                                                          \
        __syncthreads();                                                                           \
        float2 a_g[2], a_m[2], a_s[2], a_sk[2], a_k[2], a_mk[2], a_ky[2];                          \
        _Pragma("unroll") for (int h = 0; h < 2; ++h)                                              \
            a_g[h] = a_m[h] = a_s[h] = a_sk[h] = a_k[h] = a_mk[h] = a_ky[h] = bc2(0.f);            \
        {                                                                                          \
            const float* bp_ = buf_ + lane_off;                                                    \
            _Pragma("unroll") for (int t_ = 0; t_ <= T; ++t_) {                                    \
                const float2 p_ = ld2(bp_ + t_ * CC);                                              \
                const float2 k1_ = ld2(bp_ + FS + t_ * CC);                                        \
                const float2 k2_ = ld2(bp_ + 2 * FS + t_ * CC);                                    \
                const float2 pk1_ = mul2(p_, k1_), pk2_ = mul2(p_, k2_);                           \
                _Pragma("unroll") for (int h = 0; h < 2; ++h) {                                    \
                    const int tt_ = t_ - h;                                                        \
                    if (tt_ >= 0 && tt_ < T) {                                                     \
                        a_g[h] = fma2c((float)TP::g(tt_), p_, a_g[h]);                             \
                        a_m[h] = fma2c((float)TP::m(tt_), p_, a_m[h]);                             \
                        a_s[h] = fma2c((float)TP::s(tt_), p_, a_s[h]);                             \
                        a_sk[h] = fma2c((float)TP::s(tt_), pk1_, a_sk[h]);                         \
                        a_k[h] = fma2c((float)TP::s(tt_), k1_, a_k[h]);                            \
                        a_mk[h] = fma2c((float)TP::m(tt_), pk2_, a_mk[h]);                         \
                        a_ky[h] = fma2c((float)TP::m(tt_), k2_, a_ky[h]);                          \
                    }                                                                              \
                }                                                                                  \
            }                                                                                      \
        }                                                                                          \
        _Pragma("unroll") for (int h = 0; h < 2; ++h) {                                            \
            const float2 xa_ = fma2(mu_dx, a_g[h], mul2(hx, a_sk[h]));                             \
            const float2 xg_ = mul2(nu_dy, a_m[h]);                                                \
            const float2 xs_ = mul2(hy, a_mk[h]);                                                  \
            const float2 xd1_ = mul2(mhx, a_k[h]);                                                 \
            const float2 xd2_ = mul2(mhy, a_ky[h]);                                                \
            _Pragma("unroll") for (int i_ = 0; i_ < T; ++i_) {                                     \
                const int sl_ = ((SK) + i_) % T;                                                   \
                const int b_ = 2 * L - i_;                                                         \
                const float m_ = (float)TP::m(b_), gt_ = (float)TP::g(b_), s_ = (float)TP::s(b_);  \
                if (i_ == 2 * L) {                                                                 \
                    rA[h][sl_] = fma2c(m_, xa_, fma2c(gt_, xg_, mul2(bc2(s_), xs_)));              \
                    rB[h][sl_] = mul2(bc2(m_), a_s[h]);                                            \
                    rC[h][sl_] = mul2(bc2(s_), a_m[h]);                                            \
                    rD[h][sl_] = fma2c(m_, xd1_, mul2(bc2(s_), xd2_));                             \
                } else {                                                                           \
                    rA[h][sl_] = fma2c(m_, xa_, fma2c(gt_, xg_, fma2c(s_, xs_, rA[h][sl_])));      \
                    rB[h][sl_] = fma2c(m_, a_s[h], rB[h][sl_]);                                    \
                    rC[h][sl_] = fma2c(s_, a_m[h], rC[h][sl_]);                                    \
                    rD[h][sl_] = fma2c(m_, xd1_, fma2c(s_, xd2_, rD[h][sl_]));                     \
                }                                                                                  \
            }                                                                                      \
        }                                                                                          \
        if ((OUT) && (Y) < yb) {                                                                   \
            const int y_ = (Y);                                                                    \
            const int cs_ = slot >= L ? slot - L : slot - L + S;                                   \
            _Pragma("unroll") for (int h = 0; h < 2; ++h) {                                        \
                if (act[h]) {                                                                      \
                    const float* cb_ = sm + cs_ * (NF * FS) + (L + h) * CC + lane_off;             \
                    const float2 pc_ = ld2(cb_), kxc_ = ld2(cb_ + FS), kyc_ = ld2(cb_ + 2 * FS);   \
                    float2 r_ = fma2(hx, mul2(kxc_, rB[h][SK]), rA[h][SK]);                        \
                    r_ = fma2(hy, mul2(kyc_, rC[h][SK]), r_);                                      \
                    r_ = sub2(fma2(pc_, add2(rD[h][SK], sg_[h]), r_), q_[h]);                      \
                    if (SWEEP) {                                                                   \
                        const float2 d_ = mul2(beta2, add2(strm2, sg_[h]));                        \
                        const float2 inv_ = make_float2(rcp_nr(d_.x), rcp_nr(d_.y));               \
                        float2 qt_ = mul2(r_, inv_);                                               \
                        if (a.refine_div)                                                          \
                            qt_ = fma2(fma2(make_float2(-d_.x, -d_.y), qt_, r_), inv_, qt_);       \
                        st2(o_p + h * sxo + (int64_t)y_ * g.C, sub2(pc_, qt_));                    \
                    } else {                                                                       \
                        if (o_p) st2(o_p + h * sxo + (int64_t)y_ * g.C, r_);                       \
                        l1 += fabs((double)r_.x) + fabs((double)r_.y);                             \
                    }                                                                              \
                }                                                                                  \
            }                                                                                      \
        }                                                                                          \
        if (k_ + P < nsteps) {                                                                     \
            const int is_ = slot + P >= S ? slot + P - S : slot + P;                               \
            st.issue(ya - L + k_ + P, sbase + is_ * SLOTB, FSB, a.psi);                            \
        }                                                                                          \
        cp_async_commit();                                                                         \
        slot = slot + 1 == S ? 0 : slot + 1;                                                       \
    }

    // prologue: lead rows ya-L .. ya+L-1 (outputs below ya are never emitted)
#pragma unroll
    for (int k = 0; k < 2 * L; ++k) XB_STEP(k, (k + 1) % T, false, 0);

    int kbase = 2 * L;
    for (int y0 = ya; y0 < yb; y0 += T, kbase += T) {
#pragma unroll
        for (int s = 0; s < T; ++s) XB_STEP(kbase + s, s, true, y0 + s);
    }
#undef XB_STEP
    cp_async_wait<0>();
    if (!SWEEP && a.partials) {
        const double tot = block_sum(l1, red);
        if (threadIdx.x == 0 && threadIdx.y == 0)
            a.partials[((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = tot;
    }
}

}  // namespace csn
