// fp32 PG residual / fused sweep (K3 / K3E / K5) with TMA row staging and an mbarrier
// producer/consumer ring (sm_100a).
//
// Same operator, lane mapping (channel pairs, FFMA2) and arithmetic as
// pg_residual_x2_kernel — results are bit-identical — with the staging re-done the
// Blackwell way:
//   * one elected thread stages a whole cell row of every field with
//     cp.async.bulk.tensor (TMA, a 3D tensor map over the padded [x][y][channel]
//     field, box = W cells x 1 row x 64 channels); no per-thread address / vacuum-rule
//     math, no per-thread LDGSTS;
//   * slot readiness is an mbarrier with a transaction count (full[s]); slot reuse is
//     a second mbarrier that each warp arrives on after its last read of the row
//     (empty[s], 8 arrivals).  There is no CTA-wide barrier in the march: a warp only
//     waits for data, so warps drift up to P rows apart instead of lock-stepping.
// Halos are read AS STORED, like the reference's pg_residual (R/discretisation.py:
// 239-276 works on psi.data with its stored halo): the caller applies the boundary
// first (sawtooth_cycle does, R/multigrid.py:166,277,305) and k is zero outside its
// band.  The sweep's psi' = psi - delta is formed at each read (delta padded by >= L
// with its boundary applied); the frozen-cycle iterate average reads pbar_old through
// a second (8-cell) box and writes pbar from the consuming thread.
#pragma once
#include "pg_kernels_x2.cuh"
#include "tma_util.cuh"

namespace csn {

struct PGTmaMaps {
    CUtensorMap psi, kx, ky, aux;   // aux: delta (sweep) or pbar_old (EMA)
};

// ring geometry: a slot holds psi, kx, ky rows (W cells) plus delta (W cells, sweep) or
// pbar_old (the CTA's PG_TX cells, EMA); PREFETCH rows are in flight ahead of the
// lead row.  (Measured and not kept: a warp-private shared stash of each warp's centre
// psi', kx, ky that frees a row's slot right after its lead-row step, so S - 1 rows are
// in flight instead of S - L - 1 — C4 sweep 3.18 -> 3.33 ms, residual 3.04 -> 3.23 ms:
// the march does not wait on TMA latency.)
template <int L, int MODE>
struct TmaRing {
    static constexpr int FS = (PG_TX + 2 * L) * X2_CC;
    static constexpr int SLOT = 3 * FS + (MODE == PG_SWEEP ? FS : MODE == PG_RESID_EMA ? PG_TX * X2_CC : 0);
    // L = 3: S = T = 7 (4-5 rows ahead measured slower: spills, less L1); L = 1: S = 2T = 6
    // (prefetch depth 3-7 measured equal on C3, C5-weak; S a multiple of T keeps the ring
    // slot of every unrolled step a compile-time constant)
    static constexpr int PREFETCH = L > 3 ? 2 : (L == 1 ? 4 : 3);
    static constexpr int S = L + 1 + PREFETCH;
    static constexpr int T = 2 * L + 1;
    static constexpr int U = S % T == 0 ? S : T;     // steps per unrolled march iteration
};

template <int L, int MODE>
constexpr size_t pg_residual_tma_smem() {
    return (size_t)TmaRing<L, MODE>::S * TmaRing<L, MODE>::SLOT * sizeof(float) +
           128;   // + alignment slack (TMA destinations: 128 B)
}

// resident CTAs per SM the TMA residual / sweep is compiled for.  The linear (p = 1)
// march fits 80 registers (3 CTAs/SM) without spills; measured per variant: the sweep
// with generic group strides (GS = 0, e.g. the 7-group C5) gains 10% at 3 CTAs/SM
// (C5-weak 17.5 -> 15.7 ms), the residual modes and the 1-/2-group specialisations lose
// 2-4% (C3 sweep 0.237 -> 0.243 ms, residual 0.221 -> 0.230 ms), so only that variant
// takes 3.  (4 CTAs/SM, 64 registers: spills, C3 1.37 -> 1.64 ms.)
#ifndef CSN_TMA_MINB1
#define CSN_TMA_MINB1 2
#endif
template <int L, int MODE = PG_RESID, int GS = 1>
struct TmaMinBlocks {
    static constexpr bool sweep0 = (MODE == PG_SWEEP || MODE == PG_SWEEPF) && GS == 0;
    static constexpr int value = L == 1 ? (sweep0 ? 3 : CSN_TMA_MINB1) : (L <= 3 ? 2 : 1);
};

template <int L, int MODE, int KD = 0, int GS = 0>
__global__ void __launch_bounds__(32 * PG_TX, TmaMinBlocks<L, MODE, GS>::value)
pg_residual_tma_kernel(const PGResidArgs<float> a, const __grid_constant__ PGTmaMaps m) {
    // KD 0: D computed here; 1: computed and stored to a.dterm; 2: read from a.dterm
    // (bit-identical: the stored value is the one this kernel would compute).
    // GS = 1 / 2: one or two groups and a per-cell source: sigma and q of a cell are one
    // scalar (1 group) or one 8-byte pair load (2 groups: a lane's channel pair is the
    // two groups of one direction) each, at a compile-time stride in y
    constexpr bool SWEEP = MODE == PG_SWEEP || MODE == PG_SWEEPF;
    constexpr bool DSUB = MODE == PG_SWEEP;       // psi' = psi - delta formed per read
    constexpr bool EMA = MODE == PG_RESID_EMA;
    using TP = UnitTaps<L>;
    constexpr int T = 2 * L + 1;
    constexpr int CC = X2_CC;
    constexpr int W = PG_TX + 2 * L;
    constexpr int NF = (MODE == PG_RESID || MODE == PG_SWEEPF) ? 3 : 4;
    constexpr int S = TmaRing<L, MODE>::S;
    constexpr int P = TmaRing<L, MODE>::PREFETCH;   // (S - L - 1)
    constexpr int FS = W * CC;                     // floats per field row
    constexpr int SLOT = TmaRing<L, MODE>::SLOT;
    constexpr unsigned ROWB = W * CC * sizeof(float);
    constexpr unsigned TXB = 3 * ROWB + (DSUB ? ROWB : 0) + (EMA ? PG_TX * CC * sizeof(float) : 0);
    extern __shared__ __align__(128) unsigned char smraw[];
    // 128-byte aligned ring base; pointer arithmetic on smraw keeps the shared address
    // space (a uintptr_t round trip would turn every ring read into a generic LD)
    float* sm = reinterpret_cast<float*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
    __shared__ double red[32];
    __shared__ __align__(8) uint64_t full[S];
    __shared__ unsigned relc[S];                   // warps done with each slot

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
    constexpr int U = TmaRing<L, MODE>::U;
    const int nsteps = 2 * L + (int)(((yb - ya) + U - 1) / U) * U;   // lead rows ya-L ...
    const bool producer = tid == 0;

    if (producer) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            relc[s] = 0u;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // shared-window addresses of the ring and its barriers, once
    const unsigned sm_s = smem_u32(sm), full_s = smem_u32(full);
    // producer: lead row ya - L + k of every field into slot s
    auto issue = [&](int k, int s) {
        const int yy = ya - L + k;
        const unsigned dst = sm_s + s * (SLOT * 4), fb = full_s + 8 * s;
        mbar_expect_tx_s(fb, TXB);
        tma_load_3d_s(dst, &m.psi, fb, c0, yy + a.psi_h, x0 - L + a.psi_h);
        tma_load_3d_s(dst + FS * 4, &m.kx, fb, c0, yy + a.k_h, x0 - L + a.k_h);
        tma_load_3d_s(dst + 2 * FS * 4, &m.ky, fb, c0, yy + a.k_h, x0 - L + a.k_h);
        if (DSUB) tma_load_3d_s(dst + 3 * FS * 4, &m.aux, fb, c0, yy + a.delta_h, x0 - L + a.delta_h);
        if (EMA) tma_load_3d_s(dst + 3 * FS * 4, &m.aux, fb, c0, yy + a.avg_h, x0 + a.avg_h);
    };

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
    float* avg_p = EMA && act ? a.avg + fidx(x, 0, cs, g.ny, a.avg_h, g.C) : nullptr;
    const float2 beta2 = bc2(a.beta);
    const bool refine = a.refine_div != 0;
    const float2 strm2 = a.strm ? make_float2(a.strm[n0], a.strm[n1]) : bc2(0.f);
    const int oy0 = max(ya, 0), oy1 = yb;
    const int lane_off = ty * CC + 2 * tx;          // this lane's pair in a staged row

    float2 rA[T], rB[T], rC[T], rD[T];              // pending outputs, by (y - ya) mod T
#pragma unroll
    for (int i = 0; i < T; ++i) rA[i] = rB[i] = rC[i] = rD[i] = bc2(0.f);
    float* dt_p = KD ? a.dterm + fidx(xs, 0, cs, g.ny, 0, g.C) : nullptr;
    float2 dN = bc2(0.f);
    if (KD == 2 && act) dN = ld2(dt_p + (int64_t)ya * g.C);

    if (producer) {          // every slot's first row; refills come from the releases
#pragma unroll
        for (int k = 0; k < S; ++k)
            if (k < nsteps) issue(k, k);
    }
    double l1 = 0.0;
    int slot = 0;          // slot of the current step (k mod S)
    unsigned fpar = 0;     // parity of the current fill of `slot`
    float2 sgN = bc2(0.f), qN = bc2(0.f);
    if (act) {
        if (GS == 1) {
            sgN = bc2(sig0[ya]);
            qN = bc2(q0[ya]);
        } else if (GS == 2) {
            sgN = ld2(sig0 + 2 * ya);
            qN = ld2(q0 + 2 * ya);
        } else {
            sgN = make_float2(sig0[ya * g.ng], sig1[ya * g.ng]);
            qN = make_float2(q0[ya * qst], q1[ya * qst]);
        }
    }

#define TMA_STEP(K, SK, OUT, Y, SLOTC)                                                \
    {                                                                                 \
        const int k_ = (K);                                                           \
        const int ss_ = (SLOTC) >= 0 ? (SLOTC) : slot;                                \
        float2 sg_ = sgN, q_ = qN, dd_ = dN;                                          \
        if ((OUT) && act && (Y) + 1 < yb) {                                           \
            if (GS == 1) {                                                            \
                sgN = bc2(sig0[(Y) + 1]);                                             \
                qN = bc2(q0[(Y) + 1]);                                                \
            } else if (GS == 2) {                                                     \
                sgN = ld2(sig0 + 2 * ((Y) + 1));                                      \
                qN = ld2(q0 + 2 * ((Y) + 1));                                         \
            } else {                                                                  \
                sgN = make_float2(sig0[((Y) + 1) * g.ng], sig1[((Y) + 1) * g.ng]);   \
                qN = make_float2(q0[((Y) + 1) * qst], q1[((Y) + 1) * qst]);          \
            }                                                                         \
            if (KD == 2) dN = ld2(dt_p + (int64_t)((Y) + 1) * g.C);                  \
        }                                                                             \
        mbar_wait_s(full_s + 8 * ss_, fpar);                                           \
        const float* buf_ = sm + ss_ * SLOT;                                           \
        if (EMA && avg_p) {                                                           \
            const int yl_ = ya - L + k_;                                              \
            if (yl_ >= oy0 && yl_ < oy1) {                                            \
                const float2 p_ = ld2(buf_ + L * CC + lane_off);                      \
                float2 o_ = p_;                                                       \
                if (a.avg_mode == 2) {                                                \
                    const float2 b_ = ld2(buf_ + 3 * FS + lane_off);                  \
                    o_ = make_float2(__fmaf_rn(b_.x, a.omt, __fmul_rn(a.theta, p_.x)),   \
                                     __fmaf_rn(b_.y, a.omt, __fmul_rn(a.theta, p_.y)));  \
                }                                                                     \
                st2(avg_p + (int64_t)yl_ * g.C, o_);                                  \
            }                                                                         \
        }                                                                             \
        float2 a_g = bc2(0.f), a_m = a_g, a_s = a_g, a_sk = a_g, a_k = a_g, a_mk = a_g, a_ky = a_g; \
        {                                                                             \
            const float* bp_ = buf_ + lane_off;                                       \
            _Pragma("unroll") for (int t_ = 0; t_ < T; ++t_) {                        \
                float2 p_ = ld2(bp_ + t_ * CC);                                       \
                if (DSUB) p_ = sub2(p_, ld2(bp_ + 3 * FS + t_ * CC));                 \
                const float2 k1_ = ld2(bp_ + FS + t_ * CC);                          \
                const float2 k2_ = ld2(bp_ + 2 * FS + t_ * CC);                      \
                a_g = fma2c((float)TP::g(t_), p_, a_g);                               \
                a_m = fma2c((float)TP::m(t_), p_, a_m);                               \
                a_s = fma2c((float)TP::s(t_), p_, a_s);                               \
                a_sk = fma2c((float)TP::s(t_), mul2(p_, k1_), a_sk);                  \
                if (KD != 2) a_k = fma2c((float)TP::s(t_), k1_, a_k);                 \
                a_mk = fma2c((float)TP::m(t_), mul2(p_, k2_), a_mk);                  \
                if (KD != 2) a_ky = fma2c((float)TP::m(t_), k2_, a_ky);               \
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
                if (KD != 2) rD[sl_] = fma2c(m_, xd1_, mul2(bc2(s_), xd2_));          \
            } else {                                                                  \
                rA[sl_] = fma2c(m_, xa_, fma2c(gt_, xg_, fma2c(s_, xs_, rA[sl_])));   \
                rB[sl_] = fma2c(m_, a_s, rB[sl_]);                                    \
                rC[sl_] = fma2c(s_, a_m, rC[sl_]);                                    \
                if (KD != 2) rD[sl_] = fma2c(m_, xd1_, fma2c(s_, xd2_, rD[sl_]));     \
            }                                                                         \
        }                                                                             \
        const int cs_ = ss_ >= L ? ss_ - L : ss_ - L + S;  /* centre row's slot */ \
        if ((OUT) && act && (Y) < yb) {                                               \
            const int y_ = (Y);                                                       \
            const float* cb_ = sm + cs_ * SLOT + L * CC + lane_off;                    \
            float2 pc_ = ld2(cb_);                                                    \
            if (DSUB) pc_ = sub2(pc_, ld2(cb_ + 3 * FS));                             \
            const float2 kxc_ = ld2(cb_ + FS), kyc_ = ld2(cb_ + 2 * FS);             \
            float2 r_ = fma2(hx, mul2(kxc_, rB[SK]), rA[SK]);                         \
            r_ = fma2(hy, mul2(kyc_, rC[SK]), r_);                                    \
            const float2 dk_ = KD == 2 ? dd_ : rD[SK];                                \
            if (KD == 1) st2(dt_p + (int64_t)y_ * g.C, dk_);                         \
            r_ = sub2(fma2(pc_, add2(dk_, sg_), r_), q_);                             \
            if (SWEEP) {                                                              \
                const float2 d_ = mul2(beta2, add2(strm2, sg_));                      \
                const float2 inv_ = make_float2(rcp_nr(d_.x), rcp_nr(d_.y));          \
                float2 qt_ = mul2(r_, inv_);                                          \
                if (refine)                                                           \
                    qt_ = fma2(fma2(make_float2(-d_.x, -d_.y), qt_, r_), inv_, qt_);  \
                st2(o_p + (int64_t)y_ * g.C, sub2(pc_, qt_));                         \
            } else {                                                                  \
                if (o_p) st2(o_p + (int64_t)y_ * g.C, r_);                           \
                l1 += fabs((double)r_.x) + fabs((double)r_.y);                        \
            }                                                                         \
        }                                                                             \
        if ((OUT) || k_ >= L) {              /* last read of the centre row's slot */ \
            __syncwarp();                                                             \
            if (tx == 0) {                                                            \
                /* the last warp to release the slot refills it (row k - L + S): no   \
                   warp ever waits for the others to free a slot */                   \
                if (atomicAdd(&relc[cs_], 1u) == PG_TX - 1) {                         \
                    relc[cs_] = 0u;                                                   \
                    if (k_ - L + S < nsteps) {                                        \
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  \
                        issue(k_ - L + S, cs_);                                       \
                    }                                                                 \
                }                                                                     \
            }                                                                         \
        }                                                                             \
        slot = ss_ + 1; if (slot == S) { slot = 0; fpar ^= 1u; }                                 \
    }

    // prologue: lead rows ya-L .. ya+L-1 (outputs below ya are never emitted)
#pragma unroll
    for (int k = 0; k < 2 * L; ++k) TMA_STEP(k, (k + 1) % T, false, 0, k % S);

    // S == U (a multiple of T): compile-time ring slot per unrolled step
    int kbase = 2 * L;
    for (int y0 = ya; y0 < yb; y0 += U, kbase += U) {
#pragma unroll
        for (int s = 0; s < U; ++s)
            TMA_STEP(kbase + s, s % T, true, y0 + s, S == U ? (2 * L + s) % S : -1);
    }
#undef TMA_STEP
    if (!SWEEP && a.partials) {
        const double tot = block_sum(l1, red);
        if (threadIdx.x == 0 && threadIdx.y == 0)
            a.partials[((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = tot;
    }
}

}  // namespace csn

namespace csn {

// ---------------------------------------------------------------------------------
// K2b (pg_kcoef_x2_kernel) with TMA row staging: R = alpha mu (M_y M_x psi_x - psi_x)
// and k on the +-l band from the K2a workspace (psi_x, psi_y on the +-2l band, halo 2l,
// read as stored; boxes beyond it are zero-filled like the cp.async stager's band
// rule).  Same lane mapping, passes and k formula (k_coef): bit-identical k.  K2b is
// issue-bound, so the per-thread staging work the TMA producer removes is time saved.
// ---------------------------------------------------------------------------------
struct KcoefMaps {
    CUtensorMap gx, gy;
};

// ring depth of the TMA K2b: L + 1 rows held for the output's centre + CSN_K2B_PREFETCH in
// flight ahead of the lead row
#ifndef CSN_K2B_PREFETCH
#define CSN_K2B_PREFETCH (L <= 3 ? X2_PREFETCH : 2)
#endif
template <int L>
struct K2bStages { static constexpr int value = L + 1 + CSN_K2B_PREFETCH; };

template <int L>
constexpr size_t pg_kcoef_tma_smem() {
    return (size_t)K2bStages<L>::value * 2 * (PG_TX + 2 * L) * X2_CC * sizeof(float) + 128;
}

// 3 CTAs/SM (78 registers); 4 (64 registers, 36 B of spills) measured C4 K2 3.92 -> 4.07 ms
#ifndef CSN_K2B_TMA_MINB
#define CSN_K2B_TMA_MINB 3
#endif
template <int L>
__global__ void __launch_bounds__(32 * PG_TX, CSN_K2B_TMA_MINB)
pg_kcoef_tma_kernel(const PGKArgs<float> a, const __grid_constant__ KcoefMaps m, int gh) {
    using TP = UnitTaps<L>;
    constexpr int T = 2 * L + 1;
    constexpr int CC = X2_CC;
    constexpr int W = PG_TX + 2 * L;
    constexpr int S = K2bStages<L>::value;
    constexpr int P = S - L - 1;
    constexpr int FS = W * CC;
    constexpr int SLOT = 2 * FS;
    constexpr unsigned TXB = 2 * FS * sizeof(float);
    extern __shared__ __align__(128) unsigned char smraw[];
    float* sm = reinterpret_cast<float*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
    __shared__ __align__(8) uint64_t full[S];
    __shared__ unsigned relc[S];                   // warps done with each slot

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
    const int lane = ty * CC + 2 * tx;
    const bool producer = tid == 0;

    if (producer) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            relc[s] = 0u;
        }
        fence_mbarrier_init();
    }
    __syncthreads();
    auto issue = [&](int k, int s) {
        const int yy = ya - L + k;
        float* dst = sm + s * SLOT;
        mbar_expect_tx(&full[s], TXB);
        tma_load_3d(dst, &m.gx, &full[s], c0, yy + gh, x0 - L + gh);
        tma_load_3d(dst + FS, &m.gy, &full[s], c0, yy + gh, x0 - L + gh);
    };
    if (producer) {          // every slot's first row; refills come from the releases
#pragma unroll
        for (int k = 0; k < S; ++k)
            if (k < nsteps) issue(k, k);
    }
    float2 r2x[T], r2y[T];   // M_x psi_x, M_x psi_y by lead row (step mod T)
    int slot = 0;
    unsigned fpar = 0;
    // per-lane constants of the k formula, kept live (opaque to the optimiser, which
    // otherwise recomputes the six products at every output: 3% of the kernel's issue)
    float2 armu = make_float2(a.alpha_r * mu0, a.alpha_r * mu1);
    float2 arnu = make_float2(a.alpha_r * nu0, a.alpha_r * nu1);
    float capx0 = a.dx * fabsf(mu0), capx1 = a.dx * fabsf(mu1);
    float capy0 = a.dy * fabsf(nu0), capy1 = a.dy * fabsf(nu1);
    asm volatile("" : "+f"(armu.x), "+f"(armu.y), "+f"(arnu.x), "+f"(arnu.y), "+f"(capx0),
                      "+f"(capx1), "+f"(capy0), "+f"(capy1));

#define K2BT_STEP(K, KR, OUT, Y)                                                         \
    {                                                                                     \
        const int k_ = (K);                                                               \
        mbar_wait(&full[slot], fpar);                                                     \
        const float* buf_ = sm + slot * SLOT + lane;                                      \
        float2 mx_ = bc2(0.f), my_ = mx_;                                                 \
        _Pragma("unroll") for (int t = 0; t < T; ++t) {                                   \
            mx_ = fma2c((float)TP::m(t), ld2(buf_ + t * CC), mx_);                        \
            my_ = fma2c((float)TP::m(t), ld2(buf_ + FS + t * CC), my_);                   \
        }                                                                                 \
        r2x[(KR)] = mx_;                                                                  \
        r2y[(KR)] = my_;                                                                  \
        const int cs_ = slot >= L ? slot - L : slot - L + S;                              \
        if ((OUT) && act && (Y) < yb) {                                                   \
            float2 mmx = bc2(0.f), mmy = mmx;                                             \
            _Pragma("unroll") for (int b = 0; b < T; ++b) {                               \
                mmx = fma2c((float)TP::m(b), r2x[((KR) + 1 + b) % T], mmx);               \
                mmy = fma2c((float)TP::m(b), r2y[((KR) + 1 + b) % T], mmy);               \
            }                                                                             \
            const float* cb = sm + cs_ * SLOT + L * CC + lane;                            \
            const float2 pxc = ld2(cb), pyc = ld2(cb + FS);                               \
            const float2 rx = mul2(armu, sub2(mmx, pxc));                                 \
            const float2 ry = mul2(arnu, sub2(mmy, pyc));                                 \
            const float amu[2] = {fabsf(mu0), fabsf(mu1)}, anu[2] = {fabsf(nu0), fabsf(nu1)}; \
            const float capx[2] = {capx0, capx1}, capy[2] = {capy0, capy1};               \
            const float pxv[2] = {pxc.x, pxc.y}, pyv[2] = {pyc.x, pyc.y};                 \
            const float rxv[2] = {rx.x, rx.y}, ryv[2] = {ry.x, ry.y};                     \
            float kx[2], ky[2];                                                           \
            _Pragma("unroll") for (int h = 0; h < 2; ++h) {                               \
                kx[h] = k_coef(rxv[h], pxv[h], a.cax, a.csx, capx[h], amu[h], a.eps);     \
                ky[h] = k_coef(ryv[h], pyv[h], a.cay, a.csy, capy[h], anu[h], a.eps);     \
            }                                                                             \
            const int64_t o = kb0 + (int64_t)(Y) * g.C;                                   \
            st2(a.kx + o, make_float2(kx[0], kx[1]));                                     \
            st2(a.ky + o, make_float2(ky[0], ky[1]));                                     \
        }                                                                                 \
        if (k_ >= L) {                    /* last read of the centre row's slot */        \
            __syncwarp();                                                                 \
            if (tx == 0 && atomicAdd(&relc[cs_], 1u) == PG_TX - 1) {                      \
                relc[cs_] = 0u;                   /* the last releaser refills it */      \
                if (k_ - L + S < nsteps) {                                                \
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");          \
                    issue(k_ - L + S, cs_);                                               \
                }                                                                         \
            }                                                                             \
        }                                                                                 \
        if (++slot == S) { slot = 0; fpar ^= 1u; }                                        \
    }
#pragma unroll
    for (int k = 0; k < 2 * L; ++k) K2BT_STEP(k, k % T, false, 0);
    int kb = 2 * L;
    for (int y0 = ya; y0 < yb; y0 += T, kb += T) {
#pragma unroll
        for (int s = 0; s < T; ++s) K2BT_STEP(kb + s, (2 * L + s) % T, true, y0 + s);
    }
#undef K2BT_STEP
}

}  // namespace csn

namespace csn {

// ---------------------------------------------------------------------------------
// K2 in one pass with warp specialisation: iterate average + psi_x, psi_y (stage 1,
// the K2a computation) and R, k (stage 2, the K2b computation) in one CTA, psi_x and
// psi_y handed over through a shared-memory ring instead of an HBM workspace (16 B/DOF
// of traffic saved).  A CTA owns TX = PG_TX output cells x 64 channels and marches y:
//   * NW1 = TX + 2l stage-1 warps (one cell each, the output cells +- l): the cp.async
//     row stager (vacuum rule, EMA on the staged items, owned cells written back), a
//     named barrier among themselves per row, the x pass and the y ring of K2a; each
//     psi_x / psi_y row goes to ring slot u mod S2 (0 outside the +-2l band, like the
//     workspace), then the warp arrives on full2[slot];
//   * TX stage-2 warps (one output cell each): wait full2, the x pass / y ring / k
//     formula of K2b, and arrive on empty2 when a row's slot is read for the last time
//     (as the centre row, l rows later).
// Stage-1 warps are the old fused kernel's work without its idle edge warps: the two
// stages run concurrently instead of alternating at a CTA-wide barrier.  Operations
// and their order are K2a's and K2b's: k and the average are bit-identical to the
// split path.
// ---------------------------------------------------------------------------------
constexpr int WS_TX = PG_TX;      // output cells per CTA
constexpr int WS_S1 = 4;          // stage-1 input row ring (cp.async)

template <int L>
struct WsGeom {
    static constexpr int NW1 = WS_TX + 2 * L;          // stage-1 warps (cells)
    static constexpr int NW2 = WS_TX;                  // stage-2 warps
    static constexpr int W1 = WS_TX + 4 * L;           // staged input cells
    static constexpr int S2 = L + 4;                   // psi_x / psi_y row ring
    static constexpr int F2 = NW1 * X2_CC;             // floats per psi_x row
};

template <int L, bool EMA>
constexpr size_t pg_k_ws_smem() {
    using G = WsGeom<L>;
    return ((size_t)WS_S1 * (EMA ? 2 : 1) * G::W1 * X2_CC + (size_t)G::S2 * 2 * G::F2) *
           sizeof(float);
}

template <int L, bool EMA, int VEC>
__global__ void __launch_bounds__(32 * (WS_TX + WS_TX + 2 * L), 1)
pg_k_ws_kernel(const PGKArgs<float> a) {
    using TP = UnitTaps<L>;
    using G = WsGeom<L>;
    constexpr int T = 2 * L + 1;
    constexpr int CC = X2_CC;
    constexpr int NW1 = G::NW1, W1 = G::W1, S2 = G::S2, F2 = G::F2;
    constexpr int NT1 = 32 * NW1;
    constexpr int G4 = CC / VEC;
    constexpr int NI = (W1 * G4 + NT1 - 1) / NT1;
    constexpr int NF = EMA ? 2 : 1;
    constexpr int S1 = WS_S1;
    constexpr int FS = W1 * CC;
    extern __shared__ __align__(16) unsigned char smraw[];
    float* s1 = reinterpret_cast<float*>(smraw);               // [S1][NF][W1][CC]
    float* s2 = s1 + (size_t)S1 * NF * FS;                     // [S2][2][NW1][CC]
    __shared__ __align__(8) uint64_t full2[S2], empty2[S2];

    const Geo& g = a.g;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int c0 = blockIdx.y * CC;
    const int c = c0 + 2 * tx;
    const bool cval = c < g.C;
    const int cs = cval ? c : g.C - 2;
    const int x0 = -L + (int)blockIdx.x * WS_TX;              // output band x in [-l, nx+l)
    const int ya = -L + (int)blockIdx.z * a.ly;               // output band y in [-l, ny+l)
    const int yb = min(g.ny + L, ya + a.ly);
    const int nsteps2 = 2 * L + (int)(((yb - ya) + T - 1) / T) * T;   // psi_x rows consumed
    const int u0 = ya - L;                                    // first psi_x row

    if (ty == 0 && tx == 0) {
#pragma unroll
        for (int s = 0; s < S2; ++s) {
            mbar_init(&full2[s], NW1);
            mbar_init(&empty2[s], G::NW2);
        }
        fence_mbarrier_init();
    }
    __syncthreads();

    if (ty < NW1) {
        // ------------------------------------------------------------- stage 1
        const int tid = ty * 32 + tx;
        const int xs1 = x0 - L + ty;                          // this warp's cell
        const bool inb_x = xs1 >= -2 * L && xs1 < g.nx + 2 * L;
        const int ox0 = max(x0, 0), ox1 = min(x0 + WS_TX, g.nx);
        const int oy0 = max(ya, 0), oy1 = min(yb, g.ny);
        const float2 inv_dx = bc2(a.inv_dx), inv_dy = bc2(a.inv_dy);
        const float omt = a.omt, theta = a.theta;
        const bool write_avg = a.avg_mode != 0;
        // psi_x rows u0 .. u0 + nsteps2 - 1 from lead rows u0 - L ...
        const int nsteps1 = 2 * L + (int)((nsteps2 + T - 1) / T) * T;
        // the staged band is [-3l, nx+3l): the last CTA's overhang past it is never loaded
        // (past a ghost side it would run off the field)
        FieldDesc fd[2] = {{a.psi, a.psi_h, -3 * L, g.nx + 3 * L},
                           {a.avg_in, a.avg_in_h, -3 * L, g.nx + 3 * L}};
        Stager<float, VEC, NI, NF, 0, CC> st;
        st.init(g, fd, x0 - 2 * L, W1, c0, 0, a.mu, a.nu, tid, NT1);
        const unsigned sbase = (unsigned)__cvta_generic_to_shared(s1);
        constexpr unsigned FSB = FS * sizeof(float);
        float* own_ptr[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int e = tid + i * NT1;
            const int xi = e / G4, q = e % G4;
            const int xg = x0 - 2 * L + xi, cc = c0 + q * VEC;
            own_ptr[i] = (write_avg && e < W1 * G4 && cc < g.C && xg >= ox0 && xg < ox1)
                             ? a.avg_out + fidx(xg, 0, cc, g.ny, a.avg_out_h, g.C) : nullptr;
        }
        const int lane = ty * CC + 2 * tx;
        float2 rG[T], rM[T];
#pragma unroll
        for (int k = 0; k < S1 - 1; ++k) {
            if (k < nsteps1) st.issue(u0 - L + k, sbase + k * NF * FSB, FSB, a.psi);
            cp_async_commit();
        }
#define WS1_STEP(K, KR, OUT)                                                              \
        {                                                                                 \
            const int k_ = (K);                                                           \
            const int yl_ = u0 - L + k_;                                                  \
            cp_async_wait<S1 - 2>();                                                      \
            float* buf_ = s1 + (size_t)(k_ % S1) * NF * FS;                               \
            if (EMA || write_avg) {                                                       \
                const bool own_row_ = yl_ >= oy0 && yl_ < oy1;                            \
                _Pragma("unroll") for (int i = 0; i < NI; ++i) {                          \
                    const int e = tid + i * NT1;                                          \
                    if (e < W1 * G4) {                                                    \
                        float* p_ = buf_ + (e / G4) * CC + (e % G4) * VEC;                \
                        float pv_[VEC];                                                   \
                        _Pragma("unroll") for (int vv = 0; vv < VEC; ++vv) {              \
                            pv_[vv] = p_[vv];                                             \
                            if (EMA) pv_[vv] = ema_rn(p_[FS + vv], pv_[vv], omt, theta);  \
                            p_[vv] = pv_[vv];                                             \
                        }                                                                 \
                        if (own_ptr[i] && own_row_) {                                     \
                            float* o_ = own_ptr[i] + (int64_t)yl_ * g.C;                  \
                            _Pragma("unroll") for (int vv = 0; vv < VEC; ++vv) o_[vv] = pv_[vv]; \
                        }                                                                 \
                    }                                                                     \
                }                                                                         \
            }                                                                             \
            asm volatile("bar.sync 1, %0;" ::"r"(NT1) : "memory");                        \
            {                                                                             \
                float2 ag_ = bc2(0.f), am_ = ag_;                                         \
                const float* bp_ = buf_ + lane;                                           \
                _Pragma("unroll") for (int t = 0; t < T; ++t) {                           \
                    const float2 p_ = ld2(bp_ + t * CC);                                  \
                    ag_ = fma2c((float)TP::g(t), p_, ag_);                                \
                    am_ = fma2c((float)TP::m(t), p_, am_);                                \
                }                                                                         \
                rG[(KR)] = ag_;                                                           \
                rM[(KR)] = am_;                                                           \
            }                                                                             \
            const int u_ = yl_ - L;                     /* psi_x row of this step */      \
            if ((OUT) && u_ - u0 < nsteps2) {                                             \
                float2 px_ = bc2(0.f), py_ = px_;                                         \
                _Pragma("unroll") for (int b = 0; b < T; ++b) {                           \
                    px_ = fma2c((float)TP::m(b), rG[((KR) + 1 + b) % T], px_);            \
                    py_ = fma2c((float)TP::g(b), rM[((KR) + 1 + b) % T], py_);            \
                }                                                                         \
                const bool inb_ = inb_x && cval && u_ >= -2 * L && u_ < g.ny + 2 * L;     \
                const int n_ = u_ - u0;                                                   \
                const int sl_ = n_ % S2;                                                  \
                if (n_ >= S2) mbar_wait(&empty2[sl_], (unsigned)((n_ / S2 - 1) & 1));     \
                float* w_ = s2 + (size_t)sl_ * 2 * F2 + ty * CC + 2 * tx;                 \
                st2(w_, inb_ ? mul2(px_, inv_dx) : bc2(0.f));                            \
                st2(w_ + F2, inb_ ? mul2(py_, inv_dy) : bc2(0.f));                       \
                __syncwarp();                                                             \
                if (tx == 0) mbar_arrive(&full2[sl_]);                                    \
            }                                                                             \
            if (k_ + S1 - 1 < nsteps1)                                                    \
                st.issue(u0 - L + k_ + S1 - 1, sbase + ((k_ + S1 - 1) % S1) * NF * FSB, FSB, a.psi); \
            cp_async_commit();                                                            \
        }
#pragma unroll
        for (int k = 0; k < 2 * L; ++k) WS1_STEP(k, k % T, false);
        for (int kb = 2 * L; kb < nsteps1; kb += T) {
#pragma unroll
            for (int s = 0; s < T; ++s) WS1_STEP(kb + s, (2 * L + s) % T, true);
        }
#undef WS1_STEP
        cp_async_wait<0>();
    } else {
        // ------------------------------------------------------------- stage 2
        const int w2 = ty - NW1;                              // output cell x0 + w2
        const int x = x0 + w2;
        const bool act = x < g.nx + L && cval;
        const int n0 = cs / g.ng, n1 = (cs + 1) / g.ng;
        const float mu0 = a.mu[n0], mu1 = a.mu[n1], nu0 = a.nu[n0], nu1 = a.nu[n1];
        const int64_t kb0 = fidx(act ? x : 0, 0, cs, g.ny, a.k_h, g.C);
        const int lane = w2 * CC + 2 * tx;                    // x pass from stage-1 cell w2
        float2 r2x[T], r2y[T];
#define WS2_STEP(K, KR, OUT, Y)                                                           \
        {                                                                                 \
            const int k_ = (K);                                                           \
            const int sl_ = k_ % S2;                                                      \
            mbar_wait(&full2[sl_], (unsigned)((k_ / S2) & 1));                            \
            const float* buf_ = s2 + (size_t)sl_ * 2 * F2 + lane;                         \
            float2 mx_ = bc2(0.f), my_ = mx_;                                             \
            _Pragma("unroll") for (int t = 0; t < T; ++t) {                               \
                mx_ = fma2c((float)TP::m(t), ld2(buf_ + t * CC), mx_);                    \
                my_ = fma2c((float)TP::m(t), ld2(buf_ + F2 + t * CC), my_);               \
            }                                                                             \
            r2x[(KR)] = mx_;                                                              \
            r2y[(KR)] = my_;                                                              \
            if ((OUT) && act && (Y) < yb) {                                               \
                float2 mmx = bc2(0.f), mmy = mmx;                                         \
                _Pragma("unroll") for (int b = 0; b < T; ++b) {                           \
                    mmx = fma2c((float)TP::m(b), r2x[((KR) + 1 + b) % T], mmx);           \
                    mmy = fma2c((float)TP::m(b), r2y[((KR) + 1 + b) % T], mmy);           \
                }                                                                         \
                const float* cb = s2 + (size_t)((k_ - L) % S2) * 2 * F2 + (w2 + L) * CC + 2 * tx; \
                const float2 pxc = ld2(cb), pyc = ld2(cb + F2);                           \
                const float2 rx = mul2(make_float2(a.alpha_r * mu0, a.alpha_r * mu1),     \
                                       sub2(mmx, pxc));                                   \
                const float2 ry = mul2(make_float2(a.alpha_r * nu0, a.alpha_r * nu1),     \
                                       sub2(mmy, pyc));                                   \
                const float amu[2] = {fabsf(mu0), fabsf(mu1)}, anu[2] = {fabsf(nu0), fabsf(nu1)}; \
                const float pxv[2] = {pxc.x, pxc.y}, pyv[2] = {pyc.x, pyc.y};             \
                const float rxv[2] = {rx.x, rx.y}, ryv[2] = {ry.x, ry.y};                 \
                float kx[2], ky[2];                                                       \
                _Pragma("unroll") for (int h = 0; h < 2; ++h) {                           \
                    kx[h] = k_coef(rxv[h], pxv[h], a.cax, a.csx,         \
                                   a.dx * amu[h], amu[h], a.eps);                         \
                    ky[h] = k_coef(ryv[h], pyv[h], a.cay, a.csy,         \
                                   a.dy * anu[h], anu[h], a.eps);                         \
                }                                                                         \
                const int64_t o = kb0 + (int64_t)(Y) * g.C;                               \
                st2(a.kx + o, make_float2(kx[0], kx[1]));                                 \
                st2(a.ky + o, make_float2(ky[0], ky[1]));                                 \
            }                                                                             \
            if (k_ >= L) {                /* row k_ - L read for the last time (centre) */ \
                __syncwarp();                                                             \
                if (tx == 0) mbar_arrive(&empty2[(k_ - L) % S2]);                         \
            }                                                                             \
        }
#pragma unroll
        for (int k = 0; k < 2 * L; ++k) WS2_STEP(k, k % T, false, 0);
        int kb = 2 * L;
        for (int y0 = ya; y0 < yb; y0 += T, kb += T) {
#pragma unroll
            for (int s = 0; s < T; ++s) WS2_STEP(kb + s, (2 * L + s) % T, true, y0 + s);
        }
#undef WS2_STEP
    }
}

}  // namespace csn
