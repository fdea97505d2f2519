// extern "C" entry points of libconvsn_sm100.so (declared in include/convsn_sm100.h).
// Argument checking, launch geometry and float/double x ConvFEM-order dispatch.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <string.h>

#include "common.cuh"
#include "misc_kernels.cuh"
#include "pg_kernels.cuh"
#include "pg_kernels_x2.cuh"
#include "upwind_kernels.cuh"
#include "pg_kernels_tma.cuh"
#include "tail_kernels.cuh"
#include "launchers.h"

// NVTX ranges around every compute entry point (header-only nvtx3: a no-op function
// pointer check unless a profiler injects itself; nsys/ncu --nvtx show the ABI calls)
#include <nvtx3/nvToolsExt.h>
namespace {
struct NvtxScope {
    explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
};
}  // namespace
#define CSN_NVTX() NvtxScope csn_nvtx_scope_(__func__)

using namespace csn;

unsigned long long csn::g_launches = 0;

namespace {

// kernel-variant switches (csn_set_tuning), for A/B parity tests of kernel variants
int g_tune_upwind_x2 = 1;
int g_tune_upwind_div = 3;
int g_tune_sweep_div = 1;
int g_tune_pg_tma = 1;
int g_tune_upwind_tma = 1;   // TMA-staged smoother columns (last releaser refills): C4 correction 1.99 -> 1.75 ms
int g_tune_k2_tma = 1;   // TMA-staged K2b (last releaser refills its ring slot): C4 K2 4.04 -> 3.93 ms; the cp.async K2b was faster before that refill scheme (2.09 vs 2.18 ms)
int g_tune_pg_chunks = 0;   // y chunks of the PG marches: 0 = cost model (pick_ly), n = forced
int g_tune_tail_faces = 1;  // coarse tail: one CTA per (face, group) in shared memory; 0 = cluster kernel
int g_tune_tail_smem = 1;   // coarse tail: levels <= 2048 DOF in CTA 0's shared memory
int g_tune_k2_ws = 0;
int g_tune_pg_xb = 0;   // x-blocked residual / sweep (warps per CTA: 4 or 8; 0 = off)   // one-pass K2: 5.0 ms vs 4.2 ms split on C4 (stage 2 starved)

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        else
            cudaGetLastError();
    }
    return fn;
}

// tiled fp32 map of rank 2 or 3 (dims / box innermost first, strides in bytes)
bool raw_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims,
             const cuuint64_t* strides, const cuuint32_t* box) {
    auto enc = tensor_map_encoder();
    if (!enc || !base || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    for (int i = 0; i + 1 < rank; ++i)
        if (strides[i] % 16) return false;
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(base), dims, strides,
               box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

// 3D map over a padded fp32 field [nx + 2h][ny + 2h][C]: box = 64 channels x 1 row x bx
// cells, out-of-bounds boxes zero-filled, 256-byte L2 promotion
bool field_map(CUtensorMap* m, const void* base, const csn_geom* g, int h, int bx) {
    auto enc = tensor_map_encoder();
    if (!enc || !base) return false;
    const uint64_t C = (uint64_t)g->nd * g->ng;
    if ((C * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    cuuint64_t dims[3] = {C, (cuuint64_t)(g->ny + 2 * h), (cuuint64_t)(g->nx + 2 * h)};
    cuuint64_t strides[2] = {C * 4, (cuuint64_t)(g->ny + 2 * h) * C * 4};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)bx};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box,
               es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

constexpr int kVersion = 1;

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline bool geom_ok(const csn_geom* g) {
    return g && g->nx >= 1 && g->ny >= 1 && g->nd >= 1 && g->ng >= 1 && g->dx > 0 && g->dy > 0;
}

inline int grid1d(int64_t n, int block = 256) {
    int64_t b = cdiv(n, block);
    if (b > 148 * 64) b = 148 * 64;
    if (b < 1) b = 1;
    return (int)b;
}

// x chunks of the smoother march: start from 8-column chunks (the H = 3 warm-up columns
// are then 27% extra work, but small coarse levels need the parallelism: one 64-column
// chunk per strip left the 128^2 x 128 level at 32 CTAs), then merge chunks while the
// grid still holds >= 8 CTAs per SM
inline int up_chunks0(int nx) { return (int)cdiv(nx, 8); }

// x chunks of one smoother launch over `ctas_xy` (strip x channel) CTAs: 8-column chunks
// merged while the grid keeps >= 8 CTAs per SM; a grid below one wave (the coarse levels)
// is instead split down to single columns while it still fits one wave — a chunk's march
// is a serial chain of (columns + H warm-up) dependent steps of ~1.5 us each with one warp
// per SM, so a 16 x 16 level took 16 us as one 8-column chunk (11 steps) and takes 4
// steps as single columns (the 4x warm-up recompute is free at that size)
// (min_cols: the packed kernels start a non-first chunk's warm-up H columns before it
// without an x predicate, so their chunks keep >= 4 columns; the scalar kernel
// predicates every column)
inline int up_chunks(int nx, int64_t ctas_xy, int min_cols) {
    int chunks = up_chunks0(nx);
    while (chunks > 1 && ctas_xy * (chunks / 2) >= 148 * 8) chunks /= 2;
    while (chunks < nx && cdiv(nx, chunks * 2) >= min_cols && ctas_xy * chunks * 2 <= 148 * 2)
        chunks *= 2;
    return chunks;
}

// Rows per CTA chunk of the y-marching kernels: a measured cost model (tools/ab_chunks.sh).
// A CTA marches S = ly + 2l + 3 row steps (lead-in rows and start-up included) and the grid
// runs in R = CTAs / resident slots rounds of equally long CTAs; a last round at most half
// full runs ~1/0.65 faster (one CTA per SM).  Grids of fewer than 3 rounds made of 1 or 2
// chunks measured 10% / 5% slower per row than 4+ chunks (every CTA walks the same rows in
// lockstep), which the model carries as a factor.  The chunk count (a power of two, ly a
// multiple of the march's unroll T) minimises rounds x S:
//   * C4 residual / sweep: 2048 tiles = 6.9 rounds of 296 slots stay one chunk; its K2a
//     (3.6 rounds of 592 slots) takes 4 chunks (C4 K2 3.93 -> 3.76 ms);
//   * C3 fused K2: 304 tiles on 296 slots was 2 chunks = 2.05 rounds, now 4 = 4.1 rounds;
//   * a 64-column DD slab (256 tiles) takes 4 chunks instead of 1; C1 (16 tiles) splits
//     down to one unroll group per CTA.
// slots: resident CTAs of the kernel on the whole GPU.
inline int pick_ly(int64_t ctas_xy, int rows, int T, int L, int slots = 148 * 2) {
    if (g_tune_pg_chunks > 0)       // A/B: forced chunk count
        return (int)cdiv(cdiv(rows, g_tune_pg_chunks), T) * T;
    int best_ly = (int)cdiv(rows, T) * T;
    double best = 1e300;
    for (int chunks = 1; chunks <= 64 && rows / chunks >= T; chunks *= 2) {
        const int ly = (int)cdiv(cdiv(rows, chunks), T) * T;
        const int64_t ctas = ctas_xy * cdiv(rows, ly);
        const int64_t full = ctas / slots;
        const double frac = (double)(ctas - full * slots) / slots;
        double rounds = (double)full + (frac > 0.5 ? 1.0 : frac > 0.0 ? 0.65 : 0.0);
        if ((double)ctas / slots < 3.0) rounds *= chunks == 1 ? 1.10 : chunks == 2 ? 1.05 : 1.0;
        const double cost = rounds * (ly + 2 * L + 3);
        if (cost < best * 0.999) {      // ties keep the fewer, longer chunks
            best = cost;
            best_ly = ly;
        }
    }
    return best_ly;
}

// The kernels use the compile-time unit taps of taps_table.cuh; the caller's taps
// (host [3][2L+1] = mass, grad, stiff) must be the ConvFEM order-L set.
template <int L>
bool taps_match(const double* taps) {
    constexpr int T = 2 * L + 1;
    for (int a = 0; a < T; ++a) {
        const double ref[3] = {UnitTaps<L>::m(a), UnitTaps<L>::g(a), UnitTaps<L>::s(a)};
        for (int k = 0; k < 3; ++k) {
            const double v = taps[k * T + a];
            if (fabs(v - ref[k]) > 1e-12 * (1.0 + fabs(ref[k]))) return false;
        }
    }
    return true;
}

// 16-byte staging needs every aligned VEC-channel group inside one octahedron face
// (same upwind signs) and VEC | C (alignment): a face holds n_a^2 * ng channels
// (8 faces, or 4 for the z-folded hemisphere).
inline bool vec_ok(const csn_geom* g, int vec) {
    const int64_t C = (int64_t)g->nd * g->ng;
    const int64_t face = (int64_t)g->na * g->na * g->ng;
    return C % vec == 0 && face % vec == 0 && C % face == 0;
}

// workspace of the split diffusivity path: psi_x, psi_y on the +-2l band (halo 2l)
inline int64_t grad_field_elems(const csn_geom* g, int L) {
    return (int64_t)(g->nx + 4 * L) * (g->ny + 4 * L) * g->nd * g->ng;
}

// ------------------------------------------------------------------ PG residual
template <class Real, int L>
int pg_residual_impl(const csn_geom* g, const double* taps, const void* psi, int psi_h,
                     const void* delta, int delta_h, const void* kx, const void* ky, int k_h,
                     const void* sigma, const void* q, int q_per_dof, const void* mu,
                     const void* nu, const void* strm, void* r, int r_h, void* out, int out_h,
                     double beta, double* partials, double* l1, void* avg, int avg_h, int avg_mode,
                     double theta, void* dterm, int dterm_mode, cudaStream_t st) {
    constexpr int T = 2 * L + 1;
    if (k_h < L) return CSN_E_ARG;
    if (!taps_match<L>(taps)) return CSN_E_ARG;
    if (avg_mode < 0 || avg_mode > 2 || (avg_mode && (!avg || out))) return CSN_E_ARG;
    PGResidArgs<Real> a;
    a.avg = (Real*)avg; a.avg_h = avg_h; a.avg_mode = avg ? avg_mode : 0;
    a.theta = (Real)theta; a.omt = (Real)(1.0 - theta);
    a.g = make_geo(*g);
    a.psi = (const Real*)psi; a.psi_h = psi_h;
    a.delta = (const Real*)delta; a.delta_h = delta_h;
    a.kx = (const Real*)kx; a.ky = (const Real*)ky; a.k_h = k_h;
    a.sigma = (const Real*)sigma; a.q = (const Real*)q; a.q_per_dof = q_per_dof;
    a.mu = (const Real*)mu; a.nu = (const Real*)nu; a.strm = (const Real*)strm;
    a.inv_dx = (Real)(1.0 / g->dx); a.inv_dy = (Real)(1.0 / g->dy);
    a.hx = (Real)(0.5 / (g->dx * g->dx)); a.hy = (Real)(0.5 / (g->dy * g->dy));
    a.r = (Real*)r; a.r_h = r_h;
    a.out = (Real*)out; a.out_h = out_h; a.beta = (Real)beta;
    a.refine_div = g_tune_sweep_div;
    a.dterm = (Real*)dterm;
    // fp32: packed-fp32x2 kernel, a lane per channel pair (64 channels per CTA)
    constexpr bool X2 = sizeof(Real) == 4;
    const int gx = (int)cdiv(g->nx, PG_TX);
    const int gy = (int)cdiv((int64_t)g->nd * g->ng, X2 ? X2_CC : PG_CC);
    // y chunks a multiple of the TMA march's unroll (2T at L = 1, see TmaRing)
    a.ly = pick_ly((int64_t)gx * gy, g->ny, X2 && L == 1 ? 2 * T : T, L);
    const int gz = (int)cdiv(g->ny, a.ly);
    a.partials = (l1 || partials) ? partials : nullptr;
    dim3 grid(gx, gy, gz), block(PG_CC, PG_TX);
    const bool vec = vec_ok(g, 16 / (int)sizeof(Real));
    constexpr int V = 16 / sizeof(Real);
    if constexpr (X2) {
        // x-blocked kernel (two cells per lane), when enabled: any halo, 16-byte staging
        if constexpr (L <= 3) {
            if ((g_tune_pg_xb == 4 || g_tune_pg_xb == 8) && vec && dterm_mode == 0) {
                const int nw = g_tune_pg_xb;
                const int gxb = (int)cdiv(g->nx, 2 * nw);
                a.ly = pick_ly((int64_t)gxb * gy, g->ny, T, L);
                const int gzb = (int)cdiv(g->ny, a.ly);
                dim3 gridb(gxb, gy, gzb), blockb(32, nw);
                if (!out && l1 && !partials) return CSN_E_ARG;
                const int mode = out ? PG_SWEEP : (a.avg_mode ? PG_RESID_EMA : PG_RESID);
                if (nw == 4) {
                    if (mode == PG_SWEEP) launch_pg_resid_xb<L, PG_SWEEP, V, 4>(gridb, blockb, st, a);
                    else if (mode == PG_RESID_EMA) launch_pg_resid_xb<L, PG_RESID_EMA, V, 4>(gridb, blockb, st, a);
                    else launch_pg_resid_xb<L, PG_RESID, V, 4>(gridb, blockb, st, a);
                } else {
                    if (mode == PG_SWEEP) launch_pg_resid_xb<L, PG_SWEEP, V, 8>(gridb, blockb, st, a);
                    else if (mode == PG_RESID_EMA) launch_pg_resid_xb<L, PG_RESID_EMA, V, 8>(gridb, blockb, st, a);
                    else launch_pg_resid_xb<L, PG_RESID, V, 8>(gridb, blockb, st, a);
                }
                CSN_CHECK_LAUNCH();
                if (!out && l1) {
                    sum_f64_kernel<<<1, 1024, 0, st>>>(partials, (int64_t)gxb * gy * gzb, 1.0, l1);
                    CSN_CHECK_LAUNCH();
                }
                return CSN_OK;
            }
        }
        // TMA staging when every staged field is padded (halos read as stored)
        constexpr int W = PG_TX + 2 * L;
        PGTmaMaps maps;
        // a sweep without delta (the correction already folded into psi) stages 3 fields
        const bool fold = out && !delta;
        const bool tma = g_tune_pg_tma && psi_h >= L && k_h >= L &&
                         (!out || fold || (delta && delta_h >= L)) &&
                         field_map(&maps.psi, psi, g, psi_h, W) &&
                         field_map(&maps.kx, kx, g, k_h, W) && field_map(&maps.ky, ky, g, k_h, W) &&
                         (out ? (fold || field_map(&maps.aux, delta, g, delta_h, W))
                              : (!a.avg_mode || field_map(&maps.aux, avg, g, avg_h, PG_TX)));
        if (!tma) cudaGetLastError();
        if (dterm_mode && !tma) return CSN_E_SCHEME;      // the stored D needs the TMA kernel
        if (tma) {
            if (!out && l1 && !partials) return CSN_E_ARG;
            if (fold) {
                if (dterm_mode == 2) launch_pg_resid_tma<L, PG_SWEEPF, 2>(grid, block, st, a, maps);
                else if (dterm_mode == 0) launch_pg_resid_tma<L, PG_SWEEPF, 0>(grid, block, st, a, maps);
                else return CSN_E_SCHEME;
            } else if (out) {
                if (dterm_mode == 2) launch_pg_resid_tma<L, PG_SWEEP, 2>(grid, block, st, a, maps);
                else if (dterm_mode == 0) launch_pg_resid_tma<L, PG_SWEEP, 0>(grid, block, st, a, maps);
                else return CSN_E_SCHEME;
            } else if (a.avg_mode) {
                if (dterm_mode == 1) launch_pg_resid_tma<L, PG_RESID_EMA, 1>(grid, block, st, a, maps);
                else if (dterm_mode == 2) launch_pg_resid_tma<L, PG_RESID_EMA, 2>(grid, block, st, a, maps);
                else launch_pg_resid_tma<L, PG_RESID_EMA, 0>(grid, block, st, a, maps);
            } else {
                if (dterm_mode == 1) launch_pg_resid_tma<L, PG_RESID, 1>(grid, block, st, a, maps);
                else if (dterm_mode == 2) launch_pg_resid_tma<L, PG_RESID, 2>(grid, block, st, a, maps);
                else launch_pg_resid_tma<L, PG_RESID, 0>(grid, block, st, a, maps);
            }
            CSN_CHECK_LAUNCH();
            if (!out && l1) {
                sum_f64_kernel<<<1, 1024, 0, st>>>(partials, (int64_t)gx * gy * gz, 1.0, l1);
                CSN_CHECK_LAUNCH();
            }
            return CSN_OK;
        }
        if (out) {
            if (vec) launch_pg_resid_x2<L, PG_SWEEP, V>(grid, block, st, a);
            else launch_pg_resid_x2<L, PG_SWEEP, 1>(grid, block, st, a);
        } else {
            if (l1 && !partials) return CSN_E_ARG;
            if (a.avg_mode) {
                if (vec) launch_pg_resid_x2<L, PG_RESID_EMA, V>(grid, block, st, a);
                else launch_pg_resid_x2<L, PG_RESID_EMA, 1>(grid, block, st, a);
            } else {
                if (vec) launch_pg_resid_x2<L, PG_RESID, V>(grid, block, st, a);
                else launch_pg_resid_x2<L, PG_RESID, 1>(grid, block, st, a);
            }
        }
        CSN_CHECK_LAUNCH();
        if (!out && l1) {
            sum_f64_kernel<<<1, 1024, 0, st>>>(partials, (int64_t)gx * gy * gz, 1.0, l1);
            CSN_CHECK_LAUNCH();
        }
        return CSN_OK;
    } else {
    if (out) {
        if (vec) launch_pg_resid<Real, L, PG_SWEEP, V>(grid, block, st, a);
        else launch_pg_resid<Real, L, PG_SWEEP, 1>(grid, block, st, a);
        CSN_CHECK_LAUNCH();
    } else {
        if (l1 && !partials) return CSN_E_ARG;
        if (a.avg_mode) {
            if (vec) launch_pg_resid<Real, L, PG_RESID_EMA, V>(grid, block, st, a);
            else launch_pg_resid<Real, L, PG_RESID_EMA, 1>(grid, block, st, a);
        } else {
            if (vec) launch_pg_resid<Real, L, PG_RESID, V>(grid, block, st, a);
            else launch_pg_resid<Real, L, PG_RESID, 1>(grid, block, st, a);
        }
        CSN_CHECK_LAUNCH();
        if (l1) {
            sum_f64_kernel<<<1, 1024, 0, st>>>(partials, (int64_t)gx * gy * gz, 1.0, l1);
            CSN_CHECK_LAUNCH();
        }
    }
    return CSN_OK;
    }
}

template <class Real, int L>
int pg_k_impl(const csn_geom* g, const double* taps, const double* cfg, const void* psi,
              int psi_h, const void* avg_in, int avg_in_h, void* avg_out, int avg_out_h,
              int avg_mode, double theta, const void* mu, const void* nu, void* kx, void* ky,
              int k_h, void* work, cudaStream_t st) {
    constexpr int T = 2 * L + 1;
    constexpr int KT = KTile<Real, L>::value;
    constexpr int TXO = KT - 2 * L;
    if (k_h < L) return CSN_E_ARG;
    if (!taps_match<L>(taps)) return CSN_E_ARG;
    if (avg_mode < 0 || avg_mode > 2) return CSN_E_SCHEME;
    if (avg_mode >= 1 && !avg_out) return CSN_E_ARG;
    if (avg_mode == 2 && (!avg_in || avg_in == avg_out)) return CSN_E_ARG;
    PGKArgs<Real> a;
    a.g = make_geo(*g);
    a.psi = (const Real*)psi; a.psi_h = psi_h;
    a.avg_in = (const Real*)avg_in; a.avg_in_h = avg_in ? avg_in_h : 0;
    a.avg_out = (Real*)avg_out; a.avg_out_h = avg_out ? avg_out_h : 0;
    a.avg_mode = avg_mode; a.theta = (Real)theta; a.omt = (Real)(1.0 - theta);
    a.eps = (Real)cfg[0]; a.alpha_r = (Real)cfg[1]; a.a_abs = (Real)cfg[2]; a.a_sq = (Real)cfg[3];
    a.dx = (Real)g->dx; a.dy = (Real)g->dy;
    a.inv_dx = (Real)(1.0 / g->dx); a.inv_dy = (Real)(1.0 / g->dy);
    {   // single rounded products in Real, as the device multiplication gave
        volatile Real cax = a.a_abs * a.dx, csx = a.a_sq * a.dx, cay = a.a_abs * a.dy,
                      csy = a.a_sq * a.dy;
        a.cax = cax; a.csx = csx; a.cay = cay; a.csy = csy;
    }
    a.mu = (const Real*)mu; a.nu = (const Real*)nu;
    a.kx = (Real*)kx; a.ky = (Real*)ky; a.k_h = k_h;
    constexpr int V = 16 / sizeof(Real);
    const bool vec = vec_ok(g, V);
    if constexpr (sizeof(Real) == 4 && L <= 3) {
      if (work && g_tune_k2_ws) {   // one pass, warp-specialised (no workspace traffic)
        const int gx = (int)cdiv(g->nx + 2 * L, WS_TX);
        const int gy = (int)cdiv((int64_t)g->nd * g->ng, X2_CC);
        a.ly = pick_ly((int64_t)gx * gy, g->ny + 2 * L, T, 2 * L, 148);
        dim3 grid(gx, gy, (int)cdiv(g->ny + 2 * L, a.ly)), block(32, 2 * WS_TX + 2 * L);
        if (avg_mode == 2) {
            if (vec) launch_pg_k_ws<L, true, V>(grid, block, st, a);
            else launch_pg_k_ws<L, true, 1>(grid, block, st, a);
        } else {
            if (vec) launch_pg_k_ws<L, false, V>(grid, block, st, a);
            else launch_pg_k_ws<L, false, 1>(grid, block, st, a);
        }
        CSN_CHECK_LAUNCH();
        return CSN_OK;
      }
      if (work) {   // split: K2a gradients -> workspace -> K2b coefficients
        float* gxp = (float*)work;
        float* gyp = gxp + grad_field_elems(g, L);
        const int gh = 2 * L;
        const int gy = (int)cdiv((int64_t)g->nd * g->ng, X2_CC);
        dim3 block(32, PG_TX);
        {
            const int gx = (int)cdiv(g->nx + 4 * L, PG_TX);
            a.ly = pick_ly((int64_t)gx * gy, g->ny + 4 * L, T, L, 148 * (L >= 3 ? 4 : 3));
            dim3 grid(gx, gy, (int)cdiv(g->ny + 4 * L, a.ly));
            if (avg_mode == 2) {
                if (vec) launch_pg_grad_x2<L, true, V>(grid, block, st, a, gxp, gyp, gh);
                else launch_pg_grad_x2<L, true, 1>(grid, block, st, a, gxp, gyp, gh);
            } else {
                if (vec) launch_pg_grad_x2<L, false, V>(grid, block, st, a, gxp, gyp, gh);
                else launch_pg_grad_x2<L, false, 1>(grid, block, st, a, gxp, gyp, gh);
            }
            CSN_CHECK_LAUNCH();
        }
        {
            const int gx = (int)cdiv(g->nx + 2 * L, PG_TX);
            a.ly = pick_ly((int64_t)gx * gy, g->ny + 2 * L, T, L, 148 * 3);
            dim3 grid(gx, gy, (int)cdiv(g->ny + 2 * L, a.ly));
            // TMA staging of the workspace rows (k2_tma), else the cp.async stager
            KcoefMaps km;     // the workspace is a field with halo gh = 2l
            // k2_tma: 1 = TMA K2b except at L = 2 (C2: 0.159 vs 0.166 ms cp.async; C3 0.48 -> 0.45,
            // C5-weak 25.1 -> 23.1 ms at L = 1), 2 = always
            const bool tk = (g_tune_k2_tma == 2 || (g_tune_k2_tma == 1 && L != 2)) && field_map(&km.gx, gxp, g, gh, PG_TX + 2 * L) &&
                            field_map(&km.gy, gyp, g, gh, PG_TX + 2 * L);
            if (tk) launch_pg_kcoef_tma<L>(grid, block, st, a, km, gh);
            else if (vec) launch_pg_kcoef_x2<L, V>(grid, block, st, a, gxp, gyp, gh);
            else launch_pg_kcoef_x2<L, 1>(grid, block, st, a, gxp, gyp, gh);
            if (!tk) cudaGetLastError();
            CSN_CHECK_LAUNCH();
        }
        return CSN_OK;
      }
      {   // fused two-stage, packed fp32x2, a lane per channel pair
        constexpr int TXO2 = X2_KT - 2 * L;
        const int gx = (int)cdiv(g->nx + 2 * L, TXO2);
        const int gy = (int)cdiv((int64_t)g->nd * g->ng, X2_CC);
        a.ly = pick_ly((int64_t)gx * gy, g->ny + 2 * L, T, 2 * L, L == 1 ? 148 * 2 : 148);
        const int gz = (int)cdiv(g->ny + 2 * L, a.ly);
        dim3 grid(gx, gy, gz), block(32, X2_KT);
        if (avg_mode == 2) {
            if (vec) launch_pg_k_x2<L, true, V>(grid, block, st, a);
            else launch_pg_k_x2<L, true, 1>(grid, block, st, a);
        } else {
            if (vec) launch_pg_k_x2<L, false, V>(grid, block, st, a);
            else launch_pg_k_x2<L, false, 1>(grid, block, st, a);
        }
        CSN_CHECK_LAUNCH();
        return CSN_OK;
      }
    } else {
    const int gx = (int)cdiv(g->nx + 2 * L, TXO);
    const int gy = (int)cdiv((int64_t)g->nd * g->ng, PG_CC);
    a.ly = pick_ly((int64_t)gx * gy, g->ny + 2 * L, T, 2 * L, 148);
    const int gz = (int)cdiv(g->ny + 2 * L, a.ly);
    dim3 grid(gx, gy, gz), block(PG_CC, KT);
    if (avg_mode == 2) {
        if (vec) launch_pg_k<Real, L, true, V>(grid, block, st, a);
        else launch_pg_k<Real, L, true, 1>(grid, block, st, a);
    } else {
        if (vec) launch_pg_k<Real, L, false, V>(grid, block, st, a);
        else launch_pg_k<Real, L, false, 1>(grid, block, st, a);
    }
    CSN_CHECK_LAUNCH();
    return CSN_OK;
    }
}

template <class Real>
int upwind_smooth_impl(const csn_geom* g, const void* src, int q_per_dof, int init_mode,
                       const void* init, int init_h, const csn_geom* gc, const void* sigma,
                       const void* mu, const void* nu, const void* strm, int n_sweeps,
                       double diag_scale, void* out, int out_h, cudaStream_t st, int fold = 0) {
    UpSmoothArgs<Real> a;
    a.fold = fold;
    a.g = make_geo(*g);
    a.src = (const Real*)src; a.q_per_dof = q_per_dof;
    a.init_mode = init_mode; a.init = (const Real*)init; a.init_h = init_h;
    a.angle_coarsens = 0;
    if (init_mode == 2) {
        a.gc = make_geo(*gc);
        if (gc->nx * 2 != g->nx || gc->ny * 2 != g->ny || gc->ng != g->ng) return CSN_E_ARG;
        if (gc->na == g->na) a.angle_coarsens = 0;
        else if (gc->na * 2 == g->na) a.angle_coarsens = 1;
        else return CSN_E_ARG;
    } else {
        a.gc = a.g;
    }
    a.sigma = (const Real*)sigma; a.mu = (const Real*)mu; a.nu = (const Real*)nu;
    a.strm = (const Real*)strm;
    a.inv_dx = (Real)(1.0 / g->dx); a.inv_dy = (Real)(1.0 / g->dy);
    a.scale = (Real)diag_scale; a.use_scale = diag_scale != 1.0;
    a.out = (Real*)out; a.out_h = out_h;
    a.exact_div = std::is_same<Real, float>::value ? g_tune_upwind_div : 0;   // fp64: r / d
    a.keep = (Real)(1.0 - 1.0 / diag_scale);
    if constexpr (std::is_same<Real, float>::value) {
        // packed channel-pair kernel when a 64-channel CTA lies in one face (see
        // upwind_smooth_x2_kernel); the scalar kernel covers every other case
        const int64_t C = (int64_t)g->nd * g->ng;
        const int64_t face = (int64_t)g->na * g->na * g->ng;
        const bool g1 = g->ng == 1;
        if (g_tune_upwind_x2 && n_sweeps == 3 && q_per_dof &&
            (a.exact_div == 3 || a.exact_div == 0) && C % UPX_CC == 0 &&
            face % UPX_CC == 0 &&
            !(g1 && init_mode == 2 && !a.angle_coarsens)) {
            const int gx = (int)cdiv(cdiv(g->ny, UPX_UT), UPX_SPB);
            const int gy = (int)(C / UPX_CC);
            const int chunks = up_chunks(g->nx, (int64_t)gx * gy, 4);
            a.xchunk = (int)cdiv(g->nx, chunks);
            const int gz = (int)cdiv(g->nx, a.xchunk);
            dim3 grid(gx, gy, gz), block(32, UPX_SPB);
            // TMA-staged columns (upwind_smooth_tma_kernel) where its layout applies
            // (default on since the last warp to release a column slot refills it: the
            // producer thread no longer waits for every warp each step — C4 correction
            // 1.99 -> 1.75 ms; with producer waits it had measured 1.18 vs 1.15 ms for
            // the register kernel)
            if (g_tune_upwind_tma && g1 && a.exact_div == 3 && init_mode != 1 && g->na >= 8 &&
                g->na <= 32 && g->ny % 4 == 0 &&
                (init_mode == 0 || (init_h == 0 && a.angle_coarsens))) {
                UpTmaMaps maps;
                // ghost x sides: the maps start H fine / 2 coarse columns before x = 0 and
                // end as many past nx (the x-ghosted source, sigma and coarse correction of
                // a DD rank); a physical side ends at the domain and TMA zero-fills
                const int gw = g->ghost_w ? UP_H : 0, ge = g->ghost_e ? UP_H : 0;
                const int cw = g->ghost_w ? (UP_H + 1) / 2 : 0, ce = g->ghost_e ? (UP_H + 1) / 2 : 0;
                a.tma_xoff = gw;
                a.tma_cxoff = cw;
                const cuuint64_t C64 = (cuuint64_t)C;
                cuuint64_t sd[3] = {C64, (cuuint64_t)g->ny, (cuuint64_t)(g->nx + gw + ge)};
                cuuint64_t ss[2] = {C64 * 4, C64 * 4 * g->ny};
                cuuint32_t sb[3] = {UPX_CC, UPT_ROWS, 1};
                cuuint64_t gd[2] = {(cuuint64_t)g->ny, (cuuint64_t)(g->nx + gw + ge)};
                cuuint64_t gs[1] = {(cuuint64_t)g->ny * 4};
                cuuint32_t gb[2] = {UPT_SIGROWS, 1};
                bool ok = raw_map(&maps.src, (const float*)src - (int64_t)gw * g->ny * C, 3, sd,
                                  ss, sb) &&
                          raw_map(&maps.sigma, (const float*)sigma - (int64_t)gw * g->ny, 2, gd,
                                  gs, gb);
                if (ok && init_mode == 2) {
                    const cuuint64_t Cc = (cuuint64_t)gc->nd * gc->ng;
                    cuuint64_t id[3] = {Cc, (cuuint64_t)gc->ny, (cuuint64_t)(gc->nx + cw + ce)};
                    cuuint64_t is[2] = {Cc * 4, Cc * 4 * gc->ny};
                    cuuint32_t ib[3] = {UPT_CCH, UPT_CROWS, 1};
                    ok = raw_map(&maps.init, (const float*)init - (int64_t)cw * gc->ny * Cc, 3,
                                 id, is, ib);
                } else if (ok) {
                    maps.init = maps.src;   // unused (mode 0)
                }
                if (ok) {
                    upwind_smooth_tma_kernel<<<grid, block, 0, st>>>(a, maps);
                    CSN_CHECK_LAUNCH();
                    return CSN_OK;
                }
                cudaGetLastError();
            }
            auto go = [&](auto gmt, auto dmt) {
                upwind_smooth_x2_kernel<3, decltype(gmt)::value, decltype(dmt)::value>
                    <<<grid, block, 0, st>>>(a);
            };
            using G0 = std::integral_constant<int, 0>;
            using G1_ = std::integral_constant<int, 1>;
            using G2 = std::integral_constant<int, 2>;
            using D0 = std::integral_constant<int, 0>;
            using D3 = std::integral_constant<int, 3>;
            // packed update forms: 3 (Jacobi, default) and 0 (fused reciprocal); the
            // other forms run in the scalar kernel
            auto pick = [&](auto gmt) {
                if (a.exact_div == 3) go(gmt, D3());
                else go(gmt, D0());
            };
            if (g1) pick(G0()); else if (g->ng % 2 == 0) pick(G1_()); else pick(G2());
            CSN_CHECK_LAUNCH();
            return CSN_OK;
        }
    }
    if constexpr (std::is_same<Real, float>::value) {
        // single-lane face-uniform kernel: 32-channel CTAs inside one face (odd ng)
        const int64_t C = (int64_t)g->nd * g->ng;
        const int64_t face = (int64_t)g->na * g->na * g->ng;
        if (g_tune_upwind_x2 && n_sweeps == 3 && q_per_dof && a.exact_div == 3 &&
            C % UPX1_CC == 0 && face % UPX1_CC == 0) {
            const int gx = (int)cdiv(cdiv(g->ny, UPX_UT), UPX_SPB);
            const int gy = (int)(C / UPX1_CC);
            const int chunks = up_chunks(g->nx, (int64_t)gx * gy, 4);
            a.xchunk = (int)cdiv(g->nx, chunks);
            const int gz = (int)cdiv(g->nx, a.xchunk);
            upwind_smooth_x1_kernel<3><<<dim3(gx, gy, gz), dim3(32, UPX_SPB), 0, st>>>(a);
            CSN_CHECK_LAUNCH();
            return CSN_OK;
        }
    }
    const int gx = (int)cdiv(cdiv(g->ny, UT), UP_SPB);
    const int gy = (int)cdiv((int64_t)g->nd * g->ng, UP_CC);
    // x chunks: keep chunks long against the H-column warm-up, fill the machine
    const int chunks = up_chunks(g->nx, (int64_t)gx * gy, 1);
    a.xchunk = (int)cdiv(g->nx, chunks);
    const int gz = (int)cdiv(g->nx, a.xchunk);
    dim3 grid(gx, gy, gz), block(UP_CC, UP_SPB);
    switch (n_sweeps) {
        case 0: upwind_smooth_kernel<Real, 0><<<grid, block, 0, st>>>(a); break;
        case 1: upwind_smooth_kernel<Real, 1><<<grid, block, 0, st>>>(a); break;
        case 2: upwind_smooth_kernel<Real, 2><<<grid, block, 0, st>>>(a); break;
        default: upwind_smooth_kernel<Real, 3><<<grid, block, 0, st>>>(a); break;
    }
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

#define DTYPE_DISPATCH(dtype, FN, ...)                         \
    ((dtype) == CSN_F32 ? FN<float>(__VA_ARGS__)               \
     : (dtype) == CSN_F64 ? FN<double>(__VA_ARGS__) : CSN_E_DTYPE)

}  // namespace

extern "C" {

int csn_version(void) { return kVersion; }

unsigned long long csn_launch_count(void) { return g_launches; }

int csn_set_tuning(const char* key, int value, int* prev) {
    if (!key) return CSN_E_ARG;
    int* slot = nullptr;
    if (!strcmp(key, "upwind_x2")) slot = &g_tune_upwind_x2;
    if (!strcmp(key, "tail_smem")) slot = &g_tune_tail_smem;
    if (!strcmp(key, "tail_faces")) slot = &g_tune_tail_faces;
    if (!strcmp(key, "pg_chunks")) slot = &g_tune_pg_chunks;
    if (!strcmp(key, "upwind_div")) slot = &g_tune_upwind_div;
    if (!strcmp(key, "sweep_div")) slot = &g_tune_sweep_div;
    if (!strcmp(key, "pg_tma")) slot = &g_tune_pg_tma;
    if (!strcmp(key, "upwind_tma")) slot = &g_tune_upwind_tma;
    if (!strcmp(key, "k2_tma")) slot = &g_tune_k2_tma;
    if (!strcmp(key, "k2_ws")) slot = &g_tune_k2_ws;
    if (!strcmp(key, "pg_xb")) slot = &g_tune_pg_xb;
    if (!slot) return CSN_E_ARG;
    if (prev) *prev = *slot;
    *slot = value;
    return CSN_OK;
}

const char* csn_error_string(int code) {
    switch (code) {
        case CSN_OK: return "ok";
        case CSN_E_ARG: return "invalid argument";
        case CSN_E_ORDER: return "unsupported ConvFEM order (expected 1, 2, 3 or 5)";
        case CSN_E_DTYPE: return "unsupported dtype";
        case CSN_E_SCHEME: return "unsupported mode";
        default: break;
    }
    if (code < 0) return cudaGetErrorString((cudaError_t)(-code));
    return "unknown error";
}

int64_t csn_partials_size(int dtype, const csn_geom* g, int order) {
    (void)dtype;
    if (!geom_ok(g)) return -CSN_E_ARG;
    const int64_t C = (int64_t)g->nd * g->ng;
    int64_t pg = cdiv(g->nx, PG_TX) * cdiv(C, PG_CC) * (int64_t)g->ny;   // upper bound (ly >= 1)
    int64_t up = grid1d((int64_t)g->nx * g->ny * C);
    int64_t cells = grid1d((int64_t)g->nx * g->ny * g->ng);
    (void)order;
    int64_t m = pg > up ? pg : up;
    return m > cells ? m : cells;
}

int csn_apply_boundary(int dtype, const csn_geom* g, void* f, int halo, const void* mu,
                       const void* nu, void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !f || !mu || !nu || halo < 0) return CSN_E_ARG;
    if (halo == 0) return CSN_OK;
    Geo d = make_geo(*g);
    const int64_t cells = (int64_t)2 * halo * (g->ny + 2 * halo) + (int64_t)g->nx * 2 * halo;
    if (cells > INT32_MAX) return CSN_E_ARG;
    // a few CTAs per SM, each looping over halo cells (one cell per CTA is launch-bound)
    const int64_t face = (int64_t)g->na * g->na * g->ng;
    if (dtype == CSN_F32 && d.C % 4 == 0 && face % 4 == 0 &&
        (reinterpret_cast<uintptr_t>(f) & 15) == 0) {
        const int64_t gx4 = cdiv(d.C / 4, 256);
        int64_t gy4 = cdiv(148 * 8, gx4);
        if (gy4 > cells) gy4 = cells;
        if (gy4 > 65535) gy4 = 65535;
        boundary4_kernel<<<dim3((unsigned)gx4, (unsigned)(gy4 < 1 ? 1 : gy4)), 256, 0, S(stream)>>>(
            d, (float*)f, halo, (const float*)mu, (const float*)nu);
        CSN_CHECK_LAUNCH();
        return CSN_OK;
    }
    const int64_t gxb = cdiv(d.C, 256);
    int64_t gyb = cdiv(148 * 8, gxb);
    if (gyb > cells) gyb = cells;
    if (gyb > 65535) gyb = 65535;
    dim3 grid((unsigned)gxb, (unsigned)(gyb < 1 ? 1 : gyb));
    if (dtype == CSN_F32)
        boundary_kernel<float><<<grid, 256, 0, S(stream)>>>(d, (float*)f, halo, (const float*)mu,
                                                            (const float*)nu);
    else if (dtype == CSN_F64)
        boundary_kernel<double><<<grid, 256, 0, S(stream)>>>(d, (double*)f, halo,
                                                             (const double*)mu, (const double*)nu);
    else return CSN_E_DTYPE;
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

int csn_upwind_residual(int dtype, const csn_geom* g, const void* psi, int psi_halo,
                        const void* sigma, const void* q, int q_per_dof, const void* mu,
                        const void* nu, void* r, int r_halo, double* partials, double* l1,
                        void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !psi || !sigma || !q || !mu || !nu || psi_halo < 1) return CSN_E_ARG;
    if (l1 && !partials) return CSN_E_ARG;
    const int64_t total = (int64_t)g->nx * g->ny * g->nd * g->ng;
    const int nb = grid1d(total);
    auto run = [&](auto tag) -> int {
        using Real = decltype(tag);
        UpResArgs<Real> a;
        a.g = make_geo(*g);
        a.psi = (const Real*)psi; a.psi_h = psi_halo;
        a.sigma = (const Real*)sigma; a.q = (const Real*)q; a.q_per_dof = q_per_dof;
        a.mu = (const Real*)mu; a.nu = (const Real*)nu;
        a.dx = (Real)g->dx; a.dy = (Real)g->dy;
        a.r = (Real*)r; a.r_h = r_halo;
        a.partials = l1 ? partials : nullptr;
        upwind_residual_kernel<Real><<<nb, 256, 0, S(stream)>>>(a);
        CSN_CHECK_LAUNCH();
        if (l1) {
            sum_f64_kernel<<<1, 1024, 0, S(stream)>>>(partials, nb, 1.0, l1);
            CSN_CHECK_LAUNCH();
        }
        return CSN_OK;
    };
    if (dtype == CSN_F32) return run(float());
    if (dtype == CSN_F64) return run(double());
    return CSN_E_DTYPE;
}

int csn_upwind_smooth(int dtype, const csn_geom* g, const void* src, int q_per_dof,
                      int init_mode, const void* init, int init_halo, const csn_geom* gc,
                      const void* sigma, const void* mu, const void* nu, const void* strm,
                      int n_sweeps, double diag_scale, void* out, int out_halo, void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !src || !sigma || !mu || !nu || !strm || !out || n_sweeps < 0 ||
        n_sweeps > UP_H)
        return CSN_E_ARG;
    if (init_mode < 0 || init_mode > 2) return CSN_E_SCHEME;
    if (init_mode > 0 && !init) return CSN_E_ARG;
    if (init_mode == 2 && !geom_ok(gc)) return CSN_E_ARG;
    if (init_mode == 1 && init == out && n_sweeps > 0) return CSN_E_ARG;
    return DTYPE_DISPATCH(dtype, upwind_smooth_impl, g, src, q_per_dof, init_mode, init, init_halo,
                          gc, sigma, mu, nu, strm, n_sweeps, diag_scale, out, out_halo, S(stream));
}

int csn_upwind_smooth_sub(int dtype, const csn_geom* g, const void* src, int q_per_dof,
                          int init_mode, const void* init, int init_halo, const csn_geom* gc,
                          const void* sigma, const void* mu, const void* nu, const void* strm,
                          int n_sweeps, double diag_scale, void* psi, int psi_halo,
                          void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !src || !sigma || !mu || !nu || !strm || !psi || n_sweeps < 0 ||
        n_sweeps > UP_H)
        return CSN_E_ARG;
    if (init_mode < 0 || init_mode > 2) return CSN_E_SCHEME;
    if (init_mode > 0 && !init) return CSN_E_ARG;
    if (init_mode == 2 && !geom_ok(gc)) return CSN_E_ARG;
    if (init == psi || src == psi) return CSN_E_ARG;
    auto run = [&](auto tag) -> int {
        using Real = decltype(tag);
        return upwind_smooth_impl<Real>(g, src, q_per_dof, init_mode, init, init_halo, gc, sigma,
                                        mu, nu, strm, n_sweeps, diag_scale, psi, psi_halo,
                                        S(stream), 1);
    };
    if (dtype == CSN_F32) return run(float());
    if (dtype == CSN_F64) return run(double());
    return CSN_E_DTYPE;
}

int csn_restrict(int dtype, const csn_geom* gf, const csn_geom* gc, const void* fine,
                 int fine_halo, const void* w_f, const void* w_c, int normalise, void* coarse,
                 int coarse_halo, void* stream) {
    CSN_NVTX();
    if (!geom_ok(gf) || !geom_ok(gc) || !fine || !w_f || !coarse) return CSN_E_ARG;
    if (normalise && !w_c) return CSN_E_ARG;
    if (gc->nx * 2 != gf->nx || gc->ny * 2 != gf->ny || gc->ng != gf->ng) return CSN_E_ARG;
    int ac;
    if (gc->na == gf->na) ac = 0;
    else if (gc->na * 2 == gf->na) ac = 1;
    else return CSN_E_ARG;
    auto run = [&](auto tag) -> int {
        using Real = decltype(tag);
        RestrictArgs<Real> a;
        a.gf = make_geo(*gf); a.gc = make_geo(*gc);
        a.fine = (const Real*)fine; a.fine_h = fine_halo;
        a.wf = (const Real*)w_f; a.wc = (const Real*)w_c;
        a.af = (Real)(gf->dx * gf->dy); a.ac = (Real)(gc->dx * gc->dy);
        a.angle_coarsens = ac; a.normalise = normalise;
        a.coarse = (Real*)coarse; a.coarse_h = coarse_halo;
        const int64_t cells = (int64_t)gc->nx * gc->ny;
        if (cells > INT32_MAX) return CSN_E_ARG;
        // enough CTAs to fill the machine ~8 deep; each strides over coarse cells
        const int64_t gxc = cdiv((int64_t)gc->nd * gc->ng, 256);
        int64_t gyc = cdiv(148 * 16, gxc);
        if (gyc > cells) gyc = cells;
        if (gyc > 65535) gyc = 65535;
        if (gyc < 1) gyc = 1;
        restrict_kernel<Real><<<dim3((unsigned)gxc, (unsigned)gyc), 256, 0, S(stream)>>>(a);
        CSN_CHECK_LAUNCH();
        return CSN_OK;
    };
    if (dtype == CSN_F32) return run(float());
    if (dtype == CSN_F64) return run(double());
    return CSN_E_DTYPE;
}

int csn_coarse_tail(int dtype, int n, const csn_geom* geoms, const void* const* sigma,
                    const void* const* mu, const void* const* nu, const void* const* strm,
                    const void* const* w, void* const* src, void* const* delta, void* scratch,
                    int n_sweeps, void* stream) {
    CSN_NVTX();
    if (n < 1 || n > TAIL_MAX_LEVELS || !geoms || !sigma || !mu || !nu || !strm || !w || !src ||
        !delta || !scratch || n_sweeps < 0)
        return CSN_E_ARG;
    for (int i = 0; i < n; ++i) {
        const csn_geom& g = geoms[i];
        if (!geom_ok(&g) || g.ghost_w || g.ghost_e || !sigma[i] || !mu[i] || !nu[i] || !strm[i] ||
            !w[i] || !src[i] || !delta[i])
            return CSN_E_ARG;
        if ((int64_t)g.nx * g.ny * g.nd * g.ng > CSN_TAIL_MAX_DOF) return CSN_E_ARG;
        if (i > 0) {
            const csn_geom& f = geoms[i - 1];
            if (g.nx * 2 != f.nx || g.ny * 2 != f.ny || g.ng != f.ng ||
                (g.na != f.na && g.na * 2 != f.na))
                return CSN_E_ARG;
        }
    }
    auto run = [&](auto tag) -> int {
        using Real = decltype(tag);
        TailArgs<Real> t;
        t.n = n;
        for (int i = 0; i < n; ++i) {
            TailLevel<Real>& L = t.lv[i];
            L.g = make_geo(geoms[i]);
            L.dv.C = make_fastdiv(L.g.C); L.dv.ny = make_fastdiv(L.g.ny);
            L.dv.ng = make_fastdiv(L.g.ng); L.dv.per = make_fastdiv(L.g.na * L.g.na);
            L.dv.na = make_fastdiv(L.g.na);
            L.sigma = (const Real*)sigma[i];
            L.mu = (const Real*)mu[i]; L.nu = (const Real*)nu[i];
            L.strm = (const Real*)strm[i]; L.w = (const Real*)w[i];
            L.src = (Real*)src[i]; L.delta = (Real*)delta[i];
            L.inv_dx = (Real)(1.0 / geoms[i].dx); L.inv_dy = (Real)(1.0 / geoms[i].dy);
            L.area = (Real)(geoms[i].dx * geoms[i].dy);
            L.sig_stride = L.g.ng;
            const int per = L.g.na * L.g.na;
            L.fdv.C = make_fastdiv(per); L.fdv.ny = make_fastdiv(L.g.ny);
            L.fdv.ng = make_fastdiv(1); L.fdv.per = make_fastdiv(per);
            L.fdv.na = make_fastdiv(L.g.na);
            L.face_off = 0;
            L.const_off = 0;
        }
        t.scratch = (Real*)scratch;
        t.n_sweeps = n_sweeps;
        t.exact_div = std::is_same<Real, float>::value ? g_tune_upwind_div : 0;
        // one CTA per (face, group), everything in shared memory, when every level's slice
        // fits (csn_set_tuning "tail_faces", default on); else the cluster kernel
        {
            bool faces = g_tune_tail_faces != 0;
            int off = 0, coff = 0;
            for (int i = 0; i < n && faces; ++i) {
                const int per = geoms[i].na * geoms[i].na;
                const int64_t dof = (int64_t)geoms[i].nx * geoms[i].ny * per;
                if (geoms[i].nd % per || dof > TAIL_FACE_DOF) faces = false;
                t.lv[i].face_off = off;
                off += (int)((dof + 1) & ~(int64_t)1);        // even: 8-byte pair loads
                t.lv[i].const_off = coff;
                coff += 4 * per + geoms[i].nx * geoms[i].ny;
            }
            if (faces && off <= TAIL_FACE_SUM && coff <= TAIL_FACE_CONST) {
                constexpr size_t fsm = coarse_tail_face_smem<Real>();
                static bool fattr = false;
                if (!fattr) {
                    cudaFuncSetAttribute(coarse_tail_face_kernel<Real>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
                    fattr = true;
                }
                const int nfaces = geoms[0].nd / (geoms[0].na * geoms[0].na);
                coarse_tail_face_kernel<Real><<<nfaces * geoms[0].ng, TAIL_THREADS, fsm, S(stream)>>>(t);
                CSN_CHECK_LAUNCH();
                return CSN_OK;
            }
        }
        // levels of <= TAIL_SMEM_DOF unknowns (never the tail's first: its source is the
        // caller's) are solved in CTA 0's shared memory
        t.n_smem_first = n;
        for (int i = n - 1; i >= 1; --i) {
            const int64_t dof = (int64_t)geoms[i].nx * geoms[i].ny * geoms[i].nd * geoms[i].ng;
            if (dof > TAIL_SMEM_DOF || !g_tune_tail_smem) break;
            t.n_smem_first = i;
        }
        int off = 0;
        for (int i = 0; i < TAIL_MAX_LEVELS; ++i) {
            t.smem_off[i] = 0;
            if (i >= t.n_smem_first && i < n) {
                t.smem_off[i] = off;
                off += geoms[i].nx * geoms[i].ny * geoms[i].nd * geoms[i].ng;
            }
        }
        if (off > TAIL_SMEM_SUM) return CSN_E_ARG;
        constexpr size_t smem = coarse_tail_smem<Real>();
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(coarse_tail_kernel<Real>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            attr = true;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(TAIL_CTAS);
        cfg.blockDim = dim3(TAIL_THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = S(stream);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = TAIL_CTAS;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, coarse_tail_kernel<Real>, t);
        if (e != cudaSuccess) return -(int)e;
        ++g_launches;
        return CSN_OK;
    };
    if (dtype == CSN_F32) return run(float());
    if (dtype == CSN_F64) return run(double());
    return CSN_E_DTYPE;
}

int csn_prolong(int dtype, const csn_geom* gc, const csn_geom* gf, const void* coarse,
                int coarse_halo, void* fine, int fine_halo, void* stream) {
    CSN_NVTX();
    if (!geom_ok(gf) || !geom_ok(gc) || !fine || !coarse) return CSN_E_ARG;
    if (gc->nx * 2 != gf->nx || gc->ny * 2 != gf->ny || gc->ng != gf->ng) return CSN_E_ARG;
    int ac;
    if (gc->na == gf->na) ac = 0;
    else if (gc->na * 2 == gf->na) ac = 1;
    else return CSN_E_ARG;
    const int64_t total = (int64_t)gf->nx * gf->ny * gf->nd * gf->ng;
    auto run = [&](auto tag) -> int {
        using Real = decltype(tag);
        ProlongArgs<Real> a;
        a.gc = make_geo(*gc); a.gf = make_geo(*gf);
        a.coarse = (const Real*)coarse; a.coarse_h = coarse_halo;
        a.angle_coarsens = ac;
        a.fine = (Real*)fine; a.fine_h = fine_halo;
        prolong_kernel<Real><<<grid1d(total), 256, 0, S(stream)>>>(a);
        CSN_CHECK_LAUNCH();
        return CSN_OK;
    };
    if (dtype == CSN_F32) return run(float());
    if (dtype == CSN_F64) return run(double());
    return CSN_E_DTYPE;
}

#define ORDER_DISPATCH(FN, ...)                                                         \
    switch (order) {                                                                    \
        case 1: return dtype == CSN_F32 ? FN<float, 1>(__VA_ARGS__) : FN<double, 1>(__VA_ARGS__); \
        case 2: return dtype == CSN_F32 ? FN<float, 2>(__VA_ARGS__) : FN<double, 2>(__VA_ARGS__); \
        case 3: return dtype == CSN_F32 ? FN<float, 3>(__VA_ARGS__) : FN<double, 3>(__VA_ARGS__); \
        case 5: return dtype == CSN_F32 ? FN<float, 5>(__VA_ARGS__) : FN<double, 5>(__VA_ARGS__); \
        default: return CSN_E_ORDER;                                                    \
    }

int csn_pg_diffusivities(int dtype, int order, const csn_geom* g, const double* taps,
                         const double* cfg, const void* psi, int psi_halo, const void* avg_in,
                         int avg_in_halo, void* avg_out, int avg_out_halo, int avg_mode,
                         double theta, const void* mu, const void* nu, void* kx, void* ky,
                         int k_halo, void* work, void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !taps || !cfg || !psi || !mu || !nu || !kx || !ky) return CSN_E_ARG;
    if (dtype != CSN_F32 && dtype != CSN_F64) return CSN_E_DTYPE;
    ORDER_DISPATCH(pg_k_impl, g, taps, cfg, psi, psi_halo, avg_in, avg_in_halo, avg_out,
                   avg_out_halo, avg_mode, theta, mu, nu, kx, ky, k_halo, work, S(stream));
}

int64_t csn_pg_workspace_size(int dtype, const csn_geom* g, int order) {
    if (!geom_ok(g)) return -CSN_E_ARG;
    if (dtype != CSN_F32 || order < 1 || order > 3) return 0;
    return 2 * grad_field_elems(g, order) * (int64_t)sizeof(float);
}

int csn_pg_residual(int dtype, int order, const csn_geom* g, const double* taps,
                    const void* psi, int psi_halo, const void* delta, int delta_halo,
                    const void* kx, const void* ky, int k_halo, const void* sigma, const void* q,
                    int q_per_dof, const void* mu, const void* nu, const void* strm, void* r,
                    int r_halo, void* psi_out, int psi_out_halo, double beta, double* partials,
                    double* l1, void* avg, int avg_halo, int avg_mode, double theta,
                    void* dterm, int dterm_mode, void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !taps || !psi || !kx || !ky || !sigma || !q || !mu || !nu)
        return CSN_E_ARG;
    if (dterm_mode < 0 || dterm_mode > 2 || (dterm_mode && (!dterm || dtype != CSN_F32)))
        return CSN_E_ARG;
    if (psi_out && (!strm || psi_out == psi)) return CSN_E_ARG;
    if (dtype != CSN_F32 && dtype != CSN_F64) return CSN_E_DTYPE;
    ORDER_DISPATCH(pg_residual_impl, g, taps, psi, psi_halo, delta, delta_halo, kx, ky, k_halo,
                   sigma, q, q_per_dof, mu, nu, strm, r, r_halo, psi_out, psi_out_halo, beta,
                   partials, l1, avg, avg_halo, avg_mode, theta, dterm, dterm_mode, S(stream));
}

int csn_scalar_flux(int dtype, const csn_geom* g, const void* psi, int halo, const void* w,
                    double* phi, void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !psi || !w || !phi || halo < 0) return CSN_E_ARG;
    Geo d = make_geo(*g);
    if (g->ng <= 8) {      // one warp per cell (coalesced over the cell's channels)
        const int nb = grid1d((int64_t)g->nx * g->ny * 32);
        auto run = [&](auto tag) -> int {
            using Real = decltype(tag);
            const Real* p = (const Real*)psi;
            const Real* ww = (const Real*)w;
            switch (g->ng) {
                case 1: scalar_flux_cell_kernel<Real, 1><<<nb, 256, 0, S(stream)>>>(d, p, halo, ww, phi); break;
                case 2: scalar_flux_cell_kernel<Real, 2><<<nb, 256, 0, S(stream)>>>(d, p, halo, ww, phi); break;
                case 3: scalar_flux_cell_kernel<Real, 3><<<nb, 256, 0, S(stream)>>>(d, p, halo, ww, phi); break;
                case 4: scalar_flux_cell_kernel<Real, 4><<<nb, 256, 0, S(stream)>>>(d, p, halo, ww, phi); break;
                case 5: scalar_flux_cell_kernel<Real, 5><<<nb, 256, 0, S(stream)>>>(d, p, halo, ww, phi); break;
                case 6: scalar_flux_cell_kernel<Real, 6><<<nb, 256, 0, S(stream)>>>(d, p, halo, ww, phi); break;
                case 7: scalar_flux_cell_kernel<Real, 7><<<nb, 256, 0, S(stream)>>>(d, p, halo, ww, phi); break;
                default: scalar_flux_cell_kernel<Real, 8><<<nb, 256, 0, S(stream)>>>(d, p, halo, ww, phi); break;
            }
            CSN_CHECK_LAUNCH();
            return CSN_OK;
        };
        if (dtype == CSN_F32) return run(float());
        if (dtype == CSN_F64) return run(double());
        return CSN_E_DTYPE;
    }
    const int64_t warps = (int64_t)g->nx * g->ny * g->ng;
    const int nb = grid1d(warps * 32);
    if (dtype == CSN_F32)
        scalar_flux_kernel<float><<<nb, 256, 0, S(stream)>>>(d, (const float*)psi, halo, (const float*)w, phi);
    else if (dtype == CSN_F64)
        scalar_flux_kernel<double><<<nb, 256, 0, S(stream)>>>(d, (const double*)psi, halo, (const double*)w, phi);
    else return CSN_E_DTYPE;
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

int csn_group_source(int dtype, const csn_geom* g, const double* phi, const double* sigma_s,
                     const double* source, const double* fission, double lam, const double* chi,
                     const double* nsf, void* q, void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !phi || !sigma_s || !source || !q) return CSN_E_ARG;
    if (lam != 0.0 && (!chi || !nsf)) return CSN_E_ARG;
    Geo d = make_geo(*g);
    const int nb = grid1d((int64_t)g->nx * g->ny * g->ng);
    if (dtype == CSN_F32)
        group_source_kernel<float><<<nb, 256, 0, S(stream)>>>(d, phi, sigma_s, source, fission, lam, chi, nsf, (float*)q);
    else if (dtype == CSN_F64)
        group_source_kernel<double><<<nb, 256, 0, S(stream)>>>(d, phi, sigma_s, source, fission, lam, chi, nsf, (double*)q);
    else return CSN_E_DTYPE;
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

int csn_fission_source(const csn_geom* g, const double* phi, const double* chi,
                       const double* nsf, double inv_k, double* out, void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !phi || !chi || !nsf || !out) return CSN_E_ARG;
    Geo d = make_geo(*g);
    fission_source_kernel<<<grid1d((int64_t)g->nx * g->ny * g->ng), 256, 0, S(stream)>>>(d, phi, chi, nsf, inv_k, out);
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

int csn_production(const csn_geom* g, const double* phi, const double* nsf, double* partials,
                   double* out, void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !phi || !nsf || !partials || !out) return CSN_E_ARG;
    const int64_t n = (int64_t)g->nx * g->ny * g->ng;
    const int nb = grid1d(n);
    dot_partials_kernel<<<nb, 256, 0, S(stream)>>>(nsf, phi, n, partials);
    CSN_CHECK_LAUNCH();
    sum_f64_kernel<<<1, 1024, 0, S(stream)>>>(partials, nb, g->dx * g->dy, out);
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

int csn_sum_f64(const double* x, int64_t n, double* out, void* stream) {
    CSN_NVTX();
    if (!x || !out || n < 0) return CSN_E_ARG;
    sum_f64_kernel<<<1, 1024, 0, S(stream)>>>(x, n, 1.0, out);
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

int csn_scale(int dtype, void* x, int64_t n, double s, int divide, void* stream) {
    CSN_NVTX();
    if (!x || n < 0) return CSN_E_ARG;
    if (n == 0) return CSN_OK;
    if (dtype == CSN_F32)
        scale_kernel<float><<<grid1d(n), 256, 0, S(stream)>>>((float*)x, n, (float)s, divide);
    else if (dtype == CSN_F64)
        scale_kernel<double><<<grid1d(n), 256, 0, S(stream)>>>((double*)x, n, s, divide);
    else return CSN_E_DTYPE;
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

int csn_sub_interior(int dtype, const csn_geom* g, void* psi, int psi_halo, const void* delta,
                     int delta_halo, void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !psi || !delta) return CSN_E_ARG;
    Geo d = make_geo(*g);
    const int nb = grid1d((int64_t)g->nx * g->ny * d.C);
    if (dtype == CSN_F32)
        sub_interior_kernel<float><<<nb, 256, 0, S(stream)>>>(d, (float*)psi, psi_halo, (const float*)delta, delta_halo);
    else if (dtype == CSN_F64)
        sub_interior_kernel<double><<<nb, 256, 0, S(stream)>>>(d, (double*)psi, psi_halo, (const double*)delta, delta_halo);
    else return CSN_E_DTYPE;
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

int csn_ema(int dtype, const csn_geom* g, void* avg, int avg_halo, const void* psi,
            int psi_halo, double theta, int mode, void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !avg || !psi) return CSN_E_ARG;
    if (mode != 1 && mode != 2) return CSN_E_SCHEME;
    Geo d = make_geo(*g);
    const int nb = grid1d((int64_t)g->nx * g->ny * d.C);
    if (dtype == CSN_F32)
        ema_kernel<float><<<nb, 256, 0, S(stream)>>>(d, (float*)avg, avg_halo, (const float*)psi, psi_halo, (float)theta, (float)(1.0 - theta), mode);
    else if (dtype == CSN_F64)
        ema_kernel<double><<<nb, 256, 0, S(stream)>>>(d, (double*)avg, avg_halo, (const double*)psi, psi_halo, theta, 1.0 - theta, mode);
    else return CSN_E_DTYPE;
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

int csn_dir_lincomb(int dtype, int64_t n, int C, int ng, const void* x, const void* A, double ca,
                    const void* y, const void* B, double cb, double scale, void* out,
                    void* stream) {
    CSN_NVTX();
    if (!x || !out || n < 0 || C < 1 || ng < 1) return CSN_E_ARG;
    if (n == 0) return CSN_OK;
    if (dtype == CSN_F32)
        dir_lincomb_kernel<float><<<grid1d(n), 256, 0, S(stream)>>>(n, C, ng, (const float*)x, (const float*)A, (float)ca, (const float*)y, (const float*)B, (float)cb, (float)scale, (float*)out);
    else if (dtype == CSN_F64)
        dir_lincomb_kernel<double><<<grid1d(n), 256, 0, S(stream)>>>(n, C, ng, (const double*)x, (const double*)A, ca, (const double*)y, (const double*)B, cb, scale, (double*)out);
    else return CSN_E_DTYPE;
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

int csn_iso_diffusivity(int dtype, int64_t n, int C, int ng, const void* r, const void* px,
                        const void* py, const void* mu, const void* nu, const double* cfg,
                        void* k, void* stream) {
    CSN_NVTX();
    if (!r || !px || !py || !mu || !nu || !cfg || !k || n < 0) return CSN_E_ARG;
    if (n == 0) return CSN_OK;
    if (dtype == CSN_F32)
        iso_diffusivity_kernel<float><<<grid1d(n), 256, 0, S(stream)>>>(n, C, ng, (const float*)r, (const float*)px, (const float*)py, (const float*)mu, (const float*)nu, (float)cfg[0], (float)cfg[1], (float)cfg[2], (float)cfg[3], (float)cfg[4], (float)cfg[5], (float*)k);
    else if (dtype == CSN_F64)
        iso_diffusivity_kernel<double><<<grid1d(n), 256, 0, S(stream)>>>(n, C, ng, (const double*)r, (const double*)px, (const double*)py, (const double*)mu, (const double*)nu, cfg[0], cfg[1], cfg[2], cfg[3], cfg[4], cfg[5], (double*)k);
    else return CSN_E_DTYPE;
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

int csn_convolve(int dtype, const csn_geom* g, const void* src, int halo, const double* stencil,
                 int width, int margin, const void* dir_scale, void* out, void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !src || !stencil || !out || width < 1 || width > 11 || !(width & 1))
        return CSN_E_ARG;
    if (margin < 0 || margin + (width - 1) / 2 > halo) return CSN_E_ARG;
    Geo d = make_geo(*g);
    StencilW w;
    memset(&w, 0, sizeof(w));
    memcpy(w.w, stencil, sizeof(double) * width * width);
    const int64_t total = (int64_t)(g->nx + 2 * halo) * (g->ny + 2 * halo) * d.C;
    if (dtype == CSN_F32)
        convolve_kernel<float><<<grid1d(total), 256, 0, S(stream)>>>(d, (const float*)src, halo, w, width, margin, (const float*)dir_scale, (float*)out);
    else if (dtype == CSN_F64)
        convolve_kernel<double><<<grid1d(total), 256, 0, S(stream)>>>(d, (const double*)src, halo, w, width, margin, (const double*)dir_scale, (double*)out);
    else return CSN_E_DTYPE;
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

int csn_pass1d(int dtype, const csn_geom* g, const void* src, int halo, const double* taps,
               int width, int axis, int margin, void* out, void* stream) {
    CSN_NVTX();
    if (!geom_ok(g) || !src || !taps || !out || width < 1 || width > 121 || !(width & 1))
        return CSN_E_ARG;
    if (axis != 0 && axis != 1) return CSN_E_ARG;
    if (margin < 0 || margin + (width - 1) / 2 > halo) return CSN_E_ARG;
    Geo d = make_geo(*g);
    StencilW w;
    memset(&w, 0, sizeof(w));
    memcpy(w.w, taps, sizeof(double) * width);
    const int64_t total = (int64_t)(g->nx + 2 * halo) * (g->ny + 2 * halo) * d.C;
    if (dtype == CSN_F32)
        pass1d_kernel<float><<<grid1d(total), 256, 0, S(stream)>>>(d, (const float*)src, halo, w, width, axis, margin, (float*)out);
    else if (dtype == CSN_F64)
        pass1d_kernel<double><<<grid1d(total), 256, 0, S(stream)>>>(d, (const double*)src, halo, w, width, axis, margin, (double*)out);
    else return CSN_E_DTYPE;
    CSN_CHECK_LAUNCH();
    return CSN_OK;
}

}  // extern "C"
