// Coarse tail of the correction in ONE launch (R/multigrid.py:309-339 on the levels that
// hold at most a few DOF per thread of one CTA): the restriction chain down from the
// tail's finest level, then upwind Jacobi sweeps from the coarsest level up with the
// piecewise-constant prolongation as each level's initial iterate.
//
// As separate launches these levels are pure latency: a 16 x 16 level is one CTA marching
// 11 dependent column steps (~1.5 us each) behind a ~3 us launch, ~95 us for the six
// smallest levels of C3/C4 against ~0.2 us of arithmetic.  Here one thread-block cluster
// (8 CTAs x 1024 threads, co-scheduled on 8 SMs) owns every tail level: a stage is a
// cluster-stride loop over the level's DOF and a hardware cluster barrier
// (barrier.cluster, release / acquire: global writes of one CTA are visible to the others
// after it); the sweeps are plain Jacobi passes over ping-pong buffers (no temporal
// blocking: nothing to amortise when the level sits in L2).  Data produced inside the
// launch is read with ld.global.cg (L2), never through a possibly stale L1 line.
//
// Arithmetic is the marching kernels': restrict_cells (misc_kernels.cuh) and the update
// forms of upwind_kernels.cuh with the same operands — out-of-domain upwind neighbours
// are 0, as the marched warm-up columns / rows are (zero inflow, zero source) — so the
// fp32 result is bit-identical to csn_restrict + csn_upwind_smooth level by level
// (tests/test_gpu_parity.py::test_coarse_tail_matches_levels).
#pragma once
#include "misc_kernels.cuh"
#include "upwind_kernels.cuh"

namespace csn {

constexpr int TAIL_MAX_LEVELS = 12;
constexpr int TAIL_THREADS = 1024;
constexpr int TAIL_CTAS = 8;             // one portable-size cluster
constexpr int TAIL_STRIDE = TAIL_THREADS * TAIL_CTAS;

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <class Real>
struct TailLevel {
    Geo g;
    const Real* sigma;   // [nx][ny][ng]
    const Real* mu; const Real* nu; const Real* strm; const Real* w;   // [nd]
    Real* src;           // [nx][ny][C]: given on level 0 of the tail, restricted below
    Real* delta;         // [nx][ny][C]: the level's smoothed correction (output)
    Real inv_dx, inv_dy, area;
};

template <class Real>
struct TailArgs {
    int n;                                   // tail levels, finest first
    TailLevel<Real> lv[TAIL_MAX_LEVELS];
    Real* scratch;                           // >= the largest tail level's DOF
    int n_sweeps;
    int exact_div;                           // fp32 update form (csn_set_tuning "upwind_div")
};

// one update with the scalar smoother's form selection (upwind_smooth_kernel)
template <class Real>
__device__ __forceinline__ Real tail_update(int form, Real ce, Real xu, Real yu, Real amx,
                                            Real amy, Real sg, Real sv, Real inv, Real d) {
    if (form >= 3) return up_update_jac(ce, xu, yu, amx, amy, sv, inv, d, Real(0), form == 3);
    if (form == 2) return up_update_ref(ce, xu, yu, amx, amy, sg, sv, inv, d);
    if (form) return up_update_div(ce, xu, yu, amx, amy, sg, sv, d);
    return up_update(ce, xu, yu, amx, amy, sg, sv, inv, d);
}

template <class Real>
__global__ void __launch_bounds__(TAIL_THREADS, 1) coarse_tail_kernel(const TailArgs<Real> t) {
    const int tid = blockIdx.x * TAIL_THREADS + threadIdx.x;     // grid = one cluster
    // ---- restriction chain: src[i] from src[i - 1]
    for (int i = 1; i < t.n; ++i) {
        const TailLevel<Real>& lf = t.lv[i - 1];
        const TailLevel<Real>& lc = t.lv[i];
        RestrictArgs<Real> a;
        a.gf = lf.g; a.gc = lc.g;
        a.fine = lf.src; a.fine_h = 0;
        a.wf = lf.w; a.wc = lc.w;
        a.af = lf.area; a.ac = lc.area;
        a.angle_coarsens = lc.g.na != lf.g.na;
        a.normalise = 1;
        a.coarse = lc.src; a.coarse_h = 0;
        const int C = lc.g.C, total = C * lc.g.nx * lc.g.ny;
        for (int e = tid; e < total; e += TAIL_STRIDE)
            restrict_cells(a, e % C, e / C, 1 << 30);
        cluster_sync_all();
    }
    // ---- smoothing, coarsest level up; sweep s reads `in` (the prolonged coarser
    //      correction, or zero, for s = 0) and writes the buffer whose last turn is delta
    for (int i = t.n - 1; i >= 0; --i) {
        const TailLevel<Real>& L = t.lv[i];
        const Geo& g = L.g;
        const int C = g.C, ny = g.ny, nx = g.nx, total = C * nx * ny;
        const bool has_c = i + 1 < t.n;
        const Geo gc = has_c ? t.lv[i + 1].g : g;
        const Real* cd = has_c ? t.lv[i + 1].delta : nullptr;
        const bool ac = has_c && gc.na != g.na;
        if (t.n_sweeps == 0) {
            for (int e = tid; e < total; e += TAIL_STRIDE) {
                Real v = Real(0);
                if (has_c) {
                    const int c = e % C, cell = e / C, y = cell % ny, x = cell / ny;
                    int pc = c;
                    if (ac) {
                        const int n = c / g.ng, gg = c - n * g.ng;
                        const int per = g.na * g.na, f = n / per, rem = n - f * per;
                        const int row = rem / g.na, col = rem - row * g.na;
                        pc = (f * gc.na * gc.na + (row >> 1) * gc.na + (col >> 1)) * g.ng + gg;
                    }
                    v = __ldcg(cd + ((int64_t)(x >> 1) * gc.ny + (y >> 1)) * gc.C + pc);
                }
                L.delta[e] = v;
            }
            cluster_sync_all();
            continue;
        }
        for (int s = 0; s < t.n_sweeps; ++s) {
            // the last sweep writes delta: buffers alternate backwards from it
            Real* out = ((t.n_sweeps - 1 - s) & 1) ? t.scratch : L.delta;
            const Real* in = ((t.n_sweeps - 1 - s) & 1) ? L.delta : t.scratch;
            for (int e = tid; e < total; e += TAIL_STRIDE) {
                const int c = e % C, cell = e / C, y = cell % ny, x = cell / ny;
                const int n = c / g.ng, gg = c - n * g.ng;
                const Real mu = L.mu[n], nu = L.nu[n];
                const int xu_ = mu > Real(0) ? x - 1 : x + 1;
                const int yu_ = nu > Real(0) ? y - 1 : y + 1;
                const bool xin = xu_ >= 0 && xu_ < nx, yin = yu_ >= 0 && yu_ < ny;
                Real ce, xu, yu;
                if (s == 0) {
                    if (!has_c) {
                        ce = xu = yu = Real(0);
                    } else {
                        int pc = c;
                        if (ac) {
                            const int per = g.na * g.na, f = n / per, rem = n - f * per;
                            const int row = rem / g.na, col = rem - row * g.na;
                            pc = (f * gc.na * gc.na + (row >> 1) * gc.na + (col >> 1)) * g.ng + gg;
                        }
                        const Real* cp = cd + pc;
                        ce = __ldcg(cp + ((int64_t)(x >> 1) * gc.ny + (y >> 1)) * gc.C);
                        xu = xin ? __ldcg(cp + ((int64_t)(xu_ >> 1) * gc.ny + (y >> 1)) * gc.C)
                                 : Real(0);
                        yu = yin ? __ldcg(cp + ((int64_t)(x >> 1) * gc.ny + (yu_ >> 1)) * gc.C)
                                 : Real(0);
                    }
                } else {
                    ce = __ldcg(in + e);
                    xu = xin ? __ldcg(in + ((int64_t)xu_ * ny + y) * C + c) : Real(0);
                    yu = yin ? __ldcg(in + ((int64_t)x * ny + yu_) * C + c) : Real(0);
                }
                const Real amx = fabs(mu) * L.inv_dx, amy = fabs(nu) * L.inv_dy;
                const Real sg = L.sigma[(int64_t)cell * g.ng + gg];
                const Real d = Real(1) * (L.strm[n] + sg);
                const Real inv = up_div(Real(1), d);
                out[e] = tail_update(t.exact_div, ce, xu, yu, amx, amy, sg, __ldcg(L.src + e), inv, d);
            }
            cluster_sync_all();
        }
    }
}

}  // namespace csn
