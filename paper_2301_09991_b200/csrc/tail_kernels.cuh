// Coarse tail of the correction in ONE launch (R/multigrid.py:309-339 on the levels that
// hold at most a few DOF per thread of one cluster): the restriction chain down from the
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

// Exact quotient by a precomputed multiplier: for 0 <= v and v * d < 2^32 (here v, d <=
// 32768), floor(v / d) = umulhi(v, floor(2^32 / d) + 1).  An index decomposition by
// hardware-emulated division was 60% of the tail kernel's instructions.
struct FastDiv {
    unsigned m;      // 0: divisor 1
    __device__ __forceinline__ int operator()(int v) const {
        return m ? (int)__umulhi((unsigned)v, m) : v;
    }
};
inline FastDiv make_fastdiv(int d) {
    FastDiv f;
    f.m = d <= 1 ? 0u : (unsigned)((1ull << 32) / (unsigned)d) + 1u;
    return f;
}
struct FastDivs {
    FastDiv C, ny, ng, per, na;
    __device__ __forceinline__ int by_ng(int v) const { return ng(v); }
    __device__ __forceinline__ int by_per(int v) const { return per(v); }
    __device__ __forceinline__ int by_na(int v) const { return na(v); }
    __device__ __forceinline__ int by_ny(int v) const { return ny(v); }
};

template <class Real>
struct TailLevel {
    Geo g;
    FastDivs dv;         // by C, ny, ng, n_a^2, n_a of this level
    const Real* sigma;   // [nx][ny][ng]
    const Real* mu; const Real* nu; const Real* strm; const Real* w;   // [nd]
    Real* src;           // [nx][ny][C]: given on level 0 of the tail, restricted below
    Real* delta;         // [nx][ny][C]: the level's smoothed correction (output)
    Real inv_dx, inv_dy, area;
    int sig_stride;      // sigma of a cell: sigma[cell * sig_stride + group] (= ng)
    FastDivs fdv;        // face-local decomposition: by n_a^2 (as C), ny, 1, n_a^2, n_a
    int face_off;        // element offset of this level in the face kernel's shared arrays
    int const_off;       // ... of its [mu | nu | strm | w | sigma] block in the constants area
};

template <class Real>
struct TailArgs {
    int n;                                   // tail levels, finest first
    TailLevel<Real> lv[TAIL_MAX_LEVELS];
    Real* scratch;                           // >= the largest tail level's DOF
    int n_sweeps;
    int exact_div;                           // fp32 update form (csn_set_tuning "upwind_div")
    int n_smem_first;                        // first level held in CTA 0's shared memory (n: none)
    int smem_off[TAIL_MAX_LEVELS];           // element offset of a shared level in s_src / s_del
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

// loads of data produced inside the launch: L2 (ld.global.cg) for the levels shared by the
// cluster's CTAs, plain (generic) loads for the levels CTA 0 keeps in shared memory
template <bool CG, class Real>
__device__ __forceinline__ Real tail_ld(const Real* p) { return CG ? __ldcg(p) : *p; }

// parent channel of fine channel c on the next coarser level (R/multigrid.py:130-146)
__device__ __forceinline__ int tail_parent(const Geo& g, const FastDivs& dv, const Geo& gc,
                                           bool ac, int c) {
    if (!ac) return c;
    const int n = dv.ng(c), gg = c - n * g.ng;
    const int per = g.na * g.na, f = dv.per(n), rem = n - f * per;
    const int row = dv.na(rem), col = rem - row * g.na;
    return (f * gc.na * gc.na + (row >> 1) * gc.na + (col >> 1)) * g.ng + gg;
}

// Element range [first, total) with stride `stride` of level L: restriction of the finer
// source `fine` (level Lf) into `src`
template <class Real>
__device__ __forceinline__ void tail_restrict(const TailLevel<Real>& Lf, const TailLevel<Real>& Lc,
                                              const Real* fine, Real* coarse, int first, int stride) {
    RestrictArgs<Real> a;
    a.gf = Lf.g; a.gc = Lc.g;
    a.fine = fine; a.fine_h = 0;
    a.wf = Lf.w; a.wc = Lc.w;
    a.af = Lf.area; a.ac = Lc.area;
    a.angle_coarsens = Lc.g.na != Lf.g.na;
    a.normalise = 1;
    a.coarse = coarse; a.coarse_h = 0;
    const int C = Lc.g.C, total = C * Lc.g.nx * Lc.g.ny;
    for (int e = first; e < total; e += stride) {
        const int cell = Lc.dv.C(e);
        restrict_cells(a, e - cell * C, cell, 1 << 30, Lc.dv);
    }
}

// One Jacobi sweep of level L over the element range: sweep 0 starts from the prolongation
// of the coarser correction cd (zero when there is none), later sweeps from `in`
template <bool CG, class Real>
__device__ __forceinline__ void tail_sweep(const TailLevel<Real>& L, const Geo& gc, bool has_c,
                                           const Real* __restrict__ cd,
                                           const Real* __restrict__ src,
                                           const Real* __restrict__ in, Real* __restrict__ out,
                                           bool first_sweep, int form, int first, int stride) {
    const Geo& g = L.g;
    const int C = g.C, ny = g.ny, nx = g.nx, total = C * nx * ny;
    const bool ac = has_c && gc.na != g.na;
    // the iterations are independent (in, out, src, cd never alias): unrolled so the loads
    // of four elements are in flight together
#pragma unroll 4
    for (int e = first; e < total; e += stride) {
        const int cell = L.dv.C(e), c = e - cell * C;
        const int x = L.dv.ny(cell), y = cell - x * ny;
        const int n = L.dv.ng(c), gg = c - n * g.ng;
        const Real mu = L.mu[n], nu = L.nu[n];
        const int xu_ = mu > Real(0) ? x - 1 : x + 1;
        const int yu_ = nu > Real(0) ? y - 1 : y + 1;
        const bool xin = xu_ >= 0 && xu_ < nx, yin = yu_ >= 0 && yu_ < ny;
        Real ce, xu, yu;
        if (first_sweep) {
            if (!has_c) {
                ce = xu = yu = Real(0);
            } else {
                const Real* cp = cd + tail_parent(g, L.dv, gc, ac, c);
                ce = tail_ld<CG>(cp + ((int64_t)(x >> 1) * gc.ny + (y >> 1)) * gc.C);
                xu = xin ? tail_ld<CG>(cp + ((int64_t)(xu_ >> 1) * gc.ny + (y >> 1)) * gc.C) : Real(0);
                yu = yin ? tail_ld<CG>(cp + ((int64_t)(x >> 1) * gc.ny + (yu_ >> 1)) * gc.C) : Real(0);
            }
        } else {
            ce = tail_ld<CG>(in + e);
            xu = xin ? tail_ld<CG>(in + ((int64_t)xu_ * ny + y) * C + c) : Real(0);
            yu = yin ? tail_ld<CG>(in + ((int64_t)x * ny + yu_) * C + c) : Real(0);
        }
        const Real amx = fabs(mu) * L.inv_dx, amy = fabs(nu) * L.inv_dy;
        const Real sg = L.sigma[(int64_t)cell * L.sig_stride + gg];
        const Real d = Real(1) * (L.strm[n] + sg);
        const Real inv = up_div(Real(1), d);
        out[e] = tail_update(form, ce, xu, yu, amx, amy, sg, tail_ld<CG>(src + e), inv, d);
    }
}

// n_sweeps == 0: the level's correction is the prolonged coarser one (or zero)
template <bool CG, class Real>
__device__ __forceinline__ void tail_inject(const TailLevel<Real>& L, const Geo& gc, bool has_c,
                                            const Real* cd, Real* out, int first, int stride) {
    const Geo& g = L.g;
    const int C = g.C, ny = g.ny, total = C * g.nx * ny;
    const bool ac = has_c && gc.na != g.na;
    for (int e = first; e < total; e += stride) {
        Real v = Real(0);
        if (has_c) {
            const int cell = L.dv.C(e), c = e - cell * C;
            const int x = L.dv.ny(cell), y = cell - x * ny;
            v = tail_ld<CG>(cd + ((int64_t)(x >> 1) * gc.ny + (y >> 1)) * gc.C +
                            tail_parent(g, L.dv, gc, ac, c));
        }
        out[e] = v;
    }
}

// Levels of <= TAIL_SMEM_DOF unknowns live in CTA 0's shared memory (their sources, their
// corrections and one ping-pong buffer): a stage there is a loop and a __syncthreads()
// with ~30-cycle loads instead of a cluster barrier and L2 round trips, which is what the
// five or six smallest levels cost (20 stages of ~1.5 us -> ~3 us in all).
constexpr int TAIL_SMEM_DOF = 2048;
constexpr int TAIL_SMEM_SUM = 2048 + 1024;      // >= sum of the shared levels' DOF (each <= 1/2 the finer)

template <class Real>
constexpr size_t coarse_tail_smem() { return (size_t)(2 * TAIL_SMEM_SUM + TAIL_SMEM_DOF) * sizeof(Real); }

template <class Real>
__global__ void __launch_bounds__(TAIL_THREADS, 1) coarse_tail_kernel(const TailArgs<Real> t) {
    extern __shared__ __align__(16) unsigned char tail_smraw[];
    Real* s_src = reinterpret_cast<Real*>(tail_smraw);          // shared levels' sources
    Real* s_del = s_src + TAIL_SMEM_SUM;                         // ... corrections
    Real* s_tmp = s_del + TAIL_SMEM_SUM;                         // ... ping-pong buffer
    const int tid = blockIdx.x * TAIL_THREADS + threadIdx.x;     // grid = one cluster
    // ns: first level kept in shared memory (t.n when none); levels [0, ns) are the cluster's
    const int ns = t.n_smem_first;
    // ---- restriction chain on the cluster's levels: src[i] from src[i - 1]
    for (int i = 1; i < ns; ++i) {
        tail_restrict(t.lv[i - 1], t.lv[i], t.lv[i - 1].src, t.lv[i].src, tid, TAIL_STRIDE);
        cluster_sync_all();
    }
    // ---- the shared-memory levels, CTA 0 alone: restriction down, smoothing up
    if (ns < t.n && blockIdx.x == 0) {
        const int ltid = threadIdx.x;
        int off = 0;
        for (int i = ns; i < t.n; ++i) {
            const Real* fine = i == ns ? t.lv[i - 1].src : s_src + t.smem_off[i - 1];
            tail_restrict(t.lv[i - 1], t.lv[i], fine, s_src + off, ltid, TAIL_THREADS);
            off += t.lv[i].g.C * t.lv[i].g.nx * t.lv[i].g.ny;
            __syncthreads();
        }
        for (int i = t.n - 1; i >= ns; --i) {
            const TailLevel<Real>& L = t.lv[i];
            const bool has_c = i + 1 < t.n;
            const Geo gc = has_c ? t.lv[i + 1].g : L.g;
            const Real* cd = has_c ? s_del + t.smem_off[i + 1] : nullptr;
            Real* del = s_del + t.smem_off[i];
            const Real* src = s_src + t.smem_off[i];
            if (t.n_sweeps == 0) {
                tail_inject<false>(L, gc, has_c, cd, del, ltid, TAIL_THREADS);
                __syncthreads();
            }
            for (int s = 0; s < t.n_sweeps; ++s) {
                const bool odd = (t.n_sweeps - 1 - s) & 1;
                tail_sweep<false>(L, gc, has_c, cd, src, odd ? del : s_tmp, odd ? s_tmp : del,
                                  s == 0, t.exact_div, ltid, TAIL_THREADS);
                __syncthreads();
            }
            // the ABI's outputs: this level's source and correction, to global memory
            const int total = L.g.C * L.g.nx * L.g.ny;
            for (int e = ltid; e < total; e += TAIL_THREADS) {
                L.src[e] = src[e];
                L.delta[e] = del[e];
            }
        }
    }
    if (ns < t.n && ns > 0) cluster_sync_all();     // delta[ns] is visible to the cluster
    // ---- smoothing of the cluster's levels, coarsest up; sweep s reads `in` (the prolonged
    //      coarser correction, or zero, for s = 0) and writes the buffer whose last turn is delta
    for (int i = ns - 1; i >= 0; --i) {
        const TailLevel<Real>& L = t.lv[i];
        const bool has_c = i + 1 < t.n;
        const Geo gc = has_c ? t.lv[i + 1].g : L.g;
        const Real* cd = has_c ? t.lv[i + 1].delta : nullptr;
        if (t.n_sweeps == 0) {
            tail_inject<true>(L, gc, has_c, cd, L.delta, tid, TAIL_STRIDE);
            cluster_sync_all();
            continue;
        }
        for (int s = 0; s < t.n_sweeps; ++s) {
            // the last sweep writes delta: buffers alternate backwards from it
            const bool odd = (t.n_sweeps - 1 - s) & 1;
            tail_sweep<true>(L, gc, has_c, cd, L.src, odd ? L.delta : t.scratch,
                             odd ? t.scratch : L.delta, s == 0, t.exact_div, tid, TAIL_STRIDE);
            cluster_sync_all();
        }
    }
}

// ---------------------------------------------------------------------------------
// The same tail, one CTA per (octahedron face, group), no inter-CTA synchronisation.
// Every operator of the correction keeps a face's directions and a group to themselves:
// the smoother couples only spatial neighbours of one channel, restriction sums the 2 x 2
// patch children of one face (R/multigrid.py:342-353), prolongation injects a parent into
// its children (R/multigrid.py:130-146).  So the tail splits into n_faces x n_group
// independent problems of <= TAIL_FACE_DOF unknowns per level, each solved by one CTA
// entirely in shared memory (a stage = a loop + __syncthreads()): the level-0 source
// slice is gathered from global memory once, the results scattered back at the end.
// Local layout of a level: [cell][patch r of the face] (a field with nd = n_a^2, ng = 1),
// which restrict_cells / tail_sweep take as is with the face's slice of w, mu, nu, strm
// and the group's sigma — the same rounded operations, bit-identical results.
// Launch 55 us (level by level) -> 35 us (cluster) -> ~15 us.
// ---------------------------------------------------------------------------------
constexpr int TAIL_FACE_DOF = 4096;                      // per CTA and level (32768 per 8 faces)
constexpr int TAIL_FACE_SUM = TAIL_FACE_DOF + TAIL_FACE_DOF / 4 + TAIL_FACE_DOF / 8;

constexpr int TAIL_FACE_CONST = 2048;                    // per-level mu, nu, strm, w, sigma slices

template <class Real>
constexpr size_t coarse_tail_face_smem() {
    return (size_t)(2 * TAIL_FACE_SUM + TAIL_FACE_DOF + TAIL_FACE_CONST) * sizeof(Real);
}

template <class Real>
__global__ void __launch_bounds__(TAIL_THREADS, 1) coarse_tail_face_kernel(const TailArgs<Real> t) {
    extern __shared__ __align__(16) unsigned char tail_smraw[];
    Real* s_src = reinterpret_cast<Real*>(tail_smraw);
    Real* s_del = s_src + TAIL_FACE_SUM;
    Real* s_tmp = s_del + TAIL_FACE_SUM;
    Real* s_c = s_tmp + TAIL_FACE_DOF;       // every level's constants, loaded once up front
    const int ng = t.lv[0].g.ng;
    const int face = blockIdx.x / ng, gq = blockIdx.x - face * ng;
    const int tid = threadIdx.x;

    // the face's mu, nu, strm, w and the group's sigma of every level into shared memory,
    // in flight together with the source gather below (a stage otherwise starts with an
    // L2 round trip for its level's constants)
    {
        const TailLevel<Real>& Gl = t.lv[t.n - 1];
        const int total_c = Gl.const_off + 4 * Gl.g.na * Gl.g.na + Gl.g.nx * Gl.g.ny;
        for (int ee = tid; ee < total_c; ee += TAIL_THREADS) {   // one flat loop: <= 2 per thread
            int i = 0;
            while (i + 1 < t.n && t.lv[i + 1].const_off <= ee) ++i;
            const TailLevel<Real>& G = t.lv[i];
            const int per = G.g.na * G.g.na, e = ee - G.const_off;
            const int k = e < 4 * per ? G.fdv.C(e) : 4, r = e - k * per;
            s_c[ee] = k == 0 ? G.mu[face * per + r] : k == 1 ? G.nu[face * per + r]
                    : k == 2 ? G.strm[face * per + r] : k == 3 ? G.w[face * per + r]
                             : G.sigma[(int64_t)r * ng + gq];
        }
    }

    // face-local view of level i: geometry of one face and one group, constants in smem
    auto view = [&](int i) {
        TailLevel<Real> V = t.lv[i];
        const int per = V.g.na * V.g.na;
        V.g.nd = per; V.g.ng = 1; V.g.C = per;
        V.dv = V.fdv;
        const Real* c = s_c + V.const_off;
        V.mu = c; V.nu = c + per; V.strm = c + 2 * per; V.w = c + 3 * per;
        V.sigma = c + 4 * per;
        V.sig_stride = 1;
        return V;
    };
    // global element of local (cell, r) on level i
    auto gidx = [&](const TailLevel<Real>& G, int cell, int r) {
        const int per = G.g.na * G.g.na;
        return (int64_t)cell * G.g.C + (face * per + r) * ng + gq;
    };

    {   // the CTA's slice of the given source
        const TailLevel<Real>& G = t.lv[0];
        const int per = G.g.na * G.g.na, total = G.g.nx * G.g.ny * per;
        for (int e = tid; e < total; e += TAIL_THREADS) {
            const int cell = G.fdv.C(e);
            s_src[e] = G.src[gidx(G, cell, e - cell * per)];
        }
        __syncthreads();
    }
    for (int i = 1; i < t.n; ++i) {          // restriction chain
        const TailLevel<Real> Vf = view(i - 1), Vc = view(i);
        tail_restrict(Vf, Vc, s_src + Vf.face_off, s_src + Vc.face_off, tid, TAIL_THREADS);
        __syncthreads();
    }
    for (int i = t.n - 1; i >= 0; --i) {     // smoothing, coarsest level up
        const TailLevel<Real> V = view(i);
        const bool has_c = i + 1 < t.n;
        Geo gc = V.g;
        if (has_c) {
            gc = t.lv[i + 1].g;
            gc.nd = gc.na * gc.na; gc.ng = 1; gc.C = gc.nd;
        }
        const Real* cd = has_c ? s_del + t.lv[i + 1].face_off : nullptr;
        Real* del = s_del + V.face_off;
        const Real* src = s_src + V.face_off;
        if (t.n_sweeps == 0) {
            tail_inject<false>(V, gc, has_c, cd, del, tid, TAIL_THREADS);
            __syncthreads();
        }
        for (int s = 0; s < t.n_sweeps; ++s) {
            const bool odd = (t.n_sweeps - 1 - s) & 1;
            tail_sweep<false>(V, gc, has_c, cd, src, odd ? del : s_tmp, odd ? s_tmp : del, s == 0,
                              t.exact_div, tid, TAIL_THREADS);
            __syncthreads();
        }
    }
    for (int i = 0; i < t.n; ++i) {          // the ABI's outputs, back in the global layout
        const TailLevel<Real>& G = t.lv[i];
        const int per = G.g.na * G.g.na, total = G.g.nx * G.g.ny * per;
        for (int e = tid; e < total; e += TAIL_THREADS) {
            const int cell = G.fdv.C(e);
            const int64_t ge = gidx(G, cell, e - cell * per);
            if (i > 0) G.src[ge] = s_src[G.face_off + e];
            G.delta[ge] = s_del[G.face_off + e];
        }
    }
}

}  // namespace csn
