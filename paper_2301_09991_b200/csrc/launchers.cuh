// Definitions of the PG kernel launchers (launchers.h); included by pg_part.cu only.
#pragma once
#include "launchers.h"
#include "pg_kernels_x2.cuh"
#include "pg_kernels_tma.cuh"
#include "pg_kernels_xb.cuh"

namespace csn {

template <class K>
void set_smem(K kernel, size_t bytes) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <class Real, int L, int MODE, int VEC>
void launch_pg_resid(dim3 grid, dim3 block, cudaStream_t st, const PGResidArgs<Real>& a) {
    constexpr size_t sm = pg_residual_smem<Real, L, MODE>();
    static bool attr = false;
    if (!attr) { set_smem(pg_residual_kernel<Real, L, MODE, VEC>, sm); attr = true; }
    pg_residual_kernel<Real, L, MODE, VEC><<<grid, block, sm, st>>>(a);
}

template <int L, int MODE, int VEC>
void launch_pg_resid_x2(dim3 grid, dim3 block, cudaStream_t st, const PGResidArgs<float>& a) {
    constexpr size_t sm = pg_residual_x2_smem<L, MODE>();
    static bool attr = false;
    if (!attr) { set_smem(pg_residual_x2_kernel<L, MODE, VEC>, sm); attr = true; }
    pg_residual_x2_kernel<L, MODE, VEC><<<grid, block, sm, st>>>(a);
}

template <int L, int MODE, int VEC, int NW>
void launch_pg_resid_xb(dim3 grid, dim3 block, cudaStream_t st, const PGResidArgs<float>& a) {
    constexpr size_t sm = pg_residual_xb_smem<L, MODE, NW>();
    static bool attr = false;
    if (!attr) { set_smem(pg_residual_xb_kernel<L, MODE, VEC, NW>, sm); attr = true; }
    pg_residual_xb_kernel<L, MODE, VEC, NW><<<grid, block, sm, st>>>(a);
}

template <int L, int MODE, int KD>
void launch_pg_resid_tma(dim3 grid, dim3 block, cudaStream_t st, const PGResidArgs<float>& a,
                         const PGTmaMaps& maps) {
    constexpr size_t sm = pg_residual_tma_smem<L, MODE>();
    if (KD == 0 && a.g.ng == 1 && !a.q_per_dof) {       // 1 group, per-cell source
        static bool attr1 = false;
        if (!attr1) { set_smem(pg_residual_tma_kernel<L, MODE, KD, 1>, sm); attr1 = true; }
        pg_residual_tma_kernel<L, MODE, KD, 1><<<grid, block, sm, st>>>(a, maps);
        return;
    }
    if (KD == 0 && a.g.ng == 2 && !a.q_per_dof) {       // 2 groups, per-cell source
        static bool attr2 = false;
        if (!attr2) { set_smem(pg_residual_tma_kernel<L, MODE, KD, 2>, sm); attr2 = true; }
        pg_residual_tma_kernel<L, MODE, KD, 2><<<grid, block, sm, st>>>(a, maps);
        return;
    }
    static bool attr = false;
    if (!attr) { set_smem(pg_residual_tma_kernel<L, MODE, KD>, sm); attr = true; }
    pg_residual_tma_kernel<L, MODE, KD><<<grid, block, sm, st>>>(a, maps);
}

template <int L, bool EMA, int VEC>
void launch_pg_k_ws(dim3 grid, dim3 block, cudaStream_t st, const PGKArgs<float>& a) {
    constexpr size_t sm = pg_k_ws_smem<L, EMA>();
    static bool attr = false;
    if (!attr) { set_smem(pg_k_ws_kernel<L, EMA, VEC>, sm); attr = true; }
    pg_k_ws_kernel<L, EMA, VEC><<<grid, block, sm, st>>>(a);
}

template <int L>
void launch_pg_kcoef_tma(dim3 grid, dim3 block, cudaStream_t st, const PGKArgs<float>& a,
                         const KcoefMaps& maps, int gh) {
    constexpr size_t sm = pg_kcoef_tma_smem<L>();
    static bool attr = false;
    if (!attr) { set_smem(pg_kcoef_tma_kernel<L>, sm); attr = true; }
    pg_kcoef_tma_kernel<L><<<grid, block, sm, st>>>(a, maps, gh);
}

template <int L, bool EMA, int VEC>
void launch_pg_k_x2(dim3 grid, dim3 block, cudaStream_t st, const PGKArgs<float>& a) {
    constexpr size_t sm = pg_k_x2_smem<L, EMA>();
    static bool attr = false;
    if (!attr) { set_smem(pg_diffusivity_x2_kernel<L, EMA, VEC>, sm); attr = true; }
    pg_diffusivity_x2_kernel<L, EMA, VEC><<<grid, block, sm, st>>>(a);
}

template <int L, bool EMA, int VEC>
void launch_pg_grad_x2(dim3 grid, dim3 block, cudaStream_t st, const PGKArgs<float>& a, float* gx,
                       float* gy, int gh) {
    constexpr size_t sm = pg_grad_x2_smem<L, EMA>();
    static bool attr = false;
    if (!attr) { set_smem(pg_grad_x2_kernel<L, EMA, VEC>, sm); attr = true; }
    pg_grad_x2_kernel<L, EMA, VEC><<<grid, block, sm, st>>>(a, gx, gy, gh);
}

template <int L, int VEC>
void launch_pg_kcoef_x2(dim3 grid, dim3 block, cudaStream_t st, const PGKArgs<float>& a,
                        const float* gx, const float* gy, int gh) {
    constexpr size_t sm = pg_kcoef_x2_smem<L>();
    static bool attr = false;
    if (!attr) { set_smem(pg_kcoef_x2_kernel<L, VEC>, sm); attr = true; }
    pg_kcoef_x2_kernel<L, VEC><<<grid, block, sm, st>>>(a, gx, gy, gh);
}

template <class Real, int L, bool EMA, int VEC>
void launch_pg_k(dim3 grid, dim3 block, cudaStream_t st, const PGKArgs<Real>& a) {
    constexpr size_t sm = pg_k_smem<Real, L, EMA>();
    static bool attr = false;
    if (!attr) { set_smem(pg_diffusivity_kernel<Real, L, EMA, VEC>, sm); attr = true; }
    pg_diffusivity_kernel<Real, L, EMA, VEC><<<grid, block, sm, st>>>(a);
}

}  // namespace csn
