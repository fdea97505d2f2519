// Launchers of the PG stencil kernels.  Declared here, defined (launchers.cuh) and
// explicitly instantiated per ConvFEM order in pg_part.cu, so the heavy kernel
// templates compile as parallel translation units.
#pragma once
#include <cuda_runtime.h>

#include "pg_kernels.cuh"

namespace csn {
struct PGTmaMaps;
struct KcoefMaps;
}

namespace csn {

template <class Real, int L, int MODE, int VEC>
void launch_pg_resid(dim3 grid, dim3 block, cudaStream_t st, const PGResidArgs<Real>& a);
template <int L, int MODE, int VEC>
void launch_pg_resid_x2(dim3 grid, dim3 block, cudaStream_t st, const PGResidArgs<float>& a);
template <int L, int MODE, int VEC, int NW>
void launch_pg_resid_xb(dim3 grid, dim3 block, cudaStream_t st, const PGResidArgs<float>& a);
template <int L, int MODE, int KD>
void launch_pg_resid_tma(dim3 grid, dim3 block, cudaStream_t st, const PGResidArgs<float>& a,
                         const PGTmaMaps& maps);
template <int L, bool EMA, int VEC>
void launch_pg_k_ws(dim3 grid, dim3 block, cudaStream_t st, const PGKArgs<float>& a);
template <int L>
void launch_pg_kcoef_tma(dim3 grid, dim3 block, cudaStream_t st, const PGKArgs<float>& a,
                         const KcoefMaps& maps, int gh);
template <int L, bool EMA, int VEC>
void launch_pg_k_x2(dim3 grid, dim3 block, cudaStream_t st, const PGKArgs<float>& a);
template <int L, bool EMA, int VEC>
void launch_pg_grad_x2(dim3 grid, dim3 block, cudaStream_t st, const PGKArgs<float>& a, float* gx,
                       float* gy, int gh);
template <int L, int VEC>
void launch_pg_kcoef_x2(dim3 grid, dim3 block, cudaStream_t st, const PGKArgs<float>& a,
                        const float* gx, const float* gy, int gh);
template <class Real, int L, bool EMA, int VEC>
void launch_pg_k(dim3 grid, dim3 block, cudaStream_t st, const PGKArgs<Real>& a);

}  // namespace csn
