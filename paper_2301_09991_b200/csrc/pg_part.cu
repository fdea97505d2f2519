// One explicit-instantiation unit of the PG kernel launchers: ConvFEM half-width
// CSN_L (1, 2, 3, 5) and element type CSN_PART_F64 (0: the packed fp32x2 kernels, 1: fp64).
// The Makefile compiles this file once per (L, type) so the PG kernels build in
// parallel; convsn_abi.cu sees only the declarations (launchers.h).
#include "launchers.cuh"

#ifndef CSN_L
#error "CSN_L must be defined"
#endif

namespace csn {

#define CSN_ARGS_R(R) dim3, dim3, cudaStream_t, const PGResidArgs<R>&
#define CSN_ARGS_K(R) dim3, dim3, cudaStream_t, const PGKArgs<R>&

#if CSN_PART_F64
#define CSN_RES64(M, V) template void launch_pg_resid<double, CSN_L, M, V>(CSN_ARGS_R(double));
CSN_RES64(0, 1) CSN_RES64(0, 2) CSN_RES64(1, 1) CSN_RES64(1, 2) CSN_RES64(2, 1) CSN_RES64(2, 2)
#define CSN_K64(E, V) template void launch_pg_k<double, CSN_L, E, V>(CSN_ARGS_K(double));
CSN_K64(false, 1) CSN_K64(false, 2) CSN_K64(true, 1) CSN_K64(true, 2)
#else
#define CSN_RES32(M, V) template void launch_pg_resid_x2<CSN_L, M, V>(CSN_ARGS_R(float));
CSN_RES32(0, 1) CSN_RES32(0, 4) CSN_RES32(1, 1) CSN_RES32(1, 4) CSN_RES32(2, 1) CSN_RES32(2, 4)
#define CSN_TMA(M, KD) \
    template void launch_pg_resid_tma<CSN_L, M, KD>(CSN_ARGS_R(float), const PGTmaMaps&);
CSN_TMA(0, 0) CSN_TMA(0, 1) CSN_TMA(0, 2) CSN_TMA(1, 0) CSN_TMA(1, 1) CSN_TMA(1, 2) CSN_TMA(2, 0) CSN_TMA(2, 2)
CSN_TMA(3, 0) CSN_TMA(3, 2)
#if CSN_L <= 3
#define CSN_XB(M, NW) template void launch_pg_resid_xb<CSN_L, M, 4, NW>(CSN_ARGS_R(float));
CSN_XB(0, 4) CSN_XB(1, 4) CSN_XB(2, 4) CSN_XB(0, 8) CSN_XB(1, 8) CSN_XB(2, 8)
#define CSN_K32(E, V)                                                                  \
    template void launch_pg_k_x2<CSN_L, E, V>(CSN_ARGS_K(float));                     \
    template void launch_pg_grad_x2<CSN_L, E, V>(CSN_ARGS_K(float), float*, float*, int);
CSN_K32(false, 1) CSN_K32(false, 4) CSN_K32(true, 1) CSN_K32(true, 4)
template void launch_pg_kcoef_x2<CSN_L, 1>(CSN_ARGS_K(float), const float*, const float*, int);
template void launch_pg_kcoef_x2<CSN_L, 4>(CSN_ARGS_K(float), const float*, const float*, int);
template void launch_pg_kcoef_tma<CSN_L>(CSN_ARGS_K(float), const KcoefMaps&, int);
#define CSN_WS(E, V) template void launch_pg_k_ws<CSN_L, E, V>(CSN_ARGS_K(float));
CSN_WS(false, 1) CSN_WS(false, 4) CSN_WS(true, 1) CSN_WS(true, 4)
#else
#define CSN_K32S(E, V) template void launch_pg_k<float, CSN_L, E, V>(CSN_ARGS_K(float));
CSN_K32S(false, 1) CSN_K32S(false, 4) CSN_K32S(true, 1) CSN_K32S(true, 4)
#endif
#endif

}  // namespace csn
