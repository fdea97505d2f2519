/*
 * convsn_sm100.h — C ABI of the B200 (sm_100a) sawtooth space-angle multigrid kernels.
 *
 * Drop-in boundary for the reference's hot path (arXiv 2301.09991, package
 * `convsn`, /root/reference/pkg/src/convsn).  The reference has no FFI layer: its
 * boundary is the Python API in convsn/__init__.py:12-38 plus the internals used
 * by krylov.py:17-21.  Each entry point below names the reference function(s) it
 * replaces (R = /root/reference/pkg/src/convsn/).  The Python package
 * `paper_2301_09991_b200` binds these with ctypes and re-exposes the reference's
 * Python signatures.
 *
 * Conventions
 *  - dtype: CSN_F32 (float) or CSN_F64 (double).  Every `void*` field pointer is a
 *    DEVICE pointer of that type; `double*` arguments marked (device) are fp64
 *    device buffers; `const double* taps/cfg/stencil` are HOST arrays read during
 *    the call.
 *  - A field is stored like R/grid.py:47-59: `[nx + 2h][ny + 2h][nd][ng]`, C-order,
 *    x slowest, interior at [h, h+nx) x [h, h+ny).  `*_halo` gives h per pointer.
 *  - Kernels apply the vacuum rule of R/grid.py:165-190 ON LOAD (0 where the
 *    direction enters through the side, else the nearest interior value), so no
 *    halo has to be materialised between kernels.  A side flagged ghost in
 *    csn_geom (domain decomposition) is read from halo memory instead.
 *  - Return value: 0 ok; >0 invalid argument (CSN_E_*); <0 = -cudaError_t.
 *    No call allocates device memory; no call synchronises the stream.
 *  - `stream` is a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream).
 */
#ifndef CONVSN_SM100_H
#define CONVSN_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSN_F32 0
#define CSN_F64 1

#define CSN_OK 0
#define CSN_E_ARG 1        /* bad pointer / size / halo too small          */
#define CSN_E_ORDER 2      /* ConvFEM order not in {1, 2, 3, 5}            */
#define CSN_E_DTYPE 3      /* dtype not CSN_F32 / CSN_F64                   */
#define CSN_E_SCHEME 4     /* unsupported mode flag                        */

/* Geometry of one level (one rank's x-slab under domain decomposition). */
typedef struct csn_geom {
    int32_t nx, ny;        /* interior cells                               */
    int32_t nd, ng;        /* ordinates (8 n_a^2) and groups; C = nd * ng   */
    int32_t na;            /* patches per octahedron face side (n_a)       */
    int32_t ghost_w;       /* 1: west x-halo rows hold neighbour data      */
    int32_t ghost_e;       /* 1: east x-halo rows hold neighbour data      */
    int32_t pad_;
    double dx, dy;         /* cell widths (cm)                             */
} csn_geom;

int csn_version(void);
/* Kernels this library has launched since it was loaded (instrumentation). */
unsigned long long csn_launch_count(void);
const char* csn_error_string(int code);
/* Kernel-variant switches (no reference counterpart; used by the A/B parity tests):
 *   "upwind_x2"  = 1 (default): csn_upwind_smooth takes the packed channel-pair kernel
 *                  where it applies; 0 forces the scalar kernel (bit-identical results);
 *   "upwind_div" = 3 (default): fp32 smoother in Jacobi form, new = (1 - 1/s) ce +
 *                  b / (s d) with b = the upwind neighbour terms + source, the quotient
 *                  refined by one residual step (the rounded quotient); 4: the same
 *                  without refinement; 2: ce - r / (s d) with the refined quotient;
 *                  1: ce - r / (s d) by IEEE division; 0: one fused ce - r * rcp(s d)
 *                  (the face-uniform kernels implement 3 and 0, the other forms run in
 *                  the scalar kernel).  fp64 always uses the reference form ce - r / (s d).
 *   "sweep_div"  = 1 (default): the fp32 PG sweep refines r / (beta d) the same way;
 *                  0: reciprocal product;
 *   "pg_tma"     = 1 (default): fp32 csn_pg_residual stages padded fields with TMA
 *                  (mbarrier ring); 0 forces the cp.async kernel (bit-identical);
 *   "k2_tma"     = 1 (default): the fp32 diffusivity path's second pass (k from the
 *                  workspace) stages its rows with TMA except at order 2 (2: always; 0: the
 *                  cp.async stager; bit-identical);
 *   "k2_ws"      = 0 (default): 1 runs the workspace-path diffusivities as one
 *                  warp-specialised pass (psi_x, psi_y through shared memory;
 *                  bit-identical; measured slower on C4);
 *   "upwind_tma" = 1 (default): the packed smoother stages its columns with TMA where the
 *                  layout allows (one group, 8 <= n_a <= 32; ghost x sides included); 0: the
 *                  register kernel (bit-identical);
 *   "tail_faces" = 1 (default): csn_coarse_tail runs one CTA per (octahedron face, group),
 *                  each level's slice in shared memory (no inter-CTA synchronisation); 0: the
 *                  8-CTA cluster kernel (bit-identical);
 *   "tail_smem"  = 1 (default): csn_coarse_tail solves the levels of <= 2048 unknowns in one
 *                  CTA's shared memory; 0 keeps every level on the cluster (bit-identical);
 *   "pg_chunks"  = 0 (default): the y-chunk count of the PG marches comes from the cost
 *                  model; n > 0 forces n chunks (A/B timing; fields are bit-identical, the
 *                  fp64 L1 is summed in chunk order).
 * The previous value is stored in *prev (nullable). */
int csn_set_tuning(const char* key, int value, int* prev);

/* Doubles of workspace a reduction-producing call needs for its per-block partials. */
int64_t csn_partials_size(int dtype, const csn_geom* g, int order);

/* R/grid.py:165-190 apply_boundary: fill the h-wide halo (vacuum rule), in place.
 * mu, nu: device arrays [nd] of the field dtype. */
int csn_apply_boundary(int dtype, const csn_geom* g, void* f, int halo,
                       const void* mu, const void* nu, void* stream);

/* R/discretisation.py:65-94 upwind_residual (+ R/multigrid.py:292 resid_l1).
 * q: [nx][ny][1][ng] (q_per_dof = 0) or [nx][ny][nd][ng] (q_per_dof = 1).
 * r: output field (halo r_halo, only the interior is written).
 * l1: (device) fp64 sum |r| over the interior, or NULL; partials: workspace. */
int csn_upwind_residual(int dtype, const csn_geom* g, const void* psi, int psi_halo,
                        const void* sigma, const void* q, int q_per_dof,
                        const void* mu, const void* nu,
                        void* r, int r_halo, double* partials, double* l1, void* stream);

/* R/multigrid.py:149-173 jacobi_sweep(scheme="upwind") x n_sweeps, temporally
 * blocked, with the initial iterate taken from `init_mode`:
 *   0: zero;  1: the field `init` (halo init_halo);
 *   2: prolongation (R/multigrid.py:130-146) of the coarse interior `init`
 *      (geometry gc, halo init_halo).
 * src: the level source (q_per_dof as above).  diag_scale multiplies the
 * upwind Jacobi diagonal (R/discretisation.py:97-111).  0 <= n_sweeps <= 3 per call
 * (callers chain longer runs through two buffers).  Writes the interior of `out`,
 * which must not alias `init` unless n_sweeps == 0. */
int csn_upwind_smooth(int dtype, const csn_geom* g, const void* src, int q_per_dof,
                      int init_mode, const void* init, int init_halo, const csn_geom* gc,
                      const void* sigma, const void* mu, const void* nu, const void* strm,
                      int n_sweeps, double diag_scale, void* out, int out_halo,
                      void* stream);

/* The same smoother with its result folded into the iterate instead of stored:
 * psi[interior] -= delta (R/multigrid.py:335-338 on the finest level fused with
 * R/multigrid.py:301 `psi.data[interior] -= delta`), psi padded by psi_halo.  The
 * subtraction is an L2 reduction (fl(psi - delta); REDG.F32 flushes subnormals);
 * the caller re-applies the boundary to psi's halo afterwards.  psi must not alias
 * src or init. */
int csn_upwind_smooth_sub(int dtype, const csn_geom* g, const void* src, int q_per_dof,
                          int init_mode, const void* init, int init_halo, const csn_geom* gc,
                          const void* sigma, const void* mu, const void* nu, const void* strm,
                          int n_sweeps, double diag_scale, void* psi, int psi_halo,
                          void* stream);

/* R/multigrid.py:110-127,342-353 restrict / restrict_field_array and the
 * normalisation of R/multigrid.py:326 (normalise = 1). w_f, w_c: device
 * quadrature weights [nd] of fine / coarse level (field dtype). */
int csn_restrict(int dtype, const csn_geom* gf, const csn_geom* gc,
                 const void* fine, int fine_halo, const void* w_f, const void* w_c,
                 int normalise, void* coarse, int coarse_halo, void* stream);

/* R/multigrid.py:309-339 mg_correction on the coarse tail of the hierarchy, one launch:
 * n levels (finest first; level i + 1 is the spatial 2:1 / angular 1:1 or 2:1 coarsening
 * of level i, no ghost sides), each at most CSN_TAIL_MAX_DOF degrees of freedom.
 *   src[0] (given) is restricted and normalised down the chain into src[1..n-1]
 *   (R/multigrid.py:318-326); then from the coarsest level up each delta[i] is n_sweeps
 *   upwind Jacobi sweeps (diag_scale 1) on src[i] starting from the prolongation of
 *   delta[i + 1] (zero on the coarsest) (R/multigrid.py:330-338).
 * geoms: host array of n csn_geom; sigma/mu/nu/strm/w/src/delta: HOST arrays of n device
 * pointers (sigma [nx][ny][ng]; mu, nu, strm, w [nd]; src, delta unpadded [nx][ny][nd][ng]);
 * scratch: device buffer of >= the largest level's DOF (field dtype).
 * fp32 results are bit-identical to csn_restrict + csn_upwind_smooth level by level. */
#define CSN_TAIL_MAX_LEVELS 12
#define CSN_TAIL_MAX_DOF 32768
int csn_coarse_tail(int dtype, int n, const csn_geom* geoms, const void* const* sigma,
                    const void* const* mu, const void* const* nu, const void* const* strm,
                    const void* const* w, void* const* src, void* const* delta, void* scratch,
                    int n_sweeps, void* stream);

/* R/multigrid.py:130-146 prolong (piecewise-constant injection). */
int csn_prolong(int dtype, const csn_geom* gc, const csn_geom* gf,
                const void* coarse, int coarse_halo, void* fine, int fine_halo,
                void* stream);

/* Iterate averaging + diffusivities: R/multigrid.py:217-225 (PGState.averaged_iterate)
 * fused with R/discretisation.py:114-161 (_grad_fields, pg_anisotropic_diffusivities).
 *   avg_mode 0: k from psi (no averaging);  1: avg_out = psi (first call);
 *            2: avg_out = (1 - theta) avg_in + theta psi (EMA).  k from avg_out.
 * taps: host [3][2 order + 1] = mass, grad, stiff (unit spacing, R/filters.py:90-106).
 * cfg:  host [4] = epsilon_k, alpha_r, alpha_kabs, alpha_ksquare.
 * kx, ky: outputs valid on interior +- order (k_halo >= order). */
int csn_pg_diffusivities(int dtype, int order, const csn_geom* g, const double* taps,
                         const double* cfg, const void* psi, int psi_halo,
                         const void* avg_in, int avg_in_halo, void* avg_out,
                         int avg_out_halo, int avg_mode, double theta,
                         const void* mu, const void* nu, void* kx, void* ky, int k_halo,
                         void* work, void* stream);

/* Bytes of the optional csn_pg_diffusivities workspace (0: the dtype/order has no
 * split path).  With a workspace the fp32 kernel runs as two y-marches through
 * psi_x, psi_y on the +-2l band (bit-identical k); work = NULL keeps the fused one. */
int64_t csn_pg_workspace_size(int dtype, const csn_geom* g, int order);

/* R/discretisation.py:227-276 pg_residual (anisotropy "xy", given diffusivities),
 * two modes:
 *   residual (psi_out == NULL): r = pg_residual(psi) -> r (interior), l1 (device, nullable);
 *            optionally fused with the iterate average of frozen-diffusivity cycles
 *            (R/multigrid.py:217-225, in place on avg: avg_mode 1 copy, 2 EMA, 0 off);
 *   sweep    (psi_out != NULL): R/multigrid.py:301-304 fused — psi' = psi - delta
 *            (delta nullable), psi_out = psi' - pg_residual(psi') / (beta (|mu|/dx + |nu|/dy
 *            + sigma)) (R/multigrid.py:159-172).  psi_out must not alias psi.
 * strm: device [nd] = |mu|/dx + |nu|/dy.
 * Halos: like the reference (which evaluates psi.data with its stored halo), the caller
 * applies the boundary first (csn_apply_boundary; R/multigrid.py:166,277) and kx, ky are
 * zero outside their +-l band.  fp32 fields padded by >= l (delta too, in the sweep) are
 * staged with TMA as stored; otherwise the kernel re-derives the halo by the vacuum rule
 * — identical for consistent halos (tests/test_gpu_parity.py, tma_residual).
 * dterm (fp32, TMA path only; else CSN_E_SCHEME): unpadded [nx][ny][C] buffer of the k-only
 * coefficient D = -M_y(kx S_x / 2dx^2) - S_y(ky M_x / 2dy^2) of psi in r.  dterm_mode 1
 * (residual modes): compute and store it; 2: read it instead of recomputing — valid
 * while kx, ky are unchanged; results are bit-identical; 0: unused. */
int csn_pg_residual(int dtype, int order, const csn_geom* g, const double* taps,
                    const void* psi, int psi_halo, const void* delta, int delta_halo,
                    const void* kx, const void* ky, int k_halo,
                    const void* sigma, const void* q, int q_per_dof,
                    const void* mu, const void* nu, const void* strm,
                    void* r, int r_halo, void* psi_out, int psi_out_halo, double beta,
                    double* partials, double* l1, void* avg, int avg_halo, int avg_mode,
                    double theta, void* dterm, int dterm_mode, void* stream);

/* R/grid.py:193-198 scalar_flux: phi (device fp64 [nx][ny][ng]) = sum_n w_n psi. */
int csn_scalar_flux(int dtype, const csn_geom* g, const void* psi, int halo,
                    const void* w, double* phi, void* stream);

/* R/eigen.py:117-130 assemble_group_source (+ the frozen fission term of
 * R/eigen.py:232-233,500-501): q[g] = sum_{a} ss[a->g] phi_a - ss[g->g] phi_g + s_g
 * (+ fission[g] if non-NULL) (+ lam chi_g sum nsf phi if lam != 0).
 * All inputs fp64 device, per cell: sigma_s [nx][ny][ng][ng], s/chi/nsf/fission
 * [nx][ny][ng].  q: field dtype [nx][ny][1][ng]. */
int csn_group_source(int dtype, const csn_geom* g, const double* phi, const double* sigma_s,
                     const double* source, const double* fission, double lam,
                     const double* chi, const double* nsf, void* q, void* stream);

/* R/eigen.py:232-233 frozen fission source: F[g] = (inv_k chi_g) sum_g' nsf_g' phi_g'. */
int csn_fission_source(const csn_geom* g, const double* phi, const double* chi,
                       const double* nsf, double inv_k, double* out, void* stream);

/* R/eigen.py:133-135 fission_production: out (device fp64) = dx dy sum nsf phi. */
int csn_production(const csn_geom* g, const double* phi, const double* nsf,
                   double* partials, double* out, void* stream);

/* Deterministic fp64 sum of n device doubles into *out (fixed reduction tree). */
int csn_sum_f64(const double* x, int64_t n, double* out, void* stream);

/* x[i] /= s (divide = 1) or x[i] *= s, i < n, field dtype. (R/eigen.py:212-219,243-247) */
int csn_scale(int dtype, void* x, int64_t n, double s, int divide, void* stream);

/* psi interior -= delta interior (R/multigrid.py:301). */
int csn_sub_interior(int dtype, const csn_geom* g, void* psi, int psi_halo,
                     const void* delta, int delta_halo, void* stream);

/* R/multigrid.py:217-225 averaged_iterate, elementwise over the interior (the halo
 * follows from the vacuum rule): mode 1: avg = psi;  mode 2: avg = (1 - theta) avg
 * + theta psi, in place (used on frozen cycles, where no diffusivity refresh runs). */
int csn_ema(int dtype, const csn_geom* g, void* avg, int avg_halo, const void* psi,
            int psi_halo, double theta, int mode, void* stream);

/* Non-default PG modes (R/discretisation.py:164-224), elementwise over n elements of
 * same-layout arrays with C channels per cell, ng groups (ordinate = (e % C) / ng):
 *   csn_dir_lincomb:     out = scale (ca A[n] x + cb B[n] y)   (A, B, y nullable);
 *   csn_iso_diffusivity: isotropic k from the residual estimate r and psi_x, psi_y,
 *                        cfg = {epsilon_k, alpha_kabs, alpha_ksquare, (dx+dy)/2, dx, dy}. */
int csn_dir_lincomb(int dtype, int64_t n, int C, int ng, const void* x, const void* A, double ca,
                    const void* y, const void* B, double cb, double scale, void* out,
                    void* stream);
int csn_iso_diffusivity(int dtype, int64_t n, int C, int ng, const void* r, const void* px,
                        const void* py, const void* mu, const void* nu, const double* cfg,
                        void* k, void* stream);

/* R/grid.py:85-105,139-152 convolve: square (2l+1)^2 stencil, host `stencil`
 * [width][width] (fp64), on interior +- margin, reading halo memory as stored;
 * dir_scale: device [nd] or NULL.  Writes the whole padded `out` (0 outside). */
int csn_convolve(int dtype, const csn_geom* g, const void* src, int halo,
                 const double* stencil, int width, int margin, const void* dir_scale,
                 void* out, void* stream);

/* R/grid.py:108-125 _stencil_apply_1d: one 1D pass along axis (0 = x, 1 = y),
 * host taps [width], full extent on the other axis; writes the whole padded out. */
int csn_pass1d(int dtype, const csn_geom* g, const void* src, int halo, const double* taps,
               int width, int axis, int margin, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CONVSN_SM100_H */
