"""Dense-matrix verification of the GPU path (R/verification.py:1-105, R/oracle.py:38-143).

Same three checks as the reference's ``oracle compare`` on a homogeneous fissile
block (6x6, dx = 0.5, vacuum): the GPU upwind residual vs A psi - q, one GPU Jacobi
step vs the dense step, and the GPU power iteration's k_eff vs a dense power
iteration of A - S against F.  Dense operators are assembled on the host (vectorised
over the unknowns, flat index ((i ny + j) nd + n) ng + g).
"""

from dataclasses import dataclass

import numpy as np
import torch

from .discretisation import upwind_residual
from .eigen import SolverOptions, power_iteration
from .filters import build_upwind_filters
from .grid import Field, GridSpec, apply_boundary
from .materials import CrossSections
from .multigrid import build_hierarchy, jacobi_sweep
from .problems import ProblemSpec
from .quadrature import build_quadrature


@dataclass
class OracleReport:
    rows: list   # (name, err, tol, ok)

    @property
    def passed(self):
        return all(ok for *_, ok in self.rows)


def _two_group_fuel():
    return CrossSections("fuel", np.array([0.15, 1.2]), np.array([[0.0, 0.05], [0.02, 0.0]]),
                         np.array([0.02, 0.24]), np.array([0.02, 0.24]) / 2.45,
                         np.array([1.0, 0.0]))


def oracle_problem(nx=6, ny=6, n_groups=2):
    fuel = _two_group_fuel() if n_groups == 2 else CrossSections(
        "fuel", np.array([0.5]), np.zeros((1, 1)), np.array([0.6]), np.array([0.25]),
        np.array([1.0]))
    return ProblemSpec(name="oracle_block", nx=nx, ny=ny, dx=0.5, dy=0.5,
                       region_map=np.zeros((nx, ny), dtype=int), materials=[fuel],
                       n_groups=n_groups)


def dense_operators(quad, mat, dx, dy):
    """(A, S, F): upwind streaming + removal, out-of-group scatter, fission."""
    nx, ny, ng = mat.sigma_t.shape
    nd = quad.n_dir
    idx = np.arange(nx * ny * nd * ng).reshape(nx, ny, nd, ng)
    size = idx.size
    A = np.zeros((size, size))
    mu = quad.mu[None, None, :, None] * np.ones((nx, ny, nd, ng))
    nu = quad.nu[None, None, :, None] * np.ones((nx, ny, nd, ng))
    diag = np.abs(mu) / dx + np.abs(nu) / dy + mat.sigma_t[:, :, None, :]
    A[idx.ravel(), idx.ravel()] += diag.ravel()
    # upwind neighbours (inflow boundaries drop the term: vacuum)
    for axis, coef, d in ((0, mu, dx), (1, nu, dy)):
        pos = coef > 0
        lo = [slice(None)] * 4
        hi = [slice(None)] * 4
        lo[axis], hi[axis] = slice(1, None), slice(None, -1)
        rows, cols = idx[tuple(lo)], idx[tuple(hi)]               # row i uses i-1
        m = pos[tuple(lo)]
        A[rows[m], cols[m]] -= coef[tuple(lo)][m] / d
        rows, cols = idx[tuple(hi)], idx[tuple(lo)]               # row i uses i+1
        m = ~pos[tuple(hi)]
        A[rows[m], cols[m]] += coef[tuple(hi)][m] / d
    S = np.zeros((size, size))
    F = np.zeros((size, size))
    w = quad.weights
    for i in range(nx):
        for j in range(ny):
            blk = idx[i, j]                                        # (nd, ng)
            ss = mat.sigma_s[i, j].copy()                          # [from, to]
            np.fill_diagonal(ss, 0.0)
            # row (n, g), col (m, gp): ss[gp, g] w[m]
            S[np.ix_(blk.ravel(), blk.ravel())] += _block(ss.T, w, nd, ng)
            F[np.ix_(blk.ravel(), blk.ravel())] += _block(
                np.outer(mat.chi[i, j], mat.nu_sigma_f[i, j]), w, nd, ng)
    return A, S, F


def _block(gg, w, nd, ng):
    """Matrix over (n, g) x (m, gp) with entries gg[g, gp] * w[m]."""
    out = np.zeros((nd, ng, nd, ng))
    out[:] = gg[None, :, None, :] * w[None, None, :, None]
    return out.reshape(nd * ng, nd * ng)


def dense_power_iteration(A, B, iters=2000, tol=1e-13):
    inv = np.linalg.inv(A)
    phi = np.ones(A.shape[0])
    k = 1.0
    prod_old = B @ phi
    norm_old = prod_old.sum()
    for _ in range(iters):
        phi = inv @ (prod_old / k)
        norm = (B @ phi).sum()
        k_new = k * norm / norm_old
        phi /= norm
        prod_old = B @ phi
        norm_old = prod_old.sum()
        done = abs(k_new - k) < tol * abs(k_new)
        k = k_new
        if done:
            break
    return k


def compare_against_dense_oracle(nx=6, ny=6, n_a=1, n_groups=2, tol_residual=1e-12,
                                 tol_jacobi=1e-12, tol_keff=1e-6):
    problem = oracle_problem(nx, ny, n_groups)
    quad = build_quadrature(n_a)
    mat = problem.material_field()
    grid = GridSpec(nx, ny, problem.dx, problem.dy, halo=1)
    uf = build_upwind_filters(problem.dx, problem.dy)
    A, S, F = dense_operators(quad, mat, problem.dx, problem.dy)
    rng = np.random.default_rng(2718)
    psi = Field(grid, quad.n_dir, n_groups, dtype=torch.float64)
    inner = rng.random((nx, ny, quad.n_dir, n_groups))
    psi.interior.copy_(torch.as_tensor(inner))
    q = rng.random(inner.shape)
    apply_boundary(psi, quad)
    r = upwind_residual(psi, mat.sigma_t, q, quad, uf)
    r_int = r.interior.cpu().numpy().ravel()
    err_resid = float(np.max(np.abs(r_int - (A @ inner.ravel() - q.ravel()))))
    lev = build_hierarchy(grid, quad, mat.sigma_t, 1)[0]
    stepped = psi.copy()
    jacobi_sweep(stepped, q, lev, n_sweeps=1, scheme="upwind")
    dense_step = inner.ravel() - (A @ inner.ravel() - q.ravel()) / np.diag(A)
    err_jac = float(np.max(np.abs(stepped.interior.cpu().numpy().ravel() - dense_step)))
    k_dense = dense_power_iteration(A - S, F)
    state = power_iteration(problem, SolverOptions(scheme="upwind", n_a=n_a, mg_iters=25,
                                                   jacobi_sweeps=3, outer_iters=200,
                                                   dtype="float64"))
    err_k = abs(state.k_eff - k_dense)
    return OracleReport([
        ("upwind residual vs dense", err_resid, tol_residual, err_resid <= tol_residual),
        ("jacobi sweep vs dense", err_jac, tol_jacobi, err_jac <= tol_jacobi),
        (f"power-iteration k_eff vs dense ({k_dense:.8f})", err_k, tol_keff, err_k <= tol_keff),
    ])
