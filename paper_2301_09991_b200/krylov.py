"""Krylov-accelerated Picard driver on the device (R/krylov.py:1-104).

Each Picard pass freezes the diffusivities of the current iterate and solves the
resulting linear PG system with restarted GMRES, left-preconditioned by one
multigrid correction pass.  The matvec (boundary fill + PG residual with q = 0) and
the preconditioner (``CycleEngine.correction``) are the sm_100a kernels; the Arnoldi
vector algebra runs on the device in fp64 (cuBLAS-level torch vector ops) and only
the (restart+1) x restart Hessenberg least-squares problem lives on the host.  The
GMRES is the published left-preconditioned restarted algorithm with Givens rotations
and the inner/outer tolerance coupling SciPy uses (the reference calls
``scipy.sparse.linalg.gmres``, R/krylov.py:88-89).  Use ``dtype="float64"``: the
default 1e-11 GMRES tolerance is below fp32 resolution.
"""

import math

import numpy as np
import torch

from . import _lib
from .discretisation import pg_anisotropic_diffusivities, pg_residual, pg_residual_launch
from .eigen import (FixedSourceResult, SolverOptions, _run_cycles, assemble_group_source,
                    setup_transport)
from .grid import Field, apply_boundary, default_device, scalar_flux


def _givens(f, g):
    """(c, s, r) with [c s; -s c] [f; g] = [r; 0] (real LAPACK lartg convention)."""
    if g == 0.0:
        return 1.0, 0.0, f
    if f == 0.0:
        return 0.0, 1.0 if g > 0 else -1.0, abs(g)
    r = math.hypot(f, g)
    c = abs(f) / r
    s = math.copysign(1.0, f) * g / r
    return c, s, math.copysign(r, f)


def gmres(matvec, psolve, b, x0, rtol=1e-5, atol=0.0, restart=20, maxiter=None):
    """Left-preconditioned restarted GMRES on device vectors; returns (x, info)."""
    n = b.numel()
    bnrm2 = float(torch.linalg.vector_norm(b))
    if bnrm2 == 0.0:
        return b.clone(), 0
    atol = max(float(atol), rtol * bnrm2)
    eps = float(torch.finfo(b.dtype).eps)
    maxiter = n * 10 if maxiter is None else maxiter
    restart = min(restart, n)
    x = x0.clone()
    mb = float(torch.linalg.vector_norm(psolve(b)))
    ptol_max = 1.0
    ptol = mb * min(ptol_max, atol / bnrm2)
    presid = 0.0
    V = torch.empty((restart + 1, n), dtype=b.dtype, device=b.device)
    rnorm = None
    r = b - matvec(x) if bool(torch.any(x != 0)) else b.clone()
    if float(torch.linalg.vector_norm(r)) < atol:
        return x, 0
    for _ in range(maxiter):
        v0 = psolve(r)
        beta = float(torch.linalg.vector_norm(v0))
        V[0] = v0 / beta
        H = np.zeros((restart, restart + 1))
        G = np.zeros((restart, 2))
        S = np.zeros(restart + 1)
        S[0] = beta
        breakdown = False
        col = 0
        for col in range(restart):
            w = psolve(matvec(V[col]))
            h0 = float(torch.linalg.vector_norm(w))
            for k in range(col + 1):                       # modified Gram-Schmidt
                hk = float(torch.dot(V[k], w))
                H[col, k] = hk
                w -= hk * V[k]
            h1 = float(torch.linalg.vector_norm(w))
            H[col, col + 1] = h1
            V[col + 1] = w
            if h1 <= eps * h0:
                H[col, col + 1] = 0.0
                breakdown = True
            else:
                V[col + 1] *= 1.0 / h1
            for k in range(col):                            # previous rotations
                c, s = G[k]
                n0, n1 = H[col, k], H[col, k + 1]
                H[col, k], H[col, k + 1] = c * n0 + s * n1, -s * n0 + c * n1
            c, s, mag = _givens(H[col, col], H[col, col + 1])
            G[col] = c, s
            H[col, col], H[col, col + 1] = mag, 0.0
            tmp = -s * S[col]
            S[col], S[col + 1] = c * S[col], tmp
            presid = abs(tmp)
            if presid <= ptol or breakdown:
                break
        if H[col, col] == 0.0:
            S[col] = 0.0
        y = S[:col + 1].copy()
        for k in range(col, 0, -1):                          # back substitution
            if y[k] != 0.0:
                y[k] /= H[k, k]
                y[:k] -= y[k] * H[k, :k]
        if y[0] != 0.0:
            y[0] /= H[0, 0]
        x += torch.as_tensor(y, dtype=b.dtype, device=b.device) @ V[:col + 1]
        r = b - matvec(x)
        rnorm = float(torch.linalg.vector_norm(r))
        if rnorm <= atol or breakdown:
            break
        if presid <= ptol:
            ptol_max = max(eps, 0.25 * ptol_max)
        else:
            ptol_max = min(1.0, 1.5 * ptol_max)
        ptol = presid * min(ptol_max, atol / rnorm)
    return x, 0 if rnorm is not None and rnorm <= atol else maxiter


def _linear_pieces(setup, diff, q, psi_like, eng):
    """Frozen-k matvec, right-hand side and multigrid preconditioner (R/krylov.py:24-51)."""
    grid, quad = setup.grid, setup.quad
    nd, ng = quad.n_dir, setup.mat.n_groups
    lev = setup.hierarchy[0]
    opts = setup.options
    dt = psi_like.dtype
    work = Field(grid, nd, ng, dtype=dt, device=psi_like.device)
    r = torch.empty((grid.nx, grid.ny, nd, ng), dtype=dt, device=psi_like.device)
    zero_q = torch.zeros((grid.nx, grid.ny, 1, ng), dtype=dt, device=psi_like.device)
    kx, ky = diff
    shape = (grid.nx, grid.ny, nd, ng)

    def matvec(v):
        work.interior.copy_(v.view(shape))
        apply_boundary(work, quad)
        pg_residual_launch(work, lev.sigma_t, zero_q, quad, setup.filters, kx, ky, grid.halo,
                           r=r, r_halo=0)
        return r.reshape(-1).to(torch.float64)

    def precondition(v):
        src = v.view(shape).to(dt).contiguous()
        return eng.correction(src, opts.jacobi_sweeps, opts.pg.beta_diag).reshape(-1).to(
            torch.float64)

    b = torch.broadcast_to(q, shape).reshape(-1).to(torch.float64)
    return matvec, b, precondition


def solve_fixed_source_krylov(problem, options=None, picard_iters=10, picard_tol=1e-8,
                              gmres_rtol=1e-11, gmres_maxiter=400):
    """Fixed-source solve with frozen-diffusivity GMRES inner solves (R/krylov.py:54-104)."""
    options = options or SolverOptions()
    if options.scheme != "pg":
        raise ValueError("the Krylov driver targets the pg scheme")
    setup = setup_transport(problem, options)
    if setup.mat.fissile:
        raise ValueError("fixed-source driver: problem has fission")
    grid, quad = setup.grid, setup.quad
    nd, ng = quad.n_dir, setup.mat.n_groups
    dt = options.torch_dtype()
    dev = default_device()
    psi = Field(grid, nd, ng, dtype=dt, device=dev)
    if options.bootstrap() > 0:
        psi, _ = _run_cycles(psi, setup, options.bootstrap(), scheme="upwind")
    eng = setup.hierarchy.engine(ng, dt, dev)
    history = []
    converged = False
    for _ in range(picard_iters):
        apply_boundary(psi, quad)
        q = assemble_group_source(scalar_flux(psi, quad), setup.mat, dtype=dt)
        diff = pg_anisotropic_diffusivities(psi, setup.filters, quad, options.pg)
        matvec, b, prec = _linear_pieces(setup, diff, q, psi.data, eng)
        x0 = psi.interior.reshape(-1).to(torch.float64)
        x, _info = gmres(matvec, prec, b, x0, rtol=gmres_rtol, atol=0.0, restart=40,
                         maxiter=gmres_maxiter)
        move = float(torch.max(torch.abs(x - x0))) / max(float(torch.max(torch.abs(x))), 1e-300)
        psi.interior.copy_(x.view(psi.interior.shape).to(dt))
        apply_boundary(psi, quad)
        r = pg_residual(psi, setup.hierarchy[0].sigma_t, q, quad, setup.filters, options.pg)
        history.append(float(torch.sum(torch.abs(r.interior.to(torch.float64)))))
        if move < picard_tol:
            converged = True
            break
    phi = scalar_flux(psi, quad).cpu().numpy()
    return FixedSourceResult(psi=psi, phi=phi, residual_history=history, converged=converged)
