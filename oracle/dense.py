"""Dense brute-force operators for known-answer tests (TEST ORACLE ONLY).

Restates R/oracle.py:34-143 (``R`` = /root/reference/pkg/src/convsn/):
unknowns psi[i, j, n, g] are flattened C-order; the vacuum boundary drops
the upwind neighbour at inflow sides.
"""

import numpy as np


def flat(i, j, n, g, ny, nd, ng):
    return ((i * ny + j) * nd + n) * ng + g


def streaming_removal(mu, nu, sigma, dx, dy):
    """Upwind streaming + removal matrix (R/oracle.py:38-65)."""
    nx, ny, ng = sigma.shape
    nd = len(mu)
    A = np.zeros((nx * ny * nd * ng,) * 2)
    for i in range(nx):
        for j in range(ny):
            for n in range(nd):
                for g in range(ng):
                    row = flat(i, j, n, g, ny, nd, ng)
                    A[row, row] += abs(mu[n]) / dx + abs(nu[n]) / dy + sigma[i, j, g]
                    if mu[n] > 0 and i > 0:
                        A[row, flat(i - 1, j, n, g, ny, nd, ng)] -= mu[n] / dx
                    elif mu[n] < 0 and i < nx - 1:
                        A[row, flat(i + 1, j, n, g, ny, nd, ng)] += mu[n] / dx
                    if nu[n] > 0 and j > 0:
                        A[row, flat(i, j - 1, n, g, ny, nd, ng)] -= nu[n] / dy
                    elif nu[n] < 0 and j < ny - 1:
                        A[row, flat(i, j + 1, n, g, ny, nd, ng)] += nu[n] / dy
    return A


def scatter(weights, sigma_s):
    """Out-of-group in-scatter matrix (R/oracle.py:68-85)."""
    nx, ny, ng = sigma_s.shape[:3]
    nd = len(weights)
    S = np.zeros((nx * ny * nd * ng,) * 2)
    for i in range(nx):
        for j in range(ny):
            for n in range(nd):
                for g in range(ng):
                    row = flat(i, j, n, g, ny, nd, ng)
                    for m in range(nd):
                        for gp in range(ng):
                            if gp != g:
                                S[row, flat(i, j, m, gp, ny, nd, ng)] += sigma_s[i, j, gp, g] * weights[m]
    return S


def fission(weights, chi, nu_sigma_f):
    """Fission matrix (R/oracle.py:88-104)."""
    nx, ny, ng = chi.shape
    nd = len(weights)
    F = np.zeros((nx * ny * nd * ng,) * 2)
    for i in range(nx):
        for j in range(ny):
            for n in range(nd):
                for g in range(ng):
                    row = flat(i, j, n, g, ny, nd, ng)
                    for m in range(nd):
                        for gp in range(ng):
                            F[row, flat(i, j, m, gp, ny, nd, ng)] += chi[i, j, g] * nu_sigma_f[i, j, gp] * weights[m]
    return F


def jacobi_step(A, x, b, beta=1.0):
    """x - (beta diag A)^-1 (A x - b) (R/oracle.py:107-110)."""
    return x - (A @ x - b) / (beta * np.diag(A))


def power_iteration(A, B, iters=500, tol=1e-13):
    """Dominant eigenvalue of A^-1 B, production-ratio update (R/oracle.py:113-143)."""
    inv = np.linalg.inv(A)
    phi = np.ones(A.shape[0])
    k = 1.0
    prod_old = B @ phi
    norm_old = prod_old.sum()
    if norm_old == 0:
        raise ValueError("no fission production; eigenproblem is singular")
    hist = [k]
    for _ in range(iters):
        phi = inv @ (prod_old / k)
        norm = (B @ phi).sum()
        k_new = k * norm / norm_old
        phi /= norm
        prod_old = B @ phi
        norm_old = prod_old.sum()
        converged = abs(k_new - k) < tol * abs(k_new)
        k = k_new
        hist.append(k)
        if converged:
            break
    return k, phi, hist
