"""Discrete transport operators on the B200 (R/discretisation.py:1-286).

Lumped-mass-normalised residuals: upwind ``r = mu D-psi + nu D-psi + sigma psi - q``
and the ConvFEM Petrov-Galerkin residual with the residual-driven anisotropic
diffusion ``-1/2[(k psi)'' + k psi'' - psi k'']`` (stiffness filter = negated second
derivative).  Each function is one launch of a fused sm_100a kernel
(csrc/pg_kernels.cuh, csrc/upwind_kernels.cuh); fields stay on the device.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .grid import Field, geom, quad_dev


@dataclass(frozen=True)
class PGConfig:
    """Scalar knobs of the non-linear PG stabilisation (R/discretisation.py:34-58)."""

    epsilon_k: float = 1.0e-3
    alpha_r: float = 3.0
    beta_r: float = 3.0
    beta_diag: float = 3.0
    k_freeze_rel: float = 0.05

    def alpha_kabs(self, order):
        return 2.0 ** order / 16.0

    def alpha_ksquare(self, order):
        return 2.0 ** order / 2.0

    def host_cfg(self, order):
        return np.array([self.epsilon_k, self.alpha_r, self.alpha_kabs(order),
                         self.alpha_ksquare(order)], dtype=np.float64)


def _sigma_array(mat):
    return getattr(mat, "sigma_t", mat)


def sigma_tensor(mat, like):
    """Per-cell removal (nx, ny, ng) as a contiguous device tensor of like's dtype."""
    s = _sigma_array(mat)
    if isinstance(s, torch.Tensor):
        return s.to(device=like.device, dtype=like.dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(s), dtype=like.dtype, device=like.device)


def source_tensor(q, nx, ny, nd, ng, like):
    """(tensor, q_per_dof) for a source broadcastable to (nx, ny, nd, ng)."""
    if not isinstance(q, torch.Tensor):
        q = torch.as_tensor(np.asarray(q, dtype=np.float64))
    q = q.to(device=like.device, dtype=like.dtype)
    if tuple(q.shape) == (nx, ny, 1, ng):
        return q.contiguous(), 0
    if tuple(q.shape) == (nx, ny, nd, ng):
        return q.contiguous(), 1
    return torch.broadcast_to(q, (nx, ny, nd, ng)).contiguous(), 1


def upwind_residual(psi, mat, q, quad, uf):
    """Upwind residual Field with a zero halo (R/discretisation.py:65-94)."""
    d = psi.data
    _lib.require_cuda(d)
    g = psi.grid
    sig = sigma_tensor(mat, d)
    qt, per_dof = source_tensor(q, g.nx, g.ny, psi.n_dir, psi.n_group, d)
    qd = quad_dev(quad, d)
    out = psi.zeros_like()
    gm = _lib.geom(g.nx, g.ny, psi.n_dir, psi.n_group, quad.n_a, uf.dx, uf.dy)
    _lib.call("csn_upwind_residual", _lib.dtype_code(d), gm, _lib.ptr(d), g.halo, _lib.ptr(sig),
              _lib.ptr(qt), per_dof, _lib.ptr(qd["mu"]), _lib.ptr(qd["nu"]), _lib.ptr(out.data),
              g.halo, None, None, _lib.stream())
    return out


def jacobi_diagonal(mat, quad, grid, scheme="upwind", cfg=None):
    """beta (|mu|/dx + |nu|/dy + sigma_t), beta = 1 (upwind) or beta_diag (pg).

    Returned as a float64 device tensor (nx, ny, n_dir, ng); the solver kernels
    never materialise it (they form it per DOF on the fly).
    """
    beta = 1.0
    if scheme == "pg":
        beta = (cfg or PGConfig()).beta_diag
    elif scheme != "upwind":
        raise ValueError(f"unknown scheme {scheme!r}")
    from .grid import default_device
    dev = default_device()
    sig = torch.as_tensor(np.asarray(_sigma_array(mat), dtype=np.float64), device=dev)
    stream_term = torch.as_tensor(np.abs(quad.mu) / grid.dx + np.abs(quad.nu) / grid.dy,
                                  dtype=torch.float64, device=dev)
    return beta * (stream_term.reshape(1, 1, -1, 1) + sig[:, :, None, :])


def _check_order(fs, halo):
    l = fs.half_width
    if halo < 3 * l:
        raise ValueError(f"PG diffusivities need halo >= {3 * l}, field has {halo}")


def diffusivities_workspace(psi_data, gm, order):
    """Workspace tensor for the split fp32 diffusivity path (None where it has none)."""
    nbytes = _lib.load().csn_pg_workspace_size(_lib.dtype_code(psi_data), gm, order)
    if nbytes < 0:
        _lib.check(int(nbytes), "csn_pg_workspace_size")
    if nbytes == 0:
        return None
    return torch.empty(int(nbytes) // 4, dtype=torch.float32, device=psi_data.device)


def diffusivities_into(psi_data, grid, n_dir, n_group, n_a, fs, cfg, mu, nu, kx, ky, k_halo,
                       avg_in=None, avg_out=None, avg_mode=0, theta=1.0, psi_halo=None, gm=None,
                       work=None):
    """Launch the averaging + k kernels (K2; K2a + K2b through ``work`` when given)."""
    taps_arr = fs.taps()
    cfg_arr = cfg.host_cfg(fs.order)
    taps_p = taps_arr.ctypes.data_as(_lib._DP)
    cfg_p = cfg_arr.ctypes.data_as(_lib._DP)
    h = grid.halo if psi_halo is None else psi_halo
    if gm is None:
        gm = _lib.geom(grid.nx, grid.ny, n_dir, n_group, n_a, fs.dx, fs.dy)
    _lib.call("csn_pg_diffusivities", _lib.dtype_code(psi_data), fs.order, gm, taps_p, cfg_p,
              _lib.ptr(psi_data), h, _lib.ptr(avg_in), h, _lib.ptr(avg_out), h, avg_mode,
              float(theta), _lib.ptr(mu), _lib.ptr(nu), _lib.ptr(kx), _lib.ptr(ky), k_halo,
              _lib.ptr(work), _lib.stream())


def pg_anisotropic_diffusivities(psi, fs, quad, cfg, grads=None):
    """(k_x, k_y) shaped like psi.data, meaningful on interior +- l (R/discretisation.py:125-161).

    ``grads`` is accepted for signature parity; the kernel recomputes the
    gradients in registers.  Outside the +-l band the arrays hold 0.
    """
    d = psi.data
    _lib.require_cuda(d)
    _check_order(fs, psi.grid.halo)
    qd = quad_dev(quad, d)
    kx = torch.zeros_like(d)
    ky = torch.zeros_like(d)
    diffusivities_into(d, psi.grid, psi.n_dir, psi.n_group, quad.n_a, fs, cfg, qd["mu"],
                       qd["nu"], kx, ky, psi.grid.halo)
    return kx, ky


def _k_tensor(k, like):
    if isinstance(k, torch.Tensor):
        return k.to(device=like.device, dtype=like.dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(k), dtype=like.dtype, device=like.device)


def pg_residual(psi, mat, q, quad, fs, cfg, diffusivities=None, anisotropy="xy"):
    """PG residual Field with a zero halo (R/discretisation.py:239-276)."""
    d = psi.data
    _lib.require_cuda(d)
    g = psi.grid
    if diffusivities is not None:
        kx, ky = (_k_tensor(k, d) for k in diffusivities)
    elif anisotropy == "xy":
        kx, ky = pg_anisotropic_diffusivities(psi, fs, quad, cfg)
    elif anisotropy == "iso":
        from .alternatives import pg_isotropic_diffusivity
        k = pg_isotropic_diffusivity(psi, fs, quad, cfg)
        kx, ky = k, k
    else:
        raise ValueError(f"unknown anisotropy setting {anisotropy!r}")
    if tuple(kx.shape) != tuple(d.shape):
        raise ValueError("diffusivities must be shaped like the field data")
    out = psi.zeros_like()
    pg_residual_launch(psi, mat, q, quad, fs, kx, ky, g.halo, r=out.data, r_halo=g.halo)
    return out


def pg_residual_launch(psi, mat, q, quad, fs, kx, ky, k_halo, r=None, r_halo=0, psi_out=None,
                       out_halo=0, delta=None, delta_halo=0, beta=1.0, partials=None, l1=None,
                       sigma=None, qt=None, per_dof=None, consts=None, avg=None, avg_mode=0,
                       theta=1.0, gm=None, dterm=None, dterm_mode=0):
    d = psi.data
    g = psi.grid
    if sigma is None:
        sigma = sigma_tensor(mat, d)
    if qt is None:
        qt, per_dof = source_tensor(q, g.nx, g.ny, psi.n_dir, psi.n_group, d)
    qd = consts or quad.device(d.dtype, d.device, fs.dx, fs.dy)
    taps_p = fs.taps().ctypes.data_as(_lib._DP)
    if gm is None:
        gm = _lib.geom(g.nx, g.ny, psi.n_dir, psi.n_group, quad.n_a, fs.dx, fs.dy)
    _lib.call("csn_pg_residual", _lib.dtype_code(d), fs.order, gm, taps_p, _lib.ptr(d), g.halo,
              _lib.ptr(delta), delta_halo, _lib.ptr(kx), _lib.ptr(ky), k_halo, _lib.ptr(sigma),
              _lib.ptr(qt), per_dof, _lib.ptr(qd["mu"]), _lib.ptr(qd["nu"]), _lib.ptr(qd["strm"]),
              _lib.ptr(r), r_halo, _lib.ptr(psi_out), out_halo, float(beta), _lib.ptr(partials),
              _lib.ptr(l1), _lib.ptr(avg), g.halo, int(avg_mode), float(theta), _lib.ptr(dterm),
              int(dterm_mode), _lib.stream())


def pg_isotropic_diffusivity(psi, fs, quad, cfg, mode="mixed_mass", grads=None):
    from .alternatives import pg_isotropic_diffusivity as _iso
    return _iso(psi, fs, quad, cfg, mode)


def residual_estimate(psi, fs, quad, cfg, mode="mixed_mass", grads=None):
    from .alternatives import residual_estimate as _est
    return _est(psi, fs, quad, cfg, mode)


def residual_alternatives(psi, fs, quad, cfg, mode):
    """Field-valued residual estimate (R/discretisation.py:279-286)."""
    from .alternatives import residual_alternatives as _alt
    return _alt(psi, fs, quad, cfg, mode)
