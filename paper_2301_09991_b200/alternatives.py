"""Non-default PG discretisation modes on the device (R/discretisation.py:164-224,279-286).

Off the production path (the drivers use the anisotropic "xy" mode): the isotropic
diffusivity (``anisotropy="iso"``) and the residual-estimate variants ("mixed_mass",
"low_order", "high_order").  Built from the generic 1D-pass kernel (R/grid.py:108-125
semantics: full-array outputs, zero outside interior +- margin) and two elementwise
kernels, so array contents match the reference's full padded arrays.
"""

import numpy as np
import torch

from . import _lib
from .filters import averaged_stencils_1d
from .grid import Field, pass1d


def _sep(t, grid, nd, ng, tx, ty, margin):
    return pass1d(pass1d(t, grid, nd, ng, tx, 0, margin), grid, nd, ng, ty, 1, margin)


def _lincomb(x, A, ca, y=None, B=None, cb=0.0, scale=1.0):
    out = torch.empty_like(x)
    C = x.shape[2] * x.shape[3]
    _lib.call("csn_dir_lincomb", _lib.dtype_code(x), x.numel(), C, x.shape[3], _lib.ptr(x),
              _lib.ptr(A), float(ca), _lib.ptr(y), _lib.ptr(B), float(cb), float(scale),
              _lib.ptr(out), _lib.stream())
    return out


def grad_fields(psi, fs):
    """psi_x = M_y G_x psi / dx, psi_y = G_y M_x psi / dy on +-2l (R/discretisation.py:114-122)."""
    d, g = psi.data, psi.grid
    _lib.require_cuda(d)
    l = fs.half_width
    nd, ng = psi.n_dir, psi.n_group
    return (_sep(d, g, nd, ng, fs.grad1 / fs.dx, fs.mass1, 2 * l),
            _sep(d, g, nd, ng, fs.mass1, fs.grad1 / fs.dy, 2 * l))


def residual_estimate(psi, fs, quad, cfg, mode="mixed_mass", grads=None):
    """Equation-residual estimate, full padded array (R/discretisation.py:188-224)."""
    d, g = psi.data, psi.grid
    l = fs.half_width
    nd, ng = psi.n_dir, psi.n_group
    qd = quad.device(d.dtype, d.device)
    px, py = grads if grads is not None else grad_fields(psi, fs)
    adv = _lincomb(px, qd["mu"], 1.0, py, qd["nu"], 1.0)
    if mode == "mixed_mass":
        mm = _sep(adv, g, nd, ng, fs.mass1, fs.mass1, l)
        return _lincomb(mm, None, 1.0, adv, None, -1.0, cfg.beta_r)
    if mode == "low_order":
        if fs.order - 1 < 1:
            raise ValueError("low_order residual needs filter order >= 2")
        other = fs.order - 1
    elif mode == "high_order":
        other = fs.order + 1
    else:
        raise ValueError(f"unknown residual mode {mode!r}")
    mass_o, grad_o, _ = averaged_stencils_1d(other)
    margin = min(l, g.halo - other)
    if margin < 0:
        raise ValueError("field halo too small for the comparison order")
    ox = _sep(d, g, nd, ng, grad_o / fs.dx, mass_o, margin)
    oy = _sep(d, g, nd, ng, mass_o, grad_o / fs.dy, margin)
    adv_o = _lincomb(ox, qd["mu"], 1.0, oy, qd["nu"], 1.0)
    if mode == "low_order":
        return _lincomb(adv, None, 1.0, adv_o, None, -1.0)
    return _lincomb(adv_o, None, 1.0, adv, None, -1.0)


def pg_isotropic_diffusivity(psi, fs, quad, cfg, mode="mixed_mass", grads=None):
    """Single isotropic k (R/discretisation.py:164-185), full padded array."""
    d = psi.data
    px, py = grads if grads is not None else grad_fields(psi, fs)
    r = residual_estimate(psi, fs, quad, cfg, mode, (px, py))
    qd = quad.device(d.dtype, d.device)
    hh = 0.5 * (fs.dx + fs.dy)
    cf = np.array([cfg.epsilon_k, cfg.alpha_kabs(fs.order), cfg.alpha_ksquare(fs.order), hh,
                   fs.dx, fs.dy], dtype=np.float64)
    k = torch.empty_like(d)
    _lib.call("csn_iso_diffusivity", _lib.dtype_code(d), d.numel(), psi.n_dir * psi.n_group,
              psi.n_group, _lib.ptr(r), _lib.ptr(px), _lib.ptr(py), _lib.ptr(qd["mu"]),
              _lib.ptr(qd["nu"]), cf.ctypes.data_as(_lib._DP), _lib.ptr(k), _lib.stream())
    return k


def residual_alternatives(psi, fs, quad, cfg, mode):
    """Field whose interior holds the residual estimate (R/discretisation.py:279-286)."""
    r = residual_estimate(psi, fs, quad, cfg, mode)
    out = psi.zeros_like()
    out.interior.copy_(r[psi.grid.halo:psi.grid.halo + psi.grid.nx,
                         psi.grid.halo:psi.grid.halo + psi.grid.ny])
    return out
