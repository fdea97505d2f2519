"""Angular-flux fields on the B200 and the field-level operators (R/grid.py:1-198).

``Field.data`` is a contiguous CUDA tensor ``[nx + 2h, ny + 2h, n_dir, n_group]``
(float32 by default, float64 on request) — the reference's padded layout, x
slowest, so an x-slab of a field is one contiguous block.  All operators run in
libconvsn_sm100.so; there is no CPU fallback.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

DEFAULT_DTYPE = torch.float32


def default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA device (B200, sm_100a) is required: this package has no "
                           "CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True)
class GridSpec:
    """Interior node counts, spacings (cm) and halo width (R/grid.py:20-44)."""

    nx: int
    ny: int
    dx: float
    dy: float
    halo: int = 1

    def __post_init__(self):
        if self.nx < 1 or self.ny < 1:
            raise ValueError("grid must have at least one interior node per axis")
        if self.dx <= 0 or self.dy <= 0:
            raise ValueError("grid spacings must be positive")
        if self.halo < 1:
            raise ValueError("halo width must be >= 1")

    @property
    def x_centres(self):
        return (np.arange(self.nx) + 0.5) * self.dx

    @property
    def y_centres(self):
        return (np.arange(self.ny) + 0.5) * self.dy


class Field:
    """Angular flux psi[ix, iy, n, g] with halo padding, resident on the GPU."""

    __slots__ = ("grid", "data")

    def __init__(self, grid, n_dir, n_group=1, data=None, dtype=None, device=None):
        self.grid = grid
        shape = (grid.nx + 2 * grid.halo, grid.ny + 2 * grid.halo, n_dir, n_group)
        if data is None:
            data = torch.zeros(shape, dtype=dtype or DEFAULT_DTYPE,
                               device=device or default_device())
        else:
            if not isinstance(data, torch.Tensor):
                data = torch.as_tensor(np.asarray(data), dtype=dtype or DEFAULT_DTYPE)
            elif dtype is not None:
                data = data.to(dtype)
            if not data.is_cuda:
                data = data.to(device or default_device())
            data = data.contiguous()
            if tuple(data.shape) != shape:
                raise ValueError(f"field data has shape {tuple(data.shape)}, expected {shape}")
        self.data = data

    @property
    def n_dir(self):
        return self.data.shape[2]

    @property
    def n_group(self):
        return self.data.shape[3]

    @property
    def dtype(self):
        return self.data.dtype

    @property
    def interior(self):
        h = self.grid.halo
        return self.data[h:h + self.grid.nx, h:h + self.grid.ny]

    def copy(self):
        return Field(self.grid, self.n_dir, self.n_group, self.data.clone())

    def zeros_like(self):
        return Field(self.grid, self.n_dir, self.n_group, torch.zeros_like(self.data))

    def fill(self, value):
        self.data.fill_(value)
        return self

    def numpy(self):
        return self.data.detach().cpu().numpy()


def geom(grid, n_dir, n_group, n_a=None, ghost_w=0, ghost_e=0):
    if n_a is None:
        n_a = int(round((n_dir / 8) ** 0.5))
    return _lib.geom(grid.nx, grid.ny, n_dir, n_group, n_a, grid.dx, grid.dy, ghost_w, ghost_e)


def quad_dev(quad, t, grid=None):
    if grid is None:
        return quad.device(t.dtype, t.device)
    return quad.device(t.dtype, t.device, grid.dx, grid.dy)


def apply_boundary(field, quad):
    """Fill the halo band (vacuum rule of R/grid.py:165-190), in place."""
    d = field.data
    _lib.require_cuda(d)
    qd = quad_dev(quad, d)
    g = geom(field.grid, field.n_dir, field.n_group, quad.n_a)
    _lib.call("csn_apply_boundary", _lib.dtype_code(d), g, _lib.ptr(d), field.grid.halo,
              _lib.ptr(qd["mu"]), _lib.ptr(qd["nu"]), _lib.stream())
    return field


def scalar_flux(field, quad):
    """phi[i, j, g] = sum_n p_n psi[i, j, n, g] (fp64 CUDA tensor, R/grid.py:193-198)."""
    if quad.n_dir != field.n_dir:
        raise ValueError(f"quadrature has {quad.n_dir} directions, field has {field.n_dir}")
    d = field.data
    _lib.require_cuda(d)
    phi = torch.empty((field.grid.nx, field.grid.ny, field.n_group), dtype=torch.float64,
                      device=d.device)
    scalar_flux_into(field, quad, phi)
    return phi


def scalar_flux_into(field, quad, phi):
    d = field.data
    qd = quad_dev(quad, d)
    g = geom(field.grid, field.n_dir, field.n_group, quad.n_a)
    _lib.call("csn_scalar_flux", _lib.dtype_code(d), g, _lib.ptr(d), field.grid.halo,
              _lib.ptr(qd["w"]), _lib.ptr(phi), _lib.stream())
    return phi


def _dir_scale(direction_scale, t):
    if direction_scale is None:
        return None
    return torch.as_tensor(np.asarray(direction_scale, dtype=np.float64), dtype=t.dtype,
                           device=t.device).contiguous()


def convolve(field, stencil, direction_scale=None, margin=0):
    """Square-stencil correlation over interior +- margin (R/grid.py:139-152)."""
    w = np.asarray(stencil, dtype=np.float64)
    if w.ndim != 2 or w.shape[0] != w.shape[1] or w.shape[0] % 2 == 0:
        raise ValueError("stencil must be square with odd width")
    l = (w.shape[0] - 1) // 2
    if margin + l > field.grid.halo:
        raise ValueError(f"stencil half-width {l} plus margin {margin} exceeds halo "
                         f"{field.grid.halo}")
    d = field.data
    _lib.require_cuda(d)
    out = torch.empty_like(d)
    sc = _dir_scale(direction_scale, d)
    wa, wp = _lib.host_f64(w)
    _lib.call("csn_convolve", _lib.dtype_code(d), geom(field.grid, field.n_dir, field.n_group),
              _lib.ptr(d), field.grid.halo, wp, w.shape[0], margin, _lib.ptr(sc), _lib.ptr(out),
              _lib.stream())
    return Field(field.grid, field.n_dir, field.n_group, out)


def pass1d(field_data, grid, n_dir, n_group, taps, axis, margin=0):
    """One 1D correlation pass (R/grid.py:108-125) on a padded tensor."""
    taps = np.asarray(taps, dtype=np.float64)
    l = (len(taps) - 1) // 2
    if margin + l > grid.halo:
        raise ValueError("1D stencil does not fit in the halo")
    out = torch.empty_like(field_data)
    ta, tp = _lib.host_f64(taps)
    _lib.call("csn_pass1d", _lib.dtype_code(field_data), geom(grid, n_dir, n_group),
              _lib.ptr(field_data), grid.halo, tp, len(taps), axis, margin, _lib.ptr(out),
              _lib.stream())
    return out


def convolve_separable(field, row_x, row_y, direction_scale=None, margin=0):
    """Rank-one stencil outer(row_x, row_y) as x pass then y pass (R/grid.py:155-162)."""
    d = field.data
    _lib.require_cuda(d)
    tmp = pass1d(d, field.grid, field.n_dir, field.n_group, row_x, 0, margin)
    out = Field(field.grid, field.n_dir, field.n_group,
                pass1d(tmp, field.grid, field.n_dir, field.n_group, row_y, 1, margin))
    if direction_scale is not None:   # 1x1 stencil with the per-direction scale
        out = convolve(out, np.ones((1, 1)), direction_scale, margin)
    return out
