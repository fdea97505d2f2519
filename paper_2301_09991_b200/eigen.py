"""Multigroup source assembly, fixed-source and power-iteration drivers (R/eigen.py:1-251).

Group coupling is lagged Jacobi-style: each cycle rebuilds the in-scatter source
from the current scalar flux; the eigenvalue outer loop freezes the fission
source, runs a block of cycles, updates k with the production ratio and rescales
the iterate.  Scalar flux phi = sum_n p_n psi_n carries the reference's 4 pi
convention.  Everything per cycle runs on the device; the host reads one fp64
residual per cycle (PGState) and one production per outer.
"""

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .discretisation import PGConfig
from .filters import build_convfem_filters
from .grid import Field, GridSpec, apply_boundary, default_device, scalar_flux_into
from .multigrid import PGState, build_hierarchy, max_levels
from .quadrature import build_quadrature

_DTYPES = {"float32": torch.float32, "float64": torch.float64,
           torch.float32: torch.float32, torch.float64: torch.float64}


@dataclass
class SolverOptions:
    """Solver options (R/eigen.py:29-58) plus the device precision ``dtype``."""

    scheme: str = "pg"
    order: int = 2
    n_a: int = 4
    n_levels: int | None = None
    mg_iters: int = 100
    jacobi_sweeps: int = 3
    pg_sweeps: int = 1
    outer_iters: int = 100
    tol_rel: float = 0.0
    bootstrap_cycles: int | None = None
    k_avg_theta: float = 0.2
    pg: PGConfig = field(default_factory=PGConfig)
    dtype: str = "float32"          # field precision on the device ("float32" | "float64")

    def bootstrap(self):
        if self.bootstrap_cycles is not None:
            return self.bootstrap_cycles
        return 20 if self.scheme == "pg" else 0

    def filter_halo(self):
        if self.scheme == "upwind":
            return 1
        return 3 * self.order

    def torch_dtype(self):
        if self.dtype not in _DTYPES:
            raise ValueError(f"unsupported dtype {self.dtype!r}")
        return _DTYPES[self.dtype]


@dataclass
class TransportSetup:
    grid: GridSpec
    quad: object
    filters: object
    mat: object
    hierarchy: object
    options: SolverOptions


@dataclass
class FixedSourceResult:
    psi: Field
    phi: np.ndarray
    residual_history: list
    converged: bool
    bootstrap_history: list = field(default_factory=list)
    pg_log: list = field(default_factory=list)


@dataclass
class EigenState:
    psi: Field
    phi: np.ndarray
    k_eff: float
    iteration: int
    history: list
    residual_history: list = field(default_factory=list)
    pg_log: list = field(default_factory=list)

    @property
    def lam(self):
        return 1.0 / self.k_eff


def setup_transport(problem, options):
    """Grid, quadrature, filters, materials and hierarchy (R/eigen.py:98-114)."""
    if options.scheme not in ("pg", "upwind"):
        raise ValueError(f"unknown scheme {options.scheme!r}")
    grid = GridSpec(problem.nx, problem.ny, problem.dx, problem.dy, options.filter_halo())
    quad = build_quadrature(options.n_a)
    fs = build_convfem_filters(options.order, problem.dx, problem.dy) \
        if options.scheme == "pg" else None
    mat = problem.material_field()
    n_levels = options.n_levels if options.n_levels is not None else max_levels(grid.nx, grid.ny)
    hier = build_hierarchy(grid, quad, mat.sigma_t, n_levels)
    return TransportSetup(grid=grid, quad=quad, filters=fs, mat=mat, hierarchy=hier,
                          options=options)


def _geom(grid, ng, n_a):
    return _lib.geom(grid.nx, grid.ny, 8 * n_a * n_a, ng, n_a, grid.dx, grid.dy)


def assemble_group_source(phi, mat, lam=0.0, dtype=torch.float64, out=None, fission=None):
    """q_g = sum_{g' != g} s[g'->g] phi_g' + lam chi_g F + s_g, shape (nx, ny, 1, ng).

    R/eigen.py:117-130.  ``phi`` is a device (or host) fp64 array; returns a
    device tensor of ``dtype``.  ``fission`` (device fp64, nx x ny x ng) adds a
    frozen fission source (R/eigen.py:500-501).
    """
    dev = default_device()
    if not isinstance(phi, torch.Tensor):
        phi = torch.as_tensor(np.asarray(phi, dtype=np.float64), device=dev)
    phi = phi.to(device=dev, dtype=torch.float64).contiguous()
    nx, ny, ng = phi.shape
    md = mat.device(dev)
    if out is None:
        out = torch.empty((nx, ny, 1, ng), dtype=dtype, device=dev)
    g = _lib.geom(nx, ny, 1, ng, 1, 1.0, 1.0)
    _lib.call("csn_group_source", _lib.dtype_code(out), g, _lib.ptr(phi), _lib.ptr(md["sigma_s"]),
              _lib.ptr(md["source"]), _lib.ptr(fission), float(lam), _lib.ptr(md["chi"]),
              _lib.ptr(md["nu_sigma_f"]), _lib.ptr(out), _lib.stream())
    return out


def _production_dev(phi, mat, dx, dy, out, partials):
    nx, ny, ng = phi.shape
    md = mat.device(phi.device)
    g = _lib.geom(nx, ny, 1, ng, 1, dx, dy)
    _lib.call("csn_production", g, _lib.ptr(phi), _lib.ptr(md["nu_sigma_f"]), _lib.ptr(partials),
              _lib.ptr(out), _lib.stream())
    return out


def fission_production(phi, mat, dx, dy):
    """Volume-integrated fission production (R/eigen.py:133-135)."""
    dev = default_device()
    if not isinstance(phi, torch.Tensor):
        phi = torch.as_tensor(np.asarray(phi, dtype=np.float64), device=dev)
    phi = phi.to(device=dev, dtype=torch.float64).contiguous()
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    partials = torch.empty(148 * 64, dtype=torch.float64, device=dev)
    _production_dev(phi, mat, dx, dy, out, partials)
    return float(out.item())


class _CycleBuffers:
    """Per-setup device buffers for the per-cycle flux / source assembly."""

    def __init__(self, setup, dtype, dev):
        g, ng = setup.grid, setup.mat.n_groups
        self.phi = torch.zeros((g.nx, g.ny, ng), dtype=torch.float64, device=dev)
        self.q = torch.empty((g.nx, g.ny, 1, ng), dtype=dtype, device=dev)
        self.fission = torch.empty((g.nx, g.ny, ng), dtype=torch.float64, device=dev)
        self.prod = torch.zeros(1, dtype=torch.float64, device=dev)
        self.partials = torch.empty(148 * 64, dtype=torch.float64, device=dev)


def _buffers(setup, dtype, dev):
    key = ("_bufs", dtype, str(dev))
    cache = setup.__dict__.setdefault("_dev_cache", {})
    if key not in cache:
        cache[key] = _CycleBuffers(setup, dtype, dev)
    return cache[key]


def _run_cycles(psi, setup, n_iters, fission_frozen=None, pg_state=None, scheme=None):
    """n_iters cycles with lagged in-scatter sources (R/eigen.py:138-156).

    ``fission_frozen``: device fp64 (nx, ny, ng) frozen fission source or None.
    With one group the in-scatter term is identically zero (the reference's
    ``sum_a s[a->g] phi_a - s[g->g] phi_g``), so the source is assembled once.
    """
    opts = setup.options
    scheme = scheme or opts.scheme
    d = psi.data
    bufs = _buffers(setup, d.dtype, d.device)
    eng = setup.hierarchy.engine(psi.n_group, d.dtype, d.device)
    one_group = setup.mat.n_groups == 1
    if one_group:
        bufs.phi.zero_()
        assemble_group_source(bufs.phi, setup.mat, 0.0, d.dtype, bufs.q, fission_frozen)
    history = []
    for _ in range(n_iters):
        if not one_group:
            scalar_flux_into(psi, setup.quad, bufs.phi)
            assemble_group_source(bufs.phi, setup.mat, 0.0, d.dtype, bufs.q, fission_frozen)
        res = eng.cycle(psi, bufs.q, setup.filters, opts.pg, scheme, opts.jacobi_sweeps,
                        opts.pg_sweeps, pg_state)
        history.append(res)
        if not math.isfinite(res):
            break
    return psi, history


def _phi_host(psi, quad):
    bufs_phi = torch.empty((psi.grid.nx, psi.grid.ny, psi.n_group), dtype=torch.float64,
                           device=psi.data.device)
    scalar_flux_into(psi, quad, bufs_phi)
    return bufs_phi


def solve_fixed_source(problem, options=None):
    """Source-driven multigrid solve (R/eigen.py:159-191)."""
    options = options or SolverOptions()
    setup = setup_transport(problem, options)
    dtype = options.torch_dtype()
    if setup.mat.fissile:
        raise ValueError("problem has fission; use power_iteration")
    dev = default_device()
    ng = setup.mat.n_groups
    if not setup.mat.source.any():
        return FixedSourceResult(psi=Field(setup.grid, setup.quad.n_dir, ng, dtype=dtype, device=dev),
                                 phi=np.zeros((setup.grid.nx, setup.grid.ny, ng)),
                                 residual_history=[0.0], converged=True)
    psi = Field(setup.grid, setup.quad.n_dir, ng, dtype=dtype, device=dev)
    boot = []
    if options.scheme == "pg" and options.bootstrap() > 0:
        psi, boot = _run_cycles(psi, setup, options.bootstrap(), scheme="upwind")
    pgs = PGState(options.k_avg_theta)
    psi, history = _run_cycles(psi, setup, options.mg_iters, pg_state=pgs)
    phi = _phi_host(psi, setup.quad).cpu().numpy()
    converged = True
    if options.tol_rel > 0.0 and history[0] > 0.0:
        converged = history[-1] <= options.tol_rel * history[0]
    if not np.isfinite(history[-1]):
        converged = False
    return FixedSourceResult(psi=psi, phi=phi, residual_history=history, converged=converged,
                             bootstrap_history=boot, pg_log=list(pgs.log))


def _scale(t, s):
    _lib.call("csn_scale", _lib.dtype_code(t), _lib.ptr(t), t.numel(), float(s), 1, _lib.stream())


def power_iteration(problem, options=None, inner_iters=None):
    """Power method for k-effective (R/eigen.py:194-251)."""
    options = options or SolverOptions()
    setup = setup_transport(problem, options)
    mat = setup.mat
    dtype = options.torch_dtype()
    if not mat.fissile:
        raise ValueError("problem has no fission source; power iteration is undefined")
    if inner_iters is None:
        inner_iters = options.mg_iters
    dev = default_device()
    g = setup.grid
    psi = Field(g, setup.quad.n_dir, mat.n_groups, dtype=dtype, device=dev).fill(1.0)
    apply_boundary(psi, setup.quad)
    bufs = _buffers(setup, dtype, dev)
    phi = _phi_host(psi, setup.quad)
    md = mat.device(dev)
    gm = _lib.geom(g.nx, g.ny, 1, mat.n_groups, 1, g.dx, g.dy)

    def production():
        _production_dev(phi, mat, g.dx, g.dy, bufs.prod, bufs.partials)
        return float(bufs.prod.item())

    prod = production()
    if prod <= 0.0:
        raise ValueError("initial fission production is zero")
    _scale(psi.data, prod)
    _scale(phi, prod)
    k = 1.0
    history = [k]
    residual_history = []
    pgs = PGState(options.k_avg_theta)

    def frozen(inv_k):
        _lib.call("csn_fission_source", gm, _lib.ptr(phi), _lib.ptr(md["chi"]),
                  _lib.ptr(md["nu_sigma_f"]), float(inv_k), _lib.ptr(bufs.fission), _lib.stream())
        return bufs.fission

    if options.scheme == "pg" and options.bootstrap() > 0:
        psi, _ = _run_cycles(psi, setup, options.bootstrap(), fission_frozen=frozen(1.0),
                             scheme="upwind")
    for it in range(options.outer_iters):
        psi, res = _run_cycles(psi, setup, inner_iters, fission_frozen=frozen(1.0 / k),
                               pg_state=pgs)
        residual_history.extend(res)
        scalar_flux_into(psi, setup.quad, phi)
        prod = production()
        if not math.isfinite(prod) or prod <= 0.0:
            raise ValueError(f"fission production became {prod} at outer iteration {it + 1}")
        k = k * prod
        _scale(psi.data, prod)
        _scale(phi, prod)
        pgs.scale_average(prod)
        history.append(k)
    return EigenState(psi=psi, phi=phi.cpu().numpy(), k_eff=k, iteration=options.outer_iters,
                      history=history, residual_history=residual_history, pg_log=list(pgs.log))
