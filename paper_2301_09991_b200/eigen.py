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
from .quadrature import build_quadrature, fold_z

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
    fold_z: bool = False            # carry the upper hemisphere only (exact for x-y problems)

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
    if options.fold_z:
        quad = fold_z(quad)
    fs = build_convfem_filters(options.order, problem.dx, problem.dy) \
        if options.scheme == "pg" else None
    mat = problem.material_field()
    n_levels = options.n_levels if options.n_levels is not None else max_levels(grid.nx, grid.ny)
    hier = build_hierarchy(grid, quad, mat.sigma_t, n_levels)
    return TransportSetup(grid=grid, quad=quad, filters=fs, mat=mat, hierarchy=hier,
                          options=options)


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
        assemble_group_source(torch.zeros_like(bufs.phi), setup.mat, 0.0, d.dtype, bufs.q,
                              fission_frozen)
    history = []
    for _ in range(n_iters):
        if not one_group:
            scalar_flux_into(psi, setup.quad, bufs.phi)
            assemble_group_source(bufs.phi, setup.mat, 0.0, d.dtype, bufs.q, fission_frozen)
        res = eng.cycle(psi, bufs.q, setup.filters, opts.pg, scheme, opts.jacobi_sweeps,
                        opts.pg_sweeps, pg_state, halo_ok=bool(history))
        history.append(res)
        if not math.isfinite(res):
            break
    return psi, history


def _phi_host(psi, quad):
    bufs_phi = torch.empty((psi.grid.nx, psi.grid.ny, psi.n_group), dtype=torch.float64,
                           device=psi.data.device)
    scalar_flux_into(psi, quad, bufs_phi)
    return bufs_phi


def _scale(t, s):
    _lib.call("csn_scale", _lib.dtype_code(t), _lib.ptr(t), t.numel(), float(s), 1, _lib.stream())


class Solver:
    """Step-wise driver: one ``step()`` = one sawtooth cycle of the reference's solve.

    Mirrors R/eigen.py:159-251: fixed-source problems run the bootstrap (upwind) cycles
    then ``mg_iters`` cycles with a ``PGState``; fissile problems run power iteration,
    freezing the fission source per outer (``inner_iters`` cycles) and applying the
    production-ratio k update + rescale after each outer.  ``solve_fixed_source`` and
    ``power_iteration`` are ``Solver(...).run()``; the benchmark times ``step()``.
    """

    def __init__(self, problem, options=None, inner_iters=None, setup=None):
        self.options = options = options or SolverOptions()
        self.setup = setup = setup or setup_transport(problem, options)
        self.dtype = options.torch_dtype()
        self.dev = default_device()
        mat = setup.mat
        # global properties (a domain-decomposed slab may hold no fuel / no source)
        self.eigen = bool(getattr(self, "fissile_global", mat.fissile))
        g = setup.grid
        ng = mat.n_groups
        self.psi = Field(g, setup.quad.n_dir, ng, dtype=self.dtype, device=self.dev)
        self.bufs = _buffers(setup, self.dtype, self.dev)
        self.eng = setup.hierarchy.engine(ng, self.dtype, self.dev)
        self.pgs = PGState(options.k_avg_theta)
        self.history = []            # residual history of the main (PG-state) cycles
        self.boot_history = []
        self.k = 1.0
        self.k_history = [1.0]
        self.empty = False
        n_boot = options.bootstrap() if options.scheme == "pg" else 0
        if self.eigen:
            self.inner = options.mg_iters if inner_iters is None else inner_iters
            self.md = mat.device(self.dev)
            self.gm = _lib.geom(g.nx, g.ny, 1, ng, 1, g.dx, g.dy)
            # the power iteration's own phi (R/eigen.py:212-219,238-248): frozen-fission
            # input of each block, separate from the per-cycle flux of the group source
            self.phi_outer = torch.zeros_like(self.bufs.phi)
            self.psi.fill(1.0)
            apply_boundary(self.psi, setup.quad)
            scalar_flux_into(self.psi, setup.quad, self.phi_outer)
            prod = self._production()
            if prod <= 0.0:
                raise ValueError("initial fission production is zero")
            _scale(self.psi.data, prod)
            _scale(self.phi_outer, prod)
            self.phases = [("boot", n_boot)] + [("outer", self.inner)] * options.outer_iters
        else:
            self.empty = not getattr(self, "source_any", bool(mat.source.any()))
            self.phases = [] if self.empty else [("boot", n_boot), ("main", options.mg_iters)]
        self.phases = [ph for ph in self.phases if ph[1] > 0]
        self.phase = 0
        self.in_phase = 0
        self.stopped = False
        self.outer_done = 0

    # ------------------------------------------------------------------ pieces
    def _production(self):
        _production_dev(self.phi_outer, self.setup.mat, self.setup.grid.dx, self.setup.grid.dy,
                        self.bufs.prod, self.bufs.partials)
        return float(self.bufs.prod.item())

    def _frozen_fission(self, inv_k):
        _lib.call("csn_fission_source", self.gm, _lib.ptr(self.phi_outer), _lib.ptr(self.md["chi"]),
                  _lib.ptr(self.md["nu_sigma_f"]), float(inv_k), _lib.ptr(self.bufs.fission),
                  _lib.stream())
        return self.bufs.fission

    def _source(self, fission, new_block):
        """q for this cycle (R/eigen.py:145-148).

        One group: the in-scatter term sum_a s[a->g] phi_a - s[g->g] phi_g is
        identically 0, so q = s (+ frozen fission) is assembled once per block.
        """
        setup, b = self.setup, self.bufs
        if setup.mat.n_groups == 1:
            if new_block or not getattr(self, "_q_ready", False):
                if not hasattr(self, "_zphi"):
                    self._zphi = torch.zeros_like(b.phi)
                assemble_group_source(self._zphi, setup.mat, 0.0, self.dtype, b.q, fission)
                self._q_ready = True
            return b.q
        scalar_flux_into(self.psi, setup.quad, b.phi)
        assemble_group_source(b.phi, setup.mat, 0.0, self.dtype, b.q, fission)
        return b.q

    @property
    def done(self):
        return self.stopped or self.phase >= len(self.phases)

    def step(self):
        """Run one cycle (plus the outer update when an outer completes); returns res."""
        if self.done:
            raise RuntimeError("solve already finished")
        kind, n = self.phases[self.phase]
        opts = self.options
        boot = kind == "boot"
        fission = None
        if self.eigen:
            if self.in_phase == 0:       # freeze the fission source of this block
                self._fis = self._frozen_fission(1.0 if boot else 1.0 / self.k)
            fission = self._fis
        t = self.eng._t0()
        q = self._source(fission, self.in_phase == 0)
        self.eng._t1("flux+source", t)
        # psi's halo is consistent: zero start / applied boundary at setup, then every
        # cycle ends with the boundary (uniform rescaling keeps it)
        res = self.eng.cycle(self.psi, q, self.setup.filters, opts.pg,
                             "upwind" if boot else opts.scheme, opts.jacobi_sweeps,
                             opts.pg_sweeps, None if boot else self.pgs, halo_ok=True)
        (self.boot_history if boot else self.history).append(res)
        self.in_phase += 1
        finite = math.isfinite(res)
        if self.in_phase >= n or not finite:
            if self.eigen and kind == "outer":
                self._outer_update()
            self.phase += 1
            self.in_phase = 0
            if not finite and not self.eigen:
                # R/eigen.py:154-155 stops the block; fixed source then ends
                self.stopped = kind == "main"
        return res

    def _outer_update(self):
        """k <- k P; psi, phi, psi_avg /= P (R/eigen.py:238-248)."""
        scalar_flux_into(self.psi, self.setup.quad, self.phi_outer)
        prod = self._production()
        self.outer_done += 1
        if not math.isfinite(prod) or prod <= 0.0:
            raise ValueError(f"fission production became {prod} at outer iteration "
                             f"{self.outer_done}")
        self.k = self.k * prod
        _scale(self.psi.data, prod)
        _scale(self.phi_outer, prod)
        self.pgs.scale_average(prod)
        self.k_history.append(self.k)

    def run(self):
        while not self.done:
            self.step()
        return self.result()

    # ------------------------------------------------------------------ checkpoint
    # Not in the reference: a solve can stop between any two
    # cycles and resume bit-identically — psi, the PGState (decision scalars, log,
    # averaged iterate, diffusivities), the power iteration's phi and k, the phase
    # counters and the histories.  The frozen fission / group source of the current
    # block are recomputed from phi_outer and k, which do not change within a block.
    _CKPT_VERSION = 1

    def _signature(self):
        g, o = self.setup.grid, self.options
        return {"nx": g.nx, "ny": g.ny, "halo": g.halo, "n_dir": self.setup.quad.n_dir,
                "n_group": self.setup.mat.n_groups, "n_a": o.n_a, "order": o.order,
                "scheme": o.scheme, "dtype": o.dtype, "fold_z": bool(o.fold_z),
                "eigen": self.eigen}

    def state_dict(self):
        return {"version": self._CKPT_VERSION, "signature": self._signature(),
                "phase": self.phase, "in_phase": self.in_phase, "stopped": self.stopped,
                "outer_done": self.outer_done, "k": self.k, "k_history": list(self.k_history),
                "history": list(self.history), "boot_history": list(self.boot_history),
                "psi": self.psi.data.cpu().numpy(),
                "phi_outer": self.phi_outer.cpu().numpy() if self.eigen else None,
                "pgs": self.pgs.state_dict()}

    def load_state_dict(self, d):
        if d.get("version") != self._CKPT_VERSION:
            raise ValueError(f"unsupported checkpoint version {d.get('version')!r}")
        if d["signature"] != self._signature():
            raise ValueError(f"checkpoint is for {d['signature']}, solver is {self._signature()}")
        self.phase, self.in_phase = int(d["phase"]), int(d["in_phase"])
        self.stopped, self.outer_done = bool(d["stopped"]), int(d["outer_done"])
        self.k = float(d["k"])
        self.k_history = [float(v) for v in d["k_history"]]
        self.history = [float(v) for v in d["history"]]
        self.boot_history = [float(v) for v in d["boot_history"]]
        self.psi.data.copy_(torch.as_tensor(d["psi"]).reshape(self.psi.data.shape))
        if self.eigen:
            self.phi_outer.copy_(torch.as_tensor(d["phi_outer"]).reshape(self.phi_outer.shape))
            if self.in_phase > 0:        # the block's frozen fission source
                kind = self.phases[self.phase][0]
                self._fis = self._frozen_fission(1.0 if kind == "boot" else 1.0 / self.k)
        self._q_ready = False
        self.pgs.load_state_dict(d["pgs"], self.psi.data, self.setup.grid, self.setup.quad)

    def save_checkpoint(self, path):
        """Write ``state_dict`` as .npz (arrays + JSON metadata, no pickles)."""
        import json
        d = self.state_dict()
        arrays = {"psi": d.pop("psi")}
        if d["phi_outer"] is not None:
            arrays["phi_outer"] = d["phi_outer"]
        d.pop("phi_outer")
        pg = d.pop("pgs")
        for k in ("avg", "kx", "ky"):
            a = pg.pop(k)
            if a is not None:
                arrays["pgs_" + k] = a
        d["pgs"] = pg
        with open(path, "wb") as fh:
            np.savez(fh, meta=np.array(json.dumps(d)), **arrays)

    def load_checkpoint(self, path):
        import json
        with np.load(path, allow_pickle=False) as z:
            d = json.loads(str(z["meta"]))
            d["psi"] = z["psi"]
            d["phi_outer"] = z["phi_outer"] if "phi_outer" in z.files else None
            for k in ("avg", "kx", "ky"):
                d["pgs"][k] = z["pgs_" + k] if "pgs_" + k in z.files else None
        self.load_state_dict(d)
        return self

    def result(self):
        setup, ng = self.setup, self.setup.mat.n_groups
        if self.eigen:
            return EigenState(psi=self.psi, phi=self.phi_outer.cpu().numpy(), k_eff=self.k,
                              iteration=self.options.outer_iters, history=self.k_history,
                              residual_history=self.history, pg_log=list(self.pgs.log))
        if self.empty:
            return FixedSourceResult(psi=self.psi, phi=np.zeros((setup.grid.nx, setup.grid.ny, ng)),
                                     residual_history=[0.0], converged=True)
        phi = _phi_host(self.psi, setup.quad).cpu().numpy()
        hist = self.history
        converged = True
        if self.options.tol_rel > 0.0 and hist and hist[0] > 0.0:
            converged = hist[-1] <= self.options.tol_rel * hist[0]
        if hist and not np.isfinite(hist[-1]):
            converged = False
        return FixedSourceResult(psi=self.psi, phi=phi, residual_history=hist, converged=converged,
                                 bootstrap_history=self.boot_history, pg_log=list(self.pgs.log))


def solve_fixed_source(problem, options=None):
    """Source-driven multigrid solve (R/eigen.py:159-191)."""
    options = options or SolverOptions()
    setup = setup_transport(problem, options)
    if setup.mat.fissile:
        raise ValueError("problem has fission; use power_iteration")
    return Solver(problem, options, setup=setup).run()


def power_iteration(problem, options=None, inner_iters=None):
    """Power method for k-effective (R/eigen.py:194-251)."""
    options = options or SolverOptions()
    setup = setup_transport(problem, options)
    if not setup.mat.fissile:
        raise ValueError("problem has no fission source; power iteration is undefined")
    return Solver(problem, options, inner_iters, setup=setup).run()
