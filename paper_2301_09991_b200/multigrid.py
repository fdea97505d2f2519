"""Space-angle sawtooth multigrid on the B200 (R/multigrid.py:1-353).

Each level halves space and (until one patch per face) angle; removal is
coarsened harmonically.  A cycle forms the finest residual (PG or upwind),
restricts it through every level (normalised back to lumped-mass units),
Jacobi-relaxes the correction with the upwind scheme from the coarsest level up
(prolongation fused into the first sweep of each level), subtracts it, and for
the PG scheme finishes with relaxations of the full system (the subtraction is
fused into that sweep).  ``CycleEngine`` owns the device workspaces of one
hierarchy and issues the kernel sequence; the per-cycle host work is the fp64
residual read-back that drives ``PGState``.
"""

import ctypes
import gc
import itertools
import os

import numpy as np
import torch

from . import _lib
from .discretisation import (PGConfig, diffusivities_into, diffusivities_workspace,
                             jacobi_diagonal, pg_residual_launch,
                             sigma_tensor, source_tensor)
from .filters import build_upwind_filters
from .grid import Field, GridSpec, apply_boundary, default_device
from .quadrature import coarsen_quadrature

UP_MAX_SWEEPS = 3   # sweeps per temporally blocked smoother launch (csrc/upwind_kernels.cuh)


class _Nvtx:
    """NVTX range per cycle stage (host-side markers: nsys/ncu --nvtx group the kernels by
    stage; the C ABI adds one range per entry point).  A no-op without a profiler."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        torch.cuda.nvtx.range_push(self.name)

    def __exit__(self, *a):
        torch.cuda.nvtx.range_pop()


class Level:
    """One level: grid, ordinates, removal (host fp64) and upwind pieces (R/multigrid.py:32-40)."""

    def __init__(self, grid, quad, sigma_t, upwind, diag=None):
        self.grid = grid
        self.quad = quad
        self.sigma_t = sigma_t
        self.upwind = upwind
        self._diag = diag
        self._dev = {}

    @property
    def diag(self):
        """Upwind Jacobi diagonal (device fp64, built on first access only)."""
        if self._diag is None:
            self._diag = jacobi_diagonal(self.sigma_t, self.quad, self.grid, "upwind")
        return self._diag

    def sigma_dev(self, dtype, device):
        key = ("sigma", dtype, str(device))
        if key not in self._dev:
            self._dev[key] = torch.as_tensor(np.ascontiguousarray(self.sigma_t), dtype=dtype,
                                             device=device)
        return self._dev[key]

    def consts(self, dtype, device):
        return self.quad.device(dtype, device, self.grid.dx, self.grid.dy)

    def geom(self, n_group, ghost_w=0, ghost_e=0):
        g = self.grid
        return _lib.geom(g.nx, g.ny, self.quad.n_dir, n_group, self.quad.n_a, g.dx, g.dy,
                         ghost_w, ghost_e)


class MultigridHierarchy:
    """Finest-to-coarsest list of levels."""

    def __init__(self, levels):
        self.levels = levels
        self._engines = {}

    @property
    def n_levels(self):
        return len(self.levels)

    def __iter__(self):
        return iter(self.levels)

    def __getitem__(self, i):
        return self.levels[i]

    def engine(self, n_group, dtype, device):
        key = (n_group, dtype, str(device))
        if key not in self._engines:
            self._engines[key] = CycleEngine(self, n_group, dtype, device)
        return self._engines[key]


def max_levels(nx, ny):
    """Halve while both extents stay even (R/multigrid.py:60-67)."""
    n = 1
    while nx % 2 == 0 and ny % 2 == 0 and nx > 1 and ny > 1:
        nx //= 2
        ny //= 2
        n += 1
    return n


def coarsen_sigma(sigma_t, eps=1e-30):
    """Harmonic 2x2 average; a zero child forces a zero parent (R/multigrid.py:70-77)."""
    nx, ny, ng = sigma_t.shape
    blk = np.asarray(sigma_t).reshape(nx // 2, 2, ny // 2, 2, ng)
    # the sum keeps the reference's expression (NumPy's order of the 4 additions depends on
    # the shape); the zero mask is order-free, so it is OR-ed from the four strided children
    coarse = 4.0 / (1.0 / np.maximum(blk, eps)).sum(axis=(1, 3))
    zero = ((blk[:, 0, :, 0] == 0.0) | (blk[:, 0, :, 1] == 0.0) | (blk[:, 1, :, 0] == 0.0)
            | (blk[:, 1, :, 1] == 0.0))
    if zero.any():
        coarse[zero] = 0.0
    return coarse


def build_hierarchy(grid, quad, sigma_t, n_levels=None):
    """Finest-first levels; angle stops halving at n_a = 1 (R/multigrid.py:80-107)."""
    if n_levels is None:
        n_levels = max_levels(grid.nx, grid.ny)
    if n_levels < 1:
        raise ValueError("hierarchy needs at least one level")
    if grid.nx % 2 ** (n_levels - 1) or grid.ny % 2 ** (n_levels - 1):
        raise ValueError(f"grid {grid.nx}x{grid.ny} not divisible by 2**{n_levels - 1}")
    levels = []
    g, q, sig = grid, quad, np.asarray(sigma_t, dtype=np.float64)
    for i in range(n_levels):
        levels.append(Level(g, q, sig, build_upwind_filters(g.dx, g.dy)))
        if i == n_levels - 1:
            break
        sig = coarsen_sigma(sig)
        g = GridSpec(g.nx // 2, g.ny // 2, 2 * g.dx, 2 * g.dy, g.halo)
        if q.n_a > 1:
            q = coarsen_quadrature(q)
    return MultigridHierarchy(levels)


def _pair_check(fine_level, coarse_level):
    fg, cg = fine_level.grid, coarse_level.grid
    if (cg.nx * 2, cg.ny * 2) != (fg.nx, fg.ny):
        raise ValueError("levels are not a spatial 2:1 pair")
    if coarse_level.quad.n_a not in (fine_level.quad.n_a, fine_level.quad.n_a // 2):
        raise ValueError("levels are not an angular 1:1 or 2:1 pair")


def restrict(field, fine_level, coarse_level):
    """Raw integrated 2x2 (x 2x2 patch) restriction as a coarse Field (R/multigrid.py:110-127)."""
    _pair_check(fine_level, coarse_level)
    d = field.data
    _lib.require_cuda(d)
    cg = coarse_level.grid
    out = Field(cg, coarse_level.quad.n_dir, field.n_group, dtype=d.dtype, device=d.device)
    fc = fine_level.consts(d.dtype, d.device)
    cc = coarse_level.consts(d.dtype, d.device)
    _lib.call("csn_restrict", _lib.dtype_code(d), fine_level.geom(field.n_group),
              coarse_level.geom(field.n_group), _lib.ptr(d), field.grid.halo, _lib.ptr(fc["w"]),
              _lib.ptr(cc["w"]), 0, _lib.ptr(out.data), cg.halo, _lib.stream())
    return out


def restrict_field_array(arr, fine_level, coarse_level):
    """Array-in / array-out raw restriction of an interior tensor (R/multigrid.py:342-353)."""
    _pair_check(fine_level, coarse_level)
    arr = arr.contiguous()
    _lib.require_cuda(arr)
    ng = arr.shape[3]
    cg = coarse_level.grid
    out = torch.empty((cg.nx, cg.ny, coarse_level.quad.n_dir, ng), dtype=arr.dtype,
                      device=arr.device)
    fc = fine_level.consts(arr.dtype, arr.device)
    cc = coarse_level.consts(arr.dtype, arr.device)
    _lib.call("csn_restrict", _lib.dtype_code(arr), fine_level.geom(ng), coarse_level.geom(ng),
              _lib.ptr(arr), 0, _lib.ptr(fc["w"]), _lib.ptr(cc["w"]), 0, _lib.ptr(out), 0,
              _lib.stream())
    return out


def prolong(field, coarse_level, fine_level):
    """Piecewise-constant injection onto the finer level (R/multigrid.py:130-146)."""
    _pair_check(fine_level, coarse_level)
    d = field.data
    _lib.require_cuda(d)
    fg = fine_level.grid
    out = Field(fg, fine_level.quad.n_dir, field.n_group, dtype=d.dtype, device=d.device)
    _lib.call("csn_prolong", _lib.dtype_code(d), coarse_level.geom(field.n_group),
              fine_level.geom(field.n_group), _lib.ptr(d), field.grid.halo, _lib.ptr(out.data),
              fg.halo, _lib.stream())
    return out


def _smooth_chain(level, ng, src, per_dof, init, init_mode, init_halo, gc, n_sweeps, scale,
                  out, out_halo, spare, sig=None, g=None, fold=False):
    """Run n_sweeps upwind sweeps in launches of <= 3 (ping-pong through `spare`).

    fold: `out` is the iterate and the result is subtracted from its interior
    (csn_upwind_smooth_sub: the finest correction fused with psi -= delta)."""
    d = out
    c = level.consts(d.dtype, d.device)
    if sig is None:
        sig = level.sigma_dev(d.dtype, d.device)
    if g is None:
        g = level.geom(ng)
    dt = _lib.dtype_code(d)
    if fold:
        if n_sweeps > UP_MAX_SWEEPS:
            raise ValueError("the folded correction runs in one launch (<= 3 sweeps)")
        _lib.call("csn_upwind_smooth_sub", dt, g, _lib.ptr(src), per_dof, init_mode,
                  _lib.ptr(init), init_halo, gc, _lib.ptr(sig), _lib.ptr(c["mu"]),
                  _lib.ptr(c["nu"]), _lib.ptr(c["strm"]), n_sweeps, float(scale), _lib.ptr(out),
                  out_halo, _lib.stream())
        return out
    first = min(n_sweeps, UP_MAX_SWEEPS)
    bufs = [out, spare]
    k = 0
    _lib.call("csn_upwind_smooth", dt, g, _lib.ptr(src), per_dof, init_mode, _lib.ptr(init),
              init_halo, gc, _lib.ptr(sig), _lib.ptr(c["mu"]), _lib.ptr(c["nu"]),
              _lib.ptr(c["strm"]), first, float(scale), _lib.ptr(bufs[0]), out_halo,
              _lib.stream())
    done = first
    while done < n_sweeps:
        now = min(n_sweeps - done, UP_MAX_SWEEPS)
        _lib.call("csn_upwind_smooth", dt, g, _lib.ptr(src), per_dof, 1, _lib.ptr(bufs[k]),
                  out_halo, None, _lib.ptr(sig), _lib.ptr(c["mu"]), _lib.ptr(c["nu"]),
                  _lib.ptr(c["strm"]), now, float(scale), _lib.ptr(bufs[1 - k]), out_halo,
                  _lib.stream())
        k = 1 - k
        done += now
    return bufs[k]


def jacobi_sweep(psi, q, level, n_sweeps=1, scheme="upwind", cfg=None, fs=None, diag_scale=1.0,
                 diffusivities=None):
    """n_sweeps Jacobi relaxations psi <- psi - d^-1 r(psi), in place (R/multigrid.py:149-173).

    The vacuum rule is applied on load before every sweep; psi's halo is
    refreshed at the end.
    """
    cfg = cfg or PGConfig()
    if scheme not in ("pg", "upwind"):
        raise ValueError(f"unknown scheme {scheme!r}")
    d = psi.data
    _lib.require_cuda(d)
    g = psi.grid
    if scheme == "upwind":
        qt, per_dof = source_tensor(q, g.nx, g.ny, psi.n_dir, psi.n_group, d)
        if n_sweeps > 0:
            out = torch.empty_like(d)
            spare = torch.empty_like(d) if n_sweeps > UP_MAX_SWEEPS else None
            res = _smooth_chain(level, psi.n_group, qt, per_dof, d, 1, g.halo, None, n_sweeps,
                                diag_scale, out, g.halo, spare)
            psi.data = res
    else:
        if fs is None:
            raise ValueError("the pg sweep needs the filter set fs")
        from .discretisation import pg_anisotropic_diffusivities, _k_tensor
        for _ in range(n_sweeps):
            apply_boundary(psi, level.quad)
            if diffusivities is None:
                kx, ky = pg_anisotropic_diffusivities(psi, fs, level.quad, cfg)
            else:
                kx, ky = (_k_tensor(k, psi.data) for k in diffusivities)
            out = torch.empty_like(psi.data)
            pg_residual_launch(psi, level.sigma_t, q, level.quad, fs, kx, ky, g.halo,
                               psi_out=out, out_halo=g.halo, beta=cfg.beta_diag)
            psi.data = out
    apply_boundary(psi, level.quad)
    return psi


# freeze heuristics of the diffusivity Picard iteration (R/multigrid.py:176-182)
_STALL_WINDOW = 5
_STALL_FACTOR = 0.9
_UNFREEZE_GROWTH = 2.0
_MAX_FREEZE_ATTEMPTS = 3


# versions of PGState diffusivities (never reused): keys the engine's stored k-term D
_K_VERSIONS = itertools.count(1)


class PGState:
    """Across-cycle diffusivity Picard state (R/multigrid.py:185-256).

    Host logic is the reference's, decision for decision (``observe``); the
    averaged iterate and the diffusivities live on the device.  ``log`` records
    (observe call, "freeze" | "unfreeze") for parity checks.
    """

    __slots__ = ("diffusivities", "initial_residual", "frozen", "best_residual",
                 "cycles_since_best", "freeze_residual", "failed_freezes", "avg_theta",
                 "_avg", "_avg_spare", "_avg_grid", "_avg_quad", "log", "_calls", "k_version")

    def __init__(self, avg_theta=0.2):
        self.diffusivities = None
        self.initial_residual = None
        self.frozen = False
        self.best_residual = None
        self.cycles_since_best = 0
        self.freeze_residual = None
        self.failed_freezes = 0
        self.avg_theta = avg_theta
        self._avg = None
        self._avg_spare = None
        self._avg_grid = None
        self._avg_quad = None
        self.log = []
        self._calls = 0
        self.k_version = next(_K_VERSIONS)   # changes whenever the diffusivities do

    @property
    def psi_avg(self):
        """The averaged iterate as a Field (halo refreshed on access)."""
        if self._avg is None:
            return None
        f = Field(self._avg_grid, self._avg.shape[2], self._avg.shape[3], self._avg)
        apply_boundary(f, self._avg_quad)
        return f

    @psi_avg.setter
    def psi_avg(self, field):
        if field is None:
            self._avg = None
            return
        self._avg = field.data
        self._avg_grid = field.grid

    def averaged_iterate(self, psi, quad=None):
        """EMA of the iterate (R/multigrid.py:217-225); ``quad`` refreshes the halo."""
        if self.avg_theta >= 1.0:
            return psi
        d = psi.data
        first = self._avg is None
        if first:
            self._avg = torch.empty_like(d)
            self._avg_grid = psi.grid
        self._avg_quad = quad if quad is not None else self._avg_quad
        na = self._avg_quad.n_a if self._avg_quad is not None else int(round((psi.n_dir / 8) ** 0.5))
        gm = _lib.geom(psi.grid.nx, psi.grid.ny, psi.n_dir, psi.n_group, na,
                       psi.grid.dx, psi.grid.dy)
        _lib.call("csn_ema", _lib.dtype_code(d), gm, _lib.ptr(self._avg), psi.grid.halo,
                  _lib.ptr(d), psi.grid.halo, float(self.avg_theta), 1 if first else 2,
                  _lib.stream())
        if self._avg_quad is None:
            return Field(psi.grid, psi.n_dir, psi.n_group, self._avg)
        return self.psi_avg

    def observe(self, resid, k_freeze_rel):
        self._calls += 1
        if self.initial_residual is None:
            self.initial_residual = resid
            self.best_residual = resid
            return
        if self.frozen:
            if resid > _UNFREEZE_GROWTH * self.freeze_residual:
                self.frozen = False
                self.failed_freezes += 1
                self.best_residual = resid
                self.cycles_since_best = 0
                self.log.append((self._calls, "unfreeze"))
            return
        if self.failed_freezes >= _MAX_FREEZE_ATTEMPTS:
            return
        if resid <= k_freeze_rel * self.initial_residual:
            self._freeze(resid)
            return
        if resid < _STALL_FACTOR * self.best_residual:
            self.best_residual = resid
            self.cycles_since_best = 0
        else:
            self.cycles_since_best += 1
            if self.cycles_since_best >= _STALL_WINDOW:
                self._freeze(resid)

    def _freeze(self, resid):
        self.frozen = True
        self.freeze_residual = resid
        self.cycles_since_best = 0
        self.log.append((self._calls, "freeze"))

    _SCALARS = ("initial_residual", "frozen", "best_residual", "cycles_since_best",
                "freeze_residual", "failed_freezes", "avg_theta", "_calls")

    def state_dict(self):
        """Host snapshot: decision scalars, log, averaged iterate and diffusivities."""
        host = lambda t: None if t is None else t.cpu().numpy()
        d = {k: getattr(self, k) for k in self._SCALARS}
        d["log"] = [list(e) for e in self.log]
        d["avg"] = host(self._avg)
        kx, ky = self.diffusivities if self.diffusivities is not None else (None, None)
        d["kx"], d["ky"] = host(kx), host(ky)
        return d

    def load_state_dict(self, d, like, grid, quad):
        """Restore a ``state_dict``; ``like`` is a device tensor of the field shape."""
        for k in self._SCALARS:
            setattr(self, k, d[k])
        self.log = [(int(c), str(e)) for c, e in d["log"]]
        dev = lambda a: torch.as_tensor(a, dtype=like.dtype, device=like.device).reshape(like.shape)
        self._avg = None if d["avg"] is None else dev(d["avg"]).contiguous()
        self._avg_spare = None
        self._avg_grid, self._avg_quad = grid, quad
        self.diffusivities = None if d["kx"] is None else (dev(d["kx"]).contiguous(),
                                                           dev(d["ky"]).contiguous())
        self.k_version = next(_K_VERSIONS)

    def scale_average(self, s):
        """psi_avg /= s (R/eigen.py:246-247)."""
        if self._avg is not None:
            _lib.call("csn_scale", _lib.dtype_code(self._avg), _lib.ptr(self._avg),
                      self._avg.numel(), float(s), 1, _lib.stream())


GRAPH_MAX_DOF = 64 * 1024 * 1024
TAIL_MAX_DOF = 32768       # CSN_TAIL_MAX_DOF (include/convsn_sm100.h)
TAIL_MAX_LEVELS = 12


class _NoWait:
    def wait(self):
        pass


class XWindow:
    """Columns [x0, x1) of a slab as a launch geometry of their own.

    x is the slowest storage axis, so a window of any field is a narrowed view (a base
    pointer offset); a cut side is flagged ghost in the window's ``csn_geom``, so the
    kernels read the neighbouring columns of the same array there exactly as they read
    exchanged halo rows at a rank boundary.  Per-cell arithmetic does not depend on the
    tiling, so a field computed window by window is bit-identical to one launch.  Used
    by the domain-decomposed engine to run the interior columns of the PG kernels while
    the halo exchange is in flight and the edge columns after it (dd.py).
    """

    def __init__(self, gm, x0, x1, edge=False):
        self.x0, self.x1 = int(x0), int(x1)
        self.edge = edge           # reads exchanged ghost rows (runs after the exchange)
        self.gm = type(gm).from_buffer_copy(gm)
        self.gm.nx = self.x1 - self.x0
        if self.x0 > 0:
            self.gm.ghost_w = 1
        if self.x1 < gm.nx:
            self.gm.ghost_e = 1

    def pad(self, t, h):
        """Window of a field padded by h: rows [x0, x1 + 2h) of the padded array."""
        return None if t is None else t.narrow(0, self.x0, self.x1 - self.x0 + 2 * h)

    def cells(self, t):
        """Window of an unpadded per-cell array."""
        return None if t is None else t.narrow(0, self.x0, self.x1 - self.x0)


class _FullWindow:
    """The whole slab (no narrowing): what the single-domain engine launches on."""

    edge = False

    def __init__(self, gm):
        self.gm = gm

    def pad(self, t, h):
        return t

    def cells(self, t):
        return t


class CycleEngine:
    """Device workspaces + kernel sequence of one sawtooth cycle on one hierarchy."""

    def __init__(self, hierarchy, n_group, dtype, device):
        self.h = hierarchy
        self.ng = n_group
        self.dtype = dtype
        self.device = device
        L = hierarchy.levels
        self.geoms = [lev.geom(n_group) for lev in L]
        self.consts = [lev.consts(dtype, device) for lev in L]
        self.sigma = [lev.sigma_dev(dtype, device) for lev in L]
        shp = [(lev.grid.nx, lev.grid.ny, lev.quad.n_dir, n_group) for lev in L]
        e = lambda s: torch.empty(s, dtype=dtype, device=device)
        self.r0 = e(shp[0])
        self.src = [self.r0] + [e(s) for s in shp[1:]]
        self.delta = [e(s) for s in shp]
        self.spare = [None] * len(L)
        self.shapes = shp
        lib = _lib.load()
        nparts = max(lib.csn_partials_size(_lib.dtype_code(self.r0), g, 3) for g in self.geoms)
        self.partials = torch.empty(int(nparts), dtype=torch.float64, device=device)
        self.l1 = torch.zeros(1, dtype=torch.float64, device=device)
        self.l1w = None            # per-window L1 of a windowed residual (DD overlap)
        self._tail_args = False    # coarse-tail argument block (built on first use)
        self._side_stream = None   # edge windows run here beside the interior
        self._npart = int(nparts)
        self.k_work_edge = None    # (key, split-K2 workspace of the edge windows)
        self.res_host = torch.zeros(1, dtype=torch.float64, pin_memory=True)
        self.psi_alt = None
        self.k_scratch = None
        self.k_work = None         # (key, workspace of the split diffusivity kernels)
        self.probe = None          # {kernel name: [(start event, end event)]} when timing
        # replay recurring cycle plans from captured CUDA graphs where the cycle is
        # launch-bound (small levels); a C4-size cycle (12 ms of kernels) gains nothing
        # from a graph and would only pay the capture
        self.use_graphs = shp[0][0] * shp[0][1] * shp[0][2] * shp[0][3] < GRAPH_MAX_DOF
        self._graphs = {}
        self._seen = set()
        self._cap_stream = None
        self._graph_warm = False
        self._res_ev = None        # recorded after the residual L1 read-back (cycle part a)
        self.full_sync = False     # A/B switch: wait for the whole cycle (pre-split behaviour)
        # use_dterm (fp32): the residual stores the k-only coefficient D of psi whenever
        # the diffusivities change and the frozen-cycle residual and the sweep read it
        # (csn_pg_residual dterm_mode; bit-identical).  The sweep then runs in the TMA
        # kernel, which needs the finest correction padded with its boundary applied
        # (pad_delta: psi - delta is formed at each read).  Off by default: on C4 it
        # removes 23% of the sweep's FMAs but the cycle is unchanged (11.03 vs 11.04 ms:
        # K5 -2%, K3E -3%, K3 +5% for the D write, +0.03 ms delta boundary) — the PG
        # kernels are latency-bound at 16 warps/SM, not FMA-bound.
        self.use_dterm = os.environ.get("CSN_DTERM", "0") == "1" and dtype == torch.float32
        # pad_delta: the finest correction is written into a buffer padded by l with its
        # boundary applied, so the fp32 sweep runs in the TMA kernel (psi - delta formed
        # at each read; C4 sweep 3.56 -> 3.46 ms once the TMA march got compile-time ring
        # slots, for +0.02 ms of boundary fill on delta)
        self.pad_delta = self.use_dterm or dtype == torch.float32
        self.delta0p = None
        # fold_delta: the finest smoother subtracts its correction from psi in place
        # (csn_upwind_smooth_sub, an L2 reduction) and the fused sweep stages psi' alone
        # (TMA PG_SWEEPF: 3 fields, no per-read psi - delta); same DRAM bytes per cycle,
        # a quarter fewer shared-memory reads and FP adds in the sweep.  CSN_FOLD=0 turns
        # it off (A/B); domain decomposition keeps the exchanged delta.
        self.fold_delta = os.environ.get("CSN_FOLD", "1") != "0"
        self.sweep_reach = 1
        self.dterm = None
        self._dkey = None

    def _t0(self):
        if self.probe is None:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return ev

    def _t1(self, name, ev0):
        if ev0 is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.probe.setdefault(name, []).append((ev0, ev))

    # ---------------------------------------------------------------- correction
    def correction(self, r0, n_sweeps, finest_scale, out0=None, out0_halo=0, fold=False):
        """Restrict r0 through the hierarchy, smooth upward; returns the finest delta
        (into out0, a padded buffer with halo out0_halo, when given; with ``fold`` out0
        is the iterate and the finest delta is subtracted from it instead)."""
        L = self.h.levels
        dt = _lib.dtype_code(r0)
        src = [r0] + self.src[1:]
        tail = self._tail() if r0.dtype == self.dtype else None
        n_res = len(L) if tail is None else tail["start"] + 1
        for i in range(1, n_res):
            _lib.call("csn_restrict", dt, self.geoms[i - 1], self.geoms[i], _lib.ptr(src[i - 1]),
                      0, _lib.ptr(self.consts[i - 1]["w"]), _lib.ptr(self.consts[i]["w"]), 1,
                      _lib.ptr(src[i]), 0, _lib.stream())
        prev = None
        top = len(L) - 1
        if tail is not None:
            # the coarse tail (every level of <= TAIL_MAX_DOF unknowns): its restriction
            # chain and all its smoothing in one cluster launch (csrc/tail_kernels.cuh)
            _lib.call("csn_coarse_tail", dt, tail["n"], tail["geoms"], tail["sigma"], tail["mu"],
                      tail["nu"], tail["strm"], tail["w"], tail["src"], tail["delta"],
                      _lib.ptr(tail["scratch"]), int(n_sweeps), _lib.stream())
            prev = self.delta[tail["start"]]
            top = tail["start"] - 1
        for i in range(top, -1, -1):
            scale = finest_scale if i == 0 else 1.0
            if n_sweeps > UP_MAX_SWEEPS and self.spare[i] is None:
                self.spare[i] = torch.empty_like(self.delta[i])
            if prev is None:
                init, mode, gc = None, 0, None
            else:
                init, mode, gc = prev, 2, self.geoms[i + 1]
            if i == 0 and out0 is not None:
                spare = torch.empty_like(out0) if n_sweeps > UP_MAX_SWEEPS else None
                prev = _smooth_chain(L[0], self.ng, src[0], 1, init, mode, 0, gc, n_sweeps,
                                     scale, out0, out0_halo, spare, self.sigma[0], self.geoms[0],
                                     fold)
                break
            prev = _smooth_chain(L[i], self.ng, src[i], 1, init, mode, 0, gc, n_sweeps, scale,
                                 self.delta[i], 0, self.spare[i], self.sigma[i], self.geoms[i])
        return prev

    def _tail(self):
        """Argument block of the one-launch coarse tail: the levels from the first one
        (>= 1) holding <= TAIL_MAX_DOF unknowns down to the coarsest; None when fewer than
        two levels qualify or CSN_TAIL=0."""
        if self._tail_args is not False:
            return self._tail_args
        self._tail_args = None
        if os.environ.get("CSN_TAIL", "1") == "0":
            return None
        dof = [int(np.prod(s)) for s in self.shapes]
        start = next((i for i in range(1, len(dof)) if dof[i] <= TAIL_MAX_DOF), None)
        if start is None or len(dof) - start < 2 or len(dof) - start > TAIL_MAX_LEVELS:
            return None
        n = len(dof) - start
        vp = ctypes.c_void_p * n
        arr = lambda ts: vp(*[t.data_ptr() for t in ts])
        lv = range(start, len(dof))
        self._tail_args = {
            "start": start, "n": n,
            "geoms": (_lib.Geom * n)(*[self.geoms[i] for i in lv]),
            "sigma": arr([self.sigma[i] for i in lv]),
            "mu": arr([self.consts[i]["mu"] for i in lv]),
            "nu": arr([self.consts[i]["nu"] for i in lv]),
            "strm": arr([self.consts[i]["strm"] for i in lv]),
            "w": arr([self.consts[i]["w"] for i in lv]),
            "src": arr([self.src[i] for i in lv]),
            "delta": arr([self.delta[i] for i in lv]),
            "scratch": torch.empty(dof[start], dtype=self.dtype, device=self.device),
        }
        return self._tail_args

    # hooks for domain decomposition (dd.py): halo exchange / reductions; no-ops here
    def _hook_exchange(self, name, t, width):
        pass

    def _hook_exchange_many(self, items):
        """Ghost-row exchange of several padded fields [(tensor, width)] (DD ranks)."""
        for t, width in items:
            self._hook_exchange("field", t, width)

    def _hook_l1(self):
        pass

    def _hook_exchange_start(self, items):
        """Start the ghost-row exchange of [(tensor, width)]; the returned handle's
        wait() orders later launches after it.  Single domain: nothing to move."""
        self._hook_exchange_many(items)
        return _NoWait()

    def _windows(self, g, reach, n_fields=1):
        """Windows the PG kernels of one stage are launched on: the whole slab here; on
        overlapping DD ranks the interior columns first (they read no exchanged row) and
        the edge columns beside each neighbour (``edge = True``: after the exchange)."""
        return [_FullWindow(self.geoms[0])]

    def _run_windows(self, wins, exch, run):
        """run(i, window) for every window.  One window: after the exchange, on the
        current stream.  Interior + edges: the interior runs on the current stream while
        the exchange is in flight; the edge windows wait for the exchange on a side
        stream and run beside the interior (their CTAs fill the machine as the interior
        drains, where a launch of their own would leave most of a wave idle); the current
        stream then joins the side stream."""
        if len(wins) == 1:
            exch.wait()
            run(0, wins[0])
            return
        main = torch.cuda.current_stream()
        if self._side_stream is None:
            self._side_stream = torch.cuda.Stream(device=self.device)
        side = self._side_stream
        side.wait_stream(main)
        for i, w in enumerate(wins):
            if not w.edge:
                run(i, w)
        with torch.cuda.stream(side):
            exch.wait()
            for i, w in enumerate(wins):
                if w.edge:
                    run(i, w)
        main.wait_stream(side)

    # ---------------------------------------------------------------- cycle
    def cycle(self, psi, q, fs=None, cfg=None, scheme="pg", n_sweeps=3, pg_sweeps=1,
              pg_state=None, sync=True, halo_ok=False):
        """One sawtooth cycle in place; returns the fp64 L1 of the pre-update residual.

        The boundary is applied to psi first (R/multigrid.py:277) unless the caller
        asserts ``halo_ok`` (psi comes from a previous cycle or an applied boundary, as
        in the drivers): the residual kernels read halos as stored.  Host decisions (diffusivity refresh or frozen + fused EMA, buffer ping-pong) are
        planned first; the kernel sequence is then issued eagerly, or — from the second
        time the same plan and buffers recur — replayed from a captured CUDA graph.
        """
        cfg = cfg or PGConfig()
        if scheme not in ("pg", "upwind"):
            raise ValueError(f"unknown scheme {scheme!r}")
        if scheme == "pg" and fs is None:
            raise ValueError("the pg scheme needs the filter set fs")
        d = psi.data
        g = psi.grid
        qt, per_dof = source_tensor(q, g.nx, g.ny, psi.n_dir, psi.n_group, d)
        plan = self._plan(psi, fs, cfg, scheme, pg_sweeps, pg_state)
        nv_cycle = _Nvtx("csn.cycle")
        nv_cycle.__enter__()
        key = plan["key"] + (qt.data_ptr(), per_dof, n_sweeps, scheme, id(fs), cfg)

        if not halo_ok:
            c0 = self.consts[0]
            _lib.call("csn_apply_boundary", _lib.dtype_code(d), self.geoms[0], _lib.ptr(d),
                      g.halo, _lib.ptr(c0["mu"]), _lib.ptr(c0["nu"]), _lib.stream())

        # The cycle is issued in two parts: (a) up to the residual's L1 read-back, (b) the
        # correction, the sweep and the boundary.  An event between them is all the host
        # waits for: PGState.observe and the next cycle's plan need only this cycle's
        # pre-update residual, so the next cycle's launches queue behind (b) while it runs
        # instead of after an idle device (results unchanged; callers see stream order).
        if self._res_ev is None:
            self._res_ev = torch.cuda.Event()
        run_a = lambda: self._launch_a(plan, g, qt, per_dof, fs, cfg, scheme)
        run_b = lambda: self._launch_b(plan, g, qt, per_dof, fs, cfg, scheme, n_sweeps)

        if self.use_graphs and self.probe is None:
            if not self._graph_warm:      # one-time CUDA-graph machinery cost, off the cycle
                self._graph_warm = True
                self._capture(lambda: _lib.call("csn_scale", _lib.F64, _lib.ptr(self.l1), 1, 1.0,
                                                0, _lib.stream())).replay()
            graphs = self._graphs.get(key)
            if graphs is None and key in self._seen:
                graphs = (self._capture(run_a), self._capture(run_b))
                self._graphs[key] = graphs
            if graphs is not None:
                graphs[0].replay()
                self._res_ev.record()
                graphs[1].replay()
            else:
                run_a()
                self._res_ev.record()
                run_b()
                self._seen.add(key)
        else:
            run_a()
            self._res_ev.record()
            run_b()
        self._commit(plan, psi, pg_state)
        nv_cycle.__exit__()
        if not sync:
            return None
        if self.full_sync:
            torch.cuda.current_stream().synchronize()
        else:
            self._res_ev.synchronize()
        res = float(self.res_host[0])
        if self.h.levels[0].quad.folded:    # the mirrored faces carry the same |r|
            res *= 2.0
        if scheme == "pg" and pg_state is not None:
            pg_state.observe(res, cfg.k_freeze_rel)
        return res

    def _capture(self, run, error_mode="global"):
        """Capture `run` into a CUDA graph on a side stream (no GC / cache flush, unlike
        torch.cuda.graph); all buffers are preallocated, nothing allocates inside.  The
        cyclic GC is paused instead: a collection inside the capture could destroy an
        unreachable graph of another engine, and its pool release would invalidate this
        capture."""
        graph = torch.cuda.CUDAGraph()
        if self._cap_stream is None:
            self._cap_stream = torch.cuda.Stream(device=self.device)
        cur = torch.cuda.current_stream()
        self._cap_stream.wait_stream(cur)
        gc_on = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.stream(self._cap_stream):
                graph.capture_begin(capture_error_mode=error_mode)
                try:
                    run()
                finally:
                    graph.capture_end()
        finally:
            if gc_on:
                gc.enable()
        cur.wait_stream(self._cap_stream)
        return graph

    def _plan(self, psi, fs, cfg, scheme, pg_sweeps, pg_state):
        """Host-side decisions and buffer assignment of one cycle (no launches)."""
        d = psi.data
        if self.psi_alt is None or self.psi_alt.shape != d.shape or self.psi_alt.dtype != d.dtype:
            self.psi_alt = torch.empty_like(d)
        plan = {"psi": d, "alt": self.psi_alt, "k2": None, "ema": (None, 0, 1.0),
                "kx": None, "ky": None, "pg_sweeps": pg_sweeps if scheme == "pg" else 0}
        if scheme == "pg":
            l = fs.half_width
            if psi.grid.halo < 3 * l:
                raise ValueError(f"PG diffusivities need halo >= {3 * l}, field has {psi.grid.halo}")
            if pg_state is None:
                if self.k_scratch is None or self.k_scratch[0].shape != d.shape:
                    self.k_scratch = (torch.zeros_like(d), torch.zeros_like(d))
                plan["kx"], plan["ky"] = self.k_scratch
                plan["k2"] = (None, None, 0, 1.0)
            else:
                need_k = pg_state.diffusivities is None or not pg_state.frozen
                if pg_state.diffusivities is None:
                    pg_state.diffusivities = (torch.zeros_like(d), torch.zeros_like(d))
                plan["kx"], plan["ky"] = pg_state.diffusivities
                if pg_state.avg_theta >= 1.0:
                    if need_k:
                        plan["k2"] = (None, None, 0, 1.0)
                else:
                    pg_state._avg_quad = self.h.levels[0].quad
                    first = pg_state._avg is None
                    if first:
                        pg_state._avg = torch.empty_like(d)
                        pg_state._avg_grid = psi.grid
                    theta = float(pg_state.avg_theta)
                    if not need_k:      # frozen: the EMA rides in the residual kernel
                        plan["ema"] = (pg_state._avg, 1 if first else 2, theta)
                    elif first:
                        plan["k2"] = (None, pg_state._avg, 1, theta)
                    else:
                        if pg_state._avg_spare is None or pg_state._avg_spare.shape != d.shape:
                            pg_state._avg_spare = torch.empty_like(d)
                        plan["k2"] = (pg_state._avg, pg_state._avg_spare, 2, theta)
                        plan["swap_avg"] = True
        plan["kd3"], plan["kd5"], plan["dkey"] = 0, 0, None
        if scheme == "pg" and self.use_dterm:
            if self.dterm is None or self.dterm.shape != (psi.grid.nx, psi.grid.ny) + d.shape[2:]:
                self.dterm = torch.empty((psi.grid.nx, psi.grid.ny) + d.shape[2:], dtype=d.dtype,
                                         device=d.device)
                self._dkey = None
            live = plan["k2"] is not None
            ver = None if pg_state is None else pg_state.k_version
            key = (plan["kx"].data_ptr(), plan["ky"].data_ptr(), ver)
            plan["kd3"] = 2 if (not live and self._dkey == key) else 1
            plan["kd5"] = 2
            plan["dkey"] = live
        ema, k2 = plan["ema"], plan["k2"]
        plan["key"] = (d.data_ptr(), self.psi_alt.data_ptr(), plan["kd3"], plan["kd5"],
                       None if plan["kx"] is None else plan["kx"].data_ptr(),
                       None if k2 is None else tuple(None if t is None or isinstance(t, (int, float))
                                                     else t.data_ptr() for t in k2[:2]) + k2[2:],
                       (None if ema[0] is None else ema[0].data_ptr(),) + ema[1:], plan["pg_sweeps"])
        return plan

    def _launch_a(self, plan, g, qt, per_dof, fs, cfg, scheme):
        """Issue part (a) of a planned cycle on the current stream: diffusivity refresh,
        residual (+ fused EMA) and the asynchronous read-back of its L1."""
        L = self.h.levels
        f = L[0]
        c0 = self.consts[0]
        psi_in = plan["psi"]
        dt = _lib.dtype_code(psi_in)
        view = Field.__new__(Field)
        view.grid = g
        view.data = psi_in
        nd, ng, na = psi_in.shape[2], psi_in.shape[3], f.quad.n_a
        # x reach of the kernels reading psi: the diffusivity refresh needs 3l (EMA'd
        # iterate -> gradients on +-2l -> mass pass), the residual and sweep l
        if scheme == "pg":
            reach = (3 if plan["k2"] is not None else 1) * fs.half_width
        else:
            reach = 1
        avg_x = None
        if scheme == "pg" and plan["k2"] is not None and plan["k2"][0] is not None:
            avg_x = plan["k2"][0]
        # psi (and the averaged iterate before a live refresh) ghosts in one exchange
        exch = self._hook_exchange_start([(psi_in, reach)] + ([(avg_x, reach)]
                                                               if avg_x is not None else []))
        if scheme == "pg":
            kx, ky = plan["kx"], plan["ky"]
            h = g.halo
            if plan["k2"] is not None and (self.k_work is None or
                                           self.k_work[0] != (fs.order, psi_in.dtype)):
                # split K2 (two y-marches through a psi_x, psi_y workspace) from the
                # quadratic filters up; at p = 1 the fused two-stage kernel recomputes
                # only 2 of 16 stage-1 columns and runs 2 CTAs/SM, and skipping the
                # 16 B/DOF workspace round trip wins (C3 K2 0.56 -> 0.40 ms, C5-weak
                # 23.5 -> 18.5 ms); CSN_K2_SPLIT=0/1 forces either
                split = os.environ.get("CSN_K2_SPLIT", "1" if fs.order >= 2 else "0") == "1"
                self.k_work = ((fs.order, psi_in.dtype),
                               diffusivities_workspace(psi_in, self.geoms[0], fs.order)
                               if split else None)
            wins = self._windows(g, reach, 2 if avg_x is not None else 1)
            multi = len(wins) > 1
            if multi and self.l1w is None:
                self.l1w = torch.zeros(4, dtype=torch.float64, device=psi_in.device)
                # windows on two streams: one block of reduction partials per window
                self.partials = torch.empty(4 * self._npart, dtype=torch.float64,
                                            device=psi_in.device)
            work_e = None
            if multi and plan["k2"] is not None and self.k_work[1] is not None:
                ew = max(w.x1 - w.x0 for w in wins if w.edge)
                key = (fs.order, psi_in.dtype, ew)
                if self.k_work_edge is None or self.k_work_edge[0] != key:
                    ge = XWindow(self.geoms[0], 0, ew).gm
                    self.k_work_edge = (key, diffusivities_workspace(psi_in, ge, fs.order))
                work_e = self.k_work_edge[1]
            ema = plan["ema"]

            def run(i, win):
                # windowed stages are timed as a whole (below): K2 and K3 of the windows
                # interleave on two streams
                if plan["k2"] is not None:
                    avg_in, avg_out, mode, theta = plan["k2"]
                    nv = _Nvtx("csn.k_refresh")
                    nv.__enter__()
                    t = None if multi else self._t0()
                    diffusivities_into(win.pad(psi_in, h), g, nd, ng, na, fs, cfg, c0["mu"],
                                       c0["nu"], win.pad(kx, h), win.pad(ky, h), h,
                                       avg_in=win.pad(avg_in, h), avg_out=win.pad(avg_out, h),
                                       avg_mode=mode, theta=theta, gm=win.gm,
                                       work=work_e if win.edge else self.k_work[1])
                    self._t1("pg_diffusivity", t)
                    nv.__exit__()
                nv = _Nvtx("csn.residual")
                nv.__enter__()
                t = None if multi else self._t0()
                v = Field.__new__(Field)
                v.grid = g
                v.data = win.pad(psi_in, h)
                pg_residual_launch(v, None, None, f.quad, fs, win.pad(kx, h), win.pad(ky, h), h,
                                   r=win.cells(self.r0), r_halo=0,
                                   partials=self.partials[i * self._npart:] if multi
                                   else self.partials,
                                   l1=self.l1w[i:i + 1] if multi else self.l1,
                                   sigma=win.cells(self.sigma[0]), qt=win.cells(qt),
                                   per_dof=per_dof, consts=c0, avg=win.pad(ema[0], h),
                                   avg_mode=ema[1], theta=ema[2], gm=win.gm, dterm=self.dterm,
                                   dterm_mode=plan["kd3"])
                self._t1("pg_residual" if ema[1] == 0 else "pg_residual+ema", t)
                nv.__exit__()

            t = self._t0() if multi else None
            self._run_windows(wins, exch, run)
            self._t1(("pg_diffusivity+residual" if plan["k2"] is not None else "pg_residual+ema"
                      if ema[1] else "pg_residual") + " (windowed)", t)
            if multi:              # fixed-order fp64 sum of the windows' L1
                torch.sum(self.l1w[:len(wins)], dim=0, keepdim=True, out=self.l1)
        else:
            exch.wait()
            t = self._t0()
            _lib.call("csn_upwind_residual", dt, self.geoms[0], _lib.ptr(psi_in), g.halo,
                      _lib.ptr(self.sigma[0]), _lib.ptr(qt), per_dof, _lib.ptr(c0["mu"]),
                      _lib.ptr(c0["nu"]), _lib.ptr(self.r0), 0, _lib.ptr(self.partials),
                      _lib.ptr(self.l1), _lib.stream())
            self._t1("upwind_residual", t)
        self._hook_l1()
        self.res_host.copy_(self.l1, non_blocking=True)

    def _launch_b(self, plan, g, qt, per_dof, fs, cfg, scheme, n_sweeps):
        """Issue part (b): finest correction, fused PG sweep (or psi -= delta), boundary."""
        f = self.h.levels[0]
        c0 = self.consts[0]
        psi_in = plan["psi"]
        dt = _lib.dtype_code(psi_in)
        view = Field.__new__(Field)
        view.grid = g
        view.data = psi_in
        nd, ng = psi_in.shape[2], psi_in.shape[3]
        self.sweep_reach = fs.half_width if scheme == "pg" else 1    # x reach of the update
        fold = (self.fold_delta and plan["pg_sweeps"] > 0 and n_sweeps <= UP_MAX_SWEEPS)
        # field elements the (first) fused sweep moves per DOF: psi, delta, kx, ky -> psi,
        # or psi', kx, ky -> psi when the correction is folded into the iterate
        self.sweep_elems = 4 if fold else 5
        pad = self.pad_delta and plan["pg_sweeps"] > 0 and not fold
        dh = fs.half_width if pad else 0
        if pad and (self.delta0p is None or self.delta0p.shape[0] != g.nx + 2 * dh):
            self.delta0p = torch.zeros((g.nx + 2 * dh, g.ny + 2 * dh, nd, ng), dtype=psi_in.dtype,
                                       device=psi_in.device)
        nv = _Nvtx("csn.correction")
        nv.__enter__()
        t = self._t0()
        exch = _NoWait()
        if fold:
            # psi' = psi - delta in place, then its boundary (R/multigrid.py:301, :166)
            self.correction(self.r0, n_sweeps, cfg.beta_diag, psi_in, g.halo, fold=True)
            _lib.call("csn_apply_boundary", dt, self.geoms[0], _lib.ptr(psi_in), g.halo,
                      _lib.ptr(c0["mu"]), _lib.ptr(c0["nu"]), _lib.stream())
            # DD ranks: psi' ghost rows for the sweep's l-wide x reach (in flight while
            # the sweep's interior columns run)
            exch = self._hook_exchange_start([(psi_in, fs.half_width)])
            delta = None
        else:
            delta = self.correction(self.r0, n_sweeps, cfg.beta_diag if scheme == "pg" else 1.0,
                                    self.delta0p if pad else None, dh)
        if pad:
            _lib.call("csn_apply_boundary", dt, self.geoms[0], _lib.ptr(delta), dh,
                      _lib.ptr(c0["mu"]), _lib.ptr(c0["nu"]), _lib.stream())
        self._t1("correction", t)
        nv.__exit__()
        nv = _Nvtx("csn.sweep")
        nv.__enter__()
        bufs = (plan["psi"], plan["alt"])
        if plan["pg_sweeps"] > 0:
            for k in range(plan["pg_sweeps"]):
                view.data = bufs[k % 2]
                if k >= 1:
                    # the previous sweep's output: boundary (R/multigrid.py:166; the TMA
                    # sweep reads halos as stored), then its ghost rows on DD ranks (the
                    # boundary kernel also fills ghost sides; the exchange overwrites them)
                    _lib.call("csn_apply_boundary", dt, self.geoms[0], _lib.ptr(bufs[k % 2]),
                              g.halo, _lib.ptr(c0["mu"]), _lib.ptr(c0["nu"]), _lib.stream())
                    self._hook_exchange_many([(bufs[k % 2], fs.half_width)])
                t = self._t0()
                h = g.halo
                # the folded first sweep may run window by window around the exchange
                wins = (self._windows(g, fs.half_width) if k == 0 and fold
                        else [_FullWindow(self.geoms[0])])

                def run(i, win, k=k):
                    v = Field.__new__(Field)
                    v.grid = g
                    v.data = win.pad(bufs[k % 2], h)
                    pg_residual_launch(v, None, None, f.quad, fs, win.pad(plan["kx"], h),
                                       win.pad(plan["ky"], h), h,
                                       psi_out=win.pad(bufs[(k + 1) % 2], h), out_halo=h,
                                       delta=delta if k == 0 else None, delta_halo=dh,
                                       beta=cfg.beta_diag, sigma=win.cells(self.sigma[0]),
                                       qt=win.cells(qt), per_dof=per_dof, consts=c0, gm=win.gm,
                                       dterm=self.dterm, dterm_mode=plan["kd5"] if k == 0 else 0)

                self._run_windows(wins, exch, run)
                exch = _NoWait()
                self._t1("pg_sweep", t)
            view.data = bufs[plan["pg_sweeps"] % 2]
        else:
            _lib.call("csn_sub_interior", dt, self.geoms[0], _lib.ptr(psi_in), g.halo,
                      _lib.ptr(delta), 0, _lib.stream())
        nv.__exit__()
        t = self._t0()
        _lib.call("csn_apply_boundary", dt, self.geoms[0], _lib.ptr(view.data), g.halo,
                  _lib.ptr(c0["mu"]), _lib.ptr(c0["nu"]), _lib.stream())
        self._t1("boundary", t)

    def _commit(self, plan, psi, pg_state):
        """Host bookkeeping after the launches: ping-pong buffer ownership, the version of
        the diffusivities the stored k-term D belongs to."""
        if plan["k2"] is not None and pg_state is not None:
            pg_state.k_version = next(_K_VERSIONS)
        if plan["kd3"] == 1:
            self._dkey = (plan["kx"].data_ptr(), plan["ky"].data_ptr(),
                          None if pg_state is None else pg_state.k_version)
        if plan["pg_sweeps"] % 2 == 1:
            psi.data, self.psi_alt = plan["alt"], plan["psi"]
        if plan.get("swap_avg"):
            pg_state._avg, pg_state._avg_spare = pg_state._avg_spare, pg_state._avg


def sawtooth_cycle(psi, q, hierarchy, fs=None, cfg=None, scheme="pg", n_sweeps=3, pg_sweeps=1,
                   pg_state=None):
    """One sawtooth iteration; returns (psi, finest residual L1) (R/multigrid.py:259-306)."""
    _lib.require_cuda(psi.data)
    eng = hierarchy.engine(psi.n_group, psi.data.dtype, psi.data.device)
    res = eng.cycle(psi, q, fs, cfg, scheme, n_sweeps, pg_sweeps, pg_state)
    return psi, res


def mg_correction(residual_interior, hierarchy, n_sweeps=3, finest_diag_scale=1.0, cfg=None):
    """Restrict a finest residual and smooth the correction upward (R/multigrid.py:309-339).

    Returns the finest correction as a Field (to be subtracted).
    """
    r = residual_interior
    if not isinstance(r, torch.Tensor):
        r = torch.as_tensor(np.asarray(r), device=default_device())
    r = r.contiguous()
    _lib.require_cuda(r)
    eng = hierarchy.engine(r.shape[3], r.dtype, r.device)
    delta = eng.correction(r, n_sweeps, finest_diag_scale)
    f = hierarchy[0]
    out = Field(f.grid, f.quad.n_dir, r.shape[3], dtype=r.dtype, device=r.device)
    out.interior.copy_(delta)
    return out
