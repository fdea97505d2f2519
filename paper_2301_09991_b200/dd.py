"""Spatial domain decomposition: x-slabs across ranks.

Rank r owns x in [X0_r, X1_r) of the global nx x ny grid on every *distributed*
level; x is the slowest storage axis, so a slab and each of its halo bands are one
contiguous block (no packing).  Per cycle (PG scheme):

* psi ghost rows (width 3l) are refreshed before the diffusivities / residual, the
  averaged iterate's ghost rows before a live diffusivity refresh (R/multigrid.py:282-288);
* the residual's L1 (PGState input, R/multigrid.py:292) is an fp64 all-reduce;
* the correction restricts locally, refreshes each level's source ghosts (3 columns:
  the smoother's upwind warm-up), gathers the level-Lg source onto every rank,
  solves the coarse levels Lg..L-1 redundantly (they are < ~1% of the DOF), and
  smooths back up the distributed levels with the coarse correction's ghost columns
  (R/multigrid.py:309-339);
* the fused sweep reads delta's ghost rows (width l) (R/multigrid.py:301-304).

Kernels are unchanged: every launch carries ``ghost_w/ghost_e`` in its geometry, so
ghost sides read halo memory where physical sides apply the vacuum rule.

Communicators: ``TorchDistComm`` (one process per GPU, ``torch.distributed`` —
NCCL over NVLink, or gloo on CPU for tests) and ``ThreadComm`` (several ranks as
threads of one process on one device — used to verify the decomposition against
the single-domain solve on a single GPU).
"""

import os
import threading

import numpy as np
import torch

from . import _lib
from .eigen import Solver, SolverOptions, TransportSetup, setup_transport, _buffers
from .filters import build_upwind_filters
from .grid import GridSpec
from .materials import MaterialField
from .multigrid import (CycleEngine, Level, MultigridHierarchy, UP_MAX_SWEEPS, XWindow,
                        _FullWindow, _smooth_chain, build_hierarchy, coarsen_sigma, max_levels)
from .quadrature import coarsen_quadrature

GX = 5   # x-ghost columns of sources / corrections: the smoother's 3-sweep warm-up and
         # the fused sweep's l-wide read of delta (l <= 5)


# ----------------------------------------------------------------------------- comms
class SlabComm:
    """Neighbour halo exchange along x + the two collectives the solver needs."""

    rank = 0
    size = 1

    def exchange(self, t, width, hx):
        """t: dim 0 = x with interior rows [hx, t.shape[0] - hx); fill `width` ghost
        rows on each side that has a neighbour from the neighbour's interior edge."""
        raise NotImplementedError

    def exchange_many(self, items):
        """Ghost exchange of several fields [(t, width, hx)] issued together; returns a
        handle whose wait() orders the consumer after every transfer (stream-ordered on
        NCCL: the caller may queue independent work before waiting)."""
        for t, width, hx in items:
            self.exchange(t, width, hx)
        return _Done()

    def allreduce_sum_(self, t):
        raise NotImplementedError

    def allgather_x(self, t):
        """Concatenate every rank's t along dim 0 (rank order)."""
        raise NotImplementedError


class _Done:
    def wait(self):
        pass


class _Pending:
    def __init__(self, reqs, copy_back=()):
        self.reqs = reqs
        self.copy_back = list(copy_back)   # (device ghost band, host receive buffer)

    def wait(self):
        for r in self.reqs:
            r.wait()
        self.reqs = []
        for dst, src in self.copy_back:
            dst.copy_(src)
        self.copy_back = []


def _edges(t, width, hx):
    nx = t.shape[0] - 2 * hx
    if width > nx or width > hx:
        # a band wider than the slab would send the sender's own ghost rows
        raise ValueError(f"halo exchange of width {width} on a slab of {nx} rows "
                         f"(halo {hx})")
    return (t[hx:hx + width], t[hx + nx - width:hx + nx],       # west / east interior edge
            t[hx - width:hx], t[hx + nx:hx + nx + width])       # west / east ghost rows


class TorchDistComm(SlabComm):
    """torch.distributed (NCCL on GPUs, gloo on CPU); ranks ordered along x."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        # gloo moves host memory only: device bands are staged through the host (the
        # plumbing check of the N > 1 path on a single GPU; NCCL never takes this path)
        self.host_staged = dist.get_backend(group) == "gloo"

    def _ops(self, t, width, hx, copy_back=None, tag=0):
        dist = self.dist
        we, ee, wg, eg = _edges(t, width, hx)
        if self.host_staged and t.is_cuda:
            we, ee = we.cpu(), ee.cpu()
            hw, he = torch.empty_like(we), torch.empty_like(ee)
            if self.rank > 0:
                copy_back.append((wg, hw))
            if self.rank < self.size - 1:
                copy_back.append((eg, he))
            wg, eg = hw, he
        # x is the slowest axis of a contiguous field: every band is one contiguous block,
        # sent from and received into place
        ops = []
        # tags name the band (item, direction): westward sends match the west
        # neighbour's eastern receive
        if self.rank > 0:
            ops += [dist.P2POp(dist.isend, we, self.rank - 1, self.group, 2 * tag),
                    dist.P2POp(dist.irecv, wg, self.rank - 1, self.group, 2 * tag + 1)]
        if self.rank < self.size - 1:
            ops += [dist.P2POp(dist.isend, ee, self.rank + 1, self.group, 2 * tag + 1),
                    dist.P2POp(dist.irecv, eg, self.rank + 1, self.group, 2 * tag)]
        return ops

    def exchange(self, t, width, hx):
        self.exchange_many([(t, width, hx)]).wait()

    def exchange_many(self, items):
        # one grouped launch for every band (point-to-point ops to the same peer are
        # matched in issue order on both sides)
        ops, back = [], []
        for i, (t, width, hx) in enumerate(items):
            if self.size > 1 and width > 0:
                ops += self._ops(t, width, hx, back, i)
        if not ops:
            return _Done()
        return _Pending(self.dist.batch_isend_irecv(ops), back)

    def allreduce_sum_(self, t):
        if self.size > 1:
            if self.host_staged and t.is_cuda:
                h = t.cpu()
                self.dist.all_reduce(h, group=self.group)
                t.copy_(h)
            else:
                self.dist.all_reduce(t, group=self.group)
        return t

    def allgather_x(self, t):
        if self.size == 1:
            return t
        src = t.cpu() if self.host_staged and t.is_cuda else t.contiguous()
        parts = [torch.empty_like(src) for _ in range(self.size)]
        self.dist.all_gather(parts, src, group=self.group)
        return torch.cat(parts, dim=0).to(t.device)


class _Hub:
    def __init__(self, size):
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots = {}


class ThreadComm(SlabComm):
    """Ranks as threads of one process sharing one device (emulation / verification).

    Device copies are issued after a barrier on the (shared) default stream, so they
    are ordered after every rank's producing kernels and before any consumer."""

    def __init__(self, hub, rank):
        self.hub = hub
        self.rank = rank
        self.size = hub.size

    @staticmethod
    def make(size):
        hub = _Hub(size)
        return [ThreadComm(hub, r) for r in range(size)]

    def _post(self, key, t):
        self.hub.slots[(key, self.rank)] = t
        self.hub.barrier.wait()

    def _done(self):
        self.hub.barrier.wait()

    def exchange(self, t, width, hx):
        if self.size == 1 or width == 0:
            return
        self._post("x", t)
        if self.rank > 0:
            nb = self.hub.slots[("x", self.rank - 1)]
            _edges(t, width, hx)[2].copy_(_edges(nb, width, hx)[1])
        if self.rank < self.size - 1:
            nb = self.hub.slots[("x", self.rank + 1)]
            _edges(t, width, hx)[3].copy_(_edges(nb, width, hx)[0])
        self._done()

    def allreduce_sum_(self, t):
        if self.size == 1:
            return t
        self._post("r", t.clone())
        total = self.hub.slots[("r", 0)].clone()
        for r in range(1, self.size):
            total += self.hub.slots[("r", r)]
        self._done()
        t.copy_(total)
        return t

    def allgather_x(self, t):
        if self.size == 1:
            return t
        self._post("g", t)
        out = torch.cat([self.hub.slots[("g", r)] for r in range(self.size)], dim=0)
        self._done()
        return out


# ----------------------------------------------------------------------------- layout
def slab_bounds(nx, size, rank):
    if nx % size:
        raise ValueError(f"nx = {nx} is not divisible by {size} ranks")
    w = nx // size
    return rank * w, (rank + 1) * w


def distributed_levels(nx, ny, size, n_levels):
    """Levels that stay x-slab distributed: 2x2 blocks must not straddle ranks and each
    slab keeps >= 2 GX columns; the rest is gathered (>= 1 level is always gathered)."""
    w = nx // size
    lg = 0
    while lg < n_levels - 1 and (w >> lg) >= 2 * GX and (w >> lg) % 2 == 0:
        lg += 1
    return max(lg, 1)


class _XGhost:
    """A [nx + 2 GX, ...] tensor whose interior view starts at x = 0."""

    def __init__(self, shape, dtype, device, gx=GX):
        self.gx = gx
        self.full = torch.zeros((shape[0] + 2 * gx,) + tuple(shape[1:]), dtype=dtype, device=device)
        self.view = self.full[gx:gx + shape[0]]


# ----------------------------------------------------------------------------- engine
class DDCycleEngine(CycleEngine):
    """CycleEngine on one rank's slab with halo exchange, L1 all-reduce and a gathered,
    redundantly solved coarse hierarchy."""

    def __init__(self, local_h, coarse_h, comm, n_group, dtype, device, sigma_ghosted,
                 x0_levels, lg):
        self.comm = comm
        self.coarse_h = coarse_h
        self.lg = lg
        self.x0_levels = x0_levels
        super().__init__(local_h, n_group, dtype, device)
        self.pad_delta = False         # x-ghosted finest correction (see correction)
        # the finest correction folds into psi (as on one GPU); psi' ghost rows (width l)
        # are then exchanged instead of delta's
        self.use_dterm = False
        west, east = comm.rank > 0, comm.rank < comm.size - 1
        self.geoms = [lev.geom(n_group, int(west), int(east)) for lev in local_h.levels]
        self.sigma = sigma_ghosted
        # x-ghosted sources / corrections of the distributed levels
        self.src_g = [_XGhost(s, dtype, device) for s in self.shapes]
        self.delta_g = [_XGhost(s, dtype, device) for s in self.shapes]
        self.r0 = self.src_g[0].view
        self.src = [g.view for g in self.src_g]
        self.delta = [g.view for g in self.delta_g]
        self.use_graphs = False      # host barriers / NCCL calls between launches
        # overlap: the PG kernels reading exchanged psi rows (K2, K3 / K3E, the fused
        # sweep) are launched on the slab's interior columns while the exchange is in
        # flight and on the edge columns after it (XWindow); CSN_DD_OVERLAP=0 waits for
        # the exchange first and launches once (results are bit-identical either way)
        self.overlap = os.environ.get("CSN_DD_OVERLAP", "1") != "0"
        self.overlap_min_bytes = int(os.environ.get("CSN_DD_OVERLAP_MIN_MB", "32")) << 20
        cl = coarse_h.levels[0]
        self.coarse_eng = coarse_h.engine(n_group, dtype, device)
        # The gathered coarse solve and the local restriction chain are many short,
        # launch-bound kernels whose count does not shrink with the rank count: each is
        # replayed from a CUDA graph (captured on first use per sweep count) over
        # persistent buffers (one process per rank only: ThreadComm ranks launch from
        # other threads of the process while a capture would be open).  Opt-in
        # (CSN_DD_GRAPHS=1): measured 0.40 -> 0.38 ms of correction per cycle at 8 ranks
        # (compute only, tools/dd_rank_cost.py) and checked under torchrun + gloo; the
        # capture runs in thread-local mode beside NCCL's watchdog thread, which no
        # multi-GPU box has exercised yet.
        self.coarse_graphs = (isinstance(comm, TorchDistComm)
                              and os.environ.get("CSN_DD_GRAPHS", "0") == "1")
        self._cgraphs = {}
        self._local_coarse = None
        self._coarse_in = None
        self.coarse_init = _XGhost((cl.grid.nx // comm.size, cl.grid.ny, cl.quad.n_dir, n_group),
                                   dtype, device)
        self.coarse_geom = cl.geom(n_group, int(west), int(east))
        cgc = cl.grid
        self.coarse_geom.nx = cgc.nx // comm.size

    def _run_graphed(self, key, run):
        """run() eagerly on first use (allocations, kernel attributes), then capture it
        once and replay the graph from the next call on."""
        if not self.coarse_graphs or torch.cuda.is_current_stream_capturing():
            run()
            return
        g = self._cgraphs.get(key)
        if g is None:
            run()
            self._cgraphs[key] = self._capture(run, "thread_local")
        else:
            g.replay()

    def _hook_exchange(self, name, t, width):
        h = self.h.levels[0].grid.halo
        self.comm.exchange(t, width, h)

    def _hook_exchange_many(self, items):
        h = self.h.levels[0].grid.halo
        self.comm.exchange_many([(t, w, h) for t, w in items]).wait()

    def _hook_l1(self):
        self.comm.allreduce_sum_(self.l1)

    def _hook_exchange_start(self, items):
        h = self.h.levels[0].grid.halo
        return self.comm.exchange_many([(t, w, h) for t, w in items])

    def _windows(self, g, reach, n_fields=1):
        """The interior columns (they read no ghost row, so they run while the exchange is
        in flight) and the edge columns beside each neighbour (after the exchange, on the
        side stream).  The interior keeps `reach` columns plus one CTA tile's overhang
        away from a ghosted side, rounded to the 8-column tile.  Only exchanges of at least
        ``overlap_min_bytes`` per side are overlapped: the windowed launches cost ~0.1 ms
        per cycle on a 64-column C4 slab (tools/dd_rank_cost.py), which the 3l-row psi +
        averaged-iterate bands of a live cycle (78 MB per side at 8 ranks) repay and the
        l-row bands of frozen cycles and of the sweep (13 MB) do not."""
        full = [_FullWindow(self.geoms[0])]
        gm = self.geoms[0]
        h = self.h.levels[0].grid.halo
        band = reach * (gm.ny + 2 * h) * gm.nd * gm.ng * self.r0.element_size() * n_fields
        if not self.overlap or band < self.overlap_min_bytes:
            return full
        e = 8 * ((reach + 7 + 7) // 8)
        lo = e if gm.ghost_w else 0
        hi = gm.nx - e if gm.ghost_e else gm.nx
        if hi - lo < 8 or not (gm.ghost_w or gm.ghost_e):
            return full
        wins = [XWindow(gm, lo, hi)]
        if gm.ghost_w:
            wins.append(XWindow(gm, 0, lo, edge=True))
        if gm.ghost_e:
            wins.append(XWindow(gm, hi, gm.nx, edge=True))
        return wins

    def correction(self, r0, n_sweeps, finest_scale, out0=None, out0_halo=0, fold=False):
        if n_sweeps > UP_MAX_SWEEPS:
            raise ValueError("domain decomposition supports <= 3 Jacobi sweeps per level")
        L = self.h.levels
        dt = _lib.dtype_code(r0)
        comm = self.comm
        cl = self.coarse_h.levels[0]
        w = cl.grid.nx // comm.size
        x0 = comm.rank * w
        ci = self.coarse_init
        if self._local_coarse is None or self._local_coarse.dtype != r0.dtype:
            self._local_coarse = torch.empty((w,) + tuple(self.coarse_eng.shapes[0][1:]),
                                             dtype=r0.dtype, device=r0.device)
            self._coarse_in = torch.empty((cl.grid.nx,) + tuple(self.coarse_eng.shapes[0][1:]),
                                          dtype=r0.dtype, device=r0.device)
            self._cgraphs = {}

        def restrict_local():
            # local restriction down the distributed levels (2x2 blocks never straddle
            # ranks, so it reads no ghosts), then onto the coarse level's slab
            for i in range(1, len(L)):
                _lib.call("csn_restrict", dt, self.geoms[i - 1], self.geoms[i],
                          _lib.ptr(self.src[i - 1]), 0, _lib.ptr(self.consts[i - 1]["w"]),
                          _lib.ptr(self.consts[i]["w"]), 1, _lib.ptr(self.src[i]), 0,
                          _lib.stream())
            _lib.call("csn_restrict", dt, self.geoms[-1], self.coarse_geom,
                      _lib.ptr(self.src[-1]), 0, _lib.ptr(self.consts[-1]["w"]),
                      _lib.ptr(cl.consts(r0.dtype, r0.device)["w"]), 1,
                      _lib.ptr(self._local_coarse), 0, _lib.stream())

        def coarse_solve():
            # redundant solve of the gathered coarse hierarchy; this rank keeps its slab
            # of the coarse correction plus GX ghost columns
            dc = self.coarse_eng.correction(self._coarse_in, n_sweeps, 1.0)
            ci.full.zero_()
            lo, hi = max(x0 - GX, 0), min(x0 + w + GX, cl.grid.nx)
            ci.full[lo - (x0 - GX):hi - (x0 - GX)].copy_(dc[lo:hi])

        t = self._t0()
        self._run_graphed(("restrict", r0.data_ptr()), restrict_local)
        self._t1("corr.restrict", t)
        t = self._t0()
        full = comm.allgather_x(self._local_coarse)
        # every distributed level's source ghosts (the smoother's H-column warm-up) in one
        # grouped exchange, in flight while the gathered coarse levels are solved
        src_x = comm.exchange_many([(self.src_g[i].full, UP_MAX_SWEEPS, GX)
                                    for i in range(len(L))])
        self._coarse_in.copy_(full)
        self._run_graphed(("coarse", n_sweeps), coarse_solve)
        src_x.wait()
        self._t1("corr.gather+coarse", t)
        prev, gc = ci.view, self.coarse_geom
        for i in range(len(L) - 1, -1, -1):
            scale = finest_scale if i == 0 else 1.0
            t = self._t0()
            if i == 0 and fold:     # psi -= delta on the slab's interior (no delta ghosts)
                out = _smooth_chain(L[0], self.ng, self.src[0], 1, prev, 2, 0, gc, n_sweeps,
                                    scale, out0, out0_halo, None, self.sigma[0], self.geoms[0],
                                    fold=True)
                self._t1("corr.smooth0", t)
                return out
            prev = _smooth_chain(L[i], self.ng, self.src[i], 1, prev, 2, 0, gc, n_sweeps, scale,
                                 self.delta[i], 0, None, self.sigma[i], self.geoms[i])
            # ghosts the next reader needs: the finer level's warm-up prolongs from
            # (H + 1) / 2 coarse columns; the fused sweep reads l columns of the finest
            w = (UP_MAX_SWEEPS + 1) // 2 if i > 0 else min(GX, self.sweep_reach)
            comm.exchange(self.delta_g[i].full, w, GX)
            self._t1(f"corr.smooth{i}", t)
            gc = self.geoms[i]
        return prev


def _slab_material(mf, x0, x1):
    return MaterialField(mf.sigma_t[x0:x1].copy(), mf.sigma_s[x0:x1].copy(),
                         mf.nu_sigma_f[x0:x1].copy(), mf.sigma_f[x0:x1].copy(),
                         mf.chi[x0:x1].copy(), mf.source[x0:x1].copy())


class DDSolver(Solver):
    """Solver on one rank's x-slab; results (phi, histories, k) are global on every rank."""

    def __init__(self, problem, options=None, inner_iters=None, comm=None, device=None):
        options = options or SolverOptions()
        comm = comm or TorchDistComm()
        self.comm = comm
        gsetup = setup_transport(problem, options)        # global setup (host only)
        gh = gsetup.hierarchy
        nl = gh.n_levels
        lg = distributed_levels(gsetup.grid.nx, gsetup.grid.ny, comm.size, nl)
        if lg >= nl:
            raise ValueError("hierarchy too shallow to decompose")
        x0, x1 = slab_bounds(gsetup.grid.nx, comm.size, comm.rank)
        # every exchange must fit in one neighbour's slab: psi ghosts 3l on live cycles,
        # the smoother's source warm-up (UP_MAX_SWEEPS) and delta's GX columns
        l = gsetup.filters.half_width if options.scheme == "pg" else 1
        need = max(3 * l if options.scheme == "pg" else 1, UP_MAX_SWEEPS, GX)
        if x1 - x0 < need:
            raise ValueError(f"slab of {x1 - x0} columns per rank is narrower than the "
                             f"{need}-column halo exchange ({comm.size} ranks, nx = "
                             f"{gsetup.grid.nx})")
        for l in range(lg + 1):   # every distributed level and the gather level split evenly
            if (gsetup.grid.nx >> l) % comm.size:
                raise ValueError(f"level {l} extent not divisible by {comm.size} ranks")
        if device is not None:
            torch.cuda.set_device(device)
        dev = torch.device("cuda", torch.cuda.current_device())
        dtype = options.torch_dtype()
        # local distributed levels 0..lg-1 and per-level x-ghosted sigma
        levels, sig_g, x0s = [], [], []
        for l in range(lg):
            gl = gh.levels[l]
            w = gl.grid.nx // comm.size
            a0 = comm.rank * w
            grid = GridSpec(w, gl.grid.ny, gl.grid.dx, gl.grid.dy, gl.grid.halo)
            levels.append(Level(grid, gl.quad, gl.sigma_t[a0:a0 + w].copy(),
                                build_upwind_filters(gl.grid.dx, gl.grid.dy)))
            sg = _XGhost((w, gl.grid.ny, gl.sigma_t.shape[2]), dtype, dev)
            lo, hi = max(a0 - GX, 0), min(a0 + w + GX, gl.grid.nx)
            sg.full[lo - (a0 - GX):hi - (a0 - GX)].copy_(
                torch.as_tensor(gl.sigma_t[lo:hi], dtype=dtype))
            sig_g.append(sg.view)
            x0s.append(a0)
        local_h = MultigridHierarchy(levels)
        coarse_h = MultigridHierarchy(gh.levels[lg:])
        mat = _slab_material(gsetup.mat, x0, x1)
        setup = TransportSetup(grid=levels[0].grid, quad=gsetup.quad, filters=gsetup.filters,
                               mat=mat, hierarchy=local_h, options=options)
        ng = mat.n_groups
        eng = DDCycleEngine(local_h, coarse_h, comm, ng, dtype, dev, sig_g, x0s, lg)
        local_h._engines[(ng, dtype, str(dev))] = eng
        self.global_setup = gsetup
        self.fissile_global = gsetup.mat.fissile
        self.source_any = bool(gsetup.mat.source.any())
        super().__init__(problem, options, inner_iters, setup=setup)

    # global decisions must not depend on the slab's own material
    def _production(self):
        from .eigen import _production_dev
        b = self.bufs
        _production_dev(self.phi_outer, self.setup.mat, self.setup.grid.dx, self.setup.grid.dy,
                        b.prod, b.partials)
        self.comm.allreduce_sum_(b.prod)
        return float(b.prod.item())

    def result(self):
        res = super().result()
        res.phi = self.comm.allgather_x(torch.as_tensor(res.phi, device=self.bufs.phi.device)
                                        ).cpu().numpy()
        return res
