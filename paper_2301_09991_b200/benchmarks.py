"""Seeded generators for the five BASELINE.json configurations (C1-C5).

Pure NumPy, no device code: each generator returns a plain ``ProblemData``
(grid, region map, per-material cross sections, fixed source) plus the
solver options the configuration names, so the B200 solver, the CPU oracle
and the golden-vector script (which feeds the reference ``convsn`` objects)
all see identical arrays by construction.  See SURVEY.md §8(d) for the
mapping from BASELINE's wording to reference objects:

* "angle grid A x A" -> ``n_a = A / 2`` (8 n_a^2 ordinates carried);
* config "(sigma_t, sigma_s)" -> ``sigma_a = sigma_t - sum sigma_s`` with the
  scatter matrix including its diagonal, so the reference removal is
  ``sigma_t - sigma_s,gg`` (within-group scatter is inert,
  R/materials.py:3-7, R/eigen.py:124-125);
* "Petrov-Galerkin off" -> ``alpha_r = 0`` (k == 0, R/discretisation.py:145-158);
* ``bootstrap_cycles = 0`` so "N cycles" means N PG cycles (R/eigen.py:46-51).

The reference's KAIST 7-group data are not shipped (R/problems.py:14-16), so
C3 uses the bundled synthetic 2-group set (values restated from
R/data/synthetic_2group.csv:5-17) and C5 a seeded synthetic 7-group set
mapped into the reference's 4-pi scalar-flux convention.
"""

from dataclasses import dataclass, field

import numpy as np

FOUR_PI = 4.0 * np.pi


@dataclass
class MaterialData:
    name: str
    sigma_a: np.ndarray
    sigma_s: np.ndarray          # [from, to]
    nu_sigma_f: np.ndarray
    sigma_f: np.ndarray
    chi: np.ndarray


@dataclass
class ProblemData:
    name: str
    nx: int
    ny: int
    dx: float
    dy: float
    region_map: np.ndarray       # (nx, ny) material ids
    materials: list              # MaterialData per id
    source: np.ndarray | None    # (nx, ny, ng) or None
    n_groups: int
    driver: str = "fixed_source"   # or "power_iteration"
    options: dict = field(default_factory=dict)
    inner_iters: int | None = None

    @property
    def n_a(self):
        return self.options["n_a"]

    def dof(self):
        return self.nx * self.ny * 8 * self.n_a ** 2 * self.n_groups


def _mat(name, sigma_a, sigma_s, nsf=None, sf=None, chi=None):
    sa = np.asarray(sigma_a, dtype=float)
    z = np.zeros_like(sa)
    return MaterialData(name, sa, np.asarray(sigma_s, dtype=float),
                        z.copy() if nsf is None else np.asarray(nsf, float),
                        z.copy() if sf is None else np.asarray(sf, float),
                        z.copy() if chi is None else np.asarray(chi, float))


# ---------------------------------------------------------------- C1
def c1(nx=64, n_a=4, cycles=10, pg_off="alpha_r"):
    """1 group, linear, homogeneous sigma_t = 1, sigma_s = 0.5, q = 1, PG off.

    ``pg_off="alpha_r"``: scheme pg, order 1, alpha_r = 0 (k == 0);
    ``pg_off="upwind"``: the alternative reading, scheme upwind.
    """
    mat = _mat("medium", [0.5], [[0.5]])
    src = np.ones((nx, nx, 1))
    opts = dict(scheme="pg", order=1, n_a=n_a, mg_iters=cycles, bootstrap_cycles=0,
                pg=dict(alpha_r=0.0))
    if pg_off == "upwind":
        opts = dict(scheme="upwind", order=1, n_a=n_a, mg_iters=cycles, bootstrap_cycles=0)
    return ProblemData(f"c1_{pg_off}", nx, nx, 1.0 / nx, 1.0 / nx,
                       np.zeros((nx, nx), dtype=np.int64), [mat], src, 1,
                       options=opts)


# ---------------------------------------------------------------- C2 / C4
def hetero_blocks(nx, blocks, n_a, order, cycles, seed=0, name="blocks"):
    """Seeded blocks: sigma_t ~ logU[0.1, 10], c ~ U[0.1, 0.95] per block.

    Draw order: sigma_t array (blocks, blocks) then c array.  Source q = 1 on
    the central [3/8, 5/8) x [3/8, 5/8) square (1/16 of the area).
    """
    rng = np.random.default_rng(seed)
    sig = np.exp(rng.uniform(np.log(0.1), np.log(10.0), size=(blocks, blocks)))
    c = rng.uniform(0.1, 0.95, size=(blocks, blocks))
    bs = nx // blocks
    mats = []
    for bi in range(blocks):
        for bj in range(blocks):
            st, cc = sig[bi, bj], c[bi, bj]
            mats.append(_mat(f"b{bi}_{bj}", [st * (1.0 - cc)], [[st * cc]]))
    ids = np.arange(blocks * blocks).reshape(blocks, blocks)
    region = np.repeat(np.repeat(ids, bs, axis=0), bs, axis=1)
    src = np.zeros((nx, nx, 1))
    lo, hi = 3 * nx // 8, 5 * nx // 8
    src[lo:hi, lo:hi] = 1.0
    opts = dict(scheme="pg", order=order, n_a=n_a, mg_iters=cycles, bootstrap_cycles=0)
    return ProblemData(name, nx, nx, 1.0 / nx, 1.0 / nx, region, mats, src, 1,
                       options=opts)


def c2(nx=128, blocks=8, n_a=8, cycles=20, seed=0):
    """1 group, quadratic PG, 128^2, 512 ordinates, 8x8 seeded blocks."""
    return hetero_blocks(nx, blocks, n_a, 2, cycles, seed, "c2")


def c4(nx=512, blocks=32, n_a=16, cycles=20, seed=0):
    """1 group, cubic PG, 512^2, 2048 ordinates, 32x32 seeded blocks."""
    return hetero_blocks(nx, blocks, n_a, 3, cycles, seed, "c4")


# ---------------------------------------------------------------- C3 / C5
PIN_PITCH = 1.26
PIN_RADIUS = 0.4095

# R/data/synthetic_2group.csv:5-17 (group 1 fast, 2 thermal; 1->2 downscatter)
SYNTHETIC_2GROUP = {
    "fuel": dict(sigma_a=[0.15, 1.2], nsf=[0.02, 0.24], sf=[0.0081633, 0.0979592],
                 chi=[1.0, 0.0], s12=0.05),
    "moderator": dict(sigma_a=[0.01, 0.06], s12=1.0),
    "guide": dict(sigma_a=[0.005, 0.03], s12=0.9),
    "control": dict(sigma_a=[0.05, 2.5], s12=0.3),
}


def two_group_material(name):
    d = SYNTHETIC_2GROUP[name]
    ss = np.array([[0.0, d["s12"]], [0.0, 0.0]])
    return _mat(name, d["sigma_a"], ss, d.get("nsf"), d.get("sf"), d.get("chi"))


def pin_mask(cells_per_pin, radius_cells):
    """Cell-centre disc rasteriser (R/problems.py:108-112)."""
    c = (np.arange(cells_per_pin) + 0.5) - cells_per_pin / 2
    xx, yy = np.meshgrid(c, c, indexing="ij")
    return xx ** 2 + yy ** 2 <= radius_cells ** 2


def pin_lattice(n_pins, cells_per_pin, seed=0, p=(0.1, 0.8, 0.1)):
    """Region map: per pin a kind in {moderator-only, fuel, control}.

    ids: 0 moderator, 1 fuel, 2 control; the pin disc (radius 0.4095 cm at
    pitch 1.26 cm) takes the pin's kind, the rest is moderator.
    """
    rng = np.random.default_rng(seed)
    kinds = rng.choice(3, size=(n_pins, n_pins), p=list(p))
    dx = PIN_PITCH / cells_per_pin
    mask = pin_mask(cells_per_pin, PIN_RADIUS / dx)
    n = n_pins * cells_per_pin
    region = np.zeros((n, n), dtype=np.int64)
    for pi in range(n_pins):
        for pj in range(n_pins):
            blk = region[pi * cells_per_pin:(pi + 1) * cells_per_pin,
                         pj * cells_per_pin:(pj + 1) * cells_per_pin]
            blk[mask] = kinds[pi, pj]
    return region, dx


def c3(n_pins=16, cells_per_pin=16, n_a=8, outers=30, inner=5, seed=0):
    """2-group k-eigenvalue, linear PG, 16x16 seeded pin lattice, 256^2 cells."""
    region, dx = pin_lattice(n_pins, cells_per_pin, seed)
    mats = [two_group_material("moderator"), two_group_material("fuel"),
            two_group_material("control")]
    n = region.shape[0]
    opts = dict(scheme="pg", order=1, n_a=n_a, outer_iters=outers, bootstrap_cycles=0)
    return ProblemData("c3", n, n, dx, dx, region, mats, None, 2,
                       driver="power_iteration", options=opts, inner_iters=inner)


def seven_group_library(seed=0, groups=7, n_fast=3):
    """Seeded synthetic 7-group set mapped to the reference's 4-pi convention.

    Physical draws per material (moderator, fuel, control): sigma_t per group,
    scattering ratio c_g < 1, a scatter shape with a full lower-triangular
    downscatter block (g -> g' >= g) plus thermal upscatter (g' < g, both
    thermal), rows rescaled to sum to c_g sigma_t,g; fission on fast chi for
    fuel.  Mapping: sigma_s' = sigma_s / 4pi,
    nu_sigma_f' = nu_sigma_f / 4pi, sigma_f' = sigma_f / 4pi, sigma_a' =
    sigma_a + sum_{g' != g} sigma_s[g, g'] (1 - 1/4pi), which keeps the
    reference removal sigma_t - sigma_s,gg unchanged.
    """
    rng = np.random.default_rng(seed + 7000)
    G = groups
    ranges = {  # (fast sigma_t, thermal sigma_t, c range)
        "moderator": ((0.3, 0.7), (1.0, 2.5), (0.90, 0.99)),
        "fuel": ((0.2, 0.6), (0.5, 1.5), (0.50, 0.80)),
        "control": ((0.3, 0.8), (1.5, 4.0), (0.20, 0.50)),
    }
    out = []
    for name in ("moderator", "fuel", "control"):
        fr, tr, cr = ranges[name]
        st = np.concatenate([rng.uniform(*fr, size=n_fast), rng.uniform(*tr, size=G - n_fast)])
        c = rng.uniform(*cr, size=G)
        shape = np.zeros((G, G))
        for g in range(G):
            shape[g, g:] = rng.uniform(0.05, 1.0, size=G - g)
            if g > n_fast:
                shape[g, n_fast:g] = rng.uniform(0.0, 0.1, size=g - n_fast)
        ss = shape * (c * st / shape.sum(axis=1))[:, None]
        sa = st - ss.sum(axis=1)
        nsf = np.zeros(G)
        sf = np.zeros(G)
        chi = np.zeros(G)
        if name == "fuel":
            nsf = np.concatenate([rng.uniform(0.005, 0.02, size=n_fast),
                                  rng.uniform(0.05, 0.3, size=G - n_fast)])
            sf = nsf / 2.43
            chi[:n_fast] = rng.uniform(0.2, 1.0, size=n_fast)
            chi /= chi.sum()
        off = ss.sum(axis=1) - np.diag(ss)
        out.append(_mat(name, sa + off * (1.0 - 1.0 / FOUR_PI), ss / FOUR_PI,
                        nsf / FOUR_PI, sf / FOUR_PI, chi))
    return out


def c5(n_pins=64, cells_per_pin=16, n_a=16, outers=10, inner=3, seed=0, groups=7):
    """7-group k-eigenvalue, linear PG, 64x64 seeded pin lattice, 1024^2 cells.

    The weak-scaling variant is ``c5(n_pins=32 * P, ...)`` with 512 x 512 per GPU
    (use :func:`c5_weak`).
    """
    region, dx = pin_lattice(n_pins, cells_per_pin, seed)
    mats = seven_group_library(seed, groups)
    n = region.shape[0]
    opts = dict(scheme="pg", order=1, n_a=n_a, outer_iters=outers, bootstrap_cycles=0)
    return ProblemData("c5", n, n, dx, dx, region, mats, None, groups,
                       driver="power_iteration", options=opts, inner_iters=inner)


def c5_weak(world=1, n_a=16, outers=10, inner=3, seed=0, groups=7, cells_per_pin=16):
    """512 x 512 cells per GPU, stacked along x: (512 P) x 512."""
    per = 512 // cells_per_pin
    region_full, dx = pin_lattice(per * world, cells_per_pin, seed)
    region = region_full[:, :512]
    mats = seven_group_library(seed, groups)
    opts = dict(scheme="pg", order=1, n_a=n_a, outer_iters=outers, bootstrap_cycles=0)
    return ProblemData("c5_weak", region.shape[0], region.shape[1], dx, dx,
                       np.ascontiguousarray(region), mats, None, groups,
                       driver="power_iteration", options=opts, inner_iters=inner)


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}
