"""Octahedral discrete-ordinates quadrature (host setup, float64).

Same ordinate set as R/quadrature.py:112-176: eight octahedron faces, each an
``n_a x n_a`` grid of planar patches projected radially onto the unit sphere;
weight = spherical patch area, direction = patch mean of the unit vector, both in
closed form (spherical-triangle solid angles; half the arc-angle-weighted sum of
great-circle axes for the moment).  Storage is face-major, then row (equator ->
pole), then column, so 2x2 angle coarsening is a reshape.  Computed here for all
patches at once (vectorised over the patch axis) and uploaded once per level.
"""

from dataclasses import dataclass

import functools

import numpy as np

FOUR_PI = 4.0 * np.pi
N_FACES = 8
OCTANT_SIGNS = ((1, 1, 1), (-1, 1, 1), (-1, -1, 1), (1, -1, 1),
                (1, 1, -1), (-1, 1, -1), (-1, -1, -1), (1, -1, -1))


@dataclass(frozen=True, eq=False)
class AngularQuadrature:
    """Ordinate set: mean directions, patch weights and face membership."""

    n_a: int
    directions: np.ndarray   # (n_dir, 3): mu, nu, xi
    weights: np.ndarray      # (n_dir,), sum 4 pi
    face_index: np.ndarray   # (n_dir,)
    n_faces_: int = N_FACES  # 8, or 4 for the z-folded upper hemisphere (fold_z)

    def __post_init__(self):
        for arr in (self.directions, self.weights, self.face_index):
            arr.setflags(write=False)

    @property
    def n_faces(self):
        return self.n_faces_

    @property
    def folded(self):
        return self.n_faces_ != N_FACES

    @property
    def n_dir(self):
        return self.weights.shape[0]

    @property
    def mu(self):
        return self.directions[:, 0]

    @property
    def nu(self):
        return self.directions[:, 1]

    @property
    def xi(self):
        return self.directions[:, 2]

    def device(self, dtype, device, dx=None, dy=None):
        """Cached device copies: mu, nu, w (and |mu|/dx + |nu|/dy when dx, dy given)."""
        import torch
        cache = self.__dict__.setdefault("_dev", {})
        key = (str(dtype), str(device), dx, dy)
        if key not in cache:
            rows = [self.mu, self.nu, self.weights]
            if dx is not None:
                rows.append(np.abs(self.mu) / dx + np.abs(self.nu) / dy)
            # one upload per level (the rows are contiguous views of it)
            t = torch.tensor(np.stack([np.asarray(r, dtype=np.float64) for r in rows]),
                             dtype=dtype, device=device)
            d = dict(zip(("mu", "nu", "w", "strm"), t.unbind(0)))
            cache[key] = d
        return cache[key]


def _cross(a, b):
    return np.cross(a, b)


def _dot(a, b):
    return np.einsum("...i,...i->...", a, b)


def _patch_area_moment(p):
    """Area and moment of spherical quads p[k, 4, 3] (unit corners, cyclic order).

    Degenerate (pole) edges have zero length and drop out of both sums.
    """
    a, b, c, d = p[:, 0], p[:, 1], p[:, 2], p[:, 3]

    def tri(u, v, w):
        num = np.abs(_dot(u, _cross(v, w)))
        den = 1.0 + _dot(u, v) + _dot(v, w) + _dot(w, u)
        return 2.0 * np.arctan2(num, den)

    area = tri(a, b, c) + tri(a, c, d)
    mom = np.zeros_like(a)
    for u, v in ((a, b), (b, c), (c, d), (d, a)):
        ax = _cross(u, v)
        s = np.linalg.norm(ax, axis=1)
        ok = s >= 1e-15
        ang = np.arctan2(s, _dot(u, v))
        mom[ok] += (ang[ok] / s[ok])[:, None] * ax[ok]
    mom *= 0.5
    flip = _dot(mom, p.mean(axis=1)) < 0.0
    mom[flip] = -mom[flip]
    return area, mom


def build_quadrature(n_a):
    """``8 n_a^2`` ordinates with weights rescaled to sum to 4 pi (R/quadrature.py:112-151).

    The set depends on n_a alone and its arrays are read-only, so it is built once per
    n_a (and with it its coarsened chain and the device copies cached on the objects)."""
    if not isinstance(n_a, (int, np.integer)) or n_a < 1 or (n_a & (n_a - 1)) != 0:
        raise ValueError(f"n_a must be a positive power of 2, got {n_a!r}")
    return _build_quadrature(int(n_a))


@functools.lru_cache(maxsize=16)
def _build_quadrature(n_a):
    k = np.arange(n_a, dtype=float)
    t0, t1 = k / n_a, (k + 1) / n_a          # rows towards the pole
    s0, s1 = k / n_a, (k + 1) / n_a          # columns along the equator edge
    dirs = []
    for sx, sy, sz in OCTANT_SIGNS:
        va = np.array([sx, 0.0, 0.0])
        vb = np.array([0.0, sy, 0.0])
        vp = np.array([0.0, 0.0, sz])

        def pt(s, t):
            s = s[None, :, None]
            t = t[:, None, None]
            return (1.0 - t) * ((1.0 - s) * va + s * vb) + t * vp

        corners = np.stack([pt(s0, t0), pt(s1, t0), pt(s1, t1), pt(s0, t1)], axis=2)
        corners = corners.reshape(n_a * n_a, 4, 3)
        dirs.append(corners / np.linalg.norm(corners, axis=2, keepdims=True))
    # every face's patches in one elementwise pass (face-major order kept)
    weights, mom = _patch_area_moment(np.concatenate(dirs))
    directions = mom / weights[:, None]
    weights = weights * (FOUR_PI / weights.sum())
    return AngularQuadrature(n_a=n_a, directions=directions, weights=weights,
                             face_index=np.repeat(np.arange(N_FACES), n_a * n_a))


def coarsen_quadrature(quad):
    """Merge 2x2 patch blocks per face: weights add, directions weight-average."""
    if quad.n_a < 2:
        raise ValueError("cannot coarsen: already at one patch per face")
    memo = quad.__dict__.get("_coarse")          # the arrays are read-only: coarsen once
    if memo is not None:
        return memo
    m = quad.n_a // 2
    nf = quad.n_faces
    w = quad.weights.reshape(nf, m, 2, m, 2)
    d = quad.directions.reshape(nf, m, 2, m, 2, 3)
    wc = w.sum(axis=(2, 4))
    dc = (d * w[..., None]).sum(axis=(2, 4)) / wc[..., None]
    out = AngularQuadrature(n_a=m, directions=dc.reshape(-1, 3), weights=wc.reshape(-1),
                            face_index=np.repeat(np.arange(nf), m * m), n_faces_=nf)
    quad.__dict__["_coarse"] = out
    return out


def fold_z(quad):
    """Exact z-mirror fold of a 2D problem: faces 4-7 are the
    xi -> -xi mirrors of faces 0-3 with identical (mu, nu, w) (R/quadrature.py:28-31),
    and nothing in an x-y problem depends on xi, so psi stays mirror-symmetric through
    every operator.  Carrying faces 0-3 with doubled weights gives the same scalar
    flux with half the DOF.  Face-major storage keeps 2x2 coarsening a reshape."""
    if quad.folded:
        raise ValueError("quadrature is already folded")
    half = quad.n_dir // 2
    lo, hi = quad.directions[:half], quad.directions[half:]
    if not (np.array_equal(lo[:, :2], hi[:, :2]) and np.array_equal(lo[:, 2], -hi[:, 2])
            and np.array_equal(quad.weights[:half], quad.weights[half:])):
        raise ValueError("quadrature is not z-mirror symmetric")
    return AngularQuadrature(n_a=quad.n_a, directions=lo.copy(),
                             weights=2.0 * quad.weights[:half],
                             face_index=quad.face_index[:half].copy(), n_faces_=N_FACES // 2)


def quadrature_to_csv(quad, stream):
    stream.write("mu,nu,xi,weight,face\n")
    for (mu, nu, xi), w, f in zip(quad.directions, quad.weights, quad.face_index):
        stream.write(f"{mu:.17g},{nu:.17g},{xi:.17g},{w:.17g},{int(f)}\n")
