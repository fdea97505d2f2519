"""Float64 NumPy restatement of the reference sawtooth multigrid (TEST ORACLE ONLY).

Written from the reference's behaviour, not copied: plain arrays in, plain
arrays out, one function per reference operation, each citing the file:line
it restates.  ``R`` below abbreviates ``/root/reference/pkg/src/convsn/``.

Storage convention (R/grid.py:1-7,47-59): a field is a float64 array
``[nx + 2h, ny + 2h, n_dir, n_group]``, x slowest, interior at ``[h:h+nx,
h:h+ny]``.  Parity status: pinned against the reference's own outputs stored
in ``tests/golden/`` (see ``tests/test_oracle_golden.py``).
"""

import math
from types import SimpleNamespace

import numpy as np

FOUR_PI = 4.0 * math.pi
N_FACES = 8
# R/quadrature.py:28-31 — one (sx, sy, sz) sign triple per octahedron face
FACE_SIGNS = ((1, 1, 1), (-1, 1, 1), (-1, -1, 1), (1, -1, 1),
              (1, 1, -1), (-1, 1, -1), (-1, -1, -1), (1, -1, -1))

# R/multigrid.py:179-182 — diffusivity Picard freeze heuristics
STALL_WINDOW = 5
STALL_FACTOR = 0.9
UNFREEZE_GROWTH = 2.0
MAX_FREEZE_ATTEMPTS = 3


# --------------------------------------------------------------------------
# angular quadrature  (R/quadrature.py:68-176)
# --------------------------------------------------------------------------

def _unit(v):
    return v / np.linalg.norm(v)


def _spherical_patch(corners):
    """Area and vector moment of a radially projected planar polygon.

    R/quadrature.py:68-109: fan of spherical triangles (solid angle
    2*atan2(|a.(b x c)|, 1 + a.b + b.c + c.a)) for the area; half the sum of
    arc angle times great-circle axis over the boundary for the moment.
    Consecutive duplicate corners (the collapsed pole edge) are dropped.
    """
    pts = []
    for c in corners:
        u = _unit(np.asarray(c, dtype=float))
        if not pts or np.linalg.norm(u - pts[-1]) > 1e-14:
            pts.append(u)
    if len(pts) > 1 and np.linalg.norm(pts[0] - pts[-1]) < 1e-14:
        pts.pop()
    if len(pts) < 3:
        raise ValueError("degenerate patch with no area")
    area = 0.0
    a = pts[0]
    for b, c in zip(pts[1:-1], pts[2:]):
        triple = abs(np.dot(a, np.cross(b, c)))
        area += 2.0 * np.arctan2(triple, 1.0 + a @ b + b @ c + c @ a)
    mom = np.zeros(3)
    for k, p0 in enumerate(pts):
        p1 = pts[(k + 1) % len(pts)]
        axis = np.cross(p0, p1)
        s = np.linalg.norm(axis)
        if s < 1e-15:
            continue
        mom += np.arctan2(s, p0 @ p1) * (axis / s)
    mom *= 0.5
    if mom @ np.mean(pts, axis=0) < 0.0:
        mom = -mom
    return area, mom


def build_quadrature(n_a):
    """Octahedral ordinates, ``8 n_a^2`` directions (R/quadrature.py:112-151).

    Face-major, then row (equator -> pole) major, then column.  Weights are
    rescaled to sum to exactly 4 pi.
    """
    if n_a < 1 or (n_a & (n_a - 1)):
        raise ValueError("n_a must be a positive power of 2")
    nd = N_FACES * n_a * n_a
    dirs = np.empty((nd, 3))
    w = np.empty(nd)
    k = 0
    for sx, sy, sz in FACE_SIGNS:
        va, vb, vp = (np.array([sx, 0.0, 0.0]), np.array([0.0, sy, 0.0]),
                      np.array([0.0, 0.0, sz]))

        def at(s, t):
            return (1.0 - t) * ((1.0 - s) * va + s * vb) + t * vp

        for r in range(n_a):
            t0, t1 = r / n_a, (r + 1) / n_a
            for c in range(n_a):
                s0, s1 = c / n_a, (c + 1) / n_a
                area, mom = _spherical_patch(
                    (at(s0, t0), at(s1, t0), at(s1, t1), at(s0, t1)))
                w[k] = area
                dirs[k] = mom / area
                k += 1
    w *= FOUR_PI / w.sum()
    return SimpleNamespace(n_a=n_a, n_dir=nd, mu=dirs[:, 0].copy(),
                           nu=dirs[:, 1].copy(), xi=dirs[:, 2].copy(),
                           directions=dirs, weights=w,
                           face=np.repeat(np.arange(N_FACES), n_a * n_a))


def coarsen_quadrature(q):
    """Merge 2x2 patch blocks per face (R/quadrature.py:154-176)."""
    if q.n_a < 2:
        raise ValueError("cannot coarsen below one patch per face")
    m = q.n_a // 2
    w = q.weights.reshape(N_FACES, m, 2, m, 2)
    d = q.directions.reshape(N_FACES, m, 2, m, 2, 3)
    wc = w.sum(axis=(2, 4))
    dc = (d * w[..., None]).sum(axis=(2, 4)) / wc[..., None]
    dirs = dc.reshape(-1, 3)
    return SimpleNamespace(n_a=m, n_dir=N_FACES * m * m, mu=dirs[:, 0].copy(),
                           nu=dirs[:, 1].copy(), xi=dirs[:, 2].copy(),
                           directions=dirs, weights=wc.reshape(-1),
                           face=np.repeat(np.arange(N_FACES), m * m))


# --------------------------------------------------------------------------
# ConvFEM 1D stencils  (R/filters.py:36-106)
# --------------------------------------------------------------------------

def _lagrange(nodes, x):
    n = len(nodes)
    val = np.ones((n, x.size))
    der = np.zeros((n, x.size))
    for k in range(n):
        others = [m for m in range(n) if m != k]
        for m in others:
            val[k] *= (x - nodes[m]) / (nodes[k] - nodes[m])
        for m in others:
            term = np.ones_like(x) / (nodes[k] - nodes[m])
            for j in others:
                if j != m:
                    term *= (x - nodes[j]) / (nodes[k] - nodes[j])
            der[k] += term
    return val, der


def stencils_1d(p):
    """(mass, grad, stiff) unit-spacing taps, length 2p+1 (R/filters.py:59-106).

    Order-p Lagrange element on nodes 0..p, exact Gauss-Legendre (p+2 pts);
    the p distinct interior nodal rows (vertex row + p-1 element-interior
    rows) are averaged and divided by the mean nodal mass.
    """
    if p < 1:
        raise ValueError("element order must be >= 1")
    nodes = np.arange(p + 1, dtype=float)
    gx, gw = np.polynomial.legendre.leggauss(p + 2)
    x = 0.5 * p * (gx + 1.0)
    wq = 0.5 * p * gw
    v, d = _lagrange(nodes, x)
    elems = (np.einsum("iq,jq,q->ij", v, v, wq),
             np.einsum("iq,jq,q->ij", v, d, wq),
             np.einsum("iq,jq,q->ij", d, d, wq))

    def rows(e):
        out = np.zeros((p, 2 * p + 1))
        out[0, 0:p + 1] += e[p, :]
        out[0, p:] += e[0, :]
        for m in range(1, p):
            out[m, p - m:2 * p - m + 1] = e[m, :]
        return out

    mrows = rows(elems[0])
    mean_mass = mrows.sum() / p
    return tuple(rows(e).mean(axis=0) / mean_mass for e in elems)


# --------------------------------------------------------------------------
# boundary, stencil passes, scalar flux  (R/grid.py)
# --------------------------------------------------------------------------

def apply_boundary(data, h, mu, nu):
    """In-place vacuum halo fill (R/grid.py:165-190), stateless form.

    Halo value = 0 if any out-of-range side is one the direction enters
    through (west if mu > 0, east if mu <= 0, south if nu > 0, north if
    nu <= 0), else the nearest interior value psi[clamp(i), clamp(j)].  This
    equals the reference's x-then-y sequential fill, corners included.
    """
    nx, ny = data.shape[0] - 2 * h, data.shape[1] - 2 * h
    xs = np.arange(-h, nx + h)
    ys = np.arange(-h, ny + h)
    src = data[h + np.clip(xs, 0, nx - 1)][:, h + np.clip(ys, 0, ny - 1)]
    mpos = (mu > 0.0)[None, None, :, None]
    npos = (nu > 0.0)[None, None, :, None]
    west = (xs < 0)[:, None, None, None]
    east = (xs >= nx)[:, None, None, None]
    south = (ys < 0)[None, :, None, None]
    north = (ys >= ny)[None, :, None, None]
    zero = (west & mpos) | (east & ~mpos) | (south & npos) | (north & ~npos)
    data[...] = np.where(zero, 0.0, src)
    return data


def pass1d(src, taps, axis, h, margin=0):
    """One 1D correlation pass (R/grid.py:108-125).

    out = sum_a taps[a] * src[shift a - l] on (interior +- margin) along
    ``axis``, full extent along the other axis, zeros elsewhere; taps equal
    to exactly 0.0 are skipped; accumulation order tap 0 -> 2l.
    """
    taps = np.asarray(taps)
    l = (len(taps) - 1) // 2
    if margin + l > h:
        raise ValueError("1D stencil does not fit in the halo")
    n = src.shape[axis] - 2 * (h - margin)
    out = np.zeros_like(src)
    lo = h - margin
    dst = [slice(None)] * src.ndim
    dst[axis] = slice(lo, lo + n)
    acc = out[tuple(dst)]
    for a, c in enumerate(taps):
        if c == 0.0:
            continue
        sl = [slice(None)] * src.ndim
        sl[axis] = slice(lo + a - l, lo + a - l + n)
        acc += c * src[tuple(sl)]
    return out


def sep(src, tx, ty, h, margin=0):
    """x pass then y pass (R/grid.py:128-136)."""
    return pass1d(pass1d(src, tx, 0, h, margin), ty, 1, h, margin)


def convolve2d(data, stencil, h, margin=0, direction_scale=None):
    """Generic square-stencil correlation (R/grid.py:85-105,139-152)."""
    w = np.asarray(stencil)
    l = (w.shape[0] - 1) // 2
    if margin + l > h:
        raise ValueError("stencil does not fit in the halo")
    nxs = data.shape[0] - 2 * (h - margin)
    nys = data.shape[1] - 2 * (h - margin)
    out = np.zeros_like(data)
    o = h - margin
    acc = out[o:o + nxs, o:o + nys]
    for a in range(w.shape[0]):
        for b in range(w.shape[1]):
            if w[a, b] == 0.0:
                continue
            acc += w[a, b] * data[o + a - l:o + a - l + nxs,
                                  o + b - l:o + b - l + nys]
    if direction_scale is not None:
        out *= np.asarray(direction_scale).reshape(1, 1, -1, 1)
    return out


def interior(data, h):
    return data[h:data.shape[0] - h, h:data.shape[1] - h]


def scalar_flux(data, h, weights):
    """phi[i,j,g] = sum_n p_n psi[i,j,n,g] (R/grid.py:193-198)."""
    return np.einsum("xyng,n->xyg", interior(data, h), weights)


# --------------------------------------------------------------------------
# discrete operators  (R/discretisation.py)
# --------------------------------------------------------------------------

PG_DEFAULTS = dict(epsilon_k=1.0e-3, alpha_r=3.0, beta_r=3.0, beta_diag=3.0,
                   k_freeze_rel=0.05)   # R/discretisation.py:48-52


def pg_config(**kw):
    cfg = dict(PG_DEFAULTS)
    cfg.update(kw)
    return SimpleNamespace(**cfg)


def alpha_kabs(order):
    return 2.0 ** order / 16.0        # R/discretisation.py:54-55


def alpha_ksq(order):
    return 2.0 ** order / 2.0         # R/discretisation.py:57-58


def _d4(v):
    return np.asarray(v).reshape(1, 1, -1, 1)


def upwind_residual(data, h, sigma, q, mu, nu, dx, dy):
    """Upwind streaming + removal residual, interior only (R/discretisation.py:65-94)."""
    nx, ny = data.shape[0] - 2 * h, data.shape[1] - 2 * h
    c = data[h:h + nx, h:h + ny]
    w = data[h - 1:h - 1 + nx, h:h + ny]
    e = data[h + 1:h + 1 + nx, h:h + ny]
    s = data[h:h + nx, h - 1:h - 1 + ny]
    n = data[h:h + nx, h + 1:h + 1 + ny]
    ddx = np.where(_d4(mu > 0.0), c - w, e - c) / dx
    ddy = np.where(_d4(nu > 0.0), c - s, n - c) / dy
    return _d4(mu) * ddx + _d4(nu) * ddy + sigma[:, :, None, :] * c - q


def stream_diag(mu, nu, dx, dy, sigma):
    """|mu|/dx + |nu|/dy + sigma_t (R/discretisation.py:97-111, beta = 1)."""
    stream = np.abs(mu) / dx + np.abs(nu) / dy
    return 1.0 * (_d4(stream) + sigma[:, :, None, :])


def grad_fields(data, h, taps, dx, dy):
    """psi_x = M_y G_x psi / dx, psi_y = G_y M_x psi / dy on +-2l (R/discretisation.py:114-122)."""
    mass, grad, _ = taps
    l = (len(mass) - 1) // 2
    return (sep(data, grad / dx, mass, h, 2 * l),
            sep(data, mass, grad / dy, h, 2 * l))


def diffusivities(data, h, taps, order, dx, dy, mu, nu, cfg, grads=None):
    """Anisotropic PG diffusivities k_x, k_y (R/discretisation.py:125-161)."""
    mass = taps[0]
    l = (len(mass) - 1) // 2
    if h < 3 * l:
        raise ValueError(f"PG diffusivities need halo >= {3 * l}")
    px, py = grads if grads is not None else grad_fields(data, h, taps, dx, dy)
    amu, anu = _d4(np.abs(mu)), _d4(np.abs(nu))
    eps, ka, ks = cfg.epsilon_k, alpha_kabs(order), alpha_ksq(order)
    rx = cfg.alpha_r * _d4(mu) * (sep(px, mass, mass, h, l) - px)
    ry = cfg.alpha_r * _d4(nu) * (sep(py, mass, mass, h, l) - py)
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        kx = np.minimum(dx * amu, np.minimum(ka * np.abs(rx) * dx / (eps + np.abs(px)),
                                             ks * rx ** 2 * dx / (eps + amu * px ** 2)))
        ky = np.minimum(dy * anu, np.minimum(ka * np.abs(ry) * dy / (eps + np.abs(py)),
                                             ks * ry ** 2 * dy / (eps + anu * py ** 2)))
    kx = np.nan_to_num(kx, nan=0.0, posinf=0.0, neginf=0.0)
    ky = np.nan_to_num(ky, nan=0.0, posinf=0.0, neginf=0.0)
    return kx, ky


def iso_diffusivity(data, h, taps, order, dx, dy, mu, nu, cfg, mode="mixed_mass",
                    grads=None):
    """Isotropic legacy diffusivity (R/discretisation.py:164-185)."""
    px, py = grads if grads is not None else grad_fields(data, h, taps, dx, dy)
    r = residual_estimate(data, h, taps, order, dx, dy, mu, nu, cfg, mode, (px, py))
    m4, n4 = _d4(mu), _d4(nu)
    eps = cfg.epsilon_k
    hh = 0.5 * (dx + dy)
    k_abs = alpha_kabs(order) * np.abs(r) * hh / (eps + 0.5 * (np.abs(px) + np.abs(py)))
    ratio = (m4 * px + n4 * py) / (eps + px ** 2 + py ** 2)
    k_sq = (alpha_ksq(order) * r ** 2 * hh
            / (eps + 0.5 * (np.abs(ratio * px) + np.abs(ratio * py)) * (px ** 2 + py ** 2)))
    k_max = np.sqrt((dx * m4) ** 2 + (dy * n4) ** 2)
    return np.minimum(k_max, np.minimum(k_abs, k_sq))


def residual_estimate(data, h, taps, order, dx, dy, mu, nu, cfg, mode="mixed_mass",
                      grads=None):
    """Equation-residual estimate (R/discretisation.py:188-224)."""
    mass = taps[0]
    l = (len(mass) - 1) // 2
    px, py = grads if grads is not None else grad_fields(data, h, taps, dx, dy)
    adv = _d4(mu) * px + _d4(nu) * py
    if mode == "mixed_mass":
        return cfg.beta_r * (sep(adv, mass, mass, h, l) - adv)
    if mode == "low_order":
        if order - 1 < 1:
            raise ValueError("low_order residual needs filter order >= 2")
        other = order - 1
    elif mode == "high_order":
        other = order + 1
    else:
        raise ValueError(f"unknown residual mode {mode!r}")
    mo, go, _ = stencils_1d(other)
    margin = min(l, h - other)
    if margin < 0:
        raise ValueError("field halo too small for the comparison order")
    ox = sep(data, go / dx, mo, h, margin)
    oy = sep(data, mo, go / dy, h, margin)
    adv_o = _d4(mu) * ox + _d4(nu) * oy
    return adv - adv_o if mode == "low_order" else adv_o - adv


def k_diffusion(arr, k, sx, sy, h):
    """1/2 [S(k a) + k S(a) - a S(k)] (R/discretisation.py:227-236)."""
    t1 = sep(arr * k, sx, sy, h, 0)
    t2 = k * sep(arr, sx, sy, h, 0)
    t3 = arr * sep(k, sx, sy, h, 0)
    return 0.5 * (t1 + t2 - t3)


def pg_residual(data, h, sigma, q, taps, order, dx, dy, mu, nu, cfg, kxy=None,
                anisotropy="xy"):
    """PG residual, interior only (R/discretisation.py:239-276)."""
    mass, _, stiff = taps
    grads = grad_fields(data, h, taps, dx, dy)
    if kxy is not None:
        kx, ky = kxy
    elif anisotropy == "xy":
        kx, ky = diffusivities(data, h, taps, order, dx, dy, mu, nu, cfg, grads)
    elif anisotropy == "iso":
        kx = ky = iso_diffusivity(data, h, taps, order, dx, dy, mu, nu, cfg, grads=grads)
    else:
        raise ValueError(f"unknown anisotropy setting {anisotropy!r}")
    dxx = k_diffusion(data, kx, stiff / dx ** 2, mass, h)
    dyy = k_diffusion(data, ky, mass, stiff / dy ** 2, h)
    px, py = grads
    nx, ny = data.shape[0] - 2 * h, data.shape[1] - 2 * h
    sl = (slice(h, h + nx), slice(h, h + ny))
    return (_d4(mu) * px[sl] + _d4(nu) * py[sl] + dxx[sl] + dyy[sl]
            + sigma[:, :, None, :] * data[sl] - q)


# --------------------------------------------------------------------------
# hierarchy, transfers, smoothing  (R/multigrid.py)
# --------------------------------------------------------------------------

def max_levels(nx, ny):
    """R/multigrid.py:60-67."""
    n = 1
    while nx % 2 == 0 and ny % 2 == 0 and nx > 1 and ny > 1:
        nx //= 2
        ny //= 2
        n += 1
    return n


def coarsen_sigma(sig, eps=1e-30):
    """Harmonic 2x2 average, zero child => zero parent (R/multigrid.py:70-77)."""
    nx, ny, ng = sig.shape
    b = sig.reshape(nx // 2, 2, ny // 2, 2, ng)
    out = 4.0 / (1.0 / np.maximum(b, eps)).sum(axis=(1, 3))
    out[(b == 0.0).any(axis=(1, 3))] = 0.0
    return out


def build_hierarchy(nx, ny, dx, dy, h, quad, sigma, n_levels=None):
    """List of levels, finest first (R/multigrid.py:80-107)."""
    if n_levels is None:
        n_levels = max_levels(nx, ny)
    if n_levels < 1:
        raise ValueError("hierarchy needs at least one level")
    if nx % 2 ** (n_levels - 1) or ny % 2 ** (n_levels - 1):
        raise ValueError("grid not divisible by 2**(n_levels-1)")
    levels = []
    for i in range(n_levels):
        levels.append(SimpleNamespace(nx=nx, ny=ny, dx=dx, dy=dy, h=h, quad=quad,
                                      sigma=sigma,
                                      diag=stream_diag(quad.mu, quad.nu, dx, dy, sigma)))
        if i == n_levels - 1:
            break
        sigma = coarsen_sigma(sigma)
        nx, ny, dx, dy = nx // 2, ny // 2, 2 * dx, 2 * dy
        if quad.n_a > 1:
            quad = coarsen_quadrature(quad)
    return levels


def restrict_raw(arr, fine, coarse):
    """Integrated 2x2 (x 2x2 patch) restriction (R/multigrid.py:342-353)."""
    ng = arr.shape[3]
    fq, cq = fine.quad, coarse.quad
    mod = arr * _d4(fq.weights) * (fine.dx * fine.dy)
    mod = mod.reshape(coarse.nx, 2, coarse.ny, 2, fq.n_dir, ng).sum(axis=(1, 3))
    if cq.n_a != fq.n_a:
        m = fq.n_a // 2
        mod = mod.reshape(coarse.nx, coarse.ny, N_FACES, m, 2, m, 2, ng)
        mod = mod.sum(axis=(4, 6)).reshape(coarse.nx, coarse.ny, cq.n_dir, ng)
    return mod


def prolong(arr, coarse, fine):
    """Piecewise-constant injection of a coarse interior (R/multigrid.py:130-146)."""
    ng = arr.shape[3]
    if fine.quad.n_a != coarse.quad.n_a:
        na = coarse.quad.n_a
        arr = arr.reshape(coarse.nx, coarse.ny, N_FACES, na, na, ng)
        arr = np.repeat(np.repeat(arr, 2, axis=3), 2, axis=4)
        arr = arr.reshape(coarse.nx, coarse.ny, fine.quad.n_dir, ng)
    return np.repeat(np.repeat(arr, 2, axis=0), 2, axis=1)


def padded(nx, ny, h, nd, ng, inner=None):
    out = np.zeros((nx + 2 * h, ny + 2 * h, nd, ng))
    if inner is not None:
        out[h:h + nx, h:h + ny] = inner
    return out


def jacobi_upwind(data, q, lev, n_sweeps, diag_scale=1.0):
    """n upwind Jacobi sweeps, boundary before each (R/multigrid.py:149-173)."""
    d = diag_scale * lev.diag if diag_scale != 1.0 else lev.diag
    h = lev.h
    for _ in range(n_sweeps):
        apply_boundary(data, h, lev.quad.mu, lev.quad.nu)
        r = upwind_residual(data, h, lev.sigma, q, lev.quad.mu, lev.quad.nu,
                            lev.dx, lev.dy)
        data[h:h + lev.nx, h:h + lev.ny] -= r / d
    return data


def jacobi_pg(data, q, lev, taps, order, cfg, kxy, n_sweeps=1):
    """PG Jacobi sweeps with the beta_diag-enlarged diagonal (R/multigrid.py:159-172)."""
    d = cfg.beta_diag * lev.diag
    h = lev.h
    for _ in range(n_sweeps):
        apply_boundary(data, h, lev.quad.mu, lev.quad.nu)
        r = pg_residual(data, h, lev.sigma, q, taps, order, lev.dx, lev.dy,
                        lev.quad.mu, lev.quad.nu, cfg, kxy=kxy)
        data[h:h + lev.nx, h:h + lev.ny] -= r / d
    return data


class PGState:
    """Picard diffusivity state (R/multigrid.py:185-256), with a decision log."""

    def __init__(self, avg_theta=0.2):
        self.kxy = None
        self.initial = None
        self.frozen = False
        self.best = None
        self.since_best = 0
        self.freeze_res = None
        self.failed = 0
        self.theta = avg_theta
        self.psi_avg = None
        self.log = []          # (observe call index, "freeze"|"unfreeze")
        self.calls = 0

    def averaged(self, data):
        if self.theta >= 1.0:
            return data
        if self.psi_avg is None:
            self.psi_avg = data.copy()
        else:
            self.psi_avg *= 1.0 - self.theta
            self.psi_avg += self.theta * data
        return self.psi_avg

    def observe(self, res, k_freeze_rel):
        self.calls += 1
        if self.initial is None:
            self.initial = self.best = res
            return
        if self.frozen:
            if res > UNFREEZE_GROWTH * self.freeze_res:
                self.frozen = False
                self.failed += 1
                self.best = res
                self.since_best = 0
                self.log.append((self.calls, "unfreeze"))
            return
        if self.failed >= MAX_FREEZE_ATTEMPTS:
            return
        if res <= k_freeze_rel * self.initial:
            self._freeze(res)
            return
        if res < STALL_FACTOR * self.best:
            self.best = res
            self.since_best = 0
        else:
            self.since_best += 1
            if self.since_best >= STALL_WINDOW:
                self._freeze(res)

    def _freeze(self, res):
        self.frozen = True
        self.freeze_res = res
        self.since_best = 0
        self.log.append((self.calls, "freeze"))


def mg_correction(r, levels, n_sweeps=3, finest_diag_scale=1.0):
    """Restrict down, smooth up with upwind Jacobi (R/multigrid.py:309-339)."""
    src = [r]
    for i in range(1, len(levels)):
        raw = restrict_raw(src[-1], levels[i - 1], levels[i])
        lev = levels[i]
        raw /= _d4(lev.quad.weights) * (lev.dx * lev.dy)
        src.append(raw)
    ng = r.shape[3]
    lev = levels[-1]
    delta = padded(lev.nx, lev.ny, lev.h, lev.quad.n_dir, ng)
    for i in range(len(levels) - 1, -1, -1):
        scale = finest_diag_scale if i == 0 else 1.0
        jacobi_upwind(delta, src[i], levels[i], n_sweeps, scale)
        if i > 0:
            f = levels[i - 1]
            delta = padded(f.nx, f.ny, f.h, f.quad.n_dir, ng,
                           prolong(interior(delta, levels[i].h), levels[i], f))
    return delta


def sawtooth_cycle(data, q, levels, taps=None, order=None, cfg=None, scheme="pg",
                   n_sweeps=3, pg_sweeps=1, pg_state=None):
    """One sawtooth cycle in place; returns float64 L1 of the pre-update residual.

    R/multigrid.py:259-306.
    """
    cfg = cfg or pg_config()
    f = levels[0]
    h, mu, nu = f.h, f.quad.mu, f.quad.nu
    apply_boundary(data, h, mu, nu)
    if scheme == "pg":
        if pg_state is None:
            kxy = diffusivities(data, h, taps, order, f.dx, f.dy, mu, nu, cfg)
        else:
            avg = pg_state.averaged(data)
            if pg_state.kxy is None or not pg_state.frozen:
                pg_state.kxy = diffusivities(avg, h, taps, order, f.dx, f.dy, mu, nu, cfg)
            kxy = pg_state.kxy
        r = pg_residual(data, h, f.sigma, q, taps, order, f.dx, f.dy, mu, nu, cfg, kxy=kxy)
    else:
        kxy = None
        r = upwind_residual(data, h, f.sigma, q, mu, nu, f.dx, f.dy)
    res = float(np.abs(r).sum())
    if scheme == "pg" and pg_state is not None:
        pg_state.observe(res, cfg.k_freeze_rel)
    delta = mg_correction(r, levels, n_sweeps,
                          cfg.beta_diag if scheme == "pg" else 1.0)
    data[h:h + f.nx, h:h + f.ny] -= interior(delta, h)
    if scheme == "pg":
        jacobi_pg(data, q, f, taps, order, cfg, kxy, pg_sweeps)
    apply_boundary(data, h, mu, nu)
    return res


# --------------------------------------------------------------------------
# materials, sources, drivers  (R/materials.py, R/eigen.py)
# --------------------------------------------------------------------------

def material(name, sigma_a, sigma_s, nu_sigma_f=None, sigma_f=None, chi=None):
    sa = np.asarray(sigma_a, dtype=float)
    z = np.zeros_like(sa)
    return SimpleNamespace(name=name, sigma_a=sa, sigma_s=np.asarray(sigma_s, dtype=float),
                           nu_sigma_f=z if nu_sigma_f is None else np.asarray(nu_sigma_f, float),
                           sigma_f=z if sigma_f is None else np.asarray(sigma_f, float),
                           chi=z if chi is None else np.asarray(chi, float))


def removal(m):
    """sigma_t = sigma_a + out-scatter (R/materials.py:51-55)."""
    return m.sigma_a + (m.sigma_s.sum(axis=1) - np.diag(m.sigma_s))


def material_field(region_map, mats, source=None):
    """Dense per-cell arrays (R/materials.py:179-209)."""
    region_map = np.asarray(region_map)
    nx, ny = region_map.shape
    ng = mats[0].sigma_a.shape[0]
    if region_map.min() < 0 or region_map.max() >= len(mats):
        raise ValueError("region map references an undefined material id")
    out = SimpleNamespace(sigma_t=np.zeros((nx, ny, ng)), sigma_s=np.zeros((nx, ny, ng, ng)),
                          nu_sigma_f=np.zeros((nx, ny, ng)), sigma_f=np.zeros((nx, ny, ng)),
                          chi=np.zeros((nx, ny, ng)),
                          source=np.zeros((nx, ny, ng)) if source is None else np.asarray(source, float))
    for mid, m in enumerate(mats):
        mask = region_map == mid
        if not mask.any():
            continue
        out.sigma_t[mask] = removal(m)
        out.sigma_s[mask] = m.sigma_s
        out.nu_sigma_f[mask] = m.nu_sigma_f
        out.sigma_f[mask] = m.sigma_f
        out.chi[mask] = m.chi
    out.fissile = bool(out.nu_sigma_f.any())
    return out


def group_source(phi, mat, lam=0.0):
    """q_b = sum_a s[a->b] phi_a - s[b->b] phi_b + src_b (+ lam chi F) (R/eigen.py:117-130)."""
    q = np.einsum("xyab,xya->xyb", mat.sigma_s, phi)
    q -= np.einsum("xygg,xyg->xyg", mat.sigma_s, phi)
    q = q + mat.source
    if lam != 0.0:
        q = q + lam * mat.chi * np.einsum("xyg,xyg->xy", mat.nu_sigma_f, phi)[:, :, None]
    return q[:, :, None, :]


def production(phi, mat, dx, dy):
    """Volume-integrated fission production (R/eigen.py:133-135)."""
    return float(np.einsum("xyg,xyg->", mat.nu_sigma_f, phi) * dx * dy)


def solver_options(**kw):
    """Defaults of R/eigen.py:29-44."""
    opts = dict(scheme="pg", order=2, n_a=4, n_levels=None, mg_iters=100,
                jacobi_sweeps=3, pg_sweeps=1, outer_iters=100, tol_rel=0.0,
                bootstrap_cycles=None, k_avg_theta=0.2, pg=None)
    opts.update(kw)
    if opts["pg"] is None:
        opts["pg"] = pg_config()
    o = SimpleNamespace(**opts)
    return o


def n_bootstrap(o):
    """R/eigen.py:46-51."""
    if o.bootstrap_cycles is not None:
        return o.bootstrap_cycles
    return 20 if o.scheme == "pg" else 0


def setup(problem, o):
    """Grid, quadrature, taps, materials, hierarchy (R/eigen.py:98-114)."""
    if o.scheme not in ("pg", "upwind"):
        raise ValueError(f"unknown scheme {o.scheme!r}")
    h = 1 if o.scheme == "upwind" else 3 * o.order          # R/eigen.py:53-58
    quad = build_quadrature(o.n_a)
    taps = stencils_1d(o.order) if o.scheme == "pg" else None
    mat = material_field(problem.region_map, problem.materials, problem.source)
    levels = build_hierarchy(problem.nx, problem.ny, problem.dx, problem.dy, h, quad,
                             mat.sigma_t, o.n_levels)
    return SimpleNamespace(problem=problem, h=h, quad=quad, taps=taps, mat=mat,
                           levels=levels, o=o)


def run_cycles(data, st, n_iters, fission_frozen=None, pg_state=None, scheme=None,
               state_round=None):
    """Lagged-source multigrid iterations (R/eigen.py:138-156).

    ``state_round`` (oracle-only) is applied to psi and psi_avg after every
    cycle; float32 rounding measures the trajectory's fp32 noise floor.
    """
    o = st.o
    scheme = scheme or o.scheme
    hist = []
    for _ in range(n_iters):
        phi = scalar_flux(data, st.h, st.quad.weights)
        q = group_source(phi, st.mat, 0.0)
        if fission_frozen is not None:
            q = q + fission_frozen
        res = sawtooth_cycle(data, q, st.levels, st.taps, o.order, o.pg, scheme,
                             o.jacobi_sweeps, o.pg_sweeps, pg_state)
        if state_round is not None:
            data[...] = state_round(data)
            if pg_state is not None and pg_state.psi_avg is not None:
                pg_state.psi_avg[...] = state_round(pg_state.psi_avg)
        hist.append(res)
        if not math.isfinite(res):
            break
    return hist


def solve_fixed_source(problem, o, state_round=None):
    """Fixed-source driver (R/eigen.py:159-191); returns a namespace."""
    st = setup(problem, o)
    nx, ny, ng = problem.nx, problem.ny, st.mat.sigma_t.shape[2]
    if st.mat.fissile:
        raise ValueError("problem has fission; use power_iteration")
    data = padded(nx, ny, st.h, st.quad.n_dir, ng)
    if not st.mat.source.any():
        return SimpleNamespace(psi=data, phi=np.zeros((nx, ny, ng)),
                               residual_history=[0.0], converged=True,
                               bootstrap_history=[], pg_log=[])
    boot = []
    if o.scheme == "pg" and n_bootstrap(o) > 0:
        boot = run_cycles(data, st, n_bootstrap(o), scheme="upwind", state_round=state_round)
    pgs = PGState(o.k_avg_theta)
    hist = run_cycles(data, st, o.mg_iters, pg_state=pgs, state_round=state_round)
    phi = scalar_flux(data, st.h, st.quad.weights)
    converged = True
    if o.tol_rel > 0.0 and hist[0] > 0.0:
        converged = hist[-1] <= o.tol_rel * hist[0]
    if not np.isfinite(hist[-1]):
        converged = False
    return SimpleNamespace(psi=data, phi=phi, residual_history=hist, converged=converged,
                           bootstrap_history=boot, pg_log=pgs.log)


def power_iteration(problem, o, inner_iters=None, state_round=None):
    """k-eigenvalue power iteration (R/eigen.py:194-251)."""
    st = setup(problem, o)
    mat = st.mat
    if not mat.fissile:
        raise ValueError("problem has no fission source; power iteration is undefined")
    if inner_iters is None:
        inner_iters = o.mg_iters
    nx, ny, ng = problem.nx, problem.ny, mat.sigma_t.shape[2]
    h, w = st.h, st.quad.weights
    data = padded(nx, ny, h, st.quad.n_dir, ng)
    data[...] = 1.0
    apply_boundary(data, h, st.quad.mu, st.quad.nu)
    phi = scalar_flux(data, h, w)
    prod = production(phi, mat, problem.dx, problem.dy)
    if prod <= 0.0:
        raise ValueError("initial fission production is zero")
    data /= prod
    phi /= prod
    k = 1.0
    hist = [k]
    rhist = []
    pgs = PGState(o.k_avg_theta)
    if o.scheme == "pg" and n_bootstrap(o) > 0:
        fq = mat.chi * np.einsum("xyg,xyg->xy", mat.nu_sigma_f, phi)[:, :, None]
        run_cycles(data, st, n_bootstrap(o), fission_frozen=fq[:, :, None, :],
                   scheme="upwind", state_round=state_round)
    for it in range(o.outer_iters):
        fq = (1.0 / k) * mat.chi * np.einsum("xyg,xyg->xy", mat.nu_sigma_f, phi)[:, :, None]
        rhist.extend(run_cycles(data, st, inner_iters, fission_frozen=fq[:, :, None, :],
                                pg_state=pgs, state_round=state_round))
        phi = scalar_flux(data, h, w)
        prod = production(phi, mat, problem.dx, problem.dy)
        if not math.isfinite(prod) or prod <= 0.0:
            raise ValueError(f"fission production became {prod} at outer iteration {it + 1}")
        k = k * prod
        data /= prod
        phi /= prod
        if pgs.psi_avg is not None:
            pgs.psi_avg /= prod
        hist.append(k)
    return SimpleNamespace(psi=data, phi=phi, k_eff=k, iteration=o.outer_iters,
                           history=hist, residual_history=rhist, pg_log=pgs.log)


def problem(name, nx, ny, dx, dy, region_map, materials, source=None):
    ng = materials[0].sigma_a.shape[0]
    return SimpleNamespace(name=name, nx=nx, ny=ny, dx=dx, dy=dy,
                           region_map=np.asarray(region_map), materials=list(materials),
                           source=source, n_groups=ng)


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("math", "np",
                                                                   "SimpleNamespace")]
