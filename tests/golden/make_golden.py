"""Generate golden vectors by running the REAL reference (convsn) in this container.

Usage (CPU container only — /root/reference does not exist on the GPU box):

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py ops        # only per-operation fixtures

Writes ``tests/golden/*.npz``.  Inputs are stored next to outputs so the tests
replay them without the reference.  Problems come from
``paper_2301_09991_b200.benchmarks`` (pure NumPy generators) converted to the
reference's own ``ProblemSpec`` / ``SolverOptions`` objects, so the reference,
the CPU oracle and the B200 solver see identical inputs.
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import convsn  # noqa: E402  (the reference)
from convsn import discretisation as rd  # noqa: E402
from convsn import eigen as re  # noqa: E402
from convsn import filters as rf  # noqa: E402
from convsn import grid as rg  # noqa: E402
from convsn import multigrid as rm  # noqa: E402
from convsn import quadrature as rq  # noqa: E402
from convsn import verification as rv  # noqa: E402
from convsn.materials import CrossSections  # noqa: E402
from convsn.problems import ProblemSpec  # noqa: E402

from paper_2301_09991_b200 import benchmarks as B  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def ref_problem(pd):
    mats = [CrossSections(m.name, m.sigma_a, m.sigma_s, m.nu_sigma_f, m.sigma_f, m.chi)
            for m in pd.materials]
    return ProblemSpec(name=pd.name, nx=pd.nx, ny=pd.ny, dx=pd.dx, dy=pd.dy,
                       region_map=pd.region_map, materials=mats, source=pd.source,
                       n_groups=pd.n_groups)


def ref_options(pd):
    o = dict(pd.options)
    pg = o.pop("pg", None)
    if pg is not None:
        o["pg"] = rd.PGConfig(**pg)
    return re.SolverOptions(**o)


class ObserveLog:
    """Record PGState freeze/unfreeze decisions by wrapping the reference's observe."""

    def __init__(self):
        self.events = []
        self._orig = rm.PGState.observe
        self._calls = {}

    def __enter__(self):
        calls = self._calls
        orig = self._orig
        events = self.events

        def observe(state, resid, k_freeze_rel):
            n = calls.get(id(state), 0) + 1
            calls[id(state)] = n
            before = state.frozen
            orig(state, resid, k_freeze_rel)
            if state.frozen != before:
                events.append((n, 1 if state.frozen else 0))

        rm.PGState.observe = observe
        return self

    def __exit__(self, *a):
        rm.PGState.observe = self._orig


# ----------------------------------------------------------------- setup data
def make_setup():
    out = {}
    for na in (1, 2, 4, 8, 16):
        q = rq.build_quadrature(na)
        out[f"quad{na}_dirs"] = q.directions
        out[f"quad{na}_w"] = q.weights
        if na > 1:
            c = rq.coarsen_quadrature(q)
            out[f"quad{na}_coarse_dirs"] = c.directions
            out[f"quad{na}_coarse_w"] = c.weights
    for p in rf.SUPPORTED_ORDERS:
        m, g, s = rf.averaged_stencils_1d(p)
        out[f"taps{p}_mass"], out[f"taps{p}_grad"], out[f"taps{p}_stiff"] = m, g, s
    # harmonic sigma coarsening incl. the zero-child rule
    rng = np.random.default_rng(11)
    sig = rng.uniform(0.05, 5.0, size=(8, 6, 2))
    sig[0, 0, 0] = 0.0
    sig[5, 3, 1] = 0.0
    out["sigma_fine"] = sig
    out["sigma_coarse"] = rm.coarsen_sigma(sig)
    # materials: removal of the C3 / C5 libraries
    for key, mats in (("lib2", [B.two_group_material(n) for n in ("moderator", "fuel", "control")]),
                      ("lib7", B.seven_group_library(0))):
        for i, m in enumerate(mats):
            cs = CrossSections(m.name, m.sigma_a, m.sigma_s, m.nu_sigma_f, m.sigma_f, m.chi)
            out[f"{key}_{i}_sigma_t"] = cs.sigma_t
    save("setup", **out)


# ----------------------------------------------------------------- per-op
def make_ops():
    out = {}
    rng = np.random.default_rng(1234)
    nx, ny, na, ng, dx, dy = 9, 7, 2, 2, 0.3, 0.2
    quad = rq.build_quadrature(na)
    nd = quad.n_dir
    sigma = rng.uniform(0.1, 3.0, size=(nx, ny, ng))
    qcell = rng.uniform(0.0, 2.0, size=(nx, ny, 1, ng))
    qfull = rng.uniform(-1.0, 1.0, size=(nx, ny, nd, ng))
    out.update(sigma=sigma, qcell=qcell, qfull=qfull)

    # boundary on an arbitrary padded array (h = 3)
    g3 = rg.GridSpec(nx, ny, dx, dy, 3)
    raw = rng.normal(size=(nx + 6, ny + 6, nd, ng))
    f = rg.Field(g3, nd, ng, raw.copy())
    rg.apply_boundary(f, quad)
    out.update(bc_in=raw, bc_out=f.data)

    # upwind residual / diagonal / sweeps on halo 1
    g1 = rg.GridSpec(nx, ny, dx, dy, 1)
    psi1 = rg.Field(g1, nd, ng)
    psi1.interior[...] = rng.normal(size=psi1.interior.shape)
    rg.apply_boundary(psi1, quad)
    uf = rf.build_upwind_filters(dx, dy)
    out["up_psi"] = psi1.data.copy()
    out["up_r_cell"] = rd.upwind_residual(psi1, sigma, qcell, quad, uf).data
    out["up_r_full"] = rd.upwind_residual(psi1, sigma, qfull, quad, uf).data
    out["diag_up"] = rd.jacobi_diagonal(sigma, quad, g1, "upwind")
    out["diag_pg"] = rd.jacobi_diagonal(sigma, quad, g1, "pg")
    lev = rm.Level(grid=g1, quad=quad, sigma_t=sigma,
                   diag=rd.jacobi_diagonal(sigma, quad, g1), upwind=uf)
    sw = psi1.copy()
    rm.jacobi_sweep(sw, qfull, lev, n_sweeps=3, scheme="upwind", diag_scale=3.0)
    out["up_sweep3"] = sw.data

    # scalar flux + group source with fission
    out["phi"] = rg.scalar_flux(psi1, quad)
    mats = [CrossSections("a", np.array([0.2, 0.9]), np.array([[0.1, 0.3], [0.05, 0.2]]),
                          np.array([0.02, 0.3]), np.array([0.01, 0.1]), np.array([1.0, 0.0])),
            CrossSections("b", np.array([0.1, 0.4]), np.array([[0.0, 0.6], [0.02, 0.0]]),
                          np.zeros(2), np.zeros(2), np.zeros(2))]
    region = rng.integers(0, 2, size=(nx, ny))
    src = rng.uniform(0, 1, size=(nx, ny, ng))
    mf = convsn.MaterialField.from_region_map(region, mats, src)
    out["gs_region"] = region
    out["gs_src"] = src
    out["gs_q0"] = re.assemble_group_source(out["phi"], mf, 0.0)
    out["gs_q1"] = re.assemble_group_source(out["phi"], mf, 0.7)
    out["gs_prod"] = np.array(re.fission_production(out["phi"], mf, dx, dy))

    # PG operators for p = 1, 2, 3, 5
    cfg = rd.PGConfig()
    quad1 = rq.build_quadrature(1)    # 8 ordinates keep the wide-halo fixtures small
    for p in (1, 2, 3, 5):
        h = 3 * p
        gp = rg.GridSpec(nx, ny, dx, dy, h)
        quad, nd = quad1, quad1.n_dir
        psi = rg.Field(gp, nd, ng)
        psi.interior[...] = rng.normal(size=psi.interior.shape) + 2.0
        rg.apply_boundary(psi, quad)
        fs = rf.build_convfem_filters(p, dx, dy)
        kx, ky = rd.pg_anisotropic_diffusivities(psi, fs, quad, cfg)
        r_own = rd.pg_residual(psi, sigma, qcell, quad, fs, cfg)
        kx2 = np.abs(rng.normal(size=kx.shape)) * 0.01
        ky2 = np.abs(rng.normal(size=ky.shape)) * 0.01
        r_given = rd.pg_residual(psi, sigma, qcell, quad, fs, cfg, diffusivities=(kx2, ky2))
        r_iso = rd.pg_residual(psi, sigma, qcell, quad, fs, cfg, anisotropy="iso")
        levp = rm.Level(grid=gp, quad=quad, sigma_t=sigma,
                        diag=rd.jacobi_diagonal(sigma, quad, gp), upwind=rf.build_upwind_filters(dx, dy))
        sw = psi.copy()
        rm.jacobi_sweep(sw, qcell, levp, n_sweeps=1, scheme="pg", cfg=cfg, fs=fs,
                        diffusivities=(kx, ky))
        out[f"pg{p}_psi"] = psi.data
        out[f"pg{p}_kx"], out[f"pg{p}_ky"] = kx, ky
        out[f"pg{p}_r_own"] = r_own.data
        out[f"pg{p}_kx2"], out[f"pg{p}_ky2"] = kx2, ky2
        out[f"pg{p}_r_given"] = r_given.data
        out[f"pg{p}_r_iso"] = r_iso.data
        out[f"pg{p}_sweep"] = sw.data
        out[f"pg{p}_alt_mixed"] = rd.residual_alternatives(psi, fs, quad, cfg, "mixed_mass").data
        out[f"pg{p}_alt_high"] = rd.residual_alternatives(psi, fs, quad, cfg, "high_order").data
        if p >= 2:
            out[f"pg{p}_alt_low"] = rd.residual_alternatives(psi, fs, quad, cfg, "low_order").data

    # generic convolution
    g3 = rg.GridSpec(nx, ny, dx, dy, 3)
    cf = rg.Field(g3, nd, ng, rng.normal(size=(nx + 6, ny + 6, nd, ng)))
    st5 = rng.normal(size=(5, 5))
    scale = rng.normal(size=nd)
    out["conv_in"] = cf.data
    out["conv_st5"] = st5
    out["conv_scale"] = scale
    out["conv_out_m1"] = rg.convolve(cf, st5, direction_scale=scale, margin=1).data
    out["conv_out_sep"] = rg.convolve_separable(cf, st5[0], st5[1], margin=1).data
    save("ops", **out)


def make_transfer():
    out = {}
    rng = np.random.default_rng(99)
    for na, ng in ((4, 2), (1, 1), (2, 3)):
        quad = rq.build_quadrature(na)
        g = rg.GridSpec(16, 8, 0.25, 0.5, 1)
        sig = rng.uniform(0.1, 2.0, size=(16, 8, ng))
        hier = rm.build_hierarchy(g, quad, sig, n_levels=3)
        arr = rng.normal(size=(16, 8, quad.n_dir, ng))
        f = rg.Field(g, quad.n_dir, ng)
        f.interior[...] = arr
        rr = rm.restrict(f, hier[0], hier[1])
        pp = rm.prolong(rr, hier[1], hier[0])
        delta = rm.mg_correction(arr, hier, n_sweeps=3, finest_diag_scale=3.0)
        key = f"na{na}_g{ng}"
        out[f"{key}_sigma"] = sig
        out[f"{key}_r"] = arr
        out[f"{key}_restrict"] = rr.data
        out[f"{key}_prolong"] = pp.data
        out[f"{key}_mgc"] = delta.data
        for i, lev in enumerate(hier):
            out[f"{key}_lev{i}_sigma"] = lev.sigma_t
    save("transfer", **out)


# ----------------------------------------------------------------- cycles / drivers
def run_driver(pd, tag, extra=None):
    t0 = time.perf_counter()
    prob = ref_problem(pd)
    opts = ref_options(pd)
    with ObserveLog() as log:
        if pd.driver == "fixed_source":
            res = re.solve_fixed_source(prob, opts)
            arrays = dict(phi=res.phi, residual_history=np.array(res.residual_history),
                          converged=np.array(res.converged))
        else:
            res = re.power_iteration(prob, opts, inner_iters=pd.inner_iters)
            arrays = dict(phi=res.phi, residual_history=np.array(res.residual_history),
                          k_history=np.array(res.history), k_eff=np.array(res.k_eff))
    arrays["pg_log"] = np.array(log.events, dtype=np.int64).reshape(-1, 2)
    arrays["wall_s"] = np.array(time.perf_counter() - t0)
    if extra:
        arrays.update(extra)
    save(tag, **arrays)


def make_cycles(orders=(1, 2, 3, 5), upwind=True):
    # a few raw sawtooth cycles with PGState on a small heterogeneous problem
    for p in orders:
        pd = B.c2(nx=16, blocks=4, n_a=2, cycles=8)
        pd.options["order"] = p
        prob = ref_problem(pd)
        opts = ref_options(pd)
        setup = re.setup_transport(prob, opts)
        psi = rg.Field(setup.grid, setup.quad.n_dir, 1)
        rng = np.random.default_rng(5 + p)
        psi.interior[...] = rng.uniform(0.0, 1.0, size=psi.interior.shape)
        psi0 = psi.data.copy()
        st = rm.PGState(0.2)
        hist, frozen = [], []
        with ObserveLog() as log:
            for c in range(8):
                phi = rg.scalar_flux(psi, setup.quad)
                q = re.assemble_group_source(phi, setup.mat)
                psi, res = rm.sawtooth_cycle(psi, q, setup.hierarchy, fs=setup.filters,
                                             cfg=opts.pg, scheme="pg", pg_state=st)
                hist.append(res)
                frozen.append(st.frozen)
        save(f"cycle_pg{p}", psi0=psi0, psi=psi.data, psi_avg=st.psi_avg.data,
             hist=np.array(hist), frozen=np.array(frozen),
             pg_log=np.array(log.events, dtype=np.int64).reshape(-1, 2))
    if not upwind:
        return
    # upwind cycles
    pd = B.c1(nx=16, n_a=2, cycles=5, pg_off="upwind")
    prob = ref_problem(pd)
    opts = ref_options(pd)
    setup = re.setup_transport(prob, opts)
    psi = rg.Field(setup.grid, setup.quad.n_dir, 1)
    hist = []
    for c in range(5):
        q = re.assemble_group_source(rg.scalar_flux(psi, setup.quad), setup.mat)
        psi, res = rm.sawtooth_cycle(psi, q, setup.hierarchy, scheme="upwind")
        hist.append(res)
    save("cycle_upwind", psi=psi.data, hist=np.array(hist))


def make_drivers(full=True):
    run_driver(B.c1(pg_off="alpha_r"), "c1_alpha_r")
    run_driver(B.c1(pg_off="upwind"), "c1_upwind")
    run_driver(B.c2(nx=32, blocks=8, n_a=4, cycles=20), "c2_reduced")
    run_driver(B.c3(n_pins=4, cells_per_pin=16, n_a=4, outers=30, inner=5), "c3_reduced")
    run_driver(B.c4(nx=64, blocks=4, n_a=4, cycles=20), "c4_reduced")
    run_driver(B.c5(n_pins=4, cells_per_pin=16, n_a=2, outers=10, inner=3), "c5_reduced")
    # non-power-of-two grid (shallow hierarchy, odd coarsest extents)
    pd = B.c2(nx=24, blocks=4, n_a=2, cycles=6)
    pd.ny = 40
    pd.region_map = np.repeat(pd.region_map[:, :1], 40, axis=1).copy()
    pd.source = np.ones((24, 40, 1))
    run_driver(pd, "ragged_24x40")
    # dense-oracle known answers (R/verification.py:62-105)
    rep = rv.compare_against_dense_oracle()
    rep1 = rv.compare_against_dense_oracle(nx=4, ny=4, n_groups=1)
    save("dense_kat", rows=np.array([r[1] for r in rep.rows]),
         k_label=np.array(rep.rows[2][0]), k1_label=np.array(rep1.rows[2][0]))
    if full:
        run_driver(B.c2(), "c2_full")


def make_benchmarks():
    """The reference's own two benchmarks (R/problems.py) with default bootstrap cycles."""
    from convsn.problems import build_fuel_assembly, build_straight_duct, synthetic_xs_path
    with ObserveLog() as log:
        st = re.power_iteration(build_fuel_assembly(False, synthetic_xs_path(), n_pins=4),
                                re.SolverOptions(scheme="pg", order=1, n_a=1, mg_iters=2,
                                                 outer_iters=3), inner_iters=2)
    save("assembly4", phi=st.phi, k_history=np.array(st.history),
         residual_history=np.array(st.residual_history),
         pg_log=np.array(log.events, dtype=np.int64).reshape(-1, 2))
    with ObserveLog() as log:
        res = re.solve_fixed_source(build_straight_duct(0.8),
                                    re.SolverOptions(scheme="pg", order=2, n_a=1, mg_iters=6))
    save("duct08", phi=res.phi, residual_history=np.array(res.residual_history),
         boot=np.array(res.bootstrap_history),
         pg_log=np.array(log.events, dtype=np.int64).reshape(-1, 2))


def make_krylov():
    """R/krylov.py:54-104 on two tiny problems (bootstrap + frozen-k Picard/GMRES)."""
    from convsn import krylov as rk
    out = {}
    for tag, pd, kw in (("q", B.c2(nx=16, blocks=4, n_a=1, cycles=1), dict(picard_iters=3)),
                        ("l", B.c2(nx=16, blocks=2, n_a=2, cycles=1), dict(picard_iters=2))):
        pd.options.update(order=2 if tag == "q" else 1, bootstrap_cycles=3)
        t0 = time.perf_counter()
        res = rk.solve_fixed_source_krylov(ref_problem(pd), ref_options(pd), **kw)
        out[f"{tag}_phi"] = res.phi
        out[f"{tag}_hist"] = np.array(res.residual_history)
        out[f"{tag}_converged"] = np.array(res.converged)
        print(tag, "krylov", time.perf_counter() - t0, "s", res.residual_history, res.converged)
    save("krylov", **out)


# ----------------------------------------------------------------- fp32 pinning of the headline path
# C4-generator instances with >= 512 channels (the channel count the bench's fp32 kernels
# run at), and the fp32 noise floor of every driver golden: the oracle port re-run with
# psi and psi_avg rounded to float32 after every cycle (storage rounding only; SURVEY
# 8c).  The floor files hold that trajectory; tests compare GPU fp32 against
# max(1e-5, 3 x floor).
PIN = {
    "c4_64n8": lambda: B.c4(nx=64, blocks=4, n_a=8, cycles=20),
    "c4_128n8": lambda: B.c4(nx=128, blocks=8, n_a=8, cycles=20),
    "c4_256n8": lambda: B.c4(nx=256, blocks=16, n_a=8, cycles=20),
    # the linear-PG multigroup kernels at the bench's channel widths (1024 and 3584
    # channels: 2-group / generic-group TMA residual and sweep, fused K2, packed smoothers)
    "c3_64n8": lambda: B.c3(n_pins=4, cells_per_pin=16, n_a=8, outers=6, inner=5),
    "c5_64n8": lambda: B.c5(n_pins=4, cells_per_pin=16, n_a=8, outers=4, inner=3),
}
FLOOR = {
    "c1_alpha_r": lambda: B.c1(pg_off="alpha_r"),
    "c1_upwind": lambda: B.c1(pg_off="upwind"),
    "c2_reduced": lambda: B.c2(nx=32, blocks=8, n_a=4, cycles=20),
    "c3_reduced": lambda: B.c3(n_pins=4, cells_per_pin=16, n_a=4, outers=30, inner=5),
    "c4_reduced": lambda: B.c4(nx=64, blocks=4, n_a=4, cycles=20),
    "c5_reduced": lambda: B.c5(n_pins=4, cells_per_pin=16, n_a=2, outers=10, inner=3),
    "c2_full": lambda: B.c2(),
    **PIN,
}


def make_floor(tag):
    """fp32 state-rounding floor of golden `tag` (oracle port, R/eigen.py:138-156 with
    psi, psi_avg rounded after each cycle)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from _util import fp32_round, log_array, run_oracle
    pd = FLOOR[tag]()
    t0 = time.perf_counter()
    res = run_oracle(pd, state_round=fp32_round)
    gold = np.load(os.path.join(HERE, tag + ".npz"))
    floor = float(np.linalg.norm(res.phi - gold["phi"]) / np.linalg.norm(gold["phi"]))
    out = dict(phi=res.phi, residual_history=np.array(res.residual_history),
               pg_log=log_array(res.pg_log), floor=np.array(floor),
               wall_s=np.array(time.perf_counter() - t0))
    if pd.driver != "fixed_source":
        out["k_history"] = np.array(res.history)
        out["k_floor"] = np.array(abs(res.k_eff / float(gold["k_eff"]) - 1.0))
    print(tag, "fp32 floor", floor, out.get("k_floor"))
    save("floor_" + tag, **out)


def make_pin(tag):
    run_driver(PIN[tag](), tag)


if __name__ == "__main__":
    what = sys.argv[1:] or ["setup", "ops", "transfer", "cycles", "drivers"]
    for w in what:
        if w.startswith("pin:"):
            make_pin(w[4:])
            continue
        if w.startswith("floor:"):
            make_floor(w[6:])
            continue
        {"setup": make_setup, "ops": make_ops, "transfer": make_transfer,
         "cycles": make_cycles, "drivers": make_drivers,
         "drivers_small": lambda: make_drivers(False),
         "c2full": lambda: run_driver(B.c2(), "c2_full"),
         "krylov": make_krylov, "cycle5": lambda: make_cycles((5,), False), "benchmarks": make_benchmarks}[w]()
