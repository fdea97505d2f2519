"""Pin the CPU oracle (oracle/) against the real reference's golden vectors.

CPU only.  The fixtures in tests/golden/ were produced by running the
unmodified reference (tests/golden/make_golden.py); agreement here is what
licenses the oracle as the parity checker for the CUDA path.
"""

import numpy as np
import pytest

import oracle as O
from conftest import golden, rel_l2
from paper_2301_09991_b200 import benchmarks as B
from _util import log_array, run_oracle


def test_quadrature_and_coarsening():
    g = golden("setup")
    for na in (1, 2, 4, 8, 16):
        q = O.build_quadrature(na)
        np.testing.assert_allclose(q.directions, g[f"quad{na}_dirs"], rtol=0, atol=2e-15)
        np.testing.assert_allclose(q.weights, g[f"quad{na}_w"], rtol=0, atol=2e-15)
        assert abs(q.weights.sum() - 4 * np.pi) < 1e-13
        if na > 1:
            c = O.coarsen_quadrature(q)
            np.testing.assert_allclose(c.directions, g[f"quad{na}_coarse_dirs"], atol=2e-15)
            np.testing.assert_allclose(c.weights, g[f"quad{na}_coarse_w"], atol=2e-15)


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_convfem_taps(p):
    g = golden("setup")
    m, d, s = O.stencils_1d(p)
    np.testing.assert_allclose(m, g[f"taps{p}_mass"], atol=1e-14)
    np.testing.assert_allclose(d, g[f"taps{p}_grad"], atol=1e-14)
    np.testing.assert_allclose(s, g[f"taps{p}_stiff"], atol=1e-14)
    # consistency invariants (R/filters.py:4-10)
    x = np.arange(-p, p + 1, dtype=float)
    assert abs(m.sum() - 1) < 1e-14 and abs(d.sum()) < 1e-14 and abs(s.sum()) < 1e-13
    assert abs(d @ x - 1) < 1e-13 and abs(s @ x ** 2 + 2) < 1e-12


def test_sigma_coarsening_and_removal():
    g = golden("setup")
    np.testing.assert_allclose(O.coarsen_sigma(g["sigma_fine"]), g["sigma_coarse"], rtol=1e-15)
    for key, mats in (("lib2", [B.two_group_material(n) for n in ("moderator", "fuel", "control")]),
                      ("lib7", B.seven_group_library(0))):
        for i, m in enumerate(mats):
            om = O.material(m.name, m.sigma_a, m.sigma_s, m.nu_sigma_f, m.sigma_f, m.chi)
            np.testing.assert_allclose(O.removal(om), g[f"{key}_{i}_sigma_t"], rtol=1e-15)


def test_boundary_rule():
    g = golden("ops")
    q = O.build_quadrature(2)
    d = g["bc_in"].copy()
    O.apply_boundary(d, 3, q.mu, q.nu)
    np.testing.assert_array_equal(d, g["bc_out"])


def test_upwind_ops():
    g = golden("ops")
    q = O.build_quadrature(2)
    psi, sig = g["up_psi"], g["sigma"]
    for qk, rk in (("qcell", "up_r_cell"), ("qfull", "up_r_full")):
        r = O.upwind_residual(psi, 1, sig, g[qk], q.mu, q.nu, 0.3, 0.2)
        np.testing.assert_allclose(r, O.interior(g[rk], 1), rtol=0, atol=1e-13)
    np.testing.assert_allclose(O.stream_diag(q.mu, q.nu, 0.3, 0.2, sig), g["diag_up"], rtol=1e-15)
    lev = O.build_hierarchy(9, 7, 0.3, 0.2, 1, q, sig, 1)[0]
    sw = psi.copy()
    O.jacobi_upwind(sw, g["qfull"], lev, 3, 3.0)
    np.testing.assert_allclose(sw, g["up_sweep3"], atol=1e-13)


def test_flux_and_group_source():
    g = golden("ops")
    q = O.build_quadrature(2)
    phi = O.scalar_flux(g["up_psi"], 1, q.weights)
    np.testing.assert_allclose(phi, g["phi"], atol=1e-13)
    mats = [O.material("a", [0.2, 0.9], [[0.1, 0.3], [0.05, 0.2]], [0.02, 0.3], [0.01, 0.1], [1.0, 0.0]),
            O.material("b", [0.1, 0.4], [[0.0, 0.6], [0.02, 0.0]])]
    mf = O.material_field(g["gs_region"], mats, g["gs_src"])
    np.testing.assert_allclose(O.group_source(g["phi"], mf, 0.0), g["gs_q0"], atol=1e-14)
    np.testing.assert_allclose(O.group_source(g["phi"], mf, 0.7), g["gs_q1"], atol=1e-14)
    assert abs(O.production(g["phi"], mf, 0.3, 0.2) - float(g["gs_prod"])) < 1e-14


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_pg_operators(p):
    g = golden("ops")
    q = O.build_quadrature(1)
    h, l = 3 * p, p
    taps = O.stencils_1d(p)
    cfg = O.pg_config()
    psi, sig, qc = g[f"pg{p}_psi"], g["sigma"], g["qcell"]
    kx, ky = O.diffusivities(psi, h, taps, p, 0.3, 0.2, q.mu, q.nu, cfg)
    band = (slice(h - l, h + 9 + l), slice(h - l, h + 7 + l))
    np.testing.assert_allclose(kx[band], g[f"pg{p}_kx"][band], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(ky[band], g[f"pg{p}_ky"][band], rtol=1e-12, atol=1e-15)
    for key, kxy, aniso in (("r_own", None, "xy"), ("r_given", (g[f"pg{p}_kx2"], g[f"pg{p}_ky2"]), "xy"),
                            ("r_iso", None, "iso")):
        r = O.pg_residual(psi, h, sig, qc, taps, p, 0.3, 0.2, q.mu, q.nu, cfg, kxy, aniso)
        ref = O.interior(g[f"pg{p}_{key}"], h)
        assert rel_l2(r, ref) < 1e-13, key
    lev = O.build_hierarchy(9, 7, 0.3, 0.2, h, q, sig, 1)[0]
    sw = psi.copy()
    O.jacobi_pg(sw, qc, lev, taps, p, cfg, (kx, ky), 1)
    np.testing.assert_allclose(sw, g[f"pg{p}_sweep"], rtol=1e-12, atol=1e-13)
    for mode in ("mixed_mass", "high_order", "low_order"):
        if mode == "low_order" and p < 2:
            with pytest.raises(ValueError):
                O.residual_estimate(psi, h, taps, p, 0.3, 0.2, q.mu, q.nu, cfg, mode)
            continue
        key = {"mixed_mass": "alt_mixed", "high_order": "alt_high", "low_order": "alt_low"}[mode]
        est = O.residual_estimate(psi, h, taps, p, 0.3, 0.2, q.mu, q.nu, cfg, mode)
        assert rel_l2(O.interior(est, h), O.interior(g[f"pg{p}_{key}"], h)) < 1e-13


def test_generic_convolution():
    g = golden("ops")
    st5, sc = g["conv_st5"], g["conv_scale"]
    out = O.convolve2d(g["conv_in"], st5, 3, 1, sc)
    np.testing.assert_allclose(out, g["conv_out_m1"], atol=1e-13)
    out2 = O.sep(g["conv_in"], st5[0], st5[1], 3, 1)
    np.testing.assert_allclose(out2, g["conv_out_sep"], atol=1e-13)


@pytest.mark.parametrize("na,ng", [(4, 2), (1, 1), (2, 3)])
def test_transfers_and_correction(na, ng):
    g = golden("transfer")
    key = f"na{na}_g{ng}"
    q = O.build_quadrature(na)
    levels = O.build_hierarchy(16, 8, 0.25, 0.5, 1, q, g[f"{key}_sigma"], 3)
    for i, lev in enumerate(levels):
        np.testing.assert_allclose(lev.sigma, g[f"{key}_lev{i}_sigma"], rtol=1e-15)
    r = g[f"{key}_r"]
    raw = O.restrict_raw(r, levels[0], levels[1])
    np.testing.assert_allclose(raw, O.interior(g[f"{key}_restrict"], 1), rtol=1e-13, atol=1e-14)
    pro = O.prolong(raw, levels[1], levels[0])
    np.testing.assert_array_equal(pro, O.interior(g[f"{key}_prolong"], 1))
    delta = O.mg_correction(r, levels, 3, 3.0)
    assert rel_l2(delta, g[f"{key}_mgc"]) < 1e-13


@pytest.mark.parametrize("p", [1, 2, 3])
def test_pg_cycles_with_state(p):
    g = golden(f"cycle_pg{p}")
    pd = B.c2(nx=16, blocks=4, n_a=2, cycles=8)
    pd.options["order"] = p
    from _util import oracle_options, oracle_problem
    st = O.setup(oracle_problem(pd), oracle_options(pd))
    data = g["psi0"].copy()
    pgs = O.PGState(0.2)
    hist, frozen = [], []
    for _ in range(8):
        phi = O.scalar_flux(data, st.h, st.quad.weights)
        qq = O.group_source(phi, st.mat)
        hist.append(O.sawtooth_cycle(data, qq, st.levels, st.taps, p, st.o.pg, "pg", 3, 1, pgs))
        frozen.append(pgs.frozen)
    np.testing.assert_allclose(hist, g["hist"], rtol=1e-11)
    assert frozen == g["frozen"].tolist()
    assert rel_l2(data, g["psi"]) < 1e-11
    assert rel_l2(pgs.psi_avg, g["psi_avg"]) < 1e-11
    np.testing.assert_array_equal(log_array(pgs.log), g["pg_log"])


def test_upwind_cycles():
    g = golden("cycle_upwind")
    pd = B.c1(nx=16, n_a=2, cycles=5, pg_off="upwind")
    from _util import oracle_options, oracle_problem
    st = O.setup(oracle_problem(pd), oracle_options(pd))
    data = O.padded(16, 16, 1, st.quad.n_dir, 1)
    hist = []
    for _ in range(5):
        qq = O.group_source(O.scalar_flux(data, 1, st.quad.weights), st.mat)
        hist.append(O.sawtooth_cycle(data, qq, st.levels, scheme="upwind"))
    np.testing.assert_allclose(hist, g["hist"], rtol=1e-12)
    assert rel_l2(data, g["psi"]) < 1e-12


DRIVERS = {
    "c1_alpha_r": lambda: B.c1(pg_off="alpha_r"),
    "c1_upwind": lambda: B.c1(pg_off="upwind"),
    "c2_reduced": lambda: B.c2(nx=32, blocks=8, n_a=4, cycles=20),
    "c4_reduced": lambda: B.c4(nx=64, blocks=4, n_a=4, cycles=20),
    "c5_reduced": lambda: B.c5(n_pins=4, cells_per_pin=16, n_a=2, outers=10, inner=3),
}


@pytest.mark.parametrize("tag", sorted(DRIVERS))
def test_driver_trajectories(tag):
    g = golden(tag)
    pd = DRIVERS[tag]()
    res = run_oracle(pd)
    assert rel_l2(res.phi, g["phi"]) < 1e-9
    np.testing.assert_allclose(res.residual_history, g["residual_history"], rtol=1e-8)
    np.testing.assert_array_equal(log_array(res.pg_log), g["pg_log"])
    if "k_history" in g.files:
        np.testing.assert_allclose(res.history, g["k_history"], rtol=1e-11)


@pytest.mark.slow
def test_c3_reduced_trajectory():
    g = golden("c3_reduced")
    res = run_oracle(B.c3(n_pins=4, cells_per_pin=16, n_a=4, outers=30, inner=5))
    assert rel_l2(res.phi, g["phi"]) < 1e-9
    np.testing.assert_allclose(res.history, g["k_history"], rtol=1e-11)
    np.testing.assert_array_equal(log_array(res.pg_log), g["pg_log"])


def test_ragged_grid():
    g = golden("ragged_24x40")
    pd = B.c2(nx=24, blocks=4, n_a=2, cycles=6)
    pd.ny = 40
    pd.region_map = np.repeat(pd.region_map[:, :1], 40, axis=1).copy()
    pd.source = np.ones((24, 40, 1))
    res = run_oracle(pd)
    assert rel_l2(res.phi, g["phi"]) < 1e-10
    np.testing.assert_allclose(res.residual_history, g["residual_history"], rtol=1e-10)


def test_dense_known_answers():
    """R/verification.py:62-105 via the dense restatement (k = 2.79519174 at defaults)."""
    g = golden("dense_kat")
    from oracle import dense as D
    q = O.build_quadrature(1)
    fuel = O.material("fuel", [0.15, 1.2], [[0.0, 0.05], [0.02, 0.0]], [0.02, 0.24],
                      np.array([0.02, 0.24]) / 2.45, [1.0, 0.0])
    mf = O.material_field(np.zeros((6, 6), int), [fuel])
    A = D.streaming_removal(q.mu, q.nu, mf.sigma_t, 0.5, 0.5)
    S = D.scatter(q.weights, mf.sigma_s)
    F = D.fission(q.weights, mf.chi, mf.nu_sigma_f)
    k, _, _ = D.power_iteration(A - S, F, iters=2000, tol=1e-13)
    label = str(g["k_label"])
    assert f"{k:.8f}" in label and abs(k - 2.79519174) < 1e-8
    # the stencil upwind residual equals the dense operator
    rng = np.random.default_rng(2718)
    psi = O.padded(6, 6, 1, q.n_dir, 2)
    psi[1:7, 1:7] = rng.random((6, 6, q.n_dir, 2))
    qq = rng.random((6, 6, q.n_dir, 2))
    O.apply_boundary(psi, 1, q.mu, q.nu)
    r = O.upwind_residual(psi, 1, mf.sigma_t, qq, q.mu, q.nu, 0.5, 0.5)
    assert np.max(np.abs(r.ravel() - (A @ O.interior(psi, 1).ravel() - qq.ravel()))) < 1e-12
    # the oracle's own power iteration reaches the dense k
    prob = O.problem("blk", 6, 6, 0.5, 0.5, np.zeros((6, 6), int), [fuel])
    st = O.power_iteration(prob, O.solver_options(scheme="upwind", n_a=1, mg_iters=25,
                                                  outer_iters=200))
    assert abs(st.k_eff - k) < 1e-6
