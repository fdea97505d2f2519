"""CPU tests of the product's host side: setup data, PGState logic, generators, C ABI.

No GPU needed: these pin the host layer (quadrature, taps, materials, hierarchy
coarsening, the PGState decision logic) against the reference goldens / the oracle,
and check that libconvsn_sm100.so loads and exports every symbol the header
declares (no compute calls are made).
"""

import os
import re

import numpy as np
import pytest

import oracle as O
from conftest import ROOT, golden
from paper_2301_09991_b200 import benchmarks as B
from paper_2301_09991_b200 import filters as F
from paper_2301_09991_b200 import materials as M
from paper_2301_09991_b200 import multigrid as MG
from paper_2301_09991_b200 import quadrature as Q


@pytest.mark.parametrize("na", [1, 2, 4, 8, 16])
def test_quadrature_matches_reference(na):
    g = golden("setup")
    q = Q.build_quadrature(na)
    np.testing.assert_allclose(q.directions, g[f"quad{na}_dirs"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(q.weights, g[f"quad{na}_w"], rtol=1e-13)
    assert q.n_dir == 8 * na * na
    assert abs(q.weights.sum() - 4 * np.pi) < 1e-12
    assert np.all(q.mu != 0) and np.all(q.nu != 0)          # strictly inside each octant
    if na > 1:
        c = Q.coarsen_quadrature(q)
        np.testing.assert_allclose(c.directions, g[f"quad{na}_coarse_dirs"], atol=1e-13)
        np.testing.assert_allclose(c.weights, g[f"quad{na}_coarse_w"], rtol=1e-13)


def test_quadrature_mirror_symmetry():
    """Faces 4-7 mirror faces 0-3 in (mu, nu, p)."""
    q = Q.build_quadrature(4)
    h = q.n_dir // 2
    np.testing.assert_array_equal(q.mu[:h], q.mu[h:])
    np.testing.assert_array_equal(q.nu[:h], q.nu[h:])
    np.testing.assert_array_equal(q.weights[:h], q.weights[h:])


@pytest.mark.parametrize("p", F.SUPPORTED_ORDERS)
def test_taps_match_reference_and_kernel_table(p):
    g = golden("setup")
    m, d, s = F.averaged_stencils_1d(p)
    for mine, key in ((m, "mass"), (d, "grad"), (s, "stiff")):
        np.testing.assert_allclose(mine, g[f"taps{p}_{key}"], rtol=0, atol=1e-14)
    # the compile-time table baked into the kernels (tools/gen_taps.py) is this host set
    text = open(os.path.join(ROOT, "paper_2301_09991_b200", "csrc", "taps_table.cuh")).read()
    block = text[text.index(f"struct UnitTaps<{p}>"):]
    for name, arr in (("m", m), ("g", d), ("s", s)):
        line = re.search(rf"double {name}\(int i\) {{ return (.*?); }}", block).group(1)
        vals = [float(v) for v in re.findall(r"\? ([-0-9.e+]+) :", line)]
        vals.append(float(line.rsplit(":", 1)[1]))
        np.testing.assert_array_equal(np.array(vals), arr)


def test_filter_set_and_errors():
    fs = F.build_convfem_filters(2, 0.5, 0.25)
    assert fs.w_x.shape == (5, 5) and fs.half_width == 2
    np.testing.assert_allclose(fs.w_m.sum(), 1.0, atol=1e-14)
    with pytest.raises(ValueError):
        F.build_convfem_filters(4, 1.0, 1.0)
    with pytest.raises(ValueError):
        F.build_convfem_filters(1, 0.0, 1.0)
    assert F.mixed_mass_filter(fs)[2, 2] == fs.w_m[2, 2] - 1.0
    np.testing.assert_array_equal(F.from_display(F.to_display(fs.w_x)), fs.w_x)


def test_sigma_coarsening_and_materials():
    g = golden("setup")
    np.testing.assert_allclose(MG.coarsen_sigma(g["sigma_fine"]), g["sigma_coarse"], rtol=1e-15)
    for key, mats in (("lib2", [B.two_group_material(n) for n in ("moderator", "fuel", "control")]),
                      ("lib7", B.seven_group_library(0))):
        for i, m in enumerate(mats):
            cs = M.CrossSections(m.name, m.sigma_a, m.sigma_s, m.nu_sigma_f, m.sigma_f, m.chi)
            np.testing.assert_allclose(cs.sigma_t, g[f"{key}_{i}_sigma_t"], rtol=1e-15)
    with pytest.raises(M.CrossSectionDataError):
        M.CrossSections("bad", np.array([-1.0]), np.zeros((1, 1)), np.zeros(1), np.zeros(1),
                        np.zeros(1))


def test_material_field_matches_oracle():
    pd = B.c3(n_pins=2, cells_per_pin=8, n_a=1)
    from paper_2301_09991_b200.problems import problem_from_data
    mf = problem_from_data(pd).material_field()
    om = O.material_field(pd.region_map, [O.material(m.name, m.sigma_a, m.sigma_s, m.nu_sigma_f,
                                                     m.sigma_f, m.chi) for m in pd.materials])
    for k in ("sigma_t", "sigma_s", "nu_sigma_f", "chi"):
        np.testing.assert_array_equal(getattr(mf, k), getattr(om, k))


def test_csv_library_roundtrip(tmp_path):
    from paper_2301_09991_b200.problems import synthetic_xs_path
    lib = M.CrossSectionLibrary.from_csv(synthetic_xs_path())
    assert lib.n_groups == 2 and "fuel" in lib and lib["fuel"].fissile
    path = tmp_path / "lib.csv"
    with open(path, "w") as fh:
        lib.to_csv(fh)
    lib2 = M.CrossSectionLibrary.from_csv(path)
    for name in ("fuel", "moderator", "control"):
        np.testing.assert_allclose(lib2[name].sigma_t, lib[name].sigma_t, rtol=1e-5)
    with pytest.raises(M.CrossSectionDataError):
        lib["nope"]


def test_hierarchy_shapes_and_errors():
    from paper_2301_09991_b200.grid import GridSpec
    q = Q.build_quadrature(4)
    sig = np.ones((24, 40, 1))
    h = MG.build_hierarchy(GridSpec(24, 40, 0.1, 0.1, 1), q, sig)
    assert [(l.grid.nx, l.grid.ny, l.quad.n_a) for l in h] == [(24, 40, 4), (12, 20, 2), (6, 10, 1),
                                                                (3, 5, 1)]
    assert MG.max_levels(512, 512) == 10 and MG.max_levels(45, 35) == 1
    with pytest.raises(ValueError):
        MG.build_hierarchy(GridSpec(24, 40, 0.1, 0.1, 1), q, sig, n_levels=5)


def _drive(state_cls, seq, rel=0.05):
    st = state_cls(0.2)
    frozen = []
    for r in seq:
        st.observe(r, rel)
        frozen.append(st.frozen)
    return frozen, st


@pytest.mark.parametrize("seed", range(6))
def test_pgstate_decisions_match_oracle(seed):
    """Host PGState logic (R/multigrid.py:227-256) decision for decision vs the oracle."""
    rng = np.random.default_rng(seed)
    seq = list(np.abs(np.cumsum(rng.normal(0, 1, 60))) + rng.uniform(0.1, 5, 60))
    seq += [seq[-1] * 3, seq[-1] * 0.01, seq[-1] * 10] * 4
    mine, a = _drive(MG.PGState, seq)
    ref, b = _drive(O.PGState, seq)
    assert mine == ref
    assert a.failed_freezes == b.failed
    assert [e for e in a.log] == [e for e in b.log]


def test_generators_are_seeded_and_shaped():
    a, b = B.c2(), B.c2()
    np.testing.assert_array_equal(a.region_map, b.region_map)
    assert a.dof() == 128 * 128 * 512 and a.source.sum() == 32 * 32
    assert B.c4().dof() == 512 * 512 * 2048
    c5 = B.c5(n_pins=2, cells_per_pin=16, n_a=1)
    assert c5.n_groups == 7 and c5.materials[1].nu_sigma_f.any()
    for m in c5.materials:      # rows of the physical library < sigma_t; removal unchanged
        assert np.all(m.sigma_a >= 0) and np.all(m.sigma_s >= 0)


def test_library_exports_every_declared_symbol():
    """The C ABI library loads without a GPU and exports what include/*.h declares."""
    from paper_2301_09991_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = _lib.load()
    header = open(os.path.join(ROOT, "include", "convsn_sm100.h")).read()
    declared = set(re.findall(r"^\S.*?\b(csn_[a-z0-9_]+)\(", header, re.M))
    assert declared == set(_lib.EXPORTED)
    for name in declared:
        assert hasattr(lib, name)
    assert lib.csn_version() == 1
    assert lib.csn_error_string(2).decode().startswith("unsupported ConvFEM order")


def test_product_path_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import paper_2301_09991_b200 as P
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.Field(P.GridSpec(4, 4, 1.0, 1.0, 1), 8, 1)


def test_z_fold_quadrature():
    from paper_2301_09991_b200.quadrature import build_quadrature, coarsen_quadrature, fold_z
    q = build_quadrature(8)
    f = fold_z(q)
    assert f.n_dir == q.n_dir // 2 and f.n_faces == 4 and f.folded
    assert abs(f.weights.sum() - 4 * np.pi) < 1e-12
    assert np.all(f.directions[:, 2] > 0)
    # coarsening commutes with the fold (weights exactly 2x, same directions)
    cf, cq = coarsen_quadrature(f), coarsen_quadrature(q)
    np.testing.assert_array_equal(cf.weights, 2.0 * cq.weights[:cf.n_dir])
    np.testing.assert_array_equal(cf.directions, cq.directions[:cf.n_dir])
    with pytest.raises(ValueError):
        fold_z(f)


def test_xwindow_views_and_ghost_flags():
    """multigrid.XWindow (the launch geometry of an x-window of a slab, used to overlap the
    DD halo exchange with the interior columns): narrowed views start at the window's first
    column, a cut side is flagged ghost, an uncut side keeps the slab's flag."""
    import torch
    from paper_2301_09991_b200 import _lib
    from paper_2301_09991_b200.multigrid import XWindow, _FullWindow
    h, nx, ny, C = 3, 40, 6, 4
    gm = _lib.geom(nx, ny, C, 1, 1, 0.5, 0.25, ghost_w=0, ghost_e=1)
    padded = torch.arange((nx + 2 * h) * (ny + 2 * h) * C, dtype=torch.float32).reshape(
        nx + 2 * h, ny + 2 * h, C)
    cells = torch.arange(nx * ny, dtype=torch.float32).reshape(nx, ny)
    w = XWindow(gm, 16, 24)
    assert (w.gm.nx, w.gm.ny, w.gm.ghost_w, w.gm.ghost_e) == (8, ny, 1, 1)
    assert (gm.nx, gm.ghost_w, gm.ghost_e) == (nx, 0, 1)          # the slab's geometry is untouched
    v = w.pad(padded, h)
    assert v.shape[0] == 8 + 2 * h and v.data_ptr() == padded[16].data_ptr()
    assert torch.equal(v[h], padded[16 + h])                      # window column 0 = slab column 16
    assert torch.equal(w.cells(cells), cells[16:24])
    assert w.pad(None, h) is None and w.cells(None) is None
    west = XWindow(gm, 0, 16, edge=True)
    assert (west.gm.ghost_w, west.gm.ghost_e, west.edge) == (0, 1, True)   # physical west side kept
    east = XWindow(gm, 24, nx, edge=True)
    assert (east.gm.ghost_w, east.gm.ghost_e) == (1, 1)
    full = _FullWindow(gm)
    assert full.pad(padded, h) is padded and full.cells(cells) is cells and not full.edge
