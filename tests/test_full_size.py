"""Parity at BASELINE.json's full sizes, through size-independent properties.

The oracle cannot run C3/C4 at full size in test time, so the full-size
configurations are checked by properties that hold for the reference's algorithm at any
size:
  * exact homogeneity: with the diffusivities held (a frozen PG cycle) one sawtooth cycle
    is linear in (psi, averaged iterate, source), and scaling by 2 commutes with every
    IEEE rounding, so the cycle of the doubled state is bit-for-bit twice the cycle of
    the state (and its fp64 residual L1 exactly twice);
  * the fp32 trajectory tracks the fp64 one (itself pinned to the reference's goldens to
    ~1e-10 at reduced sizes) within the north-star tolerances over the first cycles;
  * mirror symmetry: a problem symmetric under x -> -x has a mirrored flux.
"""

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2301_09991_b200 as pkg
    from paper_2301_09991_b200 import _lib
    _lib.load()
    return pkg


def _opts(P, pd, dtype, cycles=None):
    o = dict(pd.options)
    pg = o.pop("pg", None)
    if cycles is not None:
        if pd.driver == "fixed_source":
            o["mg_iters"] = cycles
        else:
            o["outer_iters"] = cycles
    return P.SolverOptions(**o, pg=P.PGConfig(**(pg or {})), dtype=dtype)


def _solver(P, pd, dtype, cycles=None):
    from paper_2301_09991_b200.eigen import Solver
    from paper_2301_09991_b200.problems import problem_from_data
    inner = pd.inner_iters if pd.driver == "power_iteration" else None
    return Solver(problem_from_data(pd), _opts(P, pd, dtype, cycles), inner)


@pytest.mark.parametrize("cfg", ["c4", "c3"])
def test_frozen_cycle_is_exactly_homogeneous(P, cfg):
    """Full-size C4 / C3 (fp32): cycle(2 psi, 2 pbar, 2 q; k) == 2 cycle(psi, pbar, q; k)."""
    from paper_2301_09991_b200 import benchmarks as B
    pd = getattr(B, cfg)()
    s = _solver(P, pd, "float32")
    for _ in range(2):                  # live cycles: diffusivities and averaged iterate exist
        s.step()
    fs, cfg_pg = s.setup.filters, s.options.pg
    eng, pgs = s.eng, s.pgs
    q0 = s._source(s._fis if s.eigen else None, True).clone()
    psi0, avg0 = s.psi.data.clone(), pgs._avg.clone()
    out = []
    for scale in (1.0, 2.0):
        s.psi.data.copy_(psi0 * scale)
        pgs._avg.copy_(avg0 * scale)
        pgs.frozen = True
        pgs.freeze_residual = float("inf")
        res = eng.cycle(s.psi, q0 * scale, fs, cfg_pg, "pg", s.options.jacobi_sweeps,
                        s.options.pg_sweeps, pgs, halo_ok=True)
        torch.cuda.synchronize()
        out.append((s.psi.data.clone(), pgs._avg.clone(), res))
    (p1, a1, r1), (p2, a2, r2) = out
    assert not torch.equal(p1, psi0)                    # the cycle did update psi
    assert torch.equal(p2, 2.0 * p1)
    assert torch.equal(a2, 2.0 * a1)
    assert r2 == 2.0 * r1


@pytest.mark.parametrize("cfg,cycles", [("c4", 3), ("c3", 1)])
def test_fp32_tracks_fp64_at_full_size(P, cfg, cycles):
    """Full-size C4 (3 cycles) / C3 (one outer of 5 cycles): the fp32 solve's flux, k,
    residual history and PGState decisions match the fp64 solve's."""
    from paper_2301_09991_b200 import benchmarks as B
    pd = getattr(B, cfg)()
    res = {}
    for dt in ("float64", "float32"):
        s = _solver(P, pd, dt, cycles)
        r = s.run()
        res[dt] = (np.asarray(r.phi), list(r.residual_history), list(r.pg_log),
                   list(getattr(r, "history", [])) if s.eigen else None)
        del s, r
        torch.cuda.empty_cache()
    (p64, h64, l64, k64), (p32, h32, l32, k32) = res["float64"], res["float32"]
    err = rel_l2(p32, p64)
    print(f"{cfg}: phi rel-L2 fp32 vs fp64 {err:.3e}, residual history max rel "
          f"{np.max(np.abs(np.array(h32) / np.array(h64) - 1)):.3e}")
    assert err < 1e-5, f"phi rel-L2 fp32 vs fp64 {err:.3e}"
    np.testing.assert_allclose(h32, h64, rtol=1e-5)
    assert l32 == l64
    if k64 is not None:
        np.testing.assert_allclose(k32, k64, rtol=1e-6)


def test_mirror_symmetric_problem_has_mirrored_flux(P):
    """Full-size C4 geometry made symmetric under x -> -x (blocks and source mirrored):
    the flux is mirror-symmetric (fp64; the kernels' tap order is not mirror-invariant,
    so equality holds to rounding)."""
    from paper_2301_09991_b200 import benchmarks as B
    pd = B.c4(cycles=3)
    half = pd.nx // 2
    pd.region_map[half:] = pd.region_map[:half][::-1]
    if pd.source is not None:
        pd.source[half:] = pd.source[:half][::-1]
    s = _solver(P, pd, "float64")
    phi = np.asarray(s.run().phi)
    print(f"mirror rel-L2 {rel_l2(phi[::-1], phi):.3e}")
    assert rel_l2(phi[::-1], phi) < 1e-10
