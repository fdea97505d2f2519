"""Domain decomposition on one GPU: P x-slab ranks as threads (ThreadComm) must reproduce
the single-domain solve (same kernels; only reduction order differs)."""

import threading

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _overlap_every_exchange(monkeypatch):
    """Window every exchanged stage (the default only overlaps bands >= 32 MB per side), so
    the small test slabs exercise the interior / edge launches of K2, K3, K3E and the sweep."""
    monkeypatch.setenv("CSN_DD_OVERLAP_MIN_MB", "0")


def _opts(P, pd, dtype):
    o = dict(pd.options)
    pg = o.pop("pg", None)
    return P.SolverOptions(**o, pg=P.PGConfig(**(pg or {})), dtype=dtype)


def _run_dd(pd, opts, size):
    from paper_2301_09991_b200.dd import DDSolver, ThreadComm
    from paper_2301_09991_b200.problems import problem_from_data
    comms = ThreadComm.make(size)
    out, err = [None] * size, []

    def work(r):
        try:
            s = DDSolver(problem_from_data(pd), opts, pd.inner_iters, comm=comms[r])
            out[r] = s.run()
        except Exception as e:  # surface thread failures
            err.append(e)
            comms[r].hub.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("size", [2, 4])
@pytest.mark.parametrize("case", ["c2", "c4", "c3", "c1up"])
def test_dd_matches_single_domain(case, size):
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2301_09991_b200 as P
    from paper_2301_09991_b200 import benchmarks as B
    from paper_2301_09991_b200.problems import problem_from_data
    pd = {"c2": lambda: B.c2(nx=64, blocks=8, n_a=2, cycles=8),
          "c4": lambda: B.c4(nx=64, blocks=4, n_a=2, cycles=8),
          "c3": lambda: B.c3(n_pins=4, cells_per_pin=16, n_a=2, outers=3, inner=3),
          "c1up": lambda: B.c1(nx=64, n_a=2, cycles=6, pg_off="upwind")}[case]()
    opts = _opts(P, pd, "float64")
    prob = problem_from_data(pd)
    ref = P.solve_fixed_source(prob, opts) if pd.driver == "fixed_source" else \
        P.power_iteration(prob, opts, pd.inner_iters)
    res = _run_dd(pd, opts, size)
    for r in res:
        assert rel_l2(r.phi, ref.phi) < 1e-11
        np.testing.assert_allclose(r.residual_history, ref.residual_history, rtol=1e-11)
        assert r.pg_log == ref.pg_log
        if pd.driver != "fixed_source":
            np.testing.assert_allclose(r.history, ref.history, rtol=1e-12)


@pytest.mark.parametrize("case,nx,n_a,size", [("c4", 128, 8, 2), ("c4", 256, 8, 4),
                                              ("c3", 128, 8, 2), ("c2", 128, 8, 2)])
def test_dd_fp32_wide_channels(case, nx, n_a, size):
    """fp32 kernels (packed x2 / TMA / split K2) under x-slab ghosts with >= 256 channels:
    the last CTA's x overhang past a ghost side must not be loaded (it once faulted)."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2301_09991_b200 as P
    from paper_2301_09991_b200 import benchmarks as B
    from paper_2301_09991_b200.problems import problem_from_data
    pd = {"c4": lambda: B.c4(nx=nx, blocks=4, n_a=n_a, cycles=6),
          "c2": lambda: B.c2(nx=nx, blocks=8, n_a=n_a, cycles=6),
          "c3": lambda: B.c3(n_pins=4, cells_per_pin=nx // 4, n_a=n_a, outers=2, inner=3)}[case]()
    opts = _opts(P, pd, "float32")
    prob = problem_from_data(pd)
    ref = P.solve_fixed_source(prob, opts) if pd.driver == "fixed_source" else \
        P.power_iteration(prob, opts, pd.inner_iters)
    res = _run_dd(pd, opts, size)
    for r in res:
        assert rel_l2(r.phi, ref.phi) < 1e-6
        np.testing.assert_allclose(r.residual_history, ref.residual_history, rtol=1e-6)
        assert r.pg_log == ref.pg_log


@pytest.mark.parametrize("case,dtype,size", [("ragged", "float32", 2), ("sweeps2", "float64", 2),
                                             ("sweeps2", "float32", 4)])
def test_dd_ragged_slab_and_pg_sweeps(case, dtype, size):
    """Slabs whose width is not a multiple of the 8-cell CTA tile (nx = 200 on 2 ranks:
    the last CTA's overhang must stop at nx + l on a ghost side) and pg_sweeps = 2 (the
    second sweep reads the first sweep's output, whose ghost rows are exchanged)."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2301_09991_b200 as P
    from paper_2301_09991_b200 import benchmarks as B
    from paper_2301_09991_b200.problems import problem_from_data
    if case == "ragged":
        pd = B.c4(nx=200, blocks=8, n_a=8, cycles=5)
    else:
        pd = B.c2(nx=64, blocks=8, n_a=2 if dtype == "float64" else 8, cycles=6)
        pd.options["pg_sweeps"] = 2
    opts = _opts(P, pd, dtype)
    ref = P.solve_fixed_source(problem_from_data(pd), opts)
    res = _run_dd(pd, opts, size)
    tol = 1e-11 if dtype == "float64" else 1e-6
    for r in res:
        assert rel_l2(r.phi, ref.phi) < tol
        np.testing.assert_allclose(r.residual_history, ref.residual_history, rtol=tol)
        assert r.pg_log == ref.pg_log


@pytest.mark.parametrize("case,size", [("c4", 2), ("c4", 4), ("c3", 2), ("c2", 2)])
def test_dd_overlap_windows_bitwise(case, size, monkeypatch):
    """The PG kernels launched on interior columns while the exchange is in flight and on
    edge columns after it (XWindow, CSN_DD_OVERLAP=1, the default) give the flux of the
    one-launch path bit for bit; only the fp64 L1 is summed in window order."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2301_09991_b200 as P
    from paper_2301_09991_b200 import benchmarks as B
    pd = {"c4": lambda: B.c4(nx=256, blocks=4, n_a=8, cycles=6),
          "c2": lambda: B.c2(nx=128, blocks=8, n_a=8, cycles=6),
          "c3": lambda: B.c3(n_pins=4, cells_per_pin=32, n_a=8, outers=2, inner=3)}[case]()
    opts = _opts(P, pd, "float32")
    monkeypatch.setenv("CSN_DD_OVERLAP", "0")
    off = _run_dd(pd, opts, size)
    monkeypatch.setenv("CSN_DD_OVERLAP", "1")
    on = _run_dd(pd, opts, size)
    for a, b in zip(on, off):
        assert np.array_equal(a.phi, b.phi)
        np.testing.assert_allclose(a.residual_history, b.residual_history, rtol=1e-13)
        assert a.pg_log == b.pg_log


def test_dd_rejects_narrow_slabs():
    """A slab narrower than the widest halo exchange (3l psi rows on live cycles) is
    refused instead of sending the sender's own ghost rows."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2301_09991_b200 as P
    from paper_2301_09991_b200 import benchmarks as B
    from paper_2301_09991_b200.dd import DDSolver, ThreadComm
    from paper_2301_09991_b200.problems import problem_from_data
    pd = B.c4(nx=64, blocks=4, n_a=2, cycles=2)
    with pytest.raises(ValueError, match="narrower"):
        DDSolver(problem_from_data(pd), _opts(P, pd, "float64"), comm=ThreadComm.make(8)[0])


def test_dd_multiprocess_torchrun():
    """The N > 1 bench path as the driver launches it (torchrun, one process per rank,
    TorchDistComm), ranks sharing the one GPU over gloo (bands staged through the host):
    fp32 C4 and C3 at P = 2 reproduce the single-domain solve."""
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import os
    import random
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for graphs, args in (("1", ["c4", "64", "2", "4", "6"]), ("0", ["c3", "64", "4", "4", "3"])):
        env = dict(os.environ, CSN_DIST_BACKEND="gloo", CSN_DD_GRAPHS=graphs)
        out = subprocess.run(
            [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
             "--master-addr", "127.0.0.1", "--master-port", str(29700 + random.randrange(200)),
             os.path.join(root, "tools", "dd_torchrun_check.py")] + args,
            env=env, capture_output=True, text=True, timeout=600)
        line = [l for l in out.stdout.splitlines() if "phi rel-L2" in l]
        assert out.returncode == 0 and line, out.stdout[-2000:] + out.stderr[-2000:]
        f = line[-1].split()
        assert float(f[f.index("rel-L2") + 1]) < 1e-6 and float(f[f.index("max") + 1]) < 1e-6
        assert line[-1].endswith("log_eq True")
