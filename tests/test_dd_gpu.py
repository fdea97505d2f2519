"""Domain decomposition on one GPU: P x-slab ranks as threads (ThreadComm) must reproduce
the single-domain solve (same kernels; only reduction order differs)."""

import threading

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu


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
