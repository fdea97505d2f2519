"""Host profile of Solver construction and the first cycle (e2e overhead), cuda:0.
Usage on the GPU box: python tools/profile_setup.py [config]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2301_09991_b200 as P  # noqa: E402
from paper_2301_09991_b200 import benchmarks as B  # noqa: E402
from paper_2301_09991_b200.problems import problem_from_data  # noqa: E402


def main(cfg="c4"):
    pd = getattr(B, cfg)()
    prob = problem_from_data(pd)
    opts = bench.options_for(P, pd, "float32")
    P.solve_fixed_source(prob, opts)
    torch.cuda.synchronize()
    st = P.setup_transport(prob, opts)
    pr = cProfile.Profile()
    pr.enable()
    t0 = time.perf_counter()
    s = P.eigen.Solver(prob, opts, setup=st)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    s.step()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    pr.disable()
    print(f"Solver() {1e3 * (t1 - t0):.1f} ms, first cycle {1e3 * (t2 - t1):.1f} ms")
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main(*sys.argv[1:])
