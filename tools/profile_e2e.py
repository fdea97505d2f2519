"""Host profile of the end-to-end solve (bench.py's e2e leg) on cuda:0: where the time
outside the cycles goes (setup, uploads, allocation, read-back).  Usage on the GPU box:
    python tools/profile_e2e.py [config]"""
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
    # warm: kernels loaded, allocator populated, as in bench.py's e2e leg
    P.solve_fixed_source(prob, opts)
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        st = P.setup_transport(prob, opts)
        t1 = time.perf_counter()
        s = P.eigen.Solver(prob, opts, setup=st)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        s.step()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        while not s.done:
            s.step()
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        r = s.result()
        t5 = time.perf_counter()
        print(f"setup_transport {1e3 * (t1 - t0):.1f} ms, Solver() {1e3 * (t2 - t1):.1f} ms, "
              f"first cycle {1e3 * (t3 - t2):.1f} ms, other cycles {1e3 * (t4 - t3):.1f} ms, "
              f"result {1e3 * (t5 - t4):.1f} ms")
    pr = cProfile.Profile()
    pr.enable()
    P.solve_fixed_source(prob, opts)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(35)


if __name__ == "__main__":
    main(*sys.argv[1:])
