"""Compute-only cost of one DD rank's cycle at N ranks, on one GPU: a middle rank (both
sides ghosted) with a communicator that moves nothing (exchanges are no-ops, the L1 /
production all-reduces are identities, the coarse all-gather tiles the local slab).
It bounds the strong-scaling efficiency from the compute side: t(N=1) / (N t_rank(N))
with zero communication cost.  usage: python tools/dd_rank_cost.py N [cycles]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_09991_b200 as P
from paper_2301_09991_b200 import benchmarks as B
from paper_2301_09991_b200.problems import problem_from_data
from paper_2301_09991_b200.dd import DDSolver, SlabComm, _Done
from paper_2301_09991_b200.eigen import Solver
from paper_2301_09991_b200 import _lib
for kv in filter(None, os.environ.get("CSN_TUNE", "").split(",")):
    k, v = kv.split("=")
    _lib.set_tuning(k, int(v))


class NullComm(SlabComm):
    def __init__(self, rank, size):
        self.rank, self.size = rank, size

    def exchange(self, t, width, hx):
        pass

    def exchange_many(self, items):
        return _Done()

    def allreduce_sum_(self, t):
        return t

    def allgather_x(self, t):
        return torch.cat([t] * self.size, dim=0)


N = int(sys.argv[1])
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
W = 3
pd = B.c4()
o = dict(pd.options); pg = o.pop("pg", None); o["mg_iters"] = W + K
opts = P.SolverOptions(**o, pg=P.PGConfig(**(pg or {})), dtype="float32")
s = Solver(problem_from_data(pd), opts, None) if N == 1 else \
    DDSolver(problem_from_data(pd), opts, None, comm=NullComm(N // 2, N))
if N > 1:
    s.eng.coarse_graphs = os.environ.get("CSN_DD_GRAPHS", "0") == "1"
for _ in range(W):
    s.step()
torch.cuda.synchronize()
s.eng.probe = {} if os.environ.get("PROBE") else None
import time
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(K):
    s.step()
e1.record()
torch.cuda.synchronize()
host = (time.perf_counter() - t0) * 1e3 / K
if s.eng.probe:
    tot = {k: sum(a.elapsed_time(b) for a, b in v) / K for k, v in s.eng.probe.items()}
    print({k: round(v, 3) for k, v in tot.items()}, "sum", round(sum(tot.values()), 3))
print(f"host wall {host:.3f} ms/cycle; N={N}: {e0.elapsed_time(e1) / K:.3f} ms/cycle per rank (compute only)", flush=True)
