import sys, time, torch
sys.path.insert(0, '.')
import paper_2301_09991_b200 as P
from paper_2301_09991_b200 import benchmarks as B
from paper_2301_09991_b200.eigen import Solver
from paper_2301_09991_b200.problems import problem_from_data
pd = B.c2()
o = dict(pd.options); o["mg_iters"] = 30
opts = P.SolverOptions(**o, dtype="float32")
s = Solver(problem_from_data(pd), opts)
eng = s.eng
for i in range(30):
    n_g, n_s = len(eng._graphs), len(eng._seen)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s.step()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(i, f"{(t1-t0)*1e3:.3f} ms", "captured" if len(eng._graphs) > n_g else ("new" if len(eng._seen) > n_s else "replay"), s.pgs.frozen)
