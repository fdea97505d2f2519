"""DD (ThreadComm, one GPU) vs single domain in a chosen dtype; one case per process.

usage: python tools/dd_f32_repro.py CASE NX N_A SIZE DTYPE"""
import sys, os, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2301_09991_b200 as P
from paper_2301_09991_b200 import benchmarks as B
from paper_2301_09991_b200.problems import problem_from_data
if os.environ.get("CSN_POISON"):     # recycled allocator memory full of NaN
    _pz = [torch.full((1 << 26,), float("nan"), device="cuda") for _ in range(16)]
    del _pz
from paper_2301_09991_b200.dd import DDSolver, ThreadComm
from paper_2301_09991_b200 import _lib
for kv in filter(None, os.environ.get("CSN_TUNE", "").split(",")):
    k, v = kv.split("=")
    _lib.set_tuning(k, int(v))

case, nx, n_a, size, dtype = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
pd = {"c4": lambda: B.c4(nx=nx, blocks=4, n_a=n_a, cycles=6),
      "c2": lambda: B.c2(nx=nx, blocks=8, n_a=n_a, cycles=6),
      "c3": lambda: B.c3(n_pins=4, cells_per_pin=nx // 4, n_a=n_a, outers=2, inner=3)}[case]()
o = dict(pd.options); pg = o.pop("pg", None)
opts = P.SolverOptions(**o, pg=P.PGConfig(**(pg or {})), dtype=dtype)
prob = problem_from_data(pd)
ref = P.solve_fixed_source(prob, opts) if pd.driver == "fixed_source" else \
    P.power_iteration(prob, opts, pd.inner_iters)
comms = ThreadComm.make(size)
out, err = [None] * size, []
def work(r):
    try:
        out[r] = DDSolver(problem_from_data(pd), opts, pd.inner_iters, comm=comms[r]).run()
    except Exception as e:
        err.append(e); comms[r].hub.barrier.abort()
ts = [threading.Thread(target=work, args=(r,)) for r in range(size)]
[t.start() for t in ts]; [t.join() for t in ts]
if err:
    raise err[0]
e = float(np.linalg.norm(out[0].phi - ref.phi) / np.linalg.norm(ref.phi))
h = float(np.max(np.abs(np.array(out[0].residual_history) / np.array(ref.residual_history) - 1)))
print(f"{case} nx={nx} n_a={n_a} P={size} {dtype}: phi rel-L2 {e:.2e} hist {h:.2e} log_eq {out[0].pg_log == ref.pg_log}")
