"""N-process DD (TorchDistComm) vs the single-domain solve, one case; run under torchrun.

CSN_DIST_BACKEND=gloo lets every rank share one GPU (bands staged through the host): a
plumbing check of the N > 1 path, never a timing.
usage: torchrun --nproc-per-node N tools/dd_torchrun_check.py CASE NX N_A BLOCKS CYCLES"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import paper_2301_09991_b200 as P
from paper_2301_09991_b200 import benchmarks as B
from paper_2301_09991_b200.problems import problem_from_data
if os.environ.get("CSN_POISON"):     # recycled allocator memory full of NaN
    _pz = [torch.full((1 << 26,), float("nan"), device="cuda") for _ in range(16)]
    del _pz
from paper_2301_09991_b200.dd import DDSolver, TorchDistComm
from paper_2301_09991_b200 import _lib
for kv in filter(None, os.environ.get("CSN_TUNE", "").split(",")):
    k, v = kv.split("=")
    _lib.set_tuning(k, int(v))

case, nx, n_a, blocks, cyc = sys.argv[1], *map(int, sys.argv[2:6])
backend = os.environ.get("CSN_DIST_BACKEND", "nccl")
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
dist.init_process_group(backend)
rank = dist.get_rank()
pd = {"c4": lambda: B.c4(nx=nx, blocks=blocks, n_a=n_a, cycles=cyc),
      "c2": lambda: B.c2(nx=nx, blocks=blocks, n_a=n_a, cycles=cyc),
      "c3": lambda: B.c3(n_pins=blocks, cells_per_pin=nx // blocks, n_a=n_a, outers=2, inner=3)}[case]()
o = dict(pd.options); pg = o.pop("pg", None)
opts = P.SolverOptions(**o, pg=P.PGConfig(**(pg or {})), dtype=os.environ.get("CSN_DTYPE", "float32"))
res = DDSolver(problem_from_data(pd), opts, pd.inner_iters, comm=TorchDistComm()).run()
if rank == 0:
    prob = problem_from_data(pd)
    ref = P.solve_fixed_source(prob, opts) if pd.driver == "fixed_source" else \
        P.power_iteration(prob, opts, pd.inner_iters)
    e = float(np.linalg.norm(res.phi - ref.phi) / np.linalg.norm(ref.phi))
    h = np.array(res.residual_history) / np.array(ref.residual_history) - 1
    print(f"{case} nx={nx} n_a={n_a} P={dist.get_world_size()} {opts.dtype} {backend}: "
          f"phi rel-L2 {e:.2e} hist max {np.max(np.abs(h)):.2e} first-diff "
          f"{int(np.argmax(np.abs(h) > 1e-6)) if np.any(np.abs(h) > 1e-6) else -1} "
          f"log_eq {res.pg_log == ref.pg_log}", flush=True)
dist.destroy_process_group()
