"""Debug probe: rank 0's psi (incl. halos) after K cycles + a 3l ghost exchange vs the
single-domain psi over the same global columns; prints where they differ.  torchrun."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import paper_2301_09991_b200 as P
from paper_2301_09991_b200 import benchmarks as B
from paper_2301_09991_b200.problems import problem_from_data
from paper_2301_09991_b200.dd import DDSolver, TorchDistComm
from paper_2301_09991_b200.eigen import Solver
from paper_2301_09991_b200 import _lib
for kv in filter(None, os.environ.get("CSN_TUNE", "").split(",")):
    k, v = kv.split("=")
    _lib.set_tuning(k, int(v))

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1
torch.cuda.set_device(0)
dist.init_process_group(os.environ.get("CSN_DIST_BACKEND", "gloo"))
rank, size = dist.get_rank(), dist.get_world_size()
pd = B.c4(nx=64, blocks=4, n_a=2, cycles=6)
o = dict(pd.options); pg = o.pop("pg", None)
opts = P.SolverOptions(**o, pg=P.PGConfig(**(pg or {})), dtype="float32")
dd = DDSolver(problem_from_data(pd), opts, None, comm=TorchDistComm())
for _ in range(K):
    dd.step()
h = dd.psi.grid.halo
dd.comm.exchange_many([(dd.psi.data, h, h)]).wait()
torch.cuda.synchronize()
mine = dd.psi.data.cpu().numpy()
if rank == 0:
    s = Solver(problem_from_data(pd), opts, None)
    for _ in range(K):
        s.step()
    torch.cuda.synchronize()
    ref = s.psi.data.cpu().numpy()
    nxl = mine.shape[0] - 2 * h
    print("halo", h, "local nx", nxl, "shape", mine.shape, ref.shape)
    refc = ref[:nxl + 2 * h]            # global columns [-h, nxl + h)
    d = np.abs(mine - refc).max(axis=(2, 3))   # [x, y]
    sc = np.abs(refc).max()
    bad = np.argwhere(d > 1e-6 * sc)
    print("max |diff|", d.max(), "scale", sc, "bad cells", len(bad))
    xs = sorted(set(int(b[0]) - h for b in bad)); ys = sorted(set(int(b[1]) - h for b in bad))
    print("bad x (local, -h..)", xs[:40]); print("bad y", ys[:40])
dist.destroy_process_group()
