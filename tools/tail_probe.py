"""Event-timed csn_coarse_tail on the C1/C3-like coarse hierarchies: whole tail, its first
level alone, sweep-count dependence (where the launch's time goes)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2301_09991_b200 as P
from paper_2301_09991_b200 import _lib

def run(nx, na, ng, nlev_tail=None, sweeps=3, reps=200):
    q = P.build_quadrature(na)
    grid = P.GridSpec(nx, nx, 0.25, 0.25, 1)
    sigma = np.random.default_rng(0).uniform(0.1, 8.0, size=(nx, nx, ng))
    hier = P.build_hierarchy(grid, q, sigma)
    eng = hier.engine(ng, torch.float32, torch.device("cuda"))
    t = eng._tail()
    n = t["n"] if nlev_tail is None else nlev_tail
    for i in range(len(eng.src)):
        eng.src[i].normal_()
    args = (0, n, t["geoms"], t["sigma"], t["mu"], t["nu"], t["strm"], t["w"], t["src"], t["delta"],
            _lib.ptr(t["scratch"]), sweeps, _lib.stream())
    for _ in range(5):
        _lib.call("csn_coarse_tail", *args)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        _lib.call("csn_coarse_tail", *args)
    e1.record()
    torch.cuda.synchronize()
    dof = [int(np.prod(s)) for s in eng.shapes[t["start"]:t["start"] + n]]
    print(f"nx={nx} na={na} ng={ng} levels={n} sweeps={sweeps} dof={dof}: "
          f"{e0.elapsed_time(e1) / reps * 1e3:.1f} us per launch")

for kw in (dict(), dict(nlev_tail=1), dict(nlev_tail=2), dict(sweeps=0), dict(sweeps=1), dict(nlev_tail=1, sweeps=1)):
    run(64, 4, 1, **kw)            # C1: tail from 32x32x32
for smem in (1, 0):
    _lib.set_tuning("tail_smem", smem)
    run(64, 4, 1)
    run(256, 8, 2)                 # C3: tail from 32x32x8x2
_lib.set_tuning("tail_smem", 1)
