import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2301_09991_b200 as P
import oracle as O
g = np.load('tests/golden/transfer.npz')
for na, ng in ((4, 2), (1, 1), (2, 3), (2, 1), (1, 2)):
    key = f"na{na}_g{ng}"
    if f"{key}_r" in g.files:
        r = g[f"{key}_r"]; sig = g[f"{key}_sigma"]
    else:
        rng = np.random.default_rng(1); q0 = O.build_quadrature(na)
        r = rng.normal(size=(16, 8, q0.n_dir, ng)); sig = rng.uniform(0.1, 2, size=(16, 8, ng))
    q = P.build_quadrature(na)
    grid = P.GridSpec(16, 8, 0.25, 0.5, 1)
    hier = P.build_hierarchy(grid, q, sig, 3)
    oq = O.build_quadrature(na)
    levels = O.build_hierarchy(16, 8, 0.25, 0.5, 1, oq, sig, 3)
    for nl in (1, 2, 3):
        for sweeps in (0, 1, 3):
            hh = P.build_hierarchy(grid, q, sig, nl)
            d = P.mg_correction(torch.as_tensor(r, device='cuda'), hh, n_sweeps=sweeps, finest_diag_scale=3.0)
            ref = O.mg_correction(r, O.build_hierarchy(16, 8, 0.25, 0.5, 1, oq, sig, nl), sweeps, 3.0)
            a = d.data.cpu().numpy()
            err = np.linalg.norm(a[1:-1,1:-1] - ref[1:-1,1:-1]) / max(np.linalg.norm(ref[1:-1,1:-1]), 1e-300)
            print(key, 'levels', nl, 'sweeps', sweeps, 'err', err)
