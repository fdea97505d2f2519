import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2301_09991_b200 as P
g = np.load('tests/golden/ops.npz')
for na, ng in ((1, 2), (2, 1), (1, 4), (2, 2)):
  for p in (1, 2, 3):
    for dt in (torch.float64, torch.float32):
        q = P.build_quadrature(na)
        h, l = 3 * p, p
        grid = P.GridSpec(9, 7, 0.3, 0.2, h)
        fs = P.build_convfem_filters(p, 0.3, 0.2)
        cfg = P.PGConfig()
        rng = np.random.default_rng(0)
        psi_np = rng.normal(size=(9 + 2*h, 7 + 2*h, q.n_dir, ng)) + 2
        import oracle as O
        oq = O.build_quadrature(na)
        O.apply_boundary(psi_np, h, oq.mu, oq.nu)
        sig = rng.uniform(0.1, 3, size=(9, 7, ng)); qc = rng.uniform(0, 2, size=(9, 7, 1, ng))
        taps = O.stencils_1d(p)
        kx, ky = O.diffusivities(psi_np, h, taps, p, 0.3, 0.2, oq.mu, oq.nu, O.pg_config())
        r_ref = O.pg_residual(psi_np, h, sig, qc, taps, p, 0.3, 0.2, oq.mu, oq.nu, O.pg_config(), (kx, ky))
        psi = P.Field(grid, q.n_dir, ng, psi_np, dtype=dt)
        gkx, gky = P.pg_anisotropic_diffusivities(psi, fs, q, cfg)
        band = (slice(h - l, h + 9 + l), slice(h - l, h + 7 + l))
        ekx = np.abs(gkx.cpu().numpy()[band] - kx[band]).max() / np.abs(kx[band]).max()
        r = P.pg_residual(psi, sig, qc, q, fs, cfg, diffusivities=(kx, ky))
        er = np.abs(r.data.cpu().numpy()[h:-h, h:-h] - r_ref).max() / np.abs(r_ref).max()
        print(f"na={na} ng={ng} p={p} {str(dt)[-7:]} kx_err={ekx:.2e} r_err={er:.2e}")
