"""Three-way parity table: reference fp64 golden, the oracle's fp32
state-rounding floor, and this build's fp32 and fp64 GPU runs, for every driver golden.

    python tools/parity_table.py > profiles/r02_parity_table.md      (GPU box)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2301_09991_b200 as P  # noqa: E402
from paper_2301_09991_b200 import benchmarks as B  # noqa: E402
from paper_2301_09991_b200.problems import problem_from_data  # noqa: E402

CASES = {
    "c1_alpha_r": lambda: B.c1(pg_off="alpha_r"),
    "c1_upwind": lambda: B.c1(pg_off="upwind"),
    "c2_reduced": lambda: B.c2(nx=32, blocks=8, n_a=4, cycles=20),
    "c2_full": lambda: B.c2(),
    "c3_reduced": lambda: B.c3(n_pins=4, cells_per_pin=16, n_a=4, outers=30, inner=5),
    "c4_reduced": lambda: B.c4(nx=64, blocks=4, n_a=4, cycles=20),
    "c4_64n8": lambda: B.c4(nx=64, blocks=4, n_a=8, cycles=20),
    "c4_128n8": lambda: B.c4(nx=128, blocks=8, n_a=8, cycles=20),
    "c4_256n8": lambda: B.c4(nx=256, blocks=16, n_a=8, cycles=20),
    "c3_64n8": lambda: B.c3(n_pins=4, cells_per_pin=16, n_a=8, outers=6, inner=5),
    "c5_64n8": lambda: B.c5(n_pins=4, cells_per_pin=16, n_a=8, outers=4, inner=3),
    "c5_reduced": lambda: B.c5(n_pins=4, cells_per_pin=16, n_a=2, outers=10, inner=3),
}


def solve(pd, dtype):
    o = dict(pd.options)
    pg = o.pop("pg", None)
    opts = P.SolverOptions(**o, pg=P.PGConfig(**(pg or {})), dtype=dtype)
    prob = problem_from_data(pd)
    if pd.driver == "fixed_source":
        return P.solve_fixed_source(prob, opts)
    return P.power_iteration(prob, opts, inner_iters=pd.inner_iters)


def log(res):
    return np.array([(c, 1 if e == "freeze" else 0) for c, e in res.pg_log],
                    dtype=np.int64).reshape(-1, 2)


def main():
    gdir = os.path.join(ROOT, "tests", "golden")
    print("| case | instance | oracle fp32 floor (phi) | GPU fp32 phi | GPU fp32 / floor | "
          "fp32 bound max(1e-5, 3 floor) | GPU fp64 phi | k: floor / fp32 / fp64 | "
          "resid hist fp32 | PGState log (fp32, fp64) |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for tag, make in CASES.items():
        g = np.load(os.path.join(gdir, tag + ".npz"))
        f = np.load(os.path.join(gdir, "floor_" + tag + ".npz"))
        pd = make()
        row = {}
        for dt in ("float32", "float64"):
            r = solve(pd, dt)
            e = float(np.linalg.norm(r.phi - g["phi"]) / np.linalg.norm(g["phi"]))
            h = float(np.max(np.abs(np.array(r.residual_history) / g["residual_history"] - 1)))
            k = (abs(r.k_eff / float(g["k_eff"]) - 1.0) if "k_eff" in g.files else None)
            row[dt] = (e, h, k, np.array_equal(log(r), g["pg_log"]))
        floor = float(f["floor"])
        kf = f"{float(f['k_floor']):.1e} / {row['float32'][2]:.1e} / {row['float64'][2]:.1e}" \
            if "k_floor" in f.files else "—"
        inst = f"{pd.nx}x{pd.ny}, {8 * pd.n_a ** 2} ord, G={pd.n_groups}, p={pd.options.get('order', 1)}"
        print(f"| {tag} | {inst} | {floor:.2e} | {row['float32'][0]:.2e} | "
              f"{row['float32'][0] / floor:.2f} | {max(1e-5, 3 * floor):.2e} | "
              f"{row['float64'][0]:.1e} | {kf} | {row['float32'][1]:.1e} | "
              f"{row['float32'][3]}, {row['float64'][3]} |", flush=True)


if __name__ == "__main__":
    main()
