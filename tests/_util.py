"""Shared test helpers: convert benchmark generator output to oracle inputs."""

import numpy as np

import oracle as O


def oracle_problem(pd):
    mats = [O.material(m.name, m.sigma_a, m.sigma_s, m.nu_sigma_f, m.sigma_f, m.chi)
            for m in pd.materials]
    return O.problem(pd.name, pd.nx, pd.ny, pd.dx, pd.dy, pd.region_map, mats, pd.source)


def oracle_options(pd, **over):
    o = dict(pd.options)
    o.update(over)
    pg = o.pop("pg", None)
    if pg is not None and not hasattr(pg, "epsilon_k"):
        pg = O.pg_config(**pg)
    return O.solver_options(pg=pg, **o)


def run_oracle(pd, state_round=None, **over):
    prob = oracle_problem(pd)
    o = oracle_options(pd, **over)
    if pd.driver == "fixed_source":
        return O.solve_fixed_source(prob, o, state_round=state_round)
    return O.power_iteration(prob, o, inner_iters=pd.inner_iters, state_round=state_round)


def fp32_round(a):
    return a.astype(np.float32).astype(np.float64)


def log_array(log):
    return np.array([(c, 1 if e == "freeze" else 0) for c, e in log], dtype=np.int64).reshape(-1, 2)
