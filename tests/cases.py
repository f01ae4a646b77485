"""Shared test builders: rebuild golden recipes (tests/golden/recipes.py)
with the product's setup API, and run them through the product or the
oracle."""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from recipes import RUNS  # noqa: E402

import paper_1805_08846_b200 as P  # noqa: E402

RECIPES = {r["name"]: r for r in RUNS}


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def build_grid(r):
    """Initial StateGrid, params, solver name, BoundarySpec, initial speed."""
    problem = P.get_problem(r["problem"])
    spec = P.GridSpec(cells=tuple(r["cells"]), lower=tuple(r["lower"]), upper=tuple(r["upper"]),
                      num_states=problem.num_states)
    grid = P.create_grid(spec, np.dtype(r["dtype"]))
    P.fill_initial(grid, problem.initial_profile(r["profile"], dict(r["options"]), spec))
    params = problem.make_params({})
    sp = r["speed"]
    if sp == "bound":
        speed = problem.speed_bound(grid, params)
    elif sp[0] == "scale":
        speed = sp[1] * problem.speed_bound(grid, params)
    else:
        speed = float(sp[1])
    kind = P.BoundaryKind(r["bc"])
    bspec = P.BoundarySpec.uniform(kind, problem.normal_velocity)
    return grid, params, problem, bspec, speed


def params_dict(problem, params):
    if problem.solver_name == "acoustics":
        return {"sound_speed": params.sound_speed, "impedance": params.impedance}
    if problem.solver_name == "shallow_water":
        return {"gravity": params.gravity}
    if problem.solver_name == "advection":
        return {"speed": params.speed}
    return {}


def attempts_hex(attempts):
    return [[float(a.t_start).hex(), float(a.dt).hex(), float(a.max_speed).hex(),
             float(a.nu).hex(), bool(a.accepted), bool(a.landed)] for a in attempts]


def drive(sim, r):
    kind = r["drive"][0]
    if kind == "max_steps":
        return sim.run_until(1e30, max_steps=r["drive"][1]).attempts
    return sim.run_until(r["drive"][1], frame_times=tuple(r["drive"][2])).attempts


def oracle_sim(r, nthreads=None):
    from oracle import oracle as O
    grid, params, problem, bspec, speed = build_grid(r)
    sides = [(lo.value, hi.value) for lo, hi in bspec.sides]
    return O.OracleSimulation(
        grid.data.copy(), grid.spec.spacing, problem.solver_name, params_dict(problem, params),
        sides, bspec.normal_velocity, limiter=r["limiter"], initial_max_speed=speed,
        nthreads=nthreads or os.cpu_count() or 1), grid


def product_sim(r, **kw):
    grid, params, problem, bspec, speed = build_grid(r)
    sim = P.Simulation(grid, problem.solver, params, bspec, limiter=P.LimiterKind(r["limiter"]),
                       initial_max_speed=speed, **kw)
    return sim, grid
