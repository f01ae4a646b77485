"""Golden runs of the UNMODIFIED reference engine with user scalar solvers
registered through its plugin API (riemann.py:190-212, 259-262).

Run HERE (the build container), where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_user_solvers.py

Writes user_solvers.json: for each case, every attempt's (t_start, dt,
max_speed, nu, accepted, landed) as float.hex and the sha256 of the final
interior bytes.  tests/test_gpu_user_solver.py registers the same routines
as CUDA source (paper_1805_08846_b200/devsolver.py) and must reproduce them
bit for bit.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from clawtile import (  # noqa: E402
    BoundaryKind, BoundarySpec, LimiterKind, Simulation, create_grid, fill_initial,
)
from clawtile.grid import GridSpec  # noqa: E402
from clawtile.riemann import RiemannSolver, register_solver  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def burgers_scalar(ql, qr, normal, params, W, s):
    # inviscid Burgers, f(q) = q^2 / 2 along every axis: Roe speed
    W[0, 0] = qr[0] - ql[0]
    s[0] = 0.5 * (ql[0] + qr[0])


def pack_none(p, dtype):
    return np.zeros(1, dtype=dtype)


def burgers_profile(x, y):
    return 0.6 * np.sin(2 * math.pi * x) * np.cos(2 * math.pi * y) + 0.1


def burgers_profile_3d(x, y, z):
    return 0.5 * np.sin(2 * math.pi * x) * np.cos(2 * math.pi * y) * np.cos(2 * math.pi * z)


CASES = [
    # name, cells, profile, dtype, limiter, bc, steps
    ("burgers2d_mc_f64", (40, 32), burgers_profile, "float64", "mc", "periodic", 12),
    ("burgers2d_superbee_f32", (40, 32), burgers_profile, "float32", "superbee", "outflow", 12),
    ("burgers2d_vanleer_f64", (33, 27), burgers_profile, "float64", "vanleer", "outflow", 8),
    ("burgers3d_minmod_f64", (12, 10, 9), burgers_profile_3d, "float64", "minmod", "periodic",
     6),
]


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def main():
    solver = RiemannSolver("burgers_user", 1, burgers_scalar, pack_none,
                           normal_index=lambda axis: 0)
    register_solver(solver, overwrite=True)
    out = []
    for name, cells, prof, dtype, lim, bc, steps in CASES:
        nd = len(cells)
        spec = GridSpec(cells=cells, lower=(0.0,) * nd, upper=(1.0,) * nd, num_states=1)
        g = create_grid(spec, np.dtype(dtype))
        fill_initial(g, prof)
        speed = float(np.max(np.abs(g.interior())))
        bspec = BoundarySpec.uniform(BoundaryKind(bc), (None,) * nd)
        sim = Simulation(g, solver, None, bspec, limiter=LimiterKind(lim),
                         initial_max_speed=speed)
        rep = sim.run_until(1e30, max_steps=steps)
        out.append({
            "name": name, "cells": list(cells), "dtype": dtype, "limiter": lim, "bc": bc,
            "steps": steps, "speed": speed.hex(),
            "attempts": [[float(a.t_start).hex(), float(a.dt).hex(), float(a.max_speed).hex(),
                          float(a.nu).hex(), bool(a.accepted), bool(a.landed)]
                         for a in rep.attempts],
            "sha256": sha(sim.grid.interior()),
        })
    path = os.path.join(OUT, "user_solvers.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"wrote {path}: {len(out)} runs")


if __name__ == "__main__":
    main()
