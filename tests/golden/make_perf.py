"""Golden counters of the reference's perf model (clawtile/perf.py).

Run HERE (the build container), where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_perf.py

It imports the reference read-only and records, for a matrix of solvers,
limiters, grid shapes, tile plans and item sizes, the modeled counters of one
sweep (perf.py:404-439 sweep_counters: flops, special, bytes read/written,
stage split) and the halo read bytes (perf.py:442-452), plus the run-level
report rows of a short shallow-water run with counters on
(timestep.py:209-210, perf.py:516-553).  Writes perf.json next to this
file; tests/test_perf.py holds the product's restatement to it exactly.
"""

from __future__ import annotations

import json
import os
import sys

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np  # noqa: E402

from clawtile import (  # noqa: E402
    BoundaryKind, BoundarySpec, GridSpec, LimiterKind, Simulation, create_grid, get_solver,
    register_solver,
)
from clawtile import perf  # noqa: E402
from clawtile.riemann import RiemannSolver  # noqa: E402
from clawtile.sweep import plan_tiles  # noqa: E402

from make_golden import _vc_acoustics_scalar, _pack_vc  # noqa: E402

register_solver(RiemannSolver("vc_acoustics", 2, _vc_acoustics_scalar, _pack_vc), overwrite=True)

CASES = [
    # solver, cells, m, axis, tile shape (None = monolithic)
    ("shallow_water", (10, 6), 3, 0, None),
    ("shallow_water", (16, 12), 3, 1, (4, 4)),
    ("shallow_water", (1024, 1024), 3, 0, None),
    ("acoustics", (12, 8), 3, 0, None),
    ("acoustics", (32, 8), 3, 0, (8, 4)),
    ("acoustics", (8, 6, 5), 4, 2, (8, 2, 3)),
    ("acoustics", (96, 96, 96), 4, 1, None),
    ("advection", (16,), 1, 0, None),
    ("advection", (40,), 1, 0, (7,)),
    ("vc_acoustics", (9, 7, 6), 6, 1, None),
]
LIMITERS = ["none", "minmod", "superbee", "mc", "vanleer"]


def main():
    out = {"sweeps": [], "runs": []}
    for solver, cells, m, axis, tiles in CASES:
        spec = GridSpec(cells=cells, lower=(0.0,) * len(cells), upper=(1.0,) * len(cells),
                        num_states=m)
        plan = plan_tiles(spec, axis, tiles if tiles is not None else cells)
        for lim in LIMITERS:
            for isz in (8, 4):
                c, st = perf.sweep_counters(plan, spec, get_solver(solver), LimiterKind(lim), isz)
                out["sweeps"].append({
                    "solver": solver, "cells": list(cells), "m": m, "axis": axis,
                    "tiles": list(tiles) if tiles else None, "limiter": lim, "itemsize": isz,
                    "flops": c.flops, "special": c.special, "bytes_read": c.bytes_read,
                    "bytes_written": c.bytes_written,
                    "stages": {k: list(v) for k, v in st.items()},
                    "halo_extra": perf.halo_extra_read_bytes(plan, spec, isz),
                })
    # a run with counters: shallow water 16x12 periodic, t_end 0.05
    spec = GridSpec(cells=(16, 12), lower=(0.0, 0.0), upper=(1.0, 1.0), num_states=3)
    for tiles in (None, (8, 4)):
        g = create_grid(spec)
        rng = np.random.default_rng(8)
        g.interior()[0] = 1.0 + 0.2 * rng.random((12, 16))
        g.interior()[1:] = 0.1 * rng.standard_normal((2, 12, 16))
        sim = Simulation(g, get_solver("shallow_water"),
                         __import__("clawtile").ShallowWaterParams(1.0),
                         BoundarySpec.uniform(BoundaryKind.PERIODIC, (1, 2)),
                         initial_max_speed=2.5, collect_counters=True, tile_shape=tiles)
        rep = sim.run_until(0.05)
        report = perf.build_report(sim.counters, perf.MachineModel(1e12, 1e11))
        out["runs"].append({
            "tiles": list(tiles) if tiles else None, "attempts": len(rep.attempts),
            "sweeps": sim.counters.sweeps,
            "rows": [[r.scope, r.stage, r.flops, r.special, r.bytes, r.oi, r.bound]
                     for r in report.rows],
            "text": perf.render_text(report), "delimited": perf.render_delimited(report),
        })
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "perf.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0)
    print(f"wrote {path}: {len(out['sweeps'])} sweeps, {len(out['runs'])} runs")


if __name__ == "__main__":
    main()
