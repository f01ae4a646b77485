"""Time the UNMODIFIED reference CPU path (clawtile, Python + numba) on the
bounded C4 sample the bench's reference arm uses (the middle 1024-row band of
the 16384^2 grid, same profile and boundary kinds), serial and with
workers = cpu_count.  Build-container only: the reference
does not travel to the GPU box, so this number is reported beside the bench's
oracle-port arm (profiles/r2_reference_numba.json), never used as the arm.

    PYTHONDONTWRITEBYTECODE=1 python scripts/time_reference_numba.py [--steps 3]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import bench  # noqa: E402
import clawtile as ct  # noqa: E402


def run(inp, workers, steps):
    prob = bench.WORKLOADS["c4"][0]
    problem = ct.get_problem(prob)
    spec = inp["grid"].spec
    rspec = ct.GridSpec(cells=spec.cells, lower=spec.lower, upper=spec.upper,
                        num_states=spec.num_states)
    g = ct.create_grid(rspec, inp["dtype"])
    assert g.data.shape == inp["grid"].data.shape
    g.data[...] = inp["grid"].data
    bspec = ct.BoundarySpec.uniform(ct.BoundaryKind(inp["bspec"].sides[0][0].value),
                                    problem.normal_velocity)
    tile = None if workers == 1 else (spec.cells[0], max(8, spec.cells[1] // workers))
    with ct.Simulation(g, problem.solver, problem.make_params({}), bspec,
                       limiter=ct.LimiterKind(inp["limiter"].value), workers=workers,
                       tile_shape=tile, initial_max_speed=inp["speed"]) as sim:
        sim.attempt_step()          # numba JIT + first attempt, untimed
        acc0 = sim.steps_accepted
        t0 = time.perf_counter()
        for _ in range(steps):
            sim.attempt_step()
        el = time.perf_counter() - t0
        acc = sim.steps_accepted - acc0
    return spec.num_cells * acc / el / 1e9, el, acc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    gcells = bench.global_cells("c4", 1, "strong")
    inp, sample = bench.cpu_sample_inputs("c4", gcells)
    ncpu = os.cpu_count() or 1
    out = {"metric": bench.METRIC, "unit": bench.UNIT, "workload": "c4", "sample": sample,
           "host_cores": ncpu, "numba": __import__("numba").__version__,
           "note": "build container's cores, not the GPU box's; reference run unmodified "
                   "from /root/reference/pkg/src (clawtile.Simulation.attempt_step)"}
    for workers in (1, ncpu):
        v, el, acc = run(inp, workers, a.steps)
        out[f"workers_{workers}"] = {"value": v, "seconds": el, "steps_accepted": acc}
        print(f"workers={workers}: {v:.4f} {bench.UNIT} ({acc} steps in {el:.1f} s)", flush=True)
    path = os.path.join(ROOT, "profiles", "r2_reference_numba.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
