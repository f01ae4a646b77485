"""Generate golden vectors from the reference clawtile package.

Run HERE (the build container), where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference read-only (numba cache disabled, no bytecode) and
writes small fixtures next to this file:

* sweeps.npz   per-sweep cases: padded input after apply_boundary, axis, dt,
               solver, limiter, dtype -> reference output interior + max |s|
               (reference sweep.py:380-391 sweep_axis)
* solvers.npz  random (q_l, q_r) pairs -> waves, speeds (riemann.py:116-173)
* runs.json    per-run cases through Simulation.run_until / attempt_step:
               every attempt's (t_start, dt, max_speed, nu, accepted, landed)
               as float.hex, plus sha256 of the final interior bytes
               (timestep.py:151-285)
* runs.npz     final interiors of the small runs (for diagnostics)

The GPU box never runs this script; the fixtures travel with the repo.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF)
sys.path.insert(0, REF_TESTS)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from clawtile import (  # noqa: E402
    BoundaryKind, BoundarySpec, LimiterKind, Simulation, apply_boundary,
    build_simulation, create_grid, fill_initial, get_problem, get_solver, loads,
)
from clawtile.grid import GridSpec  # noqa: E402
from clawtile.riemann import (  # noqa: E402
    AcousticsParams, AdvectionParams, RiemannSolver, ShallowWaterParams, register_solver,
)
from clawtile.sweep import sweep_axis  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


# --------------------------------------------------------------------------
# Builder extension solver: variable-coefficient acoustics
# with (Z, c) carried as passive states.  Registered into the UNMODIFIED
# reference engine so the reference sweep/controller act as its oracle.


def _vc_acoustics_scalar(ql, qr, normal, params, W, s):
    m = W.shape[1]
    Zl = ql[m - 2]
    Zr = qr[m - 2]
    cl = ql[m - 1]
    cr = qr[m - 1]
    dp = qr[0] - ql[0]
    dun = qr[normal] - ql[normal]
    denom = Zl + Zr
    a1 = (Zr * dun - dp) / denom
    a2 = (Zl * dun + dp) / denom
    for k in range(m):
        W[0, k] = 0
        W[1, k] = 0
    W[0, 0] = -Zl * a1
    W[0, normal] = a1
    W[1, 0] = Zr * a2
    W[1, normal] = a2
    s[0] = -cl
    s[1] = cr


def _pack_vc(p, dtype):
    return np.zeros(1, dtype=dtype)


VC = RiemannSolver("vc_acoustics", 2, _vc_acoustics_scalar, _pack_vc)
register_solver(VC, overwrite=True)


def make_spec(cells, m, lower=None, upper=None):
    nd = len(cells)
    return GridSpec(cells=tuple(cells), lower=tuple(lower or (0.0,) * nd),
                    upper=tuple(upper or (1.0,) * nd), num_states=m)


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


# --------------------------------------------------------------------------
# Input builders (seeded, as pkg/tests/helpers.py:43-72)


def build_grid(solver, cells, dtype, seed):
    rng = np.random.default_rng(seed)
    nd = len(cells)
    if solver == "acoustics":
        spec = make_spec(cells, nd + 1)
        g = create_grid(spec, dtype)
        g.interior()[...] = 0.1 * rng.standard_normal(g.interior().shape)
        return g, AcousticsParams(1.3, 0.7), {"sound_speed": 1.3, "impedance": 0.7}
    if solver == "shallow_water":
        spec = make_spec(cells, 3)
        g = create_grid(spec, dtype)
        g.data[0] = 1.0
        it = g.interior()
        it[0] = 1.0 + 0.3 * rng.random(it.shape[1:])
        it[1] = 0.2 * rng.standard_normal(it.shape[1:])
        it[2] = 0.2 * rng.standard_normal(it.shape[1:])
        return g, ShallowWaterParams(1.7), {"gravity": 1.7}
    if solver == "advection":
        spec = make_spec(cells, 1)
        g = create_grid(spec, dtype)
        g.interior()[...] = rng.standard_normal(g.interior().shape)
        return g, AdvectionParams(-0.8), {"speed": -0.8}
    if solver == "vc_acoustics":
        spec = make_spec(cells, nd + 3)
        g = create_grid(spec, dtype)
        it = g.interior()
        it[: nd + 1] = 0.1 * rng.standard_normal(it[: nd + 1].shape)
        it[nd + 1] = 1.0 + rng.random(it.shape[1:])          # Z in [1, 2)
        it[nd + 2] = 0.5 + 0.5 * rng.random(it.shape[1:])    # c in [0.5, 1)
        return g, None, {}
    raise KeyError(solver)


def bspec(kind, solver, nd):
    nv = (None,) * nd if solver == "advection" else tuple(range(1, nd + 1))
    return BoundarySpec.uniform(BoundaryKind(kind), nv)


def gen_sweeps():
    cases = []
    shapes = {
        "acoustics": [(12, 7), (5, 6, 4)],
        "shallow_water": [(9, 11), (33, 5)],
        "advection": [(16,), (3,)],
        "vc_acoustics": [(7, 6), (4, 5, 6)],
    }
    seed = 100
    for solver, shp in shapes.items():
        for cells in shp:
            for dtype in (np.float64, np.float32):
                for lim in LimiterKind:
                    for kind in ("outflow", "reflective", "periodic"):
                        if solver == "advection" and kind == "reflective":
                            continue
                        seed += 1
                        grid, params, pdict = build_grid(solver, cells, dtype, seed)
                        apply_boundary(grid, bspec(kind, solver, len(cells)))
                        dt = 0.3 * min(grid.spec.spacing)
                        for axis in range(len(cells)):
                            out = create_grid(grid.spec, grid.dtype)
                            res = sweep_axis(grid, out, axis, dt, get_solver(solver), lim, params)
                            cases.append(dict(
                                solver=solver, cells=cells, dtype=np.dtype(dtype).name,
                                limiter=lim.value, bc=kind, axis=axis, dt=dt,
                                spacing=grid.spec.spacing, params=pdict,
                                qin=grid.data.copy(), qout=out.interior().copy(),
                                smax=res.max_abs_speed,
                            ))
    arrays = {}
    meta = []
    for i, c in enumerate(cases):
        arrays[f"qin_{i}"] = c.pop("qin")
        arrays[f"qout_{i}"] = c.pop("qout")
        c["cells"] = list(c["cells"])
        c["spacing"] = list(c["spacing"])
        c["dt_hex"] = float(c.pop("dt")).hex()
        c["smax_hex"] = float(c.pop("smax")).hex()
        meta.append(c)
    np.savez_compressed(os.path.join(OUT, "sweeps.npz"), **arrays)
    with open(os.path.join(OUT, "sweeps.json"), "w") as fh:
        json.dump(meta, fh, indent=0)
    print(f"sweeps: {len(meta)} cases")


def gen_solvers():
    rng = np.random.default_rng(987654321)
    out = {}
    n = 256
    for dtype in (np.float64, np.float32):
        dn = np.dtype(dtype).name
        # acoustics 3-state, axis alternating
        ql = rng.standard_normal((n, 3)).astype(dtype)
        qr = rng.standard_normal((n, 3)).astype(dtype)
        Ws, Ss = [], []
        for i in range(n):
            fan = get_solver("acoustics").solve(ql[i], qr[i], i % 2, AcousticsParams(1.3, 0.7))
            Ws.append(fan.waves); Ss.append(fan.speeds)
        out[f"acoustics_{dn}_ql"], out[f"acoustics_{dn}_qr"] = ql, qr
        out[f"acoustics_{dn}_W"], out[f"acoustics_{dn}_s"] = np.array(Ws), np.array(Ss)
        h = rng.uniform(0.3, 3.0, size=(n, 2))
        u = rng.uniform(-1.0, 1.0, size=(n, 2, 2))
        ql = np.stack([h[:, 0], h[:, 0] * u[:, 0, 0], h[:, 0] * u[:, 0, 1]], 1).astype(dtype)
        qr = np.stack([h[:, 1], h[:, 1] * u[:, 1, 0], h[:, 1] * u[:, 1, 1]], 1).astype(dtype)
        Ws, Ss = [], []
        for i in range(n):
            fan = get_solver("shallow_water").solve(ql[i], qr[i], i % 2, ShallowWaterParams(1.7))
            Ws.append(fan.waves); Ss.append(fan.speeds)
        out[f"shallow_water_{dn}_ql"], out[f"shallow_water_{dn}_qr"] = ql, qr
        out[f"shallow_water_{dn}_W"], out[f"shallow_water_{dn}_s"] = np.array(Ws), np.array(Ss)
    np.savez_compressed(os.path.join(OUT, "solvers.npz"), **out)
    print("solvers: written")


# --------------------------------------------------------------------------
# Runs


def attempts_record(report_or_list):
    recs = []
    for a in report_or_list:
        recs.append([float(a.t_start).hex(), float(a.dt).hex(), float(a.max_speed).hex(),
                     float(a.nu).hex(), bool(a.accepted), bool(a.landed)])
    return recs


def radial_dam_break(h_in=2.0, h_out=1.0, radius=0.5, center=(0.0, 0.0)):
    def profile(x, y):
        r2 = (x - center[0]) ** 2 + (y - center[1]) ** 2
        h = np.where(r2 < radius * radius, h_in, h_out)
        z = np.zeros_like(h)
        return np.stack([h, z, z])
    return profile


def two_material_pulse(nd):
    # slow coord < 0.5 (Z,c)=(1,1), else (2,0.5); gaussian
    # pulse at (0.5,0.5,0.3) width 0.1
    def profile(*coords):
        cz = coords[-1]
        cen = (0.5, 0.5, 0.3)[-nd:]
        r2 = sum((c - c0) ** 2 for c, c0 in zip(coords, cen))
        p = 1.0 * np.exp(-r2 / 0.1 ** 2)
        zero = np.zeros_like(p)
        Z = np.where(cz < 0.5, 1.0, 2.0)
        c = np.where(cz < 0.5, 1.0, 0.5)
        return np.stack([p] + [zero] * nd + [Z, c])
    return profile


def build_reference(r):
    """Reference-side construction of a recipe (tests/golden/recipes.py)."""
    cells = tuple(r["cells"])
    nd = len(cells)
    dtype = np.dtype(r["dtype"])
    if r["problem"].startswith("vc_acoustics"):
        spec = make_spec(cells, nd + 3, lower=r["lower"], upper=r["upper"])
        grid = create_grid(spec, dtype)
        fill_initial(grid, two_material_pulse(nd))
        solver, params = VC, None
        bound = None
        nv_solver = "acoustics"
    else:
        problem = get_problem(r["problem"])
        spec = make_spec(cells, problem.num_states, lower=r["lower"], upper=r["upper"])
        grid = create_grid(spec, dtype)
        if r["profile"] == "radial_dam_break":
            fill_initial(grid, radial_dam_break())
        else:
            fill_initial(grid, problem.initial_profile(r["profile"], dict(r["options"]), spec))
        params = problem.make_params({})
        solver = problem.solver
        bound = problem.speed_bound(grid, params)
        nv_solver = problem.solver_name
    sp = r["speed"]
    if sp == "bound":
        speed = bound
    elif sp[0] == "scale":
        speed = sp[1] * bound
    else:
        speed = sp[1]
    initial_sha = sha(grid.interior())
    sim = Simulation(grid, solver, params, bspec(r["bc"], nv_solver, nd),
                     limiter=LimiterKind(r["limiter"]), initial_max_speed=speed)
    return sim, initial_sha, speed


def gen_runs():
    from recipes import RUNS
    runs, arrays = [], {}
    for r in RUNS:
        sim, initial_sha, speed = build_reference(r)
        kind = r["drive"][0]
        if kind == "max_steps":
            attempts = sim.run_until(1e30, max_steps=r["drive"][1]).attempts
        else:
            attempts = sim.run_until(r["drive"][1], frame_times=tuple(r["drive"][2])).attempts
        rec = dict(name=r["name"], attempts=attempts_record(attempts), t=float(sim.t).hex(),
                   steps_accepted=sim.steps_accepted, steps_reverted=sim.steps_reverted,
                   sha256=sha(sim.grid.interior()), sha256_initial=initial_sha,
                   initial_speed=float(speed).hex())
        runs.append(rec)
        if sim.grid.interior().nbytes <= 400_000:
            arrays[r["name"]] = sim.grid.interior().copy()
        sim.close()
    with open(os.path.join(OUT, "runs.json"), "w") as fh:
        json.dump(runs, fh, indent=1)
    np.savez_compressed(os.path.join(OUT, "runs.npz"), **arrays)
    print(f"runs: {len(runs)} cases")


if __name__ == "__main__":
    gen_sweeps()
    gen_solvers()
    gen_runs()
