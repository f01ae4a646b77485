"""User device Riemann solvers (the reference's plugin ABI on the device,
riemann.py:190-212 / 259-262; paper_1805_08846_b200/devsolver.py).

A solver given as CUDA source for its scalar routine is compiled at run
time and must reproduce the UNMODIFIED reference engine running the same
scalar bit for bit (golden runs made by tests/golden/make_user_solvers.py
and, for the variable-coefficient acoustics scalar, make_golden.py)."""

from __future__ import annotations

import ctypes
import json
import os

import numpy as np
import pytest

import paper_1805_08846_b200 as P
from paper_1805_08846_b200 import devsolver

import cases

HERE = os.path.dirname(os.path.abspath(__file__))

BURGERS_CU = """
W[0][0] = qr[0] - ql[0];
s[0] = T(0.5) * (ql[0] + qr[0]);
"""

# the builder's vc-acoustics scalar (tests/golden/make_golden.py), as CUDA
VC_CU = """
const T Zl = ql[M - 2], Zr = qr[M - 2];
const T cl = ql[M - 1], cr = qr[M - 1];
const T dp = qr[0] - ql[0];
const T dun = qr[normal] - ql[normal];
const T denom = Zl + Zr;
const T a1 = (Zr * dun - dp) / denom;
const T a2 = (Zl * dun + dp) / denom;
W[0][0] = -Zl * a1;
W[0][normal] = a1;
W[1][0] = Zr * a2;
W[1][normal] = a2;
s[0] = -cl;
s[1] = cr;
"""


def _pack_none(p, dtype):
    return np.zeros(1, dtype=dtype)


def burgers():
    return P.RiemannSolver("burgers_user", 1, None, _pack_none, normal_index=lambda axis: 0,
                           device_source=BURGERS_CU)


def _profile(nd):
    if nd == 2:
        return lambda x, y: 0.6 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y) + 0.1
    return lambda x, y, z: (0.5 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y)
                            * np.cos(2 * np.pi * z))


def test_generated_source_cross_compiles():
    """The build hook itself (nvcc for sm_100a, no GPU needed)."""
    so = devsolver.compile_solver("burgers_user", BURGERS_CU, 1, 2, 1, (0, 0), (8, 4))
    L = ctypes.CDLL(so)
    for name in ("clb_user_launch_f32", "clb_user_launch_f64", "clb_user_pairs_f32",
                 "clb_user_pairs_f64"):
        assert getattr(L, name)
    with pytest.raises(ValueError, match="failed to compile"):
        devsolver.compile_solver("broken", "W[0][0] = undefined_name;", 1, 1, 1, (0,), (8,))


def test_registration_checks_the_argument_block():
    from paper_1805_08846_b200._native import lib
    L = lib()
    assert L.clb_register_device_solver(16, 2, 1, 1, L.clb_sweep_args_size() + 8, None, None,
                                        None, None) != 0
    assert L.clb_register_device_solver(3, 2, 1, 1, L.clb_sweep_args_size(), None, None,
                                        None, None) != 0


@pytest.mark.gpu
@pytest.mark.parametrize("case", json.load(open(os.path.join(HERE, "golden",
                                                             "user_solvers.json"))),
                         ids=lambda c: c["name"])
def test_user_burgers_matches_reference_engine(case):
    nd = len(case["cells"])
    spec = P.GridSpec(tuple(case["cells"]), (0.0,) * nd, (1.0,) * nd, 1)
    g = P.create_grid(spec, np.dtype(case["dtype"]))
    P.fill_initial(g, _profile(nd))
    speed = float.fromhex(case["speed"])
    assert speed == float(np.max(np.abs(g.interior())))
    bspec = P.BoundarySpec.uniform(P.BoundaryKind(case["bc"]), (None,) * nd)
    with P.Simulation(g, burgers(), None, bspec, limiter=P.LimiterKind(case["limiter"]),
                      initial_max_speed=speed) as sim:
        rep = sim.run_until(1e30, max_steps=case["steps"])
        assert cases.attempts_hex(rep.attempts) == case["attempts"]
        assert cases.sha(sim.grid.interior()) == case["sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in sorted(cases.RECIPES) if n.startswith("vc_")])
def test_user_vc_scalar_matches_reference_engine(golden_runs, name):
    """The vc-acoustics scalar registered as user CUDA (all wave components
    carried, no structural-zero elision) against the reference engine's runs
    with the Python scalar registered."""
    r = cases.RECIPES[name]
    grid, params, problem, bspec, speed = cases.build_grid(r)
    user = P.RiemannSolver("vc_user", 2, None, problem.solver.pack_params,
                           device_source=VC_CU)
    with P.Simulation(grid, user, params, bspec, limiter=P.LimiterKind(r["limiter"]),
                      initial_max_speed=speed) as sim:
        att = cases.drive(sim, r)
        g = golden_runs[name]
        assert cases.attempts_hex(att) == g["attempts"]
        assert cases.sha(sim.grid.interior()) == g["sha256"]


@pytest.mark.gpu
def test_user_solver_pairs_and_sweep_operator():
    """RiemannSolver.solve and sweep_axis through a user solver."""
    b = burgers()
    fan = b.solve(np.array([0.3]), np.array([-0.7]), 0, None)
    assert fan.waves.tolist() == [[-1.0]] and fan.speeds.tolist() == [0.5 * (0.3 + -0.7)]
    spec = P.GridSpec((24, 20), (0.0, 0.0), (1.0, 1.0), 1)
    g = P.create_grid(spec)
    P.fill_initial(g, _profile(2))
    P.apply_boundary(g, P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (None, None)))
    out = P.create_grid(spec)
    res = P.sweep_axis(g, out, 1, 0.01, b, P.LimiterKind.MC, None)
    assert res.max_abs_speed > 0.0 and np.all(np.isfinite(out.interior()))
