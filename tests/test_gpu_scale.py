"""GPU parity at the BASELINE.json sizes and on the production x-sweep
kernels: the product (C ABI, device controller) against the multithreaded
CPU oracle on the same inputs, bit for bit -- every attempt's (t, dt, max
speed, nu, accepted, landed) as float.hex and every state byte.

* C2 SW 1024^2 radial dam-break, 100 steps (one revert on the way);
* C3 3-D two-material acoustics 256^3, superbee, 5 steps;
* C4 SW 16384^2, 2 steps;
* C5 3-D acoustics 512^3 periodic, fp64 and fp32, 2 steps;
* SW 2048^2 / 8192^2 (>= 2^22 cells: the TMA tensor-map x-sweep is the
  automatic choice there) with an under-estimated initial speed, so the
  first attempt reverts and the retry is exact.

Reference semantics: /root/reference/pkg/src/clawtile/timestep.py:188-285
(attempt loop), sweep.py:183-263 (the fused sweep).  These runs take the
oracle tens of seconds each on the GPU box's host cores."""

from __future__ import annotations

import gc

import numpy as np
import pytest

import paper_1805_08846_b200 as P
from paper_1805_08846_b200._native import (XVAR_MARCH, XVAR_PAIR, XVAR_TMA, XVAR_TMA_ADAPT,
                                          XVAR_TMA_STREAM)
from oracle import oracle as O

import cases

pytestmark = pytest.mark.gpu


def _recipe(name, problem, cells, profile, dtype, bc, limiter, steps, speed="bound",
            options=None):
    nd = len(cells)
    lower = (-1.0,) * nd if profile == "radial_dam_break" else (0.0,) * nd
    return dict(name=name, problem=problem, profile=profile, options=options or {},
                cells=cells, lower=lower, upper=(1.0,) * nd, dtype=dtype, bc=bc,
                limiter=limiter, speed=speed, drive=("max_steps", steps))


def _same_bytes(a: np.ndarray, b: np.ndarray) -> bool:
    """Byte equality state by state (no whole-array temporaries)."""
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    u = np.uint64 if a.dtype.itemsize == 8 else np.uint32
    return all(np.array_equal(a[k].view(u), b[k].view(u)) for k in range(a.shape[0]))


def _run_both(r, variant=None):
    grid, params, problem, bspec, speed = cases.build_grid(r)
    sides = [(lo.value, hi.value) for lo, hi in bspec.sides]
    osim = O.OracleSimulation(grid.data.copy(), grid.spec.spacing, problem.solver_name,
                              cases.params_dict(problem, params), sides, bspec.normal_velocity,
                              limiter=r["limiter"], initial_max_speed=speed)
    oatt = cases.drive(osim, r)
    sim = P.Simulation(grid, problem.solver, params, bspec, limiter=P.LimiterKind(r["limiter"]),
                       initial_max_speed=speed)
    del grid
    gc.collect()
    with sim:
        if variant is not None:
            sim.device_grid.set_x_variant(variant)
        used = sim.device_grid.x_variant()
        att = cases.drive(sim, r)
        assert cases.attempts_hex(att) == cases.attempts_hex(oatt)
        assert float(sim.t).hex() == float(osim.t).hex()
        assert (sim.steps_accepted, sim.steps_reverted) == (osim.steps_accepted,
                                                            osim.steps_reverted)
        out = sim.device_grid.download(sim._cur)
    ref = O.interior(osim.grid)
    ok = _same_bytes(out, ref)
    if not ok:
        diff = np.abs(out.astype(np.float64) - ref.astype(np.float64))
        scale = np.maximum(np.abs(ref.astype(np.float64)).max(), 1e-300)
        pytest.fail(f"state differs: max abs {diff.max():.3e}, rel {diff.max() / scale:.3e}")
    return att, used


def test_c2_sw1024_100_steps_with_revert():
    r = _recipe("c2", "shallow_water2d", (1024, 1024), "radial_dam_break", "float64",
                "reflective", "mc", 100)
    att, _ = _run_both(r)
    assert sum(1 for a in att if not a.accepted) >= 1


@pytest.mark.parametrize("variant", [None, XVAR_MARCH, XVAR_PAIR, XVAR_TMA, XVAR_TMA_STREAM],
                         ids=["auto", "warp-march", "pair-march", "tma", "tma-stream"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_sw2048_tma_x_sweep_with_revert(dtype, variant):
    if variant == XVAR_TMA_STREAM and dtype == "float32":
        pytest.skip("the streaming x geometry is fp64 shallow water only")
    r = _recipe("sw2048", "shallow_water2d", (2048, 2048), "radial_dam_break", dtype,
                "reflective", "mc", 3, speed=("scale", 0.5))
    att, used = _run_both(r, variant)
    auto = XVAR_TMA_ADAPT if dtype == "float64" else XVAR_TMA
    assert used == (auto if variant is None else variant)
    assert not att[0].accepted and att[1].accepted


def test_sw8192_north_star_tma_x_sweep():
    r = _recipe("sw8192", "shallow_water2d", (8192, 8192), "radial_dam_break", "float64",
                "reflective", "mc", 3, speed=("scale", 0.5))
    att, used = _run_both(r)
    assert used == XVAR_TMA_ADAPT
    assert not att[0].accepted


@pytest.mark.parametrize("variant", [None, XVAR_TMA_STREAM], ids=["auto", "tma-stream"])
def test_sw8192_hump_active_flow_fp64(variant):
    # flow in every cell: the FastArith second pass is exercised in the far field
    r = _recipe("hump", "shallow_water2d", (4096, 4096), "gaussian_hump", "float64",
                "periodic", "mc", 4)
    _run_both(r, variant)


def test_c3_vc_acoustics_256cube_superbee():
    r = _recipe("c3", "vc_acoustics3d", (256, 256, 256), "two_material_pulse", "float64",
                "reflective", "superbee", 5, speed=("value", 1.0))
    _run_both(r)


def test_c4_sw16384_two_steps():
    r = _recipe("c4", "shallow_water2d", (16384, 16384), "radial_dam_break", "float64",
                "reflective", "mc", 2)
    _, used = _run_both(r)
    assert used == XVAR_TMA_ADAPT


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_c5_acoustics_512cube_periodic(dtype):
    r = _recipe("c5", "acoustics3d", (512, 512, 512), "gaussian_pressure", dtype, "periodic",
                "mc", 2, options={"width": 0.1})
    _run_both(r)


def test_c5_acoustics_pair_march_x():
    r = _recipe("c5", "acoustics3d", (512, 512, 256), "gaussian_pressure", "float64",
                "periodic", "superbee", 2, options={"width": 0.1})
    _, used = _run_both(r, XVAR_PAIR)
    assert used == XVAR_PAIR
