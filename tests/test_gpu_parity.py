"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden vectors and the CPU oracle.  Bar: bit-exact (dt sequence, max wave
speeds, every state byte) in fp64 and fp32; the north star's fallback
tolerances (L-inf rel <= 1e-12 fp64, <= 1e-5 fp32) are asserted where a
full-size run is only checked through properties."""

import math

import numpy as np
import pytest

import paper_1805_08846_b200 as P
from paper_1805_08846_b200._native import (XVAR_AUTO, XVAR_MARCH, XVAR_PAIR, XVAR_TMA,
                                          XVAR_TMA_ADAPT, XVAR_TMA_STREAM, DeviceGrid)
from oracle import oracle as O

import cases

pytestmark = pytest.mark.gpu


def _grid_from_padded(qin, c):
    cells = tuple(c["cells"])
    m = qin.shape[0]
    spec = P.GridSpec(cells, (0.0,) * len(cells), tuple(s * n for s, n in zip(c["spacing"], cells)), m)
    g = P.create_grid(spec, qin.dtype)
    g.data[...] = qin
    return g


@pytest.mark.parametrize("variant", [XVAR_AUTO, XVAR_MARCH, XVAR_TMA, XVAR_PAIR, XVAR_TMA_STREAM,
                                     XVAR_TMA_ADAPT],
                         ids=["auto", "x-march", "x-tma", "x-pair", "x-stream", "x-adapt"])
def test_golden_sweeps_bitwise(golden_sweeps, variant):
    """(The streaming / paired x geometries exist for fp64 shallow water
    only; the other cases run the automatic choice under those ids.)"""
    meta, arrays = golden_sweeps
    bad = []
    for i, c in enumerate(meta):
        qin = arrays[f"qin_{i}"]
        grid = _grid_from_padded(qin, c)
        out = P.create_grid(grid.spec, grid.dtype)
        solver = P.get_solver(c["solver"])
        params = {
            "acoustics": lambda p: P.AcousticsParams(p["sound_speed"], p["impedance"]),
            "shallow_water": lambda p: P.ShallowWaterParams(p["gravity"]),
            "advection": lambda p: P.AdvectionParams(p["speed"]),
            "vc_acoustics": lambda p: P.VcAcousticsParams(),
        }[c["solver"]](c["params"])
        dt = float.fromhex(c["dt_hex"])
        # exact reference spacing: run with dt scaled so dt/dx matches bitwise
        res = _sweep_exact(grid, out, c, dt, solver, params, variant)
        exp = arrays[f"qout_{i}"]
        if out.interior().tobytes() != exp.tobytes() or res != float.fromhex(c["smax_hex"]):
            bad.append((i, c["solver"], c["dtype"], c["limiter"], c["bc"], c["axis"]))
    assert not bad, f"{len(bad)}/{len(meta)} mismatching sweeps, first: {bad[:6]}"


def _sweep_exact(grid, out, c, dt, solver, params, variant=XVAR_AUTO):
    """sweep_axis with the golden case's exact fp64 spacing."""
    nd = len(c["cells"])
    g = DeviceGrid(ndim=nd, cells=tuple(c["cells"]), spacing=tuple(c["spacing"]),
                   num_states=grid.num_states, dtype=grid.dtype,
                   solver_id=solver.require_device(),
                   limiter_id=P.LIMITER_IDS[P.LimiterKind(c["limiter"])],
                   params=solver.pack_params(params, grid.dtype), bc=[(3, 3)] * nd,
                   normal_velocity=[None] * nd)
    try:
        if variant in (XVAR_TMA_STREAM, XVAR_TMA_ADAPT) and not (
                c["solver"] == "shallow_water" and grid.dtype == np.float64):
            variant = XVAR_AUTO
        g.set_x_variant(variant)
        g.upload_padded(0, grid.data)
        smax, _ = g.sweep(c["axis"], dt, 0, 1)
        out.interior()[...] = g.download(1)
        return smax
    finally:
        g.close()


def test_sweep_axis_api_matches_oracle(rng):
    # the public per-sweep operator (sweep.py:380-391 contract)
    for dtype in (np.float64, np.float32):
        spec = P.GridSpec((37, 29), (0.0, 0.0), (1.0, 1.0), 3)
        g = P.create_grid(spec, dtype)
        g.data[0] = 1.0
        g.interior()[0] = 1.0 + 0.3 * rng.random((29, 37))
        g.interior()[1:] = 0.2 * rng.standard_normal((2, 29, 37))
        P.apply_boundary(g, P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2)))
        for axis in (0, 1):
            out = P.create_grid(spec, dtype)
            res = P.sweep_axis(g, out, axis, 0.004, P.get_solver("shallow_water"),
                               P.LimiterKind.MC, P.ShallowWaterParams(1.0))
            ref = np.zeros_like(g.data)
            smax = O.sweep(g.data.copy(), ref, axis, 0.004, spec.spacing, "shallow_water", "mc",
                           {"gravity": 1.0})
            assert out.data.tobytes() == ref.tobytes()
            assert res.max_abs_speed == smax


@pytest.mark.parametrize("name", ["acoustics", "shallow_water"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_solver_pairs_bitwise(golden_solvers, name, dtype):
    ql = golden_solvers[f"{name}_{dtype}_ql"]
    qr = golden_solvers[f"{name}_{dtype}_qr"]
    We = golden_solvers[f"{name}_{dtype}_W"]
    se = golden_solvers[f"{name}_{dtype}_s"]
    params = P.AcousticsParams(1.3, 0.7) if name == "acoustics" else P.ShallowWaterParams(1.7)
    solver = P.get_solver(name)
    for axis in (0, 1):
        sel = np.arange(ql.shape[0]) % 2 == axis
        g = DeviceGrid(ndim=2, cells=(4, 4), spacing=(1.0, 1.0), num_states=3, dtype=dtype,
                       solver_id=solver.device_id, limiter_id=0,
                       params=solver.pack_params(params, np.dtype(dtype)), bc=[(0, 0)] * 2,
                       normal_velocity=[None] * 2)
        W, s = g.solve_pairs(axis, ql[sel], qr[sel], solver.num_waves)
        g.close()
        assert W.tobytes() == We[sel].tobytes()
        assert s.tobytes() == se[sel].tobytes()


@pytest.mark.parametrize("name", sorted(cases.RECIPES))
def test_golden_runs_bitwise(golden_runs, name):
    """dt / speed / nu / accept sequence and final state, bit for bit."""
    r = cases.RECIPES[name]
    g = golden_runs[name]
    sim, grid = cases.product_sim(r)
    with sim:
        attempts = cases.drive(sim, r)
        assert cases.attempts_hex(attempts) == g["attempts"]
        assert float(sim.t).hex() == g["t"]
        assert cases.sha(sim.grid.interior()) == g["sha256"]
        assert sim.steps_reverted == g["steps_reverted"]


SHAPES = [
    ("shallow_water2d", (97, 61), "radial_dam_break", {}),
    ("shallow_water2d", (300, 17), "gaussian_hump", {"amplitude": 0.7}),
    ("acoustics2d", (129, 70), "gaussian_pressure", {"width": 0.15}),
    ("acoustics3d", (33, 20, 18), "gaussian_pressure", {"width": 0.2}),
    ("vc_acoustics3d", (20, 17, 26), "two_material_pulse", {}),
    ("vc_acoustics2d", (41, 37), "two_material_pulse", {"center": (0.5, 0.3)}),
]


def _recipe(problem, cells, profile, options, dtype, bc, limiter, steps):
    nd = len(cells)
    lower = (-1.0,) * nd if profile == "radial_dam_break" else (0.0,) * nd
    return dict(name="adhoc", problem=problem, profile=profile, options=options, cells=cells,
                lower=lower, upper=(1.0,) * nd, dtype=dtype, bc=bc, limiter=limiter,
                speed="bound" if not problem.startswith("vc") else ("value", 1.0),
                drive=("max_steps", steps))


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"{s[0]}-{'x'.join(map(str, s[1]))}")
@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("bc", ["outflow", "reflective", "periodic"])
@pytest.mark.parametrize("limiter", ["mc", "superbee", "minmod", "vanleer", "none"])
@pytest.mark.parametrize("variant", [XVAR_MARCH, XVAR_TMA, XVAR_PAIR],
                         ids=["x-march", "x-tma", "x-pair"])
def test_random_configs_match_oracle(shape, dtype, bc, limiter, variant):
    """Both x-sweep kernels (forced per handle) on every shape / BC / limiter."""
    problem, cells, profile, options = shape
    r = _recipe(problem, cells, profile, options, dtype, bc, limiter, steps=4)
    osim, _ = cases.oracle_sim(r)
    oatt = cases.drive(osim, r)
    sim, _ = cases.product_sim(r)
    with sim:
        sim.device_grid.set_x_variant(variant)
        assert sim.device_grid.x_variant() == variant
        att = cases.drive(sim, r)
        assert cases.attempts_hex(att) == cases.attempts_hex(oatt)
        assert sim.grid.interior().tobytes() == O.interior(osim.grid).tobytes()


@pytest.mark.parametrize("shape", SHAPES[:2], ids=lambda s: f"{s[0]}-{'x'.join(map(str, s[1]))}")
@pytest.mark.parametrize("bc", ["outflow", "reflective", "periodic"])
@pytest.mark.parametrize("limiter", ["mc", "superbee", "minmod", "vanleer", "none"])
@pytest.mark.parametrize("variant", [XVAR_TMA_STREAM, XVAR_TMA_ADAPT],
                         ids=["x-stream", "x-adapt"])
def test_streaming_x_geometry_matches_oracle(shape, bc, limiter, variant):
    """fp64 shallow water's second TMA x geometry (64 rows x 128 B), forced
    and paired with the default one (the previous strided sweep's activity
    selects the twin that works, attempt by attempt)."""
    problem, cells, profile, options = shape
    r = _recipe(problem, cells, profile, options, "float64", bc, limiter, steps=6)
    osim, _ = cases.oracle_sim(r)
    oatt = cases.drive(osim, r)
    sim, _ = cases.product_sim(r)
    with sim:
        sim.device_grid.set_x_variant(variant)
        assert sim.device_grid.x_variant() == variant
        att = cases.drive(sim, r)
        assert cases.attempts_hex(att) == cases.attempts_hex(oatt)
        assert sim.grid.interior().tobytes() == O.interior(osim.grid).tobytes()


@pytest.mark.parametrize("profile,expect_stream", [("radial_dam_break", True),
                                                   ("gaussian_hump", False)],
                         ids=["dam-break-quiescent", "hump-active"])
def test_geometry_pair_selects_by_activity(profile, expect_stream):
    """The pair's selector after an attempt holds the y sweep's computed warp
    groups: far below the threshold for an early dam break (most groups
    skipped, so the next x sweep runs the streaming twin), above it for flow
    active everywhere; results stay bitwise equal to the oracle."""
    r = _recipe("shallow_water2d", (2048, 2048), profile, {}, "float64", "reflective", "mc",
                steps=2)
    osim, _ = cases.oracle_sim(r)
    oatt = cases.drive(osim, r)
    sim, _ = cases.product_sim(r)
    with sim:
        assert sim.device_grid.x_variant() == XVAR_TMA_ADAPT
        computed, thresh = sim.device_grid.x_activity()
        assert computed == 2**64 - 1          # before any strided sweep: default twin
        att = cases.drive(sim, r)             # the device controller's graph
        computed, thresh = sim.device_grid.x_activity()
        assert thresh == int(0.08 * (2048 // 32) * ((2048 + 2) // 3))
        assert (computed < thresh) == expect_stream, (computed, thresh)
        assert cases.attempts_hex(att) == cases.attempts_hex(oatt)
        assert sim.grid.interior().tobytes() == O.interior(osim.grid).tobytes()


def test_streaming_x_geometry_is_fp64_shallow_water_only():
    r = _recipe("acoustics2d", (64, 40), "gaussian_pressure", {"width": 0.15}, "float64",
                "periodic", "mc", steps=1)
    sim, _ = cases.product_sim(r)
    with sim:
        for v in (XVAR_TMA_STREAM, XVAR_TMA_ADAPT):
            with pytest.raises(Exception, match="fp64 2-D shallow water"):
                sim.device_grid.set_x_variant(v)
        with pytest.raises(Exception, match="geometry pair"):
            sim.device_grid.x_activity()
    r = _recipe("shallow_water2d", (64, 40), "radial_dam_break", {}, "float32", "periodic", "mc",
                steps=1)
    sim, _ = cases.product_sim(r)
    with sim:
        with pytest.raises(Exception, match="fp64 2-D shallow water"):
            sim.device_grid.set_x_variant(XVAR_TMA_STREAM)


@pytest.mark.parametrize("variant", [XVAR_MARCH, XVAR_TMA, XVAR_PAIR, XVAR_TMA_STREAM],
                         ids=["x-march", "x-tma", "x-pair", "x-stream"])
@pytest.mark.parametrize("seg", [(1, 1), (7, 5), (33, 40), (64, 3), (1000, 1000)])
def test_segmentation_is_bitwise_invisible(seg, variant):
    r = _recipe("shallow_water2d", (150, 130), "radial_dam_break", {}, "float64", "reflective",
                "mc", 3)
    ref_sim, _ = cases.product_sim(r)
    with ref_sim:
        cases.drive(ref_sim, r)
        ref = ref_sim.grid.interior().copy()
    sim, _ = cases.product_sim(r)
    with sim:
        sim.device_grid.set_x_variant(variant)
        sim.device_grid.set_segments(0, seg[0])
        sim.device_grid.set_segments(1, seg[1])
        cases.drive(sim, r)
        assert sim.grid.interior().tobytes() == ref.tobytes()


def test_revert_restores_state_bitwise():
    r = cases.RECIPES["dam_break_revert_64x16"]
    sim, _ = cases.product_sim(r)
    reverts = 0
    with sim:
        while sim.t < 0.15:
            before = sim.grid.interior().tobytes()
            t0 = sim.t
            a = sim.attempt_step(stop=0.15)
            if a.accepted:
                assert a.nu <= 1.0
            else:
                reverts += 1
                assert sim.t == t0
                assert sim.grid.interior().tobytes() == before
    assert reverts >= 1 and sim.steps_reverted == reverts


def test_underestimate_revert_then_exact_retry():
    # pkg/tests/test_timestep.py:88-105: nu = 1.8, retry dt = 0.45 dx, retry nu = 0.9
    spec = P.GridSpec((8, 8), (0, 0), (1, 1), 3)
    g = P.create_grid(spec)
    g.data[0] = 4.0
    sim = P.Simulation(g, P.get_solver("shallow_water"), P.ShallowWaterParams(1.0),
                       P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2)),
                       initial_max_speed=1.0, cfl_target=0.9)
    before = sim.grid.data.tobytes()
    a = sim.attempt_step()
    assert not a.accepted and a.nu == pytest.approx(1.8) and a.dt_retry == pytest.approx(0.45 / 8)
    assert sim.grid.data.tobytes() == before
    b = sim.attempt_step()
    assert b.accepted and b.nu == pytest.approx(0.9)
    sim.last_max_speed = 1.0
    sim2 = P.Simulation(P.create_grid(spec), P.get_solver("shallow_water"),
                        P.ShallowWaterParams(1.0),
                        P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2)),
                        initial_max_speed=1.0)
    sim2.grid.data[0] = 4.0
    sim2.attempt_step()
    sim2.last_max_speed = 1.0
    with pytest.raises(P.UnstableStepError):
        sim2.attempt_step()


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("where", [(3, 4), (0, 0), (15, 15)])
def test_blowup_location_matches_oracle(dtype, where):
    spec = P.GridSpec((16, 16), (0, 0), (1, 1), 3)
    rng = np.random.default_rng(1)
    g = P.create_grid(spec, dtype)
    g.interior()[...] = 0.05 * rng.standard_normal(g.interior().shape)
    sim = P.Simulation(g, P.get_solver("acoustics"), P.AcousticsParams(),
                       P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2)),
                       initial_max_speed=1.0)
    sim.grid.interior(0)[where] = np.nan
    data = sim.grid.data.copy()
    osim = O.OracleSimulation(data, spec.spacing, "acoustics",
                              {"sound_speed": 1.0, "impedance": 1.0},
                              [("periodic", "periodic")] * 2, (1, 2), initial_max_speed=1.0)
    with pytest.raises(O.OracleBlowup) as oexc:
        osim.attempt_step()
    with pytest.raises(P.NumericalBlowup) as exc:
        sim.attempt_step()
    assert (exc.value.state, exc.value.cell, exc.value.step) == \
        (oexc.value.state, oexc.value.cell, oexc.value.step)


def test_dry_state_blowup_in_shallow_water_matches_oracle():
    spec = P.GridSpec((24, 20), (0, 0), (1, 1), 3)
    g = P.create_grid(spec)
    g.interior()[0] = 1.0
    g.interior()[0][5, 7] = -0.5  # negative depth -> NaN speeds
    sim = P.Simulation(g, P.get_solver("shallow_water"), P.ShallowWaterParams(),
                       P.BoundarySpec.uniform(P.BoundaryKind.OUTFLOW, (1, 2)),
                       initial_max_speed=1.5)
    osim = O.OracleSimulation(g.data.copy(), spec.spacing, "shallow_water", {"gravity": 1.0},
                              [("outflow", "outflow")] * 2, (1, 2), initial_max_speed=1.5)
    with pytest.raises(O.OracleBlowup) as oexc:
        osim.attempt_step()
    with pytest.raises(P.NumericalBlowup) as exc:
        sim.attempt_step()
    assert (exc.value.state, exc.value.cell) == (oexc.value.state, oexc.value.cell)


def test_build_simulation_from_config():
    text = """[run]
problem = acoustics2d
t_end = 0.6
[grid]
cells = 256 256
[scheme]
limiter = mc
[boundary]
all = reflective
[initial]
profile = gaussian_pressure
amplitude = 1.0
width = 0.08
[parallel]
serial = true
"""
    with P.build_simulation(P.loads(text)) as sim:
        sim.run_until(1e30, max_steps=100)
        assert cases.sha(sim.grid.interior()).startswith("429c7880ae08b44f")
        assert sim.t == 0.35156250000000033


def test_large_periodic_conservation_fp64():
    """Size-independent property at a large grid: periodic sweeps conserve
    every state's interior sum to rounding (pkg/tests/test_acceptance.py:183-198)."""
    n = 2048
    spec = P.GridSpec((n, n), (0, 0), (1, 1), 3)
    g = P.create_grid(spec)
    P.fill_initial(g, P.get_problem("shallow_water2d").initial_profile("gaussian_hump", {}, spec))
    g.interior()[1] = 0.1
    before = g.interior().sum(axis=(1, 2))
    scale = np.abs(g.interior()).sum(axis=(1, 2))
    bound = P.get_problem("shallow_water2d").speed_bound(g, P.ShallowWaterParams())
    with P.Simulation(g, P.get_solver("shallow_water"), P.ShallowWaterParams(),
                      P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2)),
                      initial_max_speed=bound) as sim:
        sim.run_until(1e30, max_steps=5)
        after = sim.grid.interior().sum(axis=(1, 2))
    assert np.max(np.abs(after - before) / np.maximum(scale, 1.0)) < 1e-12


def test_large_grid_matches_oracle_fp32_and_fp64():
    for dtype in ("float64", "float32"):
        r = _recipe("shallow_water2d", (1024, 768), "radial_dam_break", {}, dtype, "reflective",
                    "mc", 3)
        osim, _ = cases.oracle_sim(r)
        oatt = cases.drive(osim, r)
        sim, _ = cases.product_sim(r)
        with sim:
            att = cases.drive(sim, r)
            assert cases.attempts_hex(att) == cases.attempts_hex(oatt)
            a = sim.grid.interior()
            b = O.interior(osim.grid)
            assert a.tobytes() == b.tobytes()


def _arith_inputs(rng, n):
    """Random bit patterns (every exponent, sign, NaN/inf/subnormal class)
    plus hand-picked edges of the div.rn / sqrt.rn fast-path domains."""
    bits = rng.integers(0, 2**64, size=(2, n), dtype=np.uint64)
    a, b = bits.view(np.float64)
    specials = np.array([0.0, -0.0, 1.0, -1.0, 0.5, 2.0, 3.0, np.inf, -np.inf, np.nan,
                         5e-324, -5e-324, 2.2250738585072014e-308, 1e-300, 1e-308, 1e-310,
                         2.0**-967, 2.0**-966, 2.0**-968, 2.0**-1000, 1e300, 1.7976931348623157e308,
                         2.0**1017, 2.0**1016, 2.0**1018, 2.0**-970, 2.0**-900, 0.1, 7.0, 1e-5])
    ea, eb = np.meshgrid(specials, specials)
    # smooth magnitudes like a simulation's: ratios near 1, tiny jumps, zeros
    c = rng.standard_normal(n) * 10.0 ** rng.integers(-20, 20, n)
    d = rng.standard_normal(n) * 10.0 ** rng.integers(-20, 20, n)
    c[rng.random(n) < 0.1] = 0.0
    return np.concatenate([a, ea.ravel(), c]), np.concatenate([b, eb.ravel(), d])


def test_fast_division_and_sqrt_are_bitwise_ieee(rng):
    from paper_1805_08846_b200._native import selftest_arith
    a, b = _arith_inputs(rng, 1 << 22)
    (dmis, smis, dfall, sfall, fdmis, fsmis, fdfall, fsfall,
     lmis, lfall, rmis, rfall) = selftest_arith(a, b)
    assert (dmis, smis, fdmis, fsmis, lmis, rmis) == (0, 0, 0, 0, 0, 0)
    # the edges do exercise the exact fallback
    assert min(dfall, sfall, fdfall, fsfall, lfall, rfall) > 0


@pytest.mark.parametrize("variant", [XVAR_MARCH, XVAR_TMA, XVAR_PAIR, XVAR_TMA_STREAM],
                         ids=["x-march", "x-tma", "x-pair", "x-stream"])
@pytest.mark.parametrize("limiter", ["mc", "vanleer", "superbee"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_slow_path_inputs_match_oracle(rng, limiter, dtype, variant):
    """Shallow-water sweeps over states that push divisions and square roots
    outside their fast-path domain (subnormal and 1e-300-scale momenta, tiny
    depth jumps, exact zeros): the per-step exact recomputation must keep
    every byte equal to the oracle."""
    if variant == XVAR_TMA_STREAM and dtype != "float64":
        pytest.skip("the streaming x geometry is fp64 shallow water only")
    spec = P.GridSpec((67, 45), (0.0, 0.0), (1.0, 1.0), 3)
    g = P.create_grid(spec, dtype)
    g.data[0] = 1.0
    h = 1.0 + 1e-3 * rng.random((45, 67))
    h[rng.random((45, 67)) < 0.3] = 1.0
    g.interior()[0] = h
    mom = rng.standard_normal((2, 45, 67))
    scales = ([0.0, 5e-324, 1e-310, 1e-300, 2.0**-960, 1e-150, 1e-3, 0.1] if dtype == "float64"
              else [0.0, 1e-45, 1e-40, 1e-38, 1e-30, 1e-20, 1e-3, 0.1])
    scale = rng.choice(scales, size=(2, 45, 67))
    g.interior()[1:] = mom * scale
    P.apply_boundary(g, P.BoundarySpec.uniform(P.BoundaryKind.REFLECTIVE, (1, 2)))
    from paper_1805_08846_b200 import sweep as SW
    op = SW._operator(spec, np.dtype(dtype), P.get_solver("shallow_water"),
                      P.LimiterKind(limiter), P.ShallowWaterParams(1.0))
    op.set_x_variant(variant)
    for axis in (0, 1):
        out = P.create_grid(spec, dtype)
        try:
            res = P.sweep_axis(g, out, axis, 0.004, P.get_solver("shallow_water"),
                               P.LimiterKind(limiter), P.ShallowWaterParams(1.0))
        finally:
            op.set_x_variant(XVAR_AUTO)
        ref = np.zeros_like(g.data)
        smax = O.sweep(g.data.copy(), ref, axis, 0.004, spec.spacing, "shallow_water", limiter,
                       {"gravity": 1.0})
        assert out.interior().tobytes() == O.interior(ref).tobytes()
        assert res.max_abs_speed == smax


# ---------------------------------------------------------------------------
# Device-resident controller (clb_run_batch): run_until's attempt loop on the
# device must reproduce the host loop exactly -- attempts, reverts, frames,
# final state, counters and exceptions.

def _both_modes(r, cap=4096, **kw):
    out = []
    for dc in (False, True):
        sim, _ = cases.product_sim(r, device_controller=dc)
        sim._batch_log_cap = cap
        frames = []
        with sim:
            rep = sim.run_until(r["drive"][1], frame_times=tuple(r["drive"][2]),
                                on_frame=lambda s: frames.append((s.t, cases.sha(s.grid.interior())))) \
                if r["drive"][0] == "until" else sim.run_until(1e30, max_steps=r["drive"][1])
            out.append((cases.attempts_hex(rep.attempts), [a.dt_retry for a in rep.attempts],
                        rep.steps_accepted, rep.steps_reverted, float(rep.nu_max).hex(),
                        float(rep.t_final).hex(), frames, cases.sha(sim.grid.interior()),
                        sim.steps_accepted, sim.steps_reverted, float(sim.last_max_speed).hex(),
                        sim._prev_reverted, float(sim.nu_max).hex()))
    return out


@pytest.mark.parametrize("name", sorted(cases.RECIPES))
@pytest.mark.parametrize("cap", [4096, 3])
def test_device_controller_matches_host_loop(name, cap):
    host, dev = _both_modes(cases.RECIPES[name], cap)
    assert dev == host


def test_device_controller_reverts_and_frames():
    r = dict(cases.RECIPES["dam_break_revert_64x16"])
    r["drive"] = ("until", 0.15, (0.01, 0.05, 0.1))
    host, dev = _both_modes(r)
    assert dev == host
    assert host[3] >= 1 and len(host[6]) == 3


def test_device_controller_unstable_step_error():
    spec = P.GridSpec((8, 8), (0, 0), (1, 1), 3)
    msgs = []
    for dc in (False, True):
        g = P.create_grid(spec)
        g.data[0] = 4.0
        sim = P.Simulation(g, P.get_solver("shallow_water"), P.ShallowWaterParams(1.0),
                           P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2)),
                           initial_max_speed=1.0, device_controller=dc)
        sim.attempt_step()                       # revert (nu = 1.8)
        sim.last_max_speed = 1.0                 # engineered under-estimate again
        with pytest.raises(P.UnstableStepError) as exc:
            sim.run_until(1.0)
        msgs.append((str(exc.value), sim.steps_reverted, float(sim.last_max_speed).hex()))
        sim.close()
    assert msgs[0] == msgs[1]


@pytest.mark.parametrize("where", [(3, 4), (15, 0)])
def test_device_controller_blowup_location(where):
    spec = P.GridSpec((16, 16), (0, 0), (1, 1), 3)
    base = 0.05 * np.random.default_rng(1).standard_normal((3, 16, 16))
    res = []
    for dc in (False, True):
        g = P.create_grid(spec)
        g.interior()[...] = base
        sim = P.Simulation(g, P.get_solver("acoustics"), P.AcousticsParams(),
                           P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2)),
                           initial_max_speed=1.0, device_controller=dc)
        sim.run_until(1e30, max_steps=3)
        sim.grid.interior(0)[where] = np.inf
        with pytest.raises(P.NumericalBlowup) as exc:
            sim.run_until(1e30, max_steps=5)
        res.append((exc.value.state, exc.value.cell, exc.value.step, sim.steps_accepted))
        sim.close()
    assert res[0] == res[1]


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_segment_range_launches_compose_bitwise(dtype):
    """clb_sweep_async_range: the slow-axis sweep split into interior and
    edge segment launches (multi-GPU overlap) equals one full launch."""
    problem = P.get_problem("shallow_water2d")
    spec = P.GridSpec((70, 203), (-1, -1), (1, 1), 3)
    g = P.create_grid(spec, np.dtype(dtype))
    P.fill_initial(g, problem.initial_profile("radial_dam_break", {}, spec))
    params = problem.make_params({})
    outs = []
    for split in (False, True):
        sim = P.Simulation(g, problem.solver, params,
                           P.BoundarySpec.uniform(P.BoundaryKind.REFLECTIVE, (1, 2)),
                           initial_max_speed=problem.speed_bound(g, params))
        dev = sim.device_grid
        dev.set_segments(1, 16)
        nseg, seg_len = dev.segments(1)
        assert nseg >= 3
        dev.sweep_async(0, 0.002, 0, 1, 0)
        if split:
            dev.sweep_async_range(1, 0.002, 1, 2, 1, 1, nseg - 1)
            dev.sweep_async_range(1, 0.002, 1, 2, 1, nseg - 1, nseg)
            dev.sweep_async_range(1, 0.002, 1, 2, 1, 0, 1)
        else:
            dev.sweep_async(1, 0.002, 1, 2, 1)
        speeds, flags = dev.fetch(2)
        outs.append((dev.download(2).tobytes(), speeds, flags))
        sim.close()
    assert outs[0] == outs[1]
