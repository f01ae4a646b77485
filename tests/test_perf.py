"""Perf model (§8(f) row 2).

* The reference's model (clawtile/perf.py), restated in perf.py, against
  golden counters the reference itself produced (tests/golden/make_perf.py ->
  perf.json): per-sweep flops / special / bytes / stage split / halo bytes for
  every solver, limiter, item size and tile plan of the matrix, and the
  report rows of a run with counters on.  Plus the reference's own
  contracts (pkg/tests/test_perf.py): the published OI fixtures, the byte
  and event model, transverse scaling, fp32 halving, the halo closed form,
  report shape.
* The B200 kernel model: prices of the arithmetic the kernels execute.
* On the GPU: Simulation.counters / SweepResult.counters, and the measured
  report (kernel model + reference model + measured kernel times).
"""

import json
import math
import os

import numpy as np
import pytest

import paper_1805_08846_b200 as P
from paper_1805_08846_b200 import perf as F

MIB = 2 ** 20
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def golden_perf():
    with open(os.path.join(HERE, "golden", "perf.json")) as fh:
        return json.load(fh)


def _spec(cells, m):
    return P.GridSpec(tuple(cells), (0.0,) * len(cells), (1.0,) * len(cells), m)


# ---------------------------------------------------------------------------
# the reference's model, pinned to the reference


def test_sweep_counters_match_reference(golden_perf):
    bad = []
    for c in golden_perf["sweeps"]:
        spec = _spec(c["cells"], c["m"])
        plan = P.plan_tiles(spec, c["axis"], tuple(c["tiles"]) if c["tiles"] else spec.cells)
        k, st = F.sweep_counters(plan, spec, P.get_solver(c["solver"]),
                                 P.LimiterKind(c["limiter"]), c["itemsize"])
        got = (k.flops, k.special, k.bytes_read, k.bytes_written,
               {n: list(v) for n, v in st.items()},
               F.halo_extra_read_bytes(plan, spec, c["itemsize"]))
        want = (c["flops"], c["special"], c["bytes_read"], c["bytes_written"], c["stages"],
                c["halo_extra"])
        if got != want:
            bad.append((c["solver"], c["limiter"], c["cells"], c["tiles"], got, want))
    assert not bad, f"{len(bad)} mismatches, first: {bad[:2]}"


def test_run_report_rows_match_reference(golden_perf):
    for run in golden_perf["runs"]:
        rc = F.RunCounters()
        spec = _spec((16, 12), 3)
        tiles = tuple(run["tiles"]) if run["tiles"] else spec.cells
        # the run's sweeps: 2 per attempt (x then y), every attempt counted
        for axis in (0, 1):
            plan = P.plan_tiles(spec, axis, tiles)
            c, st = F.sweep_counters(plan, spec, P.get_solver("shallow_water"),
                                     P.LimiterKind.MC, 8)
            rc.add_sweeps(axis, c, st, run["attempts"])
        assert rc.sweeps == run["sweeps"]
        rep = F.build_report(rc, F.MachineModel(1e12, 1e11))
        rows = [[r.scope, r.stage, r.flops, r.special, r.bytes, r.oi, r.bound] for r in rep.rows]
        assert rows == run["rows"]
        assert F.render_text(rep) == run["text"]
        assert F.render_delimited(rep) == run["delimited"]


def test_published_operational_intensities():
    # PAPER.md:454-488 via pkg/tests/test_perf.py:36-45
    ac = F.KernelCounters(flops=(103 + 118) * 10**6, bytes_read=int(35.1 * MIB),
                          bytes_written=int(41.4 * MIB))
    assert F.operational_intensity(ac) == pytest.approx(2.77, abs=0.02)
    sw = F.KernelCounters(flops=(153 + 175) * 10**6, bytes_read=int(27.0 * MIB),
                          bytes_written=int(37.0 * MIB))
    assert F.operational_intensity(sw) == pytest.approx(4.90, abs=0.02)


def test_roofline_arithmetic():
    m = F.MachineModel(peak_flops=1000e9, peak_bandwidth=100e9)
    assert F.roofline_bound(2.0, m) == pytest.approx(200e9)
    assert F.roofline_bound(1e6, m) == 1000e9
    ridge = m.peak_flops / m.peak_bandwidth
    assert F.roofline_bound(ridge, m) == m.peak_flops
    assert F.roofline_bound(ridge * 0.999, m) < m.peak_flops
    with pytest.raises(ValueError):
        F.roofline_bound(-1.0, m)
    with pytest.raises(ValueError):
        F.operational_intensity(F.KernelCounters(flops=10))
    with pytest.raises(ValueError):
        F.MachineModel(0.0, 1.0)
    with pytest.raises(ValueError):
        F.MachineModel(1.0, 1.0, special_function_peak=0.0)
    c = F.KernelCounters(600, 100, 200, 150)
    assert F.operational_intensity(c) == pytest.approx(2.0)
    assert c.scaled(3).total_bytes == 1050


def test_byte_and_event_model():
    spec = _spec((10, 6), 3)
    plan = P.plan_tiles(spec, 0, spec.cells)
    c, _ = F.sweep_counters(plan, spec, P.get_solver("shallow_water"), P.LimiterKind.MC, 8)
    assert c.bytes_read == (10 + 4) * 6 * 3 * 8 and c.bytes_written == 10 * 6 * 3 * 8
    ev = F.sweep_events(plan, spec)
    assert (ev.fans, ev.corrections, ev.cells) == ((10 + 3) * 6, (10 + 1) * 6, 10 * 6)
    small, large = _spec((12, 8), 3), _spec((12, 16), 3)
    cs, _ = F.sweep_counters(P.plan_tiles(small, 0, small.cells), small,
                             P.get_solver("acoustics"), P.LimiterKind.MC, 8)
    cl, _ = F.sweep_counters(P.plan_tiles(large, 0, large.cells), large,
                             P.get_solver("acoustics"), P.LimiterKind.MC, 8)
    assert (cl.flops, cl.special, cl.total_bytes) == (2 * cs.flops, 2 * cs.special,
                                                      2 * cs.total_bytes)
    adv = _spec((16,), 1)
    ca, _ = F.sweep_counters(P.plan_tiles(adv, 0, adv.cells), adv, P.get_solver("advection"),
                             P.LimiterKind.NONE, 8)
    assert ca.special == 0 and ca.flops > 0
    sq = _spec((8, 8), 3)
    c8, _ = F.sweep_counters(P.plan_tiles(sq, 0, sq.cells), sq, P.get_solver("acoustics"),
                             P.LimiterKind.MC, 8)
    c4, _ = F.sweep_counters(P.plan_tiles(sq, 0, sq.cells), sq, P.get_solver("acoustics"),
                             P.LimiterKind.MC, 4)
    assert c8.total_bytes == 2 * c4.total_bytes and c8.flops == c4.flops


@pytest.mark.parametrize("tile_shape,chunks", [((4, 8), 4), ((8, 8), 2), ((16, 8), 1),
                                               ((5, 3), 4), ((16, 1), 1)])
def test_halo_closed_form(tile_shape, chunks):
    spec = _spec((16, 8), 3)
    plan = P.plan_tiles(spec, 0, tile_shape)
    assert F.halo_extra_read_bytes(plan, spec, 8) == 4 * (chunks - 1) * 8 * 3 * 8


def test_not_collected_report():
    rep = F.build_report(F.RunCounters(), None)
    assert not rep.collected and rep.rows == ()
    assert "not collected" in F.render_text(rep)
    assert "not collected" in F.render_delimited(rep)


def test_machine_from_config():
    m = F.machine_from_config({"peak_flops": "1e12", "peak_bandwidth": "1e11"})
    assert m == F.MachineModel(1e12, 1e11)
    assert F.machine_from_config(None) is None
    with pytest.raises(P.ConfigError):
        F.machine_from_config({"peak_flops": "1e12"})


# ---------------------------------------------------------------------------
# the B200 kernel model


def test_kernel_event_prices_match_the_kernel_arithmetic():
    # shallow water, MC: per cell 1 sqrt + 2 div; per interface 27 flops
    # (23 + the 4 specials: uhat, vhat, chat, inv2c); per correction 3 limiter
    # divisions; the update accumulates 7 nonzero wave components twice
    c = F.kernel_event_costs("shallow_water", 2, 0, 3)
    assert c == {"make": (0, 3), "fan": (23, 4), "correction": (60, 3), "update": (46, 0)}
    per_cell = sum(f for f, _ in c.values()) + sum(s for _, s in c.values())
    assert per_cell == 139
    a = F.kernel_event_costs("acoustics", 3, 2, 3)
    assert a == {"make": (0, 0), "fan": (9, 0), "correction": (36, 2), "update": (28, 0)}
    assert F.kernel_event_costs("acoustics", 2, 0, 0)["correction"] == (30, 0)
    assert F.kernel_event_costs("advection", 1, 0, 4)["correction"] == (11, 2)


def test_kernel_sweep_counters_segments_and_bytes():
    d = F.kernel_sweep_counters("shallow_water", 2, (64, 40), 1, 3, 8, seg_len=16, num_states=3)
    assert d["events"]["update"] == 64 * 40
    assert d["counters"].bytes_read == 64 * 52 * 3 * 8
    assert d["counters"].bytes_written == 64 * 40 * 3 * 8
    assert d["events"]["fan"] == 64 * (19 + 19 + 11)
    rep = F.build_measured_report({1: d}, F.b200(8))
    assert rep.row("y", "full").flops == d["counters"].flops
    assert rep.row("all", "riemann").bytes == d["counters"].total_bytes
    assert "full" in F.render_measured_text(rep)


# ---------------------------------------------------------------------------
# on the device

CFG3D = """[run]
problem = acoustics3d
t_end = 0.05
[grid]
cells = 96 80 64
[scheme]
limiter = mc
[boundary]
all = periodic
[initial]
profile = gaussian_pressure
"""


@pytest.mark.gpu
def test_simulation_counters_follow_the_reference():
    """Simulation.counters (timestep.py:119,209-210): per sweep run, the
    reference's modeled counters; the device controller's batches count the
    same as the per-attempt loop; SweepResult.counters equals sweep_counters."""
    spec = _spec((16, 12), 3)
    g = P.create_grid(spec)
    rng = np.random.default_rng(8)
    g.interior()[0] = 1.0 + 0.2 * rng.random((12, 16))
    g.interior()[1:] = 0.1 * rng.standard_normal((2, 12, 16))
    out = []
    for dc in (False, True):
        sim = P.Simulation(g, P.get_solver("shallow_water"), P.ShallowWaterParams(1.0),
                           P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2)),
                           initial_max_speed=2.5, collect_counters=True,
                           device_controller=dc)
        with sim:
            rep = sim.run_until(0.05)
            out.append((len(rep.attempts), sim.counters.sweeps, sim.counters.total()))
    assert out[0] == out[1] and out[0][1] == 2 * out[0][0]
    # the per-sweep operator returns the modeled counters
    P.apply_boundary(g, P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2)))
    dst = P.create_grid(spec)
    res = P.sweep_axis(g, dst, 0, 0.01, P.get_solver("shallow_water"), P.LimiterKind.MC,
                       P.ShallowWaterParams(1.0))
    want, st = F.sweep_counters(P.plan_tiles(spec, 0, spec.cells), spec,
                                P.get_solver("shallow_water"), P.LimiterKind.MC, 8)
    assert res.counters == want and res.stage_flops == st


@pytest.mark.gpu
def test_run_perf_reference_contract():
    rep, summary = P.run_perf(P.loads(CFG3D + "[machine]\npeak_flops = 1e13\n"
                                      "peak_bandwidth = 6.5e12\n"))
    assert rep.collected and {r.scope for r in rep.rows} == {"x", "y", "z", "all"}
    assert rep.row("all", "riemann").oi < rep.row("all", "full").oi
    assert summary.steps_accepted > 0


@pytest.mark.gpu
def test_measured_report_beside_the_reference_model():
    rep, run = F.run_measured_perf(P.loads(CFG3D), ncu_bytes={0: 1.0e6})
    attempts = run.steps_accepted + run.steps_reverted
    for ax in ("x", "y", "z"):
        r = rep.row(ax, "full")
        assert r.launches == attempts
        assert r.seconds > 0 and math.isfinite(r.achieved_bandwidth)
        assert 0.0 < r.fraction_of_bound < 1.5
        ref = rep.reference.row(ax, "full")
        # the reference model prices the monolithic plan: n+4 reads per pencil
        assert ref.bytes == attempts * (ref.bytes // attempts)
    text = F.render_side_by_side(rep)
    assert "ref OI" in text and len(text.splitlines()) == 4
