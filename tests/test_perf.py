"""Perf model (§8(f) row 2): counting-float prices of the kernel arithmetic,
segment-aware traffic, roofline arithmetic (pkg/tests/test_perf.py
contracts), and measured kernel times beside them on the GPU."""

import math

import pytest

import paper_1805_08846_b200 as P
from paper_1805_08846_b200 import perf as F


def test_roofline_arithmetic():
    m = F.MachineModel(peak_flops=100.0, peak_bandwidth=10.0)
    assert F.roofline_bound(2.0, m) == 20.0
    assert F.roofline_bound(50.0, m) == 100.0
    with pytest.raises(ValueError):
        F.roofline_bound(-1.0, m)
    with pytest.raises(ValueError):
        F.operational_intensity(F.KernelCounters())
    with pytest.raises(ValueError):
        F.MachineModel(0.0, 1.0)
    c = F.KernelCounters(10, 2, 3, 3)
    assert F.operational_intensity(c) == 2.0
    assert c.scaled(3).total_bytes == 18


def test_event_prices_match_the_kernel_arithmetic():
    # shallow water, MC: per cell 1 sqrt + 2 div; per interface 27 flops
    # (23 + the 4 specials: uhat, vhat, chat, inv2c); per correction 3 limiter
    # divisions; the update accumulates 7 nonzero wave components twice
    c = F.event_costs("shallow_water", 2, 0, 3)
    assert c == {"make": (0, 3), "fan": (23, 4), "correction": (60, 3), "update": (46, 0)}
    # per cell-sweep the fp64 ops ncu counts on the x-sweep (138, profiles/)
    per_cell = sum(f for f, _ in c.values()) + sum(s for _, s in c.values())
    assert per_cell == 139
    a = F.event_costs("acoustics", 3, 2, 3)
    assert a == {"make": (0, 0), "fan": (9, 0), "correction": (36, 2), "update": (28, 0)}
    assert F.event_costs("acoustics", 2, 0, 0)["correction"] == (30, 0)   # no limiter: no divide
    assert F.event_costs("advection", 1, 0, 4)["correction"] == (11, 2)   # van Leer divides twice


def test_sweep_counters_segments_and_bytes():
    d = F.sweep_counters("shallow_water", 2, (64, 40), 1, 3, 8, seg_len=16, num_states=3)
    # y sweep: 64 pencils, segments 16,16,8 -> reads (20+20+12) cells per pencil
    assert d["events"]["update"] == 64 * 40
    assert d["counters"].bytes_read == 64 * 52 * 3 * 8
    assert d["counters"].bytes_written == 64 * 40 * 3 * 8
    assert d["events"]["fan"] == 64 * (19 + 19 + 11)
    rep = F.build_report({1: d}, F.b200(8))
    assert rep.row("y", "full").flops == d["counters"].flops
    assert rep.row("all", "riemann").bytes == d["counters"].total_bytes
    text = F.render_text(rep)
    assert "y" in text and "full" in text


@pytest.mark.gpu
def test_run_perf_measures_every_axis():
    cfg = P.loads("""[run]
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
""")
    rep, run = F.run_perf(cfg)
    for ax in ("x", "y", "z"):
        r = rep.row(ax, "full")
        assert r.launches == run.steps_accepted + run.steps_reverted
        assert r.seconds > 0 and math.isfinite(r.achieved_bandwidth)
        assert 0.0 < r.fraction_of_bound < 1.5
