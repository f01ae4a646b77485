"""Self-convergence ladder (§8(f) row 3, runner.py:149-186): the device
driver must reproduce the reference's errors and orders bit for bit on the
ladders it can run (tests/golden/make_convergence.py), and show second-order
convergence at resolutions beyond the CPU reference's reach."""

import json
import math
import os

import numpy as np
import pytest

import paper_1805_08846_b200 as P

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "convergence.json")


def test_block_mean_and_validation():
    a = np.arange(16.0).reshape(4, 4)
    assert np.array_equal(P.block_mean(a, 2), np.array([[2.5, 4.5], [10.5, 12.5]]))
    assert P.block_mean(a, 1) is a
    with pytest.raises(ValueError):
        P.block_mean(np.zeros((3, 4)), 2)
    with open(GOLD) as fh:
        cfg = P.loads(next(iter(json.load(fh).values()))["config"])
    with pytest.raises(P.ConfigError):
        P.run_convergence(cfg, 2)


@pytest.mark.gpu
def test_convergence_matches_reference():
    with open(GOLD) as fh:
        cases = json.load(fh)
    for name, c in cases.items():
        r = P.run_convergence(P.loads(c["config"]), c["levels"])
        got = [[list(lv.cells), lv.error.hex(), None if lv.order is None else lv.order.hex()]
               for lv in r.levels]
        assert got == c["result"], name
        assert list(r.reference_cells) == c["reference_cells"]


@pytest.mark.gpu
def test_second_order_at_large_resolution():
    """Acoustics pulse, periodic, 128^2 .. 1024^2 (the 1024^2 level alone is
    minutes of CPU reference time): observed orders near 2."""
    cfg = P.loads("""[run]
problem = acoustics2d
t_end = 0.25
[grid]
cells = 128 128
[scheme]
limiter = mc
[boundary]
all = periodic
[initial]
profile = gaussian_pressure
width = 0.15
""")
    r = P.run_convergence(cfg, 4)
    orders = [lv.order for lv in r.levels if lv.order is not None]
    assert all(math.isfinite(o) for o in orders)
    assert orders[0] > 1.6, orders
