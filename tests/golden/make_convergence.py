"""Convergence-ladder fixtures (§8(f) row 3) from the reference's
run_convergence (runner.py:149-186), generated in this container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_convergence.py
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from clawtile import loads  # noqa: E402
from clawtile.runner import run_convergence  # noqa: E402

CASES = {
    "acoustics_16_3levels": ("""[run]
problem = acoustics2d
t_end = 0.2
[grid]
cells = 16 16
[scheme]
limiter = mc
[boundary]
all = periodic
[initial]
profile = gaussian_pressure
width = 0.15
[parallel]
serial = true
""", 3),
    "hump_12x8_4levels_superbee": ("""[run]
problem = shallow_water2d
t_end = 0.1
[grid]
cells = 12 8
[scheme]
limiter = superbee
[boundary]
all = reflective
[initial]
profile = gaussian_hump
[parallel]
serial = true
""", 4),
}


def main():
    out = {}
    for name, (text, levels) in CASES.items():
        r = run_convergence(loads(text), levels)
        out[name] = {"config": text, "levels": levels,
                     "result": [[list(lv.cells), lv.error.hex(),
                                 None if lv.order is None else lv.order.hex()] for lv in r.levels],
                     "reference_cells": list(r.reference_cells)}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "convergence.json"),
              "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
