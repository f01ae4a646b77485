"""CPU: the oracle (oracle/clawref.c + oracle/oracle.py) is pinned to golden
vectors produced by the reference itself (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from oracle import oracle as O

import cases


def test_sweeps_match_reference_bitwise(golden_sweeps):
    meta, arrays = golden_sweeps
    bad = []
    for i, c in enumerate(meta):
        qin = np.ascontiguousarray(arrays[f"qin_{i}"])
        qout = np.zeros_like(qin)
        smax = O.sweep(qin, qout, c["axis"], float.fromhex(c["dt_hex"]), c["spacing"],
                       c["solver"], c["limiter"], c["params"], nthreads=2)
        exp = arrays[f"qout_{i}"]
        if O.interior(qout).tobytes() != exp.tobytes() or smax != float.fromhex(c["smax_hex"]):
            bad.append((i, c["solver"], c["dtype"], c["limiter"], c["bc"], c["axis"]))
    assert not bad, f"{len(bad)} mismatching sweeps, first: {bad[:5]}"
    assert len(meta) >= 400


@pytest.mark.parametrize("name", ["acoustics", "shallow_water"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_solver_pairs_match_reference_bitwise(golden_solvers, name, dtype):
    ql = golden_solvers[f"{name}_{dtype}_ql"]
    qr = golden_solvers[f"{name}_{dtype}_qr"]
    We = golden_solvers[f"{name}_{dtype}_W"]
    se = golden_solvers[f"{name}_{dtype}_s"]
    params = {"sound_speed": 1.3, "impedance": 0.7} if name == "acoustics" else {"gravity": 1.7}
    for i in range(ql.shape[0]):
        W, s = O.solve(name, ql[i], qr[i], i % 2, params, dtype=np.dtype(dtype))
        assert W.tobytes() == We[i].tobytes() and s.tobytes() == se[i].tobytes(), i


@pytest.mark.parametrize("name", sorted(cases.RECIPES))
def test_runs_match_reference(golden_runs, name):
    r = cases.RECIPES[name]
    g = golden_runs[name]
    sim, grid = cases.oracle_sim(r)
    assert cases.sha(grid.interior()) == g["sha256_initial"], "input generator drifted"
    attempts = cases.drive(sim, r)
    assert cases.attempts_hex(attempts) == g["attempts"]
    assert cases.sha(O.interior(sim.grid)) == g["sha256"]
    assert float(sim.t).hex() == g["t"]


def test_c1_known_answer(golden_runs):
    # the reference's own C1 oracle check
    g = golden_runs["c1_acoustics_pulse_256_mc_100"]
    assert g["sha256"].startswith("429c7880ae08b44f")
    assert {a[1] for a in g["attempts"]} == {(0.003515625).hex()}
    assert float.fromhex(g["t"]) == 0.35156250000000033


def _advection_line(limiter):
    data = np.zeros((1, 12))
    data[0, 2:10] = [0, 0, 0, 0, 1, 1, 1, 1]
    O.apply_boundary(data, [("outflow", "outflow")], (None,))
    out = np.zeros_like(data)
    dx = 1.0 / 8
    O.sweep(data, out, 0, 0.5 * dx, (dx,), "advection", limiter, {"speed": 1.0})
    return out[0, 2:10]


def test_hand_worked_advection_step():
    # pkg/tests/test_sweep.py:100-132
    np.testing.assert_allclose(_advection_line("none"), [0, 0, 0, -0.125, 0.625, 1, 1, 1],
                               rtol=0, atol=1e-15)
    np.testing.assert_allclose(_advection_line("minmod"), [0, 0, 0, 0, 0.5, 1, 1, 1],
                               rtol=0, atol=1e-15)


def test_thread_count_does_not_change_bits():
    rng = np.random.default_rng(3)
    data = np.ones((3, 44, 36))
    data[0, 2:-2, 2:-2] = 1.0 + 0.3 * rng.random((40, 32))
    data[1:, 2:-2, 2:-2] = 0.2 * rng.standard_normal((2, 40, 32))
    O.apply_boundary(data, [("periodic", "periodic")] * 2, (1, 2))
    outs = []
    for nt in (1, 3, 8):
        for axis in (0, 1):
            out = np.zeros_like(data)
            s = O.sweep(data, out, axis, 0.004, (1 / 32, 1 / 40), "shallow_water", "mc",
                        {"gravity": 1.0}, nthreads=nt)
            outs.append((axis, out.tobytes(), s))
    for axis in (0, 1):
        sel = [o for o in outs if o[0] == axis]
        assert all(o[1:] == sel[0][1:] for o in sel)
