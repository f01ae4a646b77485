"""CPU: host-side logic of the product package and the C-ABI library
surface (no compute without a GPU)."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_1805_08846_b200 as P
from paper_1805_08846_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "clawb200.h")) as fh:
        header = fh.read()
    declared = set(re.findall(r"\b(clb_[a-z_0-9]+)\s*\(", header))
    assert declared == set(_native.EXPORTS)
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert _native.lib().clb_version() == 1


def test_desc_struct_matches_header_layout():
    # int32 x6, int64[3], double[3], double[8], int32[3][2], int32[3], tail-padded to 8
    assert ctypes.sizeof(_native.ClbDesc) == 176
    assert _native.ClbDesc.cells.offset == 24 and _native.ClbDesc.bc.offset == 136


def test_abi_structs_match_a_c_compiler(tmp_path):
    """sizeof/offsetof of every struct the ctypes binding mirrors, as gcc
    lays them out from include/clawb200.h."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    checks = {
        "clb_desc": (_native.ClbDesc, ["cells", "spacing", "params", "bc", "normal_velocity"]),
        "clb_batch": (_native.ClbBatch, ["prev_reverted", "cur", "stop", "max_accepted",
                                         "n_attempts", "status", "fail_dt"]),
        "clb_attempt": (_native.ClbAttempt, ["dt_retry", "accepted", "landed"]),
    }
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "clawb200.h"', "int main(void){"]
    for st, (_, fields) in checks.items():
        src.append(f'printf("{st} %zu\\n", sizeof({st}));')
        for f in fields:
            src.append(f'printf("{st}.{f} %zu\\n", offsetof({st}, {f}));')
    src.append("return 0;}")
    c = tmp_path / "abi.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    out = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                       check=True).stdout.splitlines())
    for st, (cls, fields) in checks.items():
        assert int(out[st]) == ctypes.sizeof(cls), st
        for f in fields:
            assert int(out[f"{st}.{f}"]) == getattr(cls, f).offset, f"{st}.{f}"


def test_create_failure_reports_error_without_gpu_or_bad_args():
    d = _native.ClbDesc()
    d.ndim = 4
    h = ctypes.c_void_p()
    code = _native.lib().clb_create(ctypes.byref(d), ctypes.byref(h))
    assert code == _native.CLB_EINVAL
    assert b"dimensional" in _native.lib().clb_last_error(None)


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    spec = P.GridSpec((8, 8), (0, 0), (1, 1), 3)
    g = P.create_grid(spec)
    g.data[0] = 1.0
    with pytest.raises(P.DeviceError):
        P.Simulation(g, P.get_solver("shallow_water"), P.ShallowWaterParams(),
                     P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2)), initial_max_speed=1.0)


def test_python_registered_solver_is_rejected():
    solver = P.RiemannSolver("user_scalar", 1, lambda *a: None, lambda p, d: np.zeros(1, d))
    with pytest.raises(ValueError, match="no device implementation"):
        solver.require_device()


def test_limiter_ids_stable():
    assert P.LIMITER_IDS == {P.LimiterKind.NONE: 0, P.LimiterKind.MINMOD: 1,
                             P.LimiterKind.SUPERBEE: 2, P.LimiterKind.MC: 3,
                             P.LimiterKind.VANLEER: 4}


def test_pack_params_in_run_dtype():
    for dt in (np.float32, np.float64):
        pv = P.get_solver("acoustics").pack_params(P.AcousticsParams(1.3, 0.7), dt)
        assert pv.dtype == dt and pv[2] == dt(0.5) / dt(0.7)


def test_gridspec_and_indexing():
    spec = P.GridSpec((6, 4), (0, 0), (3, 2), 3)
    assert spec.spacing == (0.5, 0.5)
    assert spec.padded_array_shape == (8, 10)
    for off in (0, 17, 79):
        assert P.linear_index(spec, P.index_coords(spec, off)) == off
    with pytest.raises(ValueError):
        P.GridSpec((0,), (0,), (1,), 1)


def test_boundary_spec_validation():
    with pytest.raises(P.ConfigError):
        P.BoundarySpec(((P.BoundaryKind.PERIODIC, P.BoundaryKind.OUTFLOW),), (1,))
    with pytest.raises(P.ConfigError):
        P.BoundarySpec.uniform(P.BoundaryKind.REFLECTIVE, (None,))


def test_host_apply_boundary_matches_oracle(rng):
    from oracle import oracle as O
    for kind in ("outflow", "reflective", "periodic"):
        spec = P.GridSpec((7, 5, 4), (0, 0, 0), (1, 1, 1), 4)
        g = P.create_grid(spec)
        g.data[...] = rng.standard_normal(g.data.shape)
        ref = g.data.copy()
        P.apply_boundary(g, P.BoundarySpec.uniform(P.BoundaryKind(kind), (1, 2, 3)))
        O.apply_boundary(ref, [(kind, kind)] * 3, (1, 2, 3))
        assert g.data.tobytes() == ref.tobytes()


PULSE_CFG = """# same keys as the reference's configs/acoustics_pulse.cfg
[run]
problem = acoustics2d
t_end = 0.6
frames = 10
[grid]
cells = 256 256
lower = 0 0
upper = 1 1
[physics]
sound_speed = 1.0
impedance = 1.0
[scheme]
limiter = mc
cfl_target = 0.9
cfl_max = 1.0
[boundary]
all = reflective
[initial]
profile = gaussian_pressure
amplitude = 1.0
width = 0.08
[parallel]
tiles = 64x4
workers = 4
"""


def test_config_reference_format(tmp_path):
    path = tmp_path / "pulse.cfg"
    path.write_text(PULSE_CFG)
    cfg = P.load_config(str(path))
    assert cfg.problem == "acoustics2d" and cfg.cells == (256, 256)
    assert cfg.boundary_sides == ((P.BoundaryKind.REFLECTIVE,) * 2,) * 2
    assert cfg.frame_times()[0] == 0.06 and cfg.effective_workers() == 4
    assert cfg.with_overrides(serial=True).effective_tiles() == (256, 256)


def test_config_strictness():
    text = "[run]\nproblem = acoustics2d\nt_end = 1\n[grid]\ncells = 4 4\n[initial]\nprofile = gaussian_pressure\n"
    cfg = P.loads(text)
    assert cfg.limiter is P.LimiterKind.MC and cfg.cfl_target == 0.9
    with pytest.raises(P.ConfigError):
        P.loads(text + "[scheme]\nbogus = 1\n")
    with pytest.raises(P.ConfigError):
        P.loads(text.replace("cells = 4 4", "cells = 4"))


def test_profiles_match_recipes_initial_sha(golden_runs):
    import cases
    for name, r in cases.RECIPES.items():
        grid, *_ = cases.build_grid(r)
        assert cases.sha(grid.interior()) == golden_runs[name]["sha256_initial"], name


def test_step_order():
    assert P.step_order(3) == (0, 1, 2)
    with pytest.raises(ValueError):
        P.step_order(4)
