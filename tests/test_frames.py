"""CLAWFRM1 frames (§8(f) row 1) against fixtures written by the reference
(tests/golden/make_frames.py): host serialisation, the parser's error
contract (pkg/tests/test_frames.py), manifest; the device writer and
run_to_frames are checked byte for byte on the GPU."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_1805_08846_b200 as P
from paper_1805_08846_b200 import frames as F

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "frames")


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(GOLD, "frames.json")) as fh:
        return json.load(fh)


def _grid(g, arrays, i):
    cells = tuple(g["cells"])
    spec = P.GridSpec(cells, (0.0,) * len(cells), (1.0,) * len(cells), g["m"])
    grid = P.create_grid(spec, np.dtype(g["dtype"]))
    grid.data[...] = arrays[f"data_{i}"]
    return grid


def test_host_frame_bytes_match_reference(meta):
    arrays = np.load(os.path.join(GOLD, "grids.npz"))
    for i, g in enumerate(meta["grids"]):
        b = F.frame_bytes(_grid(g, arrays, i), g["time"], g["step"])
        assert len(b) == g["nbytes"]
        assert hashlib.sha256(b).hexdigest() == g["sha256"]
        fr = F.parse_frame(b)
        assert fr.header.dims == tuple(g["cells"]) and fr.time == g["time"] and fr.step == g["step"]
        back = P.create_grid(_grid(g, arrays, i).spec, np.dtype(g["dtype"]))
        F.load_into(back, fr)
        assert back.interior().tobytes() == _grid(g, arrays, i).interior().tobytes()


def test_reference_run_files_parse_and_match_manifest(meta):
    for name, run in meta["runs"].items():
        d = os.path.join(GOLD, name)
        man = F.read_manifest(d)
        assert [(m["index"], m["time"], m["step"]) for m in man] == \
            [(f["index"], f["time"], f["step"]) for f in run["frames"]]
        for m in man:
            fr = F.read_frame(os.path.join(d, m["file"]))
            assert fr.time == m["time"] and fr.step == m["step"]


def test_parser_error_contract():
    spec = P.GridSpec((5, 4), (0, 0), (1, 1), 3)
    g = P.create_grid(spec)
    g.interior()[...] = 1.5
    b = F.frame_bytes(g, 0.5, 7)
    with pytest.raises(P.TruncatedFrameError):
        F.parse_frame(b[:10])
    with pytest.raises(P.TruncatedFrameError):
        F.parse_frame(b[:20])
    with pytest.raises(P.TruncatedFrameError):
        F.parse_frame(b[:-1])
    with pytest.raises(P.FrameFormatError):
        F.parse_frame(b + b"\0")
    with pytest.raises(P.FrameFormatError):
        F.parse_frame(b"CLAWFRM2" + b[8:])
    bad_version = bytearray(b)
    bad_version[8] = 2
    with pytest.raises(P.FrameFormatError):
        F.parse_frame(bytes(bad_version))
    bad_ndim = bytearray(b)
    bad_ndim[12] = 4
    with pytest.raises(P.FrameFormatError):
        F.parse_frame(bytes(bad_ndim))
    other = P.create_grid(P.GridSpec((4, 5), (0, 0), (1, 1), 3))
    with pytest.raises(P.FrameFormatError):
        F.load_into(other, F.parse_frame(b))
    single = P.create_grid(spec, np.float32)
    with pytest.raises(P.FrameFormatError):
        F.load_into(single, F.parse_frame(b))


def test_manifest_round_trip(tmp_path):
    for i, (t, s) in enumerate([(0.0, 0), (0.1, 3), (0.30000000000000004, 9)]):
        F.append_manifest(str(tmp_path), i, t, s)
    rows = F.read_manifest(str(tmp_path))
    assert [(r["index"], r["time"], r["step"], r["file"]) for r in rows] == [
        (0, 0.0, 0, "frame_0000.clw"), (1, 0.1, 3, "frame_0001.clw"),
        (2, 0.30000000000000004, 9, "frame_0002.clw")]
    with pytest.raises(P.FrameFormatError):
        F.read_manifest(str(tmp_path / "missing"))


@pytest.mark.gpu
def test_run_to_frames_matches_reference_files(meta, tmp_path):
    for name, run in meta["runs"].items():
        out = tmp_path / name
        summary = P.run_to_frames(P.loads(run["config"]), str(out))
        assert float(summary.t_final).hex() == run["t_final"]
        assert summary.steps_accepted == run["steps_accepted"]
        ref = os.path.join(GOLD, name)
        assert sorted(os.listdir(out)) == sorted(os.listdir(ref))
        for f in os.listdir(ref):
            with open(os.path.join(ref, f), "rb") as a, open(out / f, "rb") as b:
                assert a.read() == b.read(), f"{name}/{f} differs"


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_device_frame_equals_host_frame(dtype):
    problem = P.get_problem("acoustics3d")
    spec = P.GridSpec((13, 9, 7), (0, 0, 0), (1, 1, 1), problem.num_states)
    g = P.create_grid(spec, np.dtype(dtype))
    P.fill_initial(g, problem.initial_profile("gaussian_pressure", {"width": 0.3}, spec))
    params = problem.make_params({})
    with P.Simulation(g, problem.solver, params,
                      P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, problem.normal_velocity),
                      initial_max_speed=problem.speed_bound(g, params)) as sim:
        sim.run_until(1e30, max_steps=3)
        dev = F.simulation_frame(sim)
        assert dev == F.frame_bytes(sim.grid, sim.t, sim.steps_accepted)
