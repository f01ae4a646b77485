"""CPU: slab decomposition host logic under gloo (world sizes 2 and 3),
computing with the oracle-backed engine.  The decomposed run must equal the
single-domain run bit for bit: every attempt (dt, max speed, nu, accept) and
every state byte, for reflective / periodic / outflow slow axes, 2-D and 3-D,
and the same first non-finite cell on blow-up."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1805_08846_b200 as P
from paper_1805_08846_b200.slab import Slab, split_counts

import cases

CASES = {
    "sw_reflective": ("shallow_water2d", (24, 21), "radial_dam_break", {}, "reflective", "mc", 8),
    "sw_periodic": ("shallow_water2d", (18, 16), "gaussian_hump", {}, "periodic", "vanleer", 6),
    "ac3d_outflow": ("acoustics3d", (8, 7, 12), "gaussian_pressure", {"width": 0.3}, "outflow",
                     "superbee", 4),
    "vc3d_periodic": ("vc_acoustics3d", (6, 5, 10), "two_material_pulse", {}, "periodic", "mc", 4),
}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _recipe(name):
    prob, cells, prof, opts, bc, lim, steps = CASES[name]
    nd = len(cells)
    lower = (-1.0,) * nd if prof == "radial_dam_break" else (0.0,) * nd
    return dict(name=name, problem=prob, profile=prof, options=opts, cells=cells, lower=lower,
                upper=(1.0,) * nd, dtype="float64", bc=bc, limiter=lim,
                speed="bound" if not prob.startswith("vc") else ("value", 1.0),
                drive=("max_steps", steps))


def _run(name, rank, world, port, nan_at=None):
    import torch.distributed as dist
    from cpu_engine import OracleEngine
    r = _recipe(name)
    grid, params, problem, bspec, speed = cases.build_grid(r)
    if nan_at is not None:
        grid.interior()[nan_at] = np.nan
    dist_mod = None
    if world > 1:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dist_mod = dist
    slab = Slab(grid.spec, bspec, rank, world, dist_mod, transport="host")
    local = P.StateGrid(slab.local_spec, grid.dtype)
    local.interior()[...] = grid.interior()[slab.local_slice()]
    sim = P.Simulation(local, problem.solver, params, bspec, limiter=P.LimiterKind(r["limiter"]),
                       initial_max_speed=speed, slab=slab, engine=OracleEngine)
    try:
        att = cases.attempts_hex(cases.drive(sim, r))
        out = ("ok", att, sim.grid.interior().copy())
    except P.NumericalBlowup as e:
        out = ("blowup", (e.state, e.cell, e.step), None)
    if world > 1:
        dist.destroy_process_group()
    return out


def _worker(rank, world, port, name, nan_at, q):
    q.put((rank, _run(name, rank, world, port, nan_at)))


def _decomposed(name, world, nan_at=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, nan_at, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    return [res[r] for r in range(world)]


def test_split_counts():
    assert split_counts(10, 3) == [4, 3, 3]
    with pytest.raises(ValueError):
        split_counts(5, 3)


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("world", [2, 3])
def test_decomposed_run_is_bitwise_single_domain(name, world):
    ref = _run(name, 0, 1, None)
    parts = _decomposed(name, world)
    assert all(p[0] == "ok" for p in parts)
    for p in parts:
        assert p[1] == ref[1], "attempt sequence differs from the single-domain run"
    nd = len(CASES[name][1])
    axis_arr = 1  # slowest axis is the first array axis after the state axis
    glued = np.concatenate([p[2] for p in parts], axis=axis_arr)
    assert glued.tobytes() == ref[2].tobytes()


def test_decomposed_blowup_reports_global_first_cell():
    nan_at = (0, 14, 5)  # state 0, y=14 (second slab), x=5
    ref = _run("sw_reflective", 0, 1, None, nan_at)
    parts = _decomposed("sw_reflective", 2, nan_at)
    assert ref[0] == "blowup"
    assert all(p == ref for p in parts)


def test_layout_neighbours_and_self_halo():
    spec = P.GridSpec((8, 12), (0, 0), (1, 1), 3)
    per = P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2))
    ref = P.BoundarySpec.uniform(P.BoundaryKind.REFLECTIVE, (1, 2))
    s = Slab(spec, per, 0, 1, None, transport="device", self_halo=True)
    assert (s.layout.lo_nbr, s.layout.hi_nbr, s.layout.exchanges) == (0, 0, True)
    assert s.local_bc([(2, 2), (2, 2)])[1] == (3, 3) and s.device_resident
    s = Slab(spec, per, 0, 1, None, transport="device")
    assert (s.layout.lo_nbr, s.layout.hi_nbr, s.layout.exchanges) == (None, None, False)
    s = Slab(spec, ref, 0, 1, None, transport="device", self_halo=True)
    assert not s.layout.exchanges            # a reflective axis never wraps
    s = Slab(spec, ref, 1, 3, None, transport="nccl")
    assert (s.layout.lo_nbr, s.layout.hi_nbr) == (0, 2) and not s.device_resident
    with pytest.raises(ValueError):
        Slab(spec, ref, 0, 2, None, transport="carrier-pigeon")
