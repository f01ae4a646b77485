"""GPU: the slab decomposition through the real device path (HALO ghost
layers written by clb_halo_copy, per-rank kernels, max-allreduce).  This
box has one GPU, so the ranks share cuda:0 and exchange halos through host
memory with gloo; the NCCL transport differs only in moving the same bytes
device-to-device.  Result must be bit-identical to the single-GPU run."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1805_08846_b200 as P
from paper_1805_08846_b200.slab import Slab

import cases

pytestmark = pytest.mark.gpu

CASES = {
    "sw_reflective": ("shallow_water2d", (200, 150), "radial_dam_break", {}, "reflective", "mc", 6),
    "sw_periodic_f32": ("shallow_water2d", (96, 130), "gaussian_hump", {}, "periodic", "superbee", 6),
    "ac3d_periodic": ("acoustics3d", (40, 33, 50), "gaussian_pressure", {"width": 0.2}, "periodic",
                      "mc", 4),
    "vc3d_reflective": ("vc_acoustics3d", (30, 20, 41), "two_material_pulse", {}, "reflective",
                        "superbee", 4),
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
                upper=(1.0,) * nd, dtype="float32" if name.endswith("f32") else "float64",
                bc=bc, limiter=lim,
                speed="bound" if not prob.startswith("vc") else ("value", 1.0),
                drive=("max_steps", steps))


def _run(name, rank, world, port):
    import torch.distributed as dist
    r = _recipe(name)
    grid, params, problem, bspec, speed = cases.build_grid(r)
    dmod = None
    if world > 1:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dmod = dist
    slab = Slab(grid.spec, bspec, rank, world, dmod, transport="host")
    local = P.StateGrid(slab.local_spec, grid.dtype)
    slab.fill_initial(local, problem.initial_profile(r["profile"], dict(r["options"]), grid.spec))
    assert local.interior().tobytes() == np.ascontiguousarray(
        grid.interior()[slab.local_slice()]).tobytes()
    with P.Simulation(local, problem.solver, params, bspec, limiter=P.LimiterKind(r["limiter"]),
                      initial_max_speed=speed, slab=slab) as sim:
        att = cases.attempts_hex(cases.drive(sim, r))
        out = (att, sim.grid.interior().copy())
    if world > 1:
        dist.destroy_process_group()
    return out


def _worker(rank, world, port, name, q):
    q.put((rank, _run(name, rank, world, port)))


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("world", [2, 3])
def test_slab_on_device_is_bitwise_single_gpu(name, world):
    ref_att, ref = _run(name, 0, 1, None)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert res[r][0] == ref_att
    glued = np.concatenate([res[r][1] for r in range(world)], axis=1)
    assert glued.tobytes() == ref.tobytes()
