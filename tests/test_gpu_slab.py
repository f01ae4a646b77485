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


# ---------------------------------------------------------------------------
# The device-resident slab path (clb_attach_comm: NCCL inside the library,
# the exchange and the max-allreduce inside the attempt graph).  One GPU, one
# rank: a periodic slow axis is exchanged with the rank itself through NCCL
# (lo/hi neighbour = rank 0, the slow-axis sides are HALO), which runs the
# same pack -> ncclSend/ncclRecv -> unpack -> overlapped slow sweep ->
# allreduce -> controller sequence as a multi-GPU run; the result must be
# bit-identical to the single-domain periodic run.

DEVICE_CASES = {
    "sw_periodic": ("shallow_water2d", (96, 130), "gaussian_hump", {}, "periodic", "mc", 8,
                    "float64"),
    "sw_periodic_f32": ("shallow_water2d", (70, 203), "gaussian_hump", {}, "periodic",
                        "superbee", 8, "float32"),
    "ac3d_periodic": ("acoustics3d", (40, 33, 50), "gaussian_pressure", {"width": 0.2},
                      "periodic", "mc", 5, "float64"),
}


def _device_recipe(name):
    prob, cells, prof, opts, bc, lim, steps, dt = DEVICE_CASES[name]
    nd = len(cells)
    return dict(name=name, problem=prob, profile=prof, options=opts, cells=cells,
                lower=(0.0,) * nd, upper=(1.0,) * nd, dtype=dt, bc=bc, limiter=lim,
                speed="bound", drive=("max_steps", steps))


@pytest.mark.parametrize("device_controller", [True, False], ids=["graph", "host-loop"])
@pytest.mark.parametrize("name", sorted(DEVICE_CASES))
def test_device_slab_exchange_with_itself_is_bitwise(name, device_controller):
    r = _device_recipe(name)
    ref_sim, _ = cases.product_sim(r)
    with ref_sim:
        ref_att = cases.attempts_hex(cases.drive(ref_sim, r))
        ref = ref_sim.grid.interior().copy()
    grid, params, problem, bspec, speed = cases.build_grid(r)
    slab = Slab(grid.spec, bspec, 0, 1, None, transport="device", self_halo=True)
    assert slab.layout.lo_nbr == 0 and slab.layout.hi_nbr == 0
    with P.Simulation(grid, problem.solver, params, bspec, limiter=P.LimiterKind(r["limiter"]),
                      initial_max_speed=speed, slab=slab,
                      device_controller=device_controller) as sim:
        att = cases.attempts_hex(cases.drive(sim, r))
        assert att == ref_att
        assert sim.grid.interior().tobytes() == ref.tobytes()


def test_device_slab_blowup_location_through_the_exchange():
    spec = P.GridSpec((40, 36), (0, 0), (1, 1), 3)
    base = 0.05 * np.random.default_rng(3).standard_normal((3, 36, 40))
    res = []
    for use_slab in (False, True):
        g = P.create_grid(spec)
        g.interior()[...] = base
        bspec = P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2))
        slab = Slab(spec, bspec, 0, 1, None, transport="device", self_halo=True) \
            if use_slab else None
        sim = P.Simulation(g, P.get_solver("acoustics"), P.AcousticsParams(), bspec,
                           initial_max_speed=1.0, slab=slab)
        sim.run_until(1e30, max_steps=2)
        sim.grid.interior(0)[35, 7] = np.nan
        with pytest.raises(P.NumericalBlowup) as exc:
            sim.run_until(1e30, max_steps=3)
        res.append((exc.value.state, exc.value.cell, exc.value.step))
        sim.close()
    assert res[0] == res[1]
