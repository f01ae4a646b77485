"""Benchmark of the time-step hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4]
                    [--scaling strong|weak] [--impl reference]

One JSON line on rank 0.  A "step" is one ``Simulation.attempt_step`` (all
ndim fused sweeps + the fp64 CFL controller) over the workload's grid.  The
default workload is C4 (BASELINE.json configs[3]: 2-D shallow water
16384^2, fp64), strong-scaled over N GPUs; ``--workload c5`` (512^3
acoustics per GPU) weak-scales.

* ``value``: cell-updates/s with the state resident in HBM, each step timed
  with CUDA events on the launch stream (host controller gaps included),
  L2 flushed (1 GiB write) between steps, summed over K steps, max over
  ranks.  Counts accepted steps only, as the reference metric does.
* ``e2e``: the same metric through the public API from pinned host memory:
  upload of the initial state, ``run_until(max_steps=K)`` (the attempt loop
  runs on the device controller; the K attempt records come back with one
  D2H), download of the final state; wall clock.
* ``roofline``: the dominant sweep kernel's algorithmic bytes per launch
  (m states read + m written per cell) / its mean CUDA-event
  duration, against MEASURED_PEAKS.json ``hbm_gbs``.
* ``cpu_baseline``: the oracle (C restatement of the reference path, all host
  threads) on a bounded sample of the same workload: the middle band of the
  global grid holding about 2^24 cells.
* ``--impl reference``: the reference's CPU path (oracle port) timed on the
  host cores, rank 0 only, each step one attempt over that same band; the
  line's ``config`` is identical to the B200 arm's.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gcell-updates/s and achieved HBM GB/s vs peak at 1/2/4/8 B200 vs CPU ref"
UNIT = "Gcell-updates/s"
# CUDACLAW SW 1000^2 fp64 average step 9.2 ms on a Tesla C2050
PUBLISHED_SW_FP64 = 1.0e6 / 9.2e-3 / 1e9

WORKLOADS = {
    # name: (problem, cells, lower, upper, profile, options, bc, limiter, precision, label)
    "c1": ("acoustics2d", (256, 256), (0, 0), (1, 1), "gaussian_pressure",
           {"amplitude": 1.0, "width": 0.08}, "reflective", "mc", "double",
           "C1: 2D acoustics 256x256 radial pressure pulse, MC, fp64"),
    "c2": ("shallow_water2d", (1024, 1024), (-1, -1), (1, 1), "radial_dam_break", {},
           "reflective", "mc", "double",
           "C2: 2D shallow water 1024x1024 radial dam-break, reflective, MC, adaptive CFL dt, fp64"),
    "c3": ("vc_acoustics3d", (256, 256, 256), (0, 0, 0), (1, 1, 1), "two_material_pulse", {},
           "reflective", "superbee", "double",
           "C3: 3D acoustics 256^3 two-material medium, superbee, fp64"),
    "c4": ("shallow_water2d", (16384, 16384), (-1, -1), (1, 1), "radial_dam_break", {},
           "reflective", "mc", "double",
           "C4: 2D shallow water 16384x16384 radial dam-break, reflective, MC, adaptive CFL dt, fp64"),
    "c5": ("acoustics3d", (512, 512, 512), (0, 0, 0), (1, 1, 1), "gaussian_pressure",
           {"width": 0.1}, "periodic", "mc", "double",
           "C5: 3D acoustics 512^3 per GPU, MC, periodic, fp64"),
    "c5f32": ("acoustics3d", (512, 512, 512), (0, 0, 0), (1, 1, 1), "gaussian_pressure",
              {"width": 0.1}, "periodic", "mc", "single",
              "C5: 3D acoustics 512^3 per GPU, MC, periodic, fp32"),
    "sw8192": ("shallow_water2d", (8192, 8192), (-1, -1), (1, 1), "radial_dam_break", {},
               "reflective", "mc", "double",
               "north-star: 2D shallow water 8192^2 radial dam-break, fp64"),
    "c4lake": ("shallow_water2d", (16384, 16384), (-1, -1), (1, 1), "lake_at_rest", {},
               "reflective", "mc", "double",
               "SW 16384^2 lake at rest (every cell uniform: the sweeps' pure streaming limit), fp64"),
    "sw8192hump": ("shallow_water2d", (8192, 8192), (0, 0), (1, 1), "gaussian_hump", {},
                   "reflective", "mc", "double",
                   "2D shallow water 8192^2 gaussian hump (flow active in every cell), fp64"),
    "sw8192f32": ("shallow_water2d", (8192, 8192), (-1, -1), (1, 1), "radial_dam_break", {},
                  "reflective", "mc", "single",
                  "north-star: 2D shallow water 8192^2 radial dam-break, fp32"),
}


#: default scaling mode per workload (BASELINE.json: C4 strong, C5 weak)
DEFAULT_SCALING = {"c4": "strong"}
#: cells of the bounded CPU sample (one band of the workload's grid)
CPU_SAMPLE_CELLS = 1 << 24


def global_cells(name, world, scaling):
    """Global grid of the run: weak scaling grows the slowest axis by `world`
    (each rank keeps the workload's size), strong scaling splits the
    workload's own grid over the ranks."""
    cells = WORKLOADS[name][1]
    if scaling == "weak":
        return tuple(cells[:-1]) + (cells[-1] * world,)
    return tuple(cells)


def config_of(args, world, scaling):
    """The run's `config`, identical in both arms (same_config)."""
    prob, cells, lower, upper, profile, options, bc, lim, prec, label = WORKLOADS[args.workload]
    gcells = global_cells(args.workload, world, scaling)
    return {
        "workload": label,
        "name": args.workload,
        "cells": list(gcells),
        "scaling": scaling,
        "parallelism": (f"slab x{world} along the slowest axis, NCCL halo exchange "
                        "(overlapped with the slow sweep) + max-allreduce on the device"
                        if world > 1 else "single GPU"),
        "l2": "flushed between steps (1 GiB write, untimed); the grid is larger than L2"
              if int(np.prod(gcells)) * 8 > 126e6 else
              "flushed between steps (1 GiB write, untimed); the working set fits L2",
        "step": "one Simulation.attempt_step (all ndim fused sweeps + the fp64 CFL "
                "controller); Gcell-updates counts accepted steps only",
    }


def build_inputs(name, gcells, world=1, rank=0, dist=None, transport="nccl", band=None):
    """Workload inputs on the global grid `gcells`.  world > 1: this rank's
    slab (global cell centres, so every byte equals the 1-GPU layout).
    band=(index, count): one slab of the global grid, alone (the bounded CPU
    sample), with the workload's physical boundaries on its faces."""
    import paper_1805_08846_b200 as P
    from paper_1805_08846_b200.slab import Slab
    prob, _, lower, upper, profile, options, bc, lim, prec, label = WORKLOADS[name]
    problem = P.get_problem(prob)
    spec = P.GridSpec(tuple(gcells), lower, upper, problem.num_states)
    bspec = P.BoundarySpec.uniform(P.BoundaryKind(bc), problem.normal_velocity)
    params = problem.make_params({})
    prof = problem.initial_profile(profile, dict(options), spec)
    slab = None
    if band is not None:
        part = Slab(spec, bspec, band[0], band[1], None)
        grid = P.create_grid(part.local_spec, P.grid.DTYPES[prec])
        part.fill_initial(grid, prof)
        speed = problem.speed_bound(grid, params)
    elif world > 1:
        slab = Slab(spec, bspec, rank, world, dist, transport=transport)
        grid = P.create_grid(slab.local_spec, P.grid.DTYPES[prec])
        slab.fill_initial(grid, prof)
        speed = float(slab.allreduce_max(np.array([problem.speed_bound(grid, params)]))[0])
    else:
        grid = P.create_grid(spec, P.grid.DTYPES[prec])
        P.fill_initial(grid, prof)
        speed = problem.speed_bound(grid, params)
    return dict(P=P, problem=problem, spec=spec, grid=grid, params=params, speed=speed,
                bspec=bspec, limiter=P.LimiterKind(lim), label=label, dtype=grid.dtype,
                slab=slab, local_cells=grid.spec.num_cells)


def cpu_sample_inputs(name, gcells):
    """The bounded CPU sample: the middle band of the global grid holding
    about CPU_SAMPLE_CELLS cells (the whole grid if it is smaller)."""
    n = int(np.prod(gcells))
    parts = max(1, min(gcells[-1] // 2, n // CPU_SAMPLE_CELLS))
    if parts == 1:
        return build_inputs(name, gcells), "the whole grid"
    inp = build_inputs(name, gcells, band=(parts // 2, parts))
    c = inp["grid"].spec.cells
    return inp, (f"the middle {c[-1]}-{'row' if len(c) == 2 else 'plane'} band "
                 f"({'x'.join(map(str, c))} cells) of the {'x'.join(map(str, gcells))} grid, "
                 "same profile and boundary kinds")


# ---------------------------------------------------------------------------
# CPU leg (oracle port of the reference path)


def oracle_from_inputs(inp, nthreads):
    from oracle import oracle as O
    problem = inp["problem"]
    pd = {"acoustics": lambda p: {"sound_speed": p.sound_speed, "impedance": p.impedance},
          "shallow_water": lambda p: {"gravity": p.gravity},
          "advection": lambda p: {"speed": p.speed},
          "vc_acoustics": lambda p: {}}[problem.solver_name](inp["params"])
    sides = [(lo.value, hi.value) for lo, hi in inp["bspec"].sides]
    return O.OracleSimulation(inp["grid"].data.copy(), inp["spec"].spacing, problem.solver_name,
                              pd, sides, inp["bspec"].normal_velocity,
                              limiter=inp["limiter"].value, initial_max_speed=inp["speed"],
                              nthreads=nthreads)


def cpu_rate(inp, budget_s=12.0, max_steps=None, warmup=1):
    """Oracle throughput on all host threads: `warmup` untimed attempts, then
    `max_steps` attempts (or as many as fit `budget_s`)."""
    nthreads = os.cpu_count() or 1
    sim = oracle_from_inputs(inp, nthreads)
    for _ in range(warmup):
        sim.attempt_step()
    cells = inp["grid"].spec.num_cells
    acc0 = sim.steps_accepted
    t0 = time.perf_counter()
    steps = 0
    while True:
        sim.attempt_step()
        steps += 1
        el = time.perf_counter() - t0
        if (max_steps is not None and steps >= max_steps) or (max_steps is None and el >= budget_s):
            break
    el = time.perf_counter() - t0
    acc = sim.steps_accepted - acc0
    return cells * acc / el / 1e9, nthreads, steps, el


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._nv = pynvml
        except Exception:
            self._nv = None
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self._nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
        }
        while True:
            try:
                # every sample of the timed region counts (short regions would
                # otherwise record nothing: utilisation is a 1/6 s average)
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                self.samples.append(mhz)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            if self._stop.wait(0.02):
                break

    def stop(self):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=2)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(workload, kernel):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)
        return d.get(workload, {}).get(kernel)
    except Exception:
        return None


def run_reference(args, rank, world, scaling):
    """The reference arm: the reference's CPU path (oracle port) on the host
    cores, rank 0 only, each step one attempt over the bounded sample of this
    run's global workload."""
    if rank != 0:
        return 0
    gcells = global_cells(args.workload, world, scaling)
    inp, sample = cpu_sample_inputs(args.workload, gcells)
    rate, nthreads, steps, el = cpu_rate(inp, max_steps=args.steps, warmup=args.warmup)
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * el / max(steps, 1),
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f64" if inp["dtype"] == np.float64 else "f32", "data": "synthetic",
        "impl": "reference",
        "config": config_of(args, world, scaling),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "sample": f"each step: one attempt_step over {sample}; {steps} timed "
                                   f"steps after {args.warmup} warm-up on {nthreads} threads "
                                   "(oracle/clawref.c sweeps + oracle/oracle.py controller)"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def flush_l2(buf):
    buf.zero_()


def run_gpu(args, rank, world, scaling):
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist = None
    rdev = "cuda"
    if world > 1:
        import torch.distributed as tdist
        if args.transport == "host":   # several ranks on one GPU (code-path check only)
            tdist.init_process_group("gloo")
            rdev = "cpu"
        else:
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist
        import logging
        logging.basicConfig(level=logging.WARNING, stream=sys.stderr,
                            format="[rank %d] %%(name)s: %%(message)s" % rank)
        logging.getLogger("clawtile.slab").setLevel(logging.INFO)
    gcells = global_cells(args.workload, world, scaling)
    inp = build_inputs(args.workload, gcells, world, rank, dist, args.transport)
    P = inp["P"]
    sim = P.Simulation(inp["grid"], inp["problem"].solver, inp["params"], inp["bspec"],
                       limiter=inp["limiter"], initial_max_speed=inp["speed"], device=local,
                       slab=inp["slab"])
    dev = sim.device_grid
    # a real (non-legacy) stream: the library maps handle 0 to its own stream,
    # so the L2 flush, the step events and the sweeps must share this one
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    dev.set_stream(stream.cuda_stream)
    flush = torch.empty(1024 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    ndim = inp["spec"].ndim
    m = inp["spec"].num_states
    isz = inp["dtype"].itemsize
    cells = inp["spec"].num_cells        # global cells (all ranks)
    lcells = inp["local_cells"]

    for _ in range(args.warmup):
        sim.attempt_step()
    dev.timing()  # drain
    dev.enable_timing(True)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    sampler = ClockSampler(local).start()
    total_ms = 0.0
    acc0, rev0 = sim.steps_accepted, sim.steps_reverted
    for _ in range(args.steps):
        flush_l2(flush)
        # the device idles before the step starts: the first sweep's launch
        # latency is inside the timed region
        stream.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.attempt_step()
        e1.record(stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    acc = sim.steps_accepted - acc0
    rev = sim.steps_reverted - rev0
    ms_axis, n_axis = dev.timing()
    dev.enable_timing(False)
    launches_timed = int(sum(n_axis))
    if dev.x_variant() == 5:
        # the x geometry pair: two sweep kernels per x sweep (one exits at entry)
        launches_timed += int(n_axis[0])
    # Kernel durations for the roofline: per-launch CUDA events recorded by the
    # library on the launch stream around every sweep of the timed region.
    per_axis = [ms_axis[a] / max(n_axis[a], 1) for a in range(ndim)]
    total_ms_local = total_ms
    if dist:
        t = torch.tensor([total_ms], device=rdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = cells * acc / (total_ms / 1e3) / 1e9

    # roofline: dominant kernel (largest time per launch)
    dom = max(range(ndim), key=lambda a: per_axis[a])
    bytes_per_launch = lcells * m * 2 * isz
    mean_ms = per_axis[dom]
    achieved = bytes_per_launch / (mean_ms / 1e3) / 1e9
    peak, peak_kind = measured_peaks()
    xvar = dev.x_variant() if hasattr(dev, "x_variant") else None
    xname = {2: "TMA tensor-map transpose", 3: "pair warp-march",
             4: "TMA tensor-map transpose, 64 rows x 128 B",
             5: "TMA tensor-map transpose, geometry pair selected per attempt"}.get(xvar,
                                                                                   "warp-march")
    kname = (("x-sweep (contiguous axis, " + xname + ")") if dom == 0
             else f"axis-{dom} sweep (strided, bulk-copy ring)")
    traffic = ncu_traffic(args.workload, f"axis{dom}")
    sim.close()
    del flush

    # e2e through the public API with pinned host buffers
    from paper_1805_08846_b200._native import PinnedBuffer
    pin_in = PinnedBuffer(inp["grid"].interior().shape, inp["dtype"])
    pin_in.array[...] = inp["grid"].interior()
    pin_out = PinnedBuffer(inp["grid"].interior().shape, inp["dtype"])
    if inp["slab"] is not None:
        inp["slab"].dev = None
    sim2 = P.Simulation(inp["grid"], inp["problem"].solver, inp["params"], inp["bspec"],
                        limiter=inp["limiter"], initial_max_speed=inp["speed"], device=local,
                        slab=inp["slab"])
    # warm-up: builds the device controller's attempt graph (one-time setup)
    sim2.run_until(1e30, max_steps=args.warmup)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    sim2.device_grid.upload(sim2._cur, pin_in.array)
    rep = sim2.run_until(1e30, max_steps=args.steps)
    sim2.device_grid.download(sim2._cur, pin_out.array)
    e2e_s = time.perf_counter() - t0
    e2e_acc = rep.steps_accepted
    e2e_att = len(rep.attempts)
    sim2.close()
    pin_in.free()
    pin_out.free()
    if dist:
        t = torch.tensor([e2e_s], device=rdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    state_bytes = inp["grid"].interior().nbytes
    rec_bytes = 48  # clb_attempt record read back per attempt
    e2e = {"value": cells * e2e_acc / e2e_s / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": int(state_bytes / args.steps),
           "d2h_bytes_per_step": int(state_bytes / args.steps + rec_bytes * e2e_att / args.steps),
           "api": "Simulation.run_until(max_steps=K)"
                  + (" (device-resident controller, one batch)" if world == 1 else
                     " (device-resident controller; halo exchange and max-allreduce over "
                     "NCCL inside the attempt graph)" if args.transport == "device" else
                     " (per-attempt host loop with NCCL halo exchange + max-allreduce)")
                  + ": pinned H2D upload of the state, K steps, D2H of the state and the "
                    "attempt records; wall clock, max over ranks",
           "steps_accepted": e2e_acc, "attempts": e2e_att}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu:
        del inp["grid"]
        sinp, sample = cpu_sample_inputs(args.workload, gcells)
        rate, nthreads, steps, el = cpu_rate(sinp, budget_s=args.cpu_budget)
        cpu = {"value": rate, "unit": UNIT, "cores": nthreads, "kind": "port",
               "sample": f"{steps} attempt_steps over {sample} in {el:.1f} s on {nthreads} "
                         "host threads (oracle/clawref.c)"}
    is_sw64 = inp["problem"].solver_name == "shallow_water" and inp["dtype"] == np.float64
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": (value / PUBLISHED_SW_FP64) if is_sw64 else None,
        "dtype": "f64" if inp["dtype"] == np.float64 else "f32", "data": "synthetic",
        "config": config_of(args, world, scaling),
        "run": {"steps_accepted": acc, "steps_reverted": rev,
                "vs_baseline_ref": "CUDACLAW SW 1000^2 fp64 9.2 ms/step, C2050 (BASELINE.md)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": f"{kname} (axis {dom})",
                     "bytes_per_launch": bytes_per_launch, "mean_launch_ms": mean_ms,
                     "peak_kind": peak_kind,
                     "algorithmic_bytes": "m states read + m written per cell per sweep "
                                          f"({m} x 2 x {isz} B) x {lcells} cells per launch",
                     "method": "CUDA events recorded on the launch stream around every "
                               "sweep launch of the timed region (clb_enable_timing)",
                     "per_axis_ms_in_step": per_axis,
                     "kernel_share_of_step": sum(ms_axis[:ndim]) / max(total_ms_local, 1e-9)},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches_timed,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", choices=["strong", "weak"], default=None,
                    help="strong: the workload's grid split over the ranks; weak: each rank "
                         "owns one workload-sized slab (default: strong for c4, else weak)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--transport", default="device", choices=["device", "nccl", "host"],
                    help="halo transport for N>1: device (NCCL inside the library, exchange "
                         "and max-allreduce in the attempt graph), nccl (torch NCCL per "
                         "attempt), host (gloo, for ranks sharing one GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    scaling = args.scaling or DEFAULT_SCALING.get(args.workload, "weak")
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        return run_reference(args, rank, world, scaling)
    return run_gpu(args, rank, world, scaling)


if __name__ == "__main__":
    sys.exit(main())
