"""Directional sweep operator (mirrors clawtile/sweep.py public API).

``sweep_axis`` / ``sweep_axis_tiled`` are the reference's per-sweep operator
(sweep.py:307-391): read ``q_in`` (ghost cells as the caller filled them),
write the updated interior of ``q_out``, return the max wave speed.  Here the
arrays are uploaded to a device handle, the fused sm_100a sweep kernel runs
with the swept axis in HALO mode (ghosts read as-is, exactly what the
reference kernel does, sweep.py:206-212), and the interior is read back.

Tile plans are kept for API compatibility and validated like the reference,
but the device ignores their shape: CTA/warp segments recompute shared fans
exactly as tiles do, so the result is bitwise the same for any plan
(pkg/tests/test_sweep.py:191-226 property).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

from . import perf
from ._native import DeviceGrid
from .boundary import BC_HALO
from .grid import GridSpec, StateGrid
from .limiter import LIMITER_IDS, LimiterKind
from .riemann import RiemannSolver


@dataclass(frozen=True)
class Tile:
    """Owned cell ranges per logical axis, interior coordinates (sweep.py:34-65)."""

    owned: tuple

    def __post_init__(self):
        object.__setattr__(self, "owned", tuple(tuple(r) for r in self.owned))

    def width(self, axis: int) -> int:
        lo, hi = self.owned[axis]
        return hi - lo

    def num_cells(self) -> int:
        n = 1
        for lo, hi in self.owned:
            n *= hi - lo
        return n

    def halo(self, sweep_axis: int):
        return tuple((lo - 2, hi + 2) if ax == sweep_axis else (lo, hi)
                     for ax, (lo, hi) in enumerate(self.owned))


@dataclass(frozen=True)
class TilePlan:
    """Disjoint tiles covering the interior exactly (sweep.py:68-100)."""

    axis: int
    tile_shape: tuple
    cells: tuple
    tiles: tuple = field(repr=False)

    def __post_init__(self):
        total = 0
        for t in self.tiles:
            if len(t.owned) != len(self.cells):
                raise ValueError("tile dimensionality does not match the grid")
            for axis, (lo, hi) in enumerate(t.owned):
                if not 0 <= lo < hi <= self.cells[axis]:
                    raise ValueError(f"tile range {(lo, hi)} outside axis {axis}")
            total += t.num_cells()
        expect = 1
        for c in self.cells:
            expect *= c
        if total != expect:
            raise ValueError("tiles do not cover the interior exactly")

    @property
    def num_tiles(self) -> int:
        return len(self.tiles)

    def redundant_fractions(self):
        return tuple(4.0 / (t.width(self.axis) + 4.0) for t in self.tiles)


def _chunk(n: int, w: int):
    return [(lo, min(lo + w, n)) for lo in range(0, n, w)]


def plan_tiles(spec: GridSpec, axis: int, tile_shape) -> TilePlan:
    """Partition the interior into tiles (sweep.py:107-130)."""
    if not 0 <= axis < spec.ndim:
        raise ValueError(f"sweep axis {axis} out of range for {spec.ndim}-D grid")
    tile_shape = tuple(int(w) for w in tile_shape)
    if len(tile_shape) != spec.ndim:
        raise ValueError(f"tile shape has {len(tile_shape)} axes, grid has {spec.ndim}")
    if any(w < 1 for w in tile_shape):
        raise ValueError("tile extents must be positive")
    per_axis = [_chunk(n, w) for n, w in zip(spec.cells, tile_shape)]
    tiles = tuple(Tile(owned=tuple(reversed(combo)))
                  for combo in itertools.product(*reversed(per_axis)))
    return TilePlan(axis=axis, tile_shape=tile_shape, cells=spec.cells, tiles=tiles)


@dataclass(frozen=True)
class SweepResult:
    max_abs_speed: float
    counters: object = None
    stage_flops: dict = field(default_factory=dict)


_OPERATORS: dict = {}


def _operator(spec: GridSpec, dtype, solver: RiemannSolver, limiter: LimiterKind, params):
    pv = solver.pack_params(params, dtype)
    key = (spec, np.dtype(dtype).name, solver.name, limiter, pv.tobytes())
    g = _OPERATORS.get(key)
    if g is None:
        if len(_OPERATORS) > 16:
            for k in list(_OPERATORS)[:8]:
                _OPERATORS.pop(k).close()
        nd = spec.ndim
        g = DeviceGrid(ndim=nd, cells=spec.cells, spacing=spec.spacing,
                       num_states=spec.num_states, dtype=dtype,
                       solver_id=solver.require_device(spec.num_states, nd, dtype),
                       limiter_id=LIMITER_IDS[limiter],
                       params=pv, bc=[(BC_HALO, BC_HALO)] * nd, normal_velocity=[None] * nd)
        _OPERATORS[key] = g
    return g


def _copy_ghost(dst: StateGrid, src: StateGrid) -> None:
    """sweep.py:294-304 (host data movement of the ghost slabs)."""
    g = dst.spec.ghost
    nd = dst.spec.ndim
    for axis in range(nd):
        arr_axis = 1 + (nd - 1 - axis)
        n = dst.spec.cells[axis]
        for rng in (slice(0, g), slice(n + g, n + 2 * g)):
            idx = [slice(None)] * (nd + 1)
            idx[arr_axis] = rng
            dst.data[tuple(idx)] = src.data[tuple(idx)]


def sweep_axis_tiled(q_in: StateGrid, q_out: StateGrid, axis: int, dt: float,
                     solver: RiemannSolver, limiter: LimiterKind, params: object,
                     plan: TilePlan, workers: int = 1, executor=None) -> SweepResult:
    """One directional sweep on the device (sweep.py:307-377 contract)."""
    spec = q_in.spec
    if q_out.spec != spec or q_out.dtype != q_in.dtype:
        raise ValueError("input and output grids must share spec and dtype")
    if q_out is q_in or q_out.data is q_in.data:
        raise ValueError("sweep cannot run in place")
    if plan.axis != axis or plan.cells != spec.cells:
        raise ValueError("tile plan does not match this grid/axis")
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    normal = solver.normal_index(axis)
    if spec.num_states > 1 and not 0 <= normal < spec.num_states:
        raise ValueError(f"normal index {normal} out of range")
    g = _operator(spec, q_in.dtype, solver, limiter, params)
    g.upload_padded(0, q_in.data)
    smax, _ = g.sweep(axis, float(dt), 0, 1)
    _copy_ghost(q_out, q_in)
    q_out.interior()[...] = g.download(1)
    # the reference's modeled counters of this sweep (sweep.py:370-377)
    try:
        counters, stage_flops = perf.sweep_counters(plan, spec, solver, limiter,
                                                    q_in.dtype.itemsize)
    except ValueError:   # a device-only user solver has no scalar to price
        counters, stage_flops = None, {}
    return SweepResult(max_abs_speed=float(smax), counters=counters, stage_flops=stage_flops)


def sweep_axis(q_in: StateGrid, q_out: StateGrid, axis: int, dt: float,
               solver: RiemannSolver, limiter: LimiterKind, params: object) -> SweepResult:
    """Untiled sweep (sweep.py:380-391)."""
    plan = plan_tiles(q_in.spec, axis, q_in.spec.cells)
    return sweep_axis_tiled(q_in, q_out, axis, dt, solver, limiter, params, plan)
