"""CPU oracle for the time-step hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker and the CPU baseline.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it; the product package never does.

It restates the reference clawtile path (paths relative to
/root/reference/pkg/src/clawtile):

* ``pack_params``      riemann.py:235-253
* ``apply_boundary``   boundary.py:87-122 (numpy, same face order)
* ``sweep``            sweep.py:307-377 / 380-391 driving the C kernel
                       ``oracle/clawref.c`` (sweep.py:183-263)
* ``OracleSimulation`` timestep.py:75-285 (estimate_dt, attempt_step,
                       run_until, buffer rotation, revert bookkeeping)

Parity pin: tests/test_oracle.py checks this module byte-for-byte against
golden vectors produced by the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libclawref.so")

SOLVER_IDS = {"advection": 0, "acoustics": 1, "shallow_water": 2, "vc_acoustics": 3}
NUM_WAVES = {"advection": 1, "acoustics": 2, "shallow_water": 3, "vc_acoustics": 2}
LIMITER_IDS = {"none": 0, "minmod": 1, "superbee": 2, "mc": 3, "vanleer": 4}
GHOST = 2

_lib = None


def build() -> str:
    """Compile the C restatement (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.clawref_sweep.restype = ctypes.c_double
        L.clawref_sweep.argtypes = [
            ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_double,
            ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
            ctypes.c_int,
        ]
        L.clawref_solve.restype = None
        L.clawref_solve.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
            ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
        ]
        L.clawref_limiter.restype = ctypes.c_double
        L.clawref_limiter.argtypes = [ctypes.c_double, ctypes.c_int]
        _lib = L
    return _lib


# ---------------------------------------------------------------------------
# riemann.py:235-253


def pack_params(solver: str, params: dict, dtype) -> np.ndarray:
    dt = np.dtype(dtype)
    if solver == "acoustics":
        out = np.zeros(3, dtype=dt)
        out[0] = params["sound_speed"]
        out[1] = params["impedance"]
        out[2] = dt.type(0.5) / out[1]
        return out
    if solver == "shallow_water":
        out = np.zeros(2, dtype=dt)
        out[0] = params["gravity"]
        out[1] = 0.5
        return out
    if solver == "advection":
        out = np.zeros(1, dtype=dt)
        out[0] = params["speed"]
        return out
    if solver == "vc_acoustics":
        return np.zeros(1, dtype=dt)
    raise KeyError(solver)


def normal_index(solver: str, axis: int) -> int:
    # riemann.py:187 default 1+axis; advection maps to 0 (riemann.py:280-284)
    return 0 if solver == "advection" else 1 + axis


# ---------------------------------------------------------------------------
# boundary.py:87-122


def apply_boundary(data: np.ndarray, sides, normal_velocity) -> None:
    """Fill ghost layers of a padded (m, [nz+4,] [ny+4,] nx+4) array in place.

    ``sides[axis] = (lo, hi)`` with kinds "outflow" | "reflective" | "periodic".
    """
    nd = data.ndim - 1
    g = GHOST
    for axis in range(nd):
        arr_axis = 1 + (nd - 1 - axis)
        n = data.shape[arr_axis] - 2 * g

        def sl(rng, state=None):
            idx = [slice(None)] * (nd + 1)
            idx[arr_axis] = rng
            if state is not None:
                idx[0] = state
            return tuple(idx)

        lo, hi = sides[axis]
        nvel = normal_velocity[axis]
        if lo == "outflow":
            data[sl(slice(0, g))] = data[sl(slice(g, g + 1))]
        elif lo == "periodic":
            data[sl(slice(0, g))] = data[sl(slice(n, n + g))]
        else:
            data[sl(slice(0, g))] = data[sl(slice(2 * g - 1, g - 1, -1))]
            data[sl(slice(0, g), nvel)] *= -1.0
        if hi == "outflow":
            data[sl(slice(n + g, n + 2 * g))] = data[sl(slice(n + g - 1, n + g))]
        elif hi == "periodic":
            data[sl(slice(n + g, n + 2 * g))] = data[sl(slice(g, 2 * g))]
        else:
            data[sl(slice(n + g, n + 2 * g))] = data[sl(slice(n + g - 1, n - 1, -1))]
            data[sl(slice(n + g, n + 2 * g), nvel)] *= -1.0


def copy_ghost(dst: np.ndarray, src: np.ndarray) -> None:
    """sweep.py:294-304"""
    nd = dst.ndim - 1
    g = GHOST
    for axis in range(nd):
        arr_axis = 1 + (nd - 1 - axis)
        n = dst.shape[arr_axis] - 2 * g
        for rng in (slice(0, g), slice(n + g, n + 2 * g)):
            idx = [slice(None)] * (nd + 1)
            idx[arr_axis] = rng
            dst[tuple(idx)] = src[tuple(idx)]


def interior(data: np.ndarray) -> np.ndarray:
    nd = data.ndim - 1
    return data[(slice(None),) + (slice(GHOST, -GHOST),) * nd]


# ---------------------------------------------------------------------------
# sweep.py:307-391


def sweep(qin: np.ndarray, qout: np.ndarray, axis: int, dt: float, spacing,
          solver: str, limiter: str, params: dict, nthreads: int = 1) -> float:
    """One monolithic directional sweep; returns max |s| (Python float)."""
    if qin.shape != qout.shape or qin.dtype != qout.dtype:
        raise ValueError("input and output grids must share spec and dtype")
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    assert qin.flags.c_contiguous and qout.flags.c_contiguous
    nd = qin.ndim - 1
    m = qin.shape[0]
    cells = np.array([qin.shape[1 + (nd - 1 - ax)] - 2 * GHOST for ax in range(nd)],
                     dtype=np.int64)
    dtype = qin.dtype
    dtdx = dtype.type(dt / spacing[axis])  # sweep.py:336-337
    pvec = pack_params(solver, params, dtype)
    copy_ghost(qout, qin)
    smax = lib().clawref_sweep(
        nd, cells.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), m, dtype.itemsize,
        qin.ctypes.data, qout.ctypes.data, axis, float(dtdx), SOLVER_IDS[solver],
        normal_index(solver, axis), pvec.ctypes.data, LIMITER_IDS[limiter],
        NUM_WAVES[solver], int(nthreads),
    )
    if smax < 0.0:
        raise ValueError("oracle sweep rejected its arguments")
    return float(smax)


def solve(solver: str, ql, qr, axis: int, params: dict, dtype=np.float64):
    dt = np.dtype(dtype)
    ql = np.ascontiguousarray(ql, dtype=dt)
    qr = np.ascontiguousarray(qr, dtype=dt)
    m = ql.shape[0]
    nw = NUM_WAVES[solver]
    W = np.zeros((nw, m), dtype=dt)
    s = np.zeros(nw, dtype=dt)
    pv = pack_params(solver, params, dt)
    lib().clawref_solve(SOLVER_IDS[solver], dt.itemsize, ql.ctypes.data, qr.ctypes.data, m,
                        normal_index(solver, axis), pv.ctypes.data, W.ctypes.data,
                        s.ctypes.data)
    return W, s


# ---------------------------------------------------------------------------
# timestep.py:45-285


@dataclass(frozen=True)
class Attempt:
    t_start: float
    dt: float
    max_speed: float
    nu: float
    accepted: bool
    landed: bool
    dt_retry: float | None = None


@dataclass
class Report:
    steps_accepted: int = 0
    steps_reverted: int = 0
    t_final: float = 0.0
    nu_max: float = 0.0
    attempts: list = field(default_factory=list)


class OracleBlowup(Exception):
    def __init__(self, state, cell, step):
        self.state, self.cell, self.step = state, cell, step
        super().__init__(f"non-finite value in state {state} at interior cell {cell} during step {step}")


class OracleUnstable(Exception):
    pass


class OracleSimulation:
    """Restatement of clawtile.timestep.Simulation over plain padded arrays."""

    def __init__(self, data: np.ndarray, spacing, solver: str, params: dict, sides,
                 normal_velocity, *, limiter="mc", cfl_target=0.9, cfl_max=1.0,
                 dt_cap=math.inf, initial_max_speed=None, nthreads=1):
        if not 0.0 < cfl_target <= cfl_max <= 1.0:
            raise ValueError("need 0 < cfl_target <= cfl_max <= 1")
        if dt_cap <= 0.0:
            raise ValueError("dt_cap must be positive")
        self.grid = np.ascontiguousarray(data)
        self.spacing = tuple(float(s) for s in spacing)
        self.solver, self.params = solver, params
        self.sides, self.normal_velocity = sides, normal_velocity
        self.limiter = limiter
        self.cfl_target, self.cfl_max, self.dt_cap = float(cfl_target), float(cfl_max), float(dt_cap)
        self.nthreads = nthreads
        self.ndim = data.ndim - 1
        self._scratch = [np.zeros_like(self.grid) for _ in range(2)]
        self._min_spacing = min(self.spacing)
        self.t = 0.0
        self.steps_accepted = 0
        self.steps_reverted = 0
        self.nu_max = 0.0
        self._prev_reverted = False
        self._prev_nu = math.inf
        self.last_max_speed = float(initial_max_speed or 0.0)

    def estimate_dt(self, stop=None):
        s = self.last_max_speed
        if s > 0.0:
            dt = self.cfl_target * self._min_spacing / s
            dt = min(dt, self.dt_cap)
        else:
            dt = self.dt_cap
        landed = False
        if stop is not None:
            remaining = stop - self.t
            if remaining <= 0.0:
                raise ValueError(f"stop time {stop} is not ahead of t={self.t}")
            if dt >= remaining:
                dt = remaining
                landed = True
        if not math.isfinite(dt):
            raise ValueError("cannot size a step: no wave activity, no dt cap, no stop time")
        return dt, landed

    def _check_finite(self, out):
        inner = interior(out)
        if np.all(np.isfinite(inner)):
            return
        bad = np.argwhere(~np.isfinite(inner))[0]
        raise OracleBlowup(int(bad[0]), tuple(int(c) for c in reversed(bad[1:])),
                           self.steps_accepted)

    def attempt_step(self, stop=None) -> Attempt:
        dt, landed = self.estimate_dt(stop)
        t_start = self.t
        src = self.grid
        step_speed = 0.0
        for j, axis in enumerate(range(self.ndim)):
            apply_boundary(src, self.sides, self.normal_velocity)
            dst = self._scratch[j % 2]
            smax = sweep(src, dst, axis, dt, self.spacing, self.solver, self.limiter,
                         self.params, self.nthreads)
            self._check_finite(dst)
            step_speed = max(step_speed, smax)
            src = dst
        nu = dt * step_speed / self._min_spacing
        accepted = nu <= self.cfl_max
        dt_retry = None
        if accepted:
            last = (self.ndim - 1) % 2
            final = src
            self._scratch = [self.grid, self._scratch[1 - last]]
            self.grid = final
            self.t = stop if (landed and stop is not None) else t_start + dt
            self.steps_accepted += 1
            self.nu_max = max(self.nu_max, nu)
            self._prev_reverted = False
        else:
            self.steps_reverted += 1
            dt_retry = self.cfl_target * self._min_spacing / step_speed
            if self._prev_reverted and nu >= self._prev_nu:
                raise OracleUnstable("two consecutive reverted steps without improvement")
            self._prev_reverted = True
            self._prev_nu = nu
        self.last_max_speed = step_speed
        return Attempt(t_start, dt, step_speed, nu, accepted, landed and accepted, dt_retry)

    def run_until(self, t_end, frame_times=(), on_frame=None, max_steps=None) -> Report:
        if t_end < self.t:
            raise ValueError(f"t_end {t_end} is behind current t {self.t}")
        frames = sorted(frame_times)
        for ft in frames:
            if ft <= self.t or ft > t_end:
                raise ValueError(f"frame time {ft} outside the run window ({self.t}, {t_end}]")
        report = Report(t_final=self.t)
        fi = 0
        start = self.steps_accepted
        while self.t < t_end:
            if max_steps is not None and self.steps_accepted - start >= max_steps:
                break
            stop = frames[fi] if fi < len(frames) else t_end
            a = self.attempt_step(stop=stop)
            report.attempts.append(a)
            if a.accepted:
                report.steps_accepted += 1
                report.nu_max = max(report.nu_max, a.nu)
                while fi < len(frames) and self.t >= frames[fi]:
                    if on_frame is not None:
                        on_frame(self)
                    fi += 1
            else:
                report.steps_reverted += 1
        report.t_final = self.t
        return report
