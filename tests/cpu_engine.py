"""Test double with DeviceGrid's interface whose arithmetic is the CPU oracle
(TEST INFRASTRUCTURE): lets the slab decomposition's host logic (halo
exchange, HALO boundary mapping, max-allreduce, blow-up location) run under
gloo on CPU and be checked bit-for-bit against a single-domain run."""

from __future__ import annotations

import numpy as np

from oracle import oracle as O

_SOLVERS = {0: "advection", 1: "acoustics", 2: "shallow_water", 3: "vc_acoustics"}
_LIMS = {0: "none", 1: "minmod", 2: "superbee", 3: "mc", 4: "vanleer"}
_KINDS = {0: "outflow", 1: "reflective", 2: "periodic", 3: "halo"}


class OracleEngine:
    def __init__(self, *, ndim, cells, spacing, num_states, dtype, solver_id, limiter_id, params,
                 bc, normal_velocity, device=0):
        self.ndim = ndim
        self.cells = tuple(int(c) for c in cells[:ndim])
        self.spacing = tuple(float(s) for s in spacing[:ndim])
        self.m = num_states
        self.dtype = np.dtype(dtype)
        self.solver = _SOLVERS[solver_id]
        self.limiter = _LIMS[limiter_id]
        p = np.asarray(params, dtype=self.dtype)
        self.params = {"acoustics": lambda: {"sound_speed": float(p[0]), "impedance": float(p[1])},
                       "shallow_water": lambda: {"gravity": float(p[0])},
                       "advection": lambda: {"speed": float(p[0])},
                       "vc_acoustics": lambda: {}}[self.solver]()
        self.bc = [tuple(b) for b in bc]
        self.nv = list(normal_velocity)
        shape = (self.m,) + tuple(c + 4 for c in reversed(self.cells))
        self.bufs = [np.zeros(shape, dtype=self.dtype) for _ in range(3)]
        self.speeds = [0.0] * 4
        self.flags = [False] * 4

    def _isl(self):
        return (slice(None),) + (slice(2, -2),) * self.ndim

    def upload(self, buf, interior):
        self.bufs[buf][self._isl()] = interior

    def download(self, buf, out=None):
        return np.ascontiguousarray(self.bufs[buf][self._isl()])

    def set_stream(self, s):
        pass

    def close(self):
        pass

    def _fill(self, data, axis):
        nd = self.ndim
        arr_axis = 1 + (nd - 1 - axis)
        n = self.cells[axis]

        def sl(a, b, step=None, state=None):
            idx = [slice(None)] * (nd + 1)
            idx[arr_axis] = slice(a, b, step)
            if state is not None:
                idx[0] = state
            return tuple(idx)

        lo, hi = (_KINDS[k] for k in self.bc[axis])
        nv = self.nv[axis]
        if lo == "outflow":
            data[sl(0, 2)] = data[sl(2, 3)]
        elif lo == "periodic":
            data[sl(0, 2)] = data[sl(n, n + 2)]
        elif lo == "reflective":
            data[sl(0, 2)] = data[sl(3, 1, -1)]
            data[sl(0, 2, state=nv)] *= -1.0
        if hi == "outflow":
            data[sl(n + 2, n + 4)] = data[sl(n + 1, n + 2)]
        elif hi == "periodic":
            data[sl(n + 2, n + 4)] = data[sl(2, 4)]
        elif hi == "reflective":
            data[sl(n + 2, n + 4)] = data[sl(n + 1, n - 1, -1)]
            data[sl(n + 2, n + 4, state=nv)] *= -1.0

    def sweep_async(self, axis, dt, src, dst, slot, literal=False):
        s = self.bufs[src]
        self._fill(s, axis)
        smax = O.sweep(s, self.bufs[dst], axis, dt, self.spacing, self.solver, self.limiter,
                       self.params)
        self.speeds[slot] = max(self.speeds[slot], smax)
        self.flags[slot] = self.flags[slot] or not np.all(np.isfinite(self.bufs[dst][self._isl()]))

    # segment-range launches: the oracle sweeps whole pencils, so ranges are
    # collected and the sweep runs once all segments of the axis were
    # requested (interior segments read no ghost row, so running them after
    # the halo exchange gives the same bytes as the device's early launch)
    def segments(self, axis):
        n = self.cells[axis]
        seg_len = max(4, -(-n // 4))
        return -(-n // seg_len), seg_len

    def sweep_async_range(self, axis, dt, src, dst, slot, seg_begin, seg_end, literal=False):
        nseg, _ = self.segments(axis)
        pend = self.__dict__.setdefault("_pending", {})
        key = (axis, dt, src, dst, slot)
        got = pend.setdefault(key, set())
        got.update(range(seg_begin, seg_end))
        if len(got) == nseg:
            del pend[key]
            self.sweep_async(axis, dt, src, dst, slot, literal)

    def fetch(self, n):
        out = (self.speeds[:n], self.flags[:n])
        self.speeds = [0.0] * 4
        self.flags = [False] * 4
        return out

    def attempt_step(self, dt, src, s0, s1):
        cur = src
        for j in range(self.ndim):
            dst = s0 if j % 2 == 0 else s1
            self.sweep_async(j, dt, cur, dst, j)
            cur = dst
        return self.fetch(self.ndim)

    def first_nonfinite(self, buf):
        inner = self.bufs[buf][self._isl()]
        bad = np.argwhere(~np.isfinite(inner))
        if bad.size == 0:
            return None
        return int(bad[0][0]), tuple(int(c) for c in reversed(bad[0][1:]))

    def _rows(self, side, ghost):
        nd = self.ndim
        n = self.cells[nd - 1]
        if side == 0:
            rng = slice(0, 2) if ghost else slice(2, 4)
        else:
            rng = slice(n + 2, n + 4) if ghost else slice(n, n + 2)
        return (slice(None), rng)

    def halo_read(self, buf, side):
        blk = np.ascontiguousarray(self.bufs[buf][self._rows(side, False)])
        return blk.reshape(self.m, -1).view(np.uint8)

    def halo_write(self, buf, side, data):
        tgt = self.bufs[buf][self._rows(side, True)]
        tgt[...] = np.asarray(data).view(self.dtype).reshape(tgt.shape)
