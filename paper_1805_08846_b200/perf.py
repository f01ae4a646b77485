"""Operation and traffic accounting for the sweeps (§8(f) row 2).

Two models, side by side:

* **The reference's model** (clawtile/perf.py:1-588, restated): every
  event -- an interface solve, a fan's fluctuation sums, a correction, a cell
  update -- is priced by shadow-executing the reference's scalar routines on
  a counting float (adds, multiplies, negations, abs are flops; divisions and
  square roots are "special"), and multiplied by the event counts of the
  tile plan (a tile of ``w`` cells reads ``w + 4`` per pencil).  The names
  and signatures are the reference's: ``sweep_counters(plan, spec, solver,
  limiter, itemsize)``, ``RunCounters``, ``build_report``, ``render_text``,
  ``render_delimited``; ``SweepResult.counters`` and ``Simulation.counters``
  carry them exactly as the reference does.  The scalar routines priced are
  restated below from riemann.py:116-173 (the device runs functors, not
  Python scalars).
* **The B200 kernel model** (``kernel_event_costs``, ``kernel_sweep_counters``):
  the arithmetic the sm_100a kernels actually execute (structural zeros
  elided, per-cell hoisting, segment halos of the library's own
  decomposition), put beside measured kernel times by ``run_measured_perf``
  and beside ncu DRAM bytes when a capture is supplied.
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

_AXES = ("x", "y", "z")


@dataclass
class KernelCounters:
    """Accumulated operation and byte counts (perf.py:35-63)."""

    flops: int = 0
    special: int = 0
    bytes_read: int = 0
    bytes_written: int = 0

    @property
    def total_flops(self) -> int:
        return self.flops + self.special

    @property
    def total_bytes(self) -> int:
        return self.bytes_read + self.bytes_written

    def add(self, other: "KernelCounters") -> None:
        self.flops += other.flops
        self.special += other.special
        self.bytes_read += other.bytes_read
        self.bytes_written += other.bytes_written

    def scaled(self, n: int) -> "KernelCounters":
        return KernelCounters(self.flops * n, self.special * n, self.bytes_read * n,
                              self.bytes_written * n)


@dataclass(frozen=True)
class MachineModel:
    """Peak rates for roofline bounds (perf.py:66-82)."""

    peak_flops: float       # flop/s
    peak_bandwidth: float   # bytes/s
    special_function_peak: float | None = None

    def __post_init__(self):
        if self.peak_flops <= 0.0 or self.peak_bandwidth <= 0.0:
            raise ValueError("machine peaks must be positive")
        if self.special_function_peak is not None and self.special_function_peak <= 0.0:
            raise ValueError("special_function_peak must be positive")


def operational_intensity(c: KernelCounters) -> float:
    """Flops per byte of modeled traffic; zero traffic is an error."""
    if c.total_bytes == 0:
        raise ValueError("operational intensity undefined for zero bytes")
    return c.total_flops / c.total_bytes


def roofline_bound(oi: float, machine: MachineModel) -> float:
    """Attainable flops/s: compute plateau or bandwidth diagonal."""
    if oi < 0.0:
        raise ValueError("operational intensity cannot be negative")
    return min(machine.peak_flops, oi * machine.peak_bandwidth)


# ---------------------------------------------------------------------------
# The reference's model (perf.py:100-439): counting float + event prices


class _RTally:
    __slots__ = ("adds", "muls", "divs", "sqrts", "negs", "abses", "minmaxes")

    def __init__(self):
        self.adds = self.muls = self.divs = self.sqrts = 0
        self.negs = self.abses = self.minmaxes = 0

    @property
    def flops(self) -> int:
        return self.adds + self.muls + self.negs + self.abses + self.minmaxes

    @property
    def special(self) -> int:
        return self.divs + self.sqrts


class _RCF:
    """The reference's counting float (perf.py:113-190)."""

    __slots__ = ("v", "t")

    def __init__(self, v, t):
        self.v = float(v)
        self.t = t

    def _w(self, v):
        return _RCF(v, self.t)

    @staticmethod
    def _val(o):
        return o.v if isinstance(o, _RCF) else float(o)

    def __add__(self, o):
        self.t.adds += 1
        return self._w(self.v + self._val(o))

    __radd__ = __add__

    def __sub__(self, o):
        self.t.adds += 1
        return self._w(self.v - self._val(o))

    def __rsub__(self, o):
        self.t.adds += 1
        return self._w(self._val(o) - self.v)

    def __mul__(self, o):
        self.t.muls += 1
        return self._w(self.v * self._val(o))

    __rmul__ = __mul__

    def __truediv__(self, o):
        self.t.divs += 1
        return self._w(self.v / self._val(o))

    def __rtruediv__(self, o):
        self.t.divs += 1
        return self._w(self._val(o) / self.v)

    def __neg__(self):
        self.t.negs += 1
        return self._w(-self.v)

    def __abs__(self):
        self.t.abses += 1
        return self._w(abs(self.v))

    def sqrt(self):
        self.t.sqrts += 1
        return self._w(math.sqrt(self.v))

    def __lt__(self, o): return self.v < self._val(o)
    def __le__(self, o): return self.v <= self._val(o)
    def __gt__(self, o): return self.v > self._val(o)
    def __ge__(self, o): return self.v >= self._val(o)
    def __float__(self): return self.v


def _cf_array(values, t):
    out = np.empty(len(values), dtype=object)
    for i, v in enumerate(values):
        out[i] = _RCF(v, t)
    return out


# The reference's scalar routines (riemann.py:116-173), restated for pricing
# only; vc_acoustics is the builder's registered scalar (make_golden.py).
def _sc_acoustics(ql, qr, normal, params, W, s):
    c, Z, inv2z = params[0], params[1], params[2]
    dp = qr[0] - ql[0]
    dun = qr[normal] - ql[normal]
    b1 = (Z * dun - dp) * inv2z
    b2 = (Z * dun + dp) * inv2z
    for k in range(W.shape[1]):
        W[0, k] = 0
        W[1, k] = 0
    W[0, 0] = -Z * b1
    W[0, normal] = b1
    W[1, 0] = Z * b2
    W[1, normal] = b2
    s[0] = -c
    s[1] = c


def _sc_shallow_water(ql, qr, normal, params, W, s):
    g, half = params[0], params[1]
    trans = 3 - normal
    hl, hr = ql[0], qr[0]
    sl, sr = hl.sqrt(), hr.sqrt()
    denom = sl + sr
    uhat = (ql[normal] / sl + qr[normal] / sr) / denom
    vhat = (ql[trans] / sl + qr[trans] / sr) / denom
    chat = (g * (half * (hl + hr))).sqrt()
    dh = qr[0] - ql[0]
    dhun = qr[normal] - ql[normal]
    dhut = qr[trans] - ql[trans]
    inv2c = half / chat
    a1 = ((uhat + chat) * dh - dhun) * inv2c
    a3 = (dhun - (uhat - chat) * dh) * inv2c
    a2 = dhut - vhat * dh
    W[0, 0] = a1
    W[0, normal] = a1 * (uhat - chat)
    W[0, trans] = a1 * vhat
    W[1, 0] = 0
    W[1, normal] = 0
    W[1, trans] = a2
    W[2, 0] = a3
    W[2, normal] = a3 * (uhat + chat)
    W[2, trans] = a3 * vhat
    s[0] = uhat - chat
    s[1] = uhat
    s[2] = uhat + chat


def _sc_advection(ql, qr, normal, params, W, s):
    W[0, 0] = qr[0] - ql[0]
    s[0] = params[0]


def _sc_vc_acoustics(ql, qr, normal, params, W, s):
    m = W.shape[1]
    Zl, Zr, cl, cr = ql[m - 2], qr[m - 2], ql[m - 1], qr[m - 1]
    dp = qr[0] - ql[0]
    dun = qr[normal] - ql[normal]
    denom = Zl + Zr
    a1 = (Zr * dun - dp) / denom
    a2 = (Zl * dun + dp) / denom
    for k in range(m):
        W[0, k] = 0
        W[1, k] = 0
    W[0, 0] = -Zl * a1
    W[0, normal] = a1
    W[1, 0] = Zr * a2
    W[1, normal] = a2
    s[0] = -cl
    s[1] = cr


_MODEL_SCALARS = {"acoustics": (_sc_acoustics, 2), "shallow_water": (_sc_shallow_water, 3),
                  "advection": (_sc_advection, 1), "vc_acoustics": (_sc_vc_acoustics, 2)}

# Representative interface states and parameters (perf.py:196-233).
_SAMPLE_STATES = {
    "acoustics": ([1.2, 0.3, -0.4, 0.2], [0.7, -0.1, 0.5, -0.3]),
    "shallow_water": ([1.5, 0.4, -0.3], [0.9, -0.2, 0.6]),
    "advection": ([1.3], [0.4]),
}
_SAMPLE_PACKED = {
    "acoustics": [1.1, 0.9, 0.5 / 0.9],   # AcousticsParams(1.1, 0.9) packed
    "shallow_water": [1.3, 0.5],          # ShallowWaterParams(1.3) packed
    "advection": [0.8],                   # AdvectionParams(0.8) packed
    "vc_acoustics": [0.0],
}


def _sample_pair(name: str, m: int):
    if name in _SAMPLE_STATES:
        ql, qr = (list(v) for v in _SAMPLE_STATES[name])
        while len(ql) < m:
            ql.append(0.15)
            qr.append(-0.25)
        return ql[:m], qr[:m]
    rng = np.random.default_rng(1234)
    return list(0.5 + rng.random(m)), list(0.5 + rng.random(m))


@lru_cache(maxsize=None)
def _solve_cost(solver_name: str, m: int) -> tuple[int, int]:
    """(flops, special) of one interface solve (perf.py:236-253)."""
    scalar, nw = _MODEL_SCALARS[solver_name]
    t = _RTally()
    ql_v, qr_v = _sample_pair(solver_name, m)
    ql, qr = _cf_array(ql_v, t), _cf_array(qr_v, t)
    params = _cf_array(_SAMPLE_PACKED[solver_name], t)
    W = np.empty((nw, m), dtype=object)
    s = np.empty(nw, dtype=object)
    # solver.normal_index(1 if m > 1 else 0) (perf.py:247): 1 + axis, or 0
    # for advection
    normal = 0 if solver_name == "advection" or m == 1 else 2
    scalar(ql, qr, normal, params, W, s)
    return t.flops, t.special


def _kernel_fan_cost(m: int, num_waves: int) -> tuple[int, int]:
    """Fluctuation accumulation per fan (perf.py:256-282)."""
    t = _RTally()
    rng = np.random.default_rng(7)
    W = np.empty((num_waves, m), dtype=object)
    for p in range(num_waves):
        for k in range(m):
            W[p, k] = _RCF(rng.standard_normal(), t)
    S = _cf_array(rng.standard_normal(num_waves) + 1.5, t)
    zero = _RCF(0.0, t)
    am = [zero] * m
    ap = [zero] * m
    smax = zero
    for p in range(num_waves):
        sp = S[p]
        asp = abs(sp)
        if asp > smax:
            smax = asp
        if sp < 0.0:
            for k in range(m):
                am[k] = am[k] + sp * W[p, k]
        elif sp > 0.0:
            for k in range(m):
                ap[k] = ap[k] + sp * W[p, k]
    return t.flops, t.special


def _phi_cost_tally(theta, kind_id: int, t):
    one = _RCF(1.0, t)
    if kind_id == 1:
        v = theta if theta < 1.0 else one
        return v if v > 0.0 else _RCF(0.0, t)
    if kind_id == 2:
        a = 2.0 * theta
        if a > 1.0:
            a = one
        b = theta if theta < 2.0 else _RCF(2.0, t)
        v = a if a > b else b
        return v if v > 0.0 else _RCF(0.0, t)
    if kind_id == 3:
        v = 0.5 * (1.0 + theta)
        if v > 2.0:
            v = _RCF(2.0, t)
        tt = 2.0 * theta
        if tt < v:
            v = tt
        return v if v > 0.0 else _RCF(0.0, t)
    if kind_id == 4:
        a = abs(theta)
        return (theta + a) / (1.0 + a)
    return one


def _correction_cost(m: int, num_waves: int, limiter_id: int) -> tuple[int, int]:
    """Limiting plus second-order flux for one interface (perf.py:311-342)."""
    t = _RTally()
    rng = np.random.default_rng(11)
    Wm = np.empty((num_waves, m), dtype=object)
    Wu = np.empty((num_waves, m), dtype=object)
    for p in range(num_waves):
        for k in range(m):
            Wm[p, k] = _RCF(rng.standard_normal() + 0.1, t)
            Wu[p, k] = _RCF(rng.standard_normal() + 0.1, t)
    S = _cf_array(rng.standard_normal(num_waves) + 1.5, t)
    dtdx = _RCF(0.4, t)
    zero = _RCF(0.0, t)
    ft = [zero] * m
    for p in range(num_waves):
        sp = S[p]
        wn = zero
        wu = zero
        for k in range(m):
            wk = Wm[p, k]
            wn = wn + wk * wk
            wu = wu + Wu[p, k] * wk
        if limiter_id == 0 or wn.v == 0.0:
            lim = _RCF(1.0, t)
        else:
            lim = _phi_cost_tally(wu / wn, limiter_id, t)
        asp = abs(sp)
        coef = 0.5 * asp * (1.0 - dtdx * asp) * lim
        for k in range(m):
            ft[k] = ft[k] + coef * Wm[p, k]
    return t.flops, t.special


def _update_cost(m: int) -> tuple[int, int]:
    """Final cell write (perf.py:345-358)."""
    t = _RTally()
    rng = np.random.default_rng(13)
    q = _cf_array(rng.standard_normal(m), t)
    ap = _cf_array(rng.standard_normal(m), t)
    am = _cf_array(rng.standard_normal(m), t)
    ftn = _cf_array(rng.standard_normal(m), t)
    ftp = _cf_array(rng.standard_normal(m), t)
    dtdx = _RCF(0.4, t)
    for k in range(m):
        _ = q[k] - dtdx * (ap[k] + am[k]) - dtdx * (ftn[k] - ftp[k])
    return t.flops, t.special


@dataclass(frozen=True)
class SweepEvents:
    """Structural event counts for one sweep over one tile plan."""

    fans: int
    corrections: int
    cells: int
    pencil_reads: int  # cells read, halo included
    cells_written: int


def sweep_events(plan, spec) -> SweepEvents:
    """perf.py:372-387."""
    fans = corrections = cells = reads = writes = 0
    for tile in plan.tiles:
        w = tile.width(plan.axis)
        pencils = 1
        for axis, (lo, hi) in enumerate(tile.owned):
            if axis != plan.axis:
                pencils *= hi - lo
        fans += (w + 3) * pencils
        corrections += (w + 1) * pencils
        cells += w * pencils
        reads += (w + 4) * pencils
        writes += w * pencils
    return SweepEvents(fans, corrections, cells, reads, writes)


@lru_cache(maxsize=None)
def _stage_costs(solver_name: str, m: int, num_waves: int, limiter_id: int):
    return (_solve_cost(solver_name, m), _kernel_fan_cost(m, num_waves),
            _correction_cost(m, num_waves, limiter_id), _update_cost(m))


def sweep_counters(plan, spec, solver, limiter, itemsize: int) -> tuple[KernelCounters, dict]:
    """Modeled counters for one sweep plus a per-stage flop split
    (perf.py:404-439): "riemann" = solves + fluctuation sums + updates,
    "second_order" = limiting and correction fluxes."""
    from .limiter import LIMITER_IDS

    name = solver if isinstance(solver, str) else solver.name
    if name not in _MODEL_SCALARS:
        # a user solver is priced by shadow-executing its own Python scalar,
        # exactly as the reference prices every registered solver
        scalar = getattr(solver, "scalar", None)
        if scalar is None:
            raise ValueError(f"no pricing scalar for solver {name!r} (give its Python "
                             "scalar routine to price it)")
        _MODEL_SCALARS[name] = (scalar, solver.num_waves)
        _SAMPLE_PACKED.setdefault(name, [0.0] * 4)
    nw = _MODEL_SCALARS[name][1]
    lim_id = limiter if isinstance(limiter, int) else LIMITER_IDS[limiter]
    ev = sweep_events(plan, spec)
    m = spec.num_states
    solve, fan, corr, upd = _stage_costs(name, m, nw, lim_id)
    riemann_f = solve[0] * ev.fans + fan[0] * ev.fans + upd[0] * ev.cells
    riemann_s = solve[1] * ev.fans + fan[1] * ev.fans + upd[1] * ev.cells
    second_f = corr[0] * ev.corrections
    second_s = corr[1] * ev.corrections
    counters = KernelCounters(flops=riemann_f + second_f, special=riemann_s + second_s,
                              bytes_read=ev.pencil_reads * m * itemsize,
                              bytes_written=ev.cells_written * m * itemsize)
    return counters, {"riemann": (riemann_f, riemann_s), "second_order": (second_f, second_s)}


def plan_events_monolithic(spec, axis: int) -> SweepEvents:
    from .sweep import plan_tiles
    return sweep_events(plan_tiles(spec, axis, spec.cells), spec)


def halo_extra_read_bytes(plan, spec, itemsize: int) -> int:
    """Read traffic added by tiling relative to one tile (perf.py:442-452)."""
    mono = plan_events_monolithic(spec, plan.axis)
    tiled = sweep_events(plan, spec)
    return (tiled.pencil_reads - mono.pencil_reads) * spec.num_states * itemsize


class RunCounters:
    """Per-axis accumulation of sweep counters across a run (perf.py:466-490)."""

    def __init__(self):
        self.per_axis: dict[int, dict] = {}
        self.sweeps = 0

    def add_sweep(self, axis: int, counters: KernelCounters, stage_flops: dict) -> None:
        slot = self.per_axis.setdefault(axis, {"counters": KernelCounters(), "stages": {}})
        slot["counters"].add(counters)
        for name, (f, s) in stage_flops.items():
            f0, s0 = slot["stages"].get(name, (0, 0))
            slot["stages"][name] = (f0 + f, s0 + s)
        self.sweeps += 1

    def add_sweeps(self, axis: int, counters: KernelCounters, stage_flops: dict, n: int) -> None:
        """n identical sweeps at once (the device controller's batches)."""
        if n <= 0:
            return
        self.add_sweep(axis, counters.scaled(n),
                       {k: (f * n, s * n) for k, (f, s) in stage_flops.items()})
        self.sweeps += n - 1

    def total(self) -> KernelCounters:
        out = KernelCounters()
        for slot in self.per_axis.values():
            out.add(slot["counters"])
        return out


@dataclass(frozen=True)
class PerfRow:
    scope: str  # axis name or "all"
    stage: str  # "riemann" or "full"
    flops: int
    special: int
    bytes: int
    oi: float
    bound: float | None


@dataclass(frozen=True)
class PerfReport:
    rows: tuple
    machine: MachineModel | None
    collected: bool = True

    def row(self, scope: str, stage: str) -> PerfRow:
        for r in self.rows:
            if r.scope == scope and r.stage == stage:
                return r
        raise KeyError(f"no row for {scope}/{stage}")


def build_report(counters: RunCounters, machine: MachineModel | None,
                 collected: bool | None = None) -> PerfReport:
    """Per sweep axis and overall, at both stage depths (perf.py:516-553)."""
    if collected is None:
        collected = counters.sweeps > 0
    if not collected:
        return PerfReport(rows=(), machine=machine, collected=False)
    rows: list = []

    def emit(scope, stages, c):
        rf, rs = stages.get("riemann", (0, 0))
        sf, ss = stages.get("second_order", (0, 0))
        b = c.total_bytes
        for stage, f, s in (("riemann", rf, rs), ("full", rf + sf, rs + ss)):
            oi = (f + s) / b if b else 0.0
            bound = roofline_bound(oi, machine) if machine is not None else None
            rows.append(PerfRow(scope, stage, f, s, b, oi, bound))

    agg_stages: dict = {}
    agg = KernelCounters()
    for axis in sorted(counters.per_axis):
        slot = counters.per_axis[axis]
        emit(_AXES[axis], slot["stages"], slot["counters"])
        for name, (f, s) in slot["stages"].items():
            f0, s0 = agg_stages.get(name, (0, 0))
            agg_stages[name] = (f0 + f, s0 + s)
        agg.add(slot["counters"])
    emit("all", agg_stages, agg)
    return PerfReport(rows=tuple(rows), machine=machine)


def render_text(report: PerfReport) -> str:
    """Human-readable aligned table (perf.py:556-575)."""
    if not report.collected:
        return "not collected (run executed without operation counters)"
    header = ("scope", "stage", "flops", "special", "bytes", "flops/byte", "bound flop/s")
    body = []
    for r in report.rows:
        bound = f"{r.bound:.4g}" if r.bound is not None else "-"
        body.append((r.scope, r.stage, str(r.flops), str(r.special), str(r.bytes),
                     f"{r.oi:.4f}", bound))
    widths = [max(len(row[i]) for row in [header] + body) for i in range(len(header))]
    lines = ["  ".join(h.ljust(w) for h, w in zip(header, widths))]
    for row in body:
        lines.append("  ".join(c.ljust(w) for c, w in zip(row, widths)))
    if report.machine is None:
        lines.append("roofline bounds omitted: no machine model configured")
    return "\n".join(lines)


def render_delimited(report: PerfReport, sep: str = "\t") -> str:
    """Machine-readable flat table (perf.py:578-588)."""
    if not report.collected:
        return "not collected\n"
    lines = [sep.join(("scope", "stage", "flops", "special", "bytes", "oi", "bound"))]
    for r in report.rows:
        bound = repr(r.bound) if r.bound is not None else ""
        lines.append(sep.join((r.scope, r.stage, str(r.flops), str(r.special), str(r.bytes),
                               repr(r.oi), bound)))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# The B200 kernel model and measured rows


def machine_from_config(machine) -> MachineModel | None:
    """The [machine] section of a run config (a dict of strings, or already
    a MachineModel) as a MachineModel (config.py:280-297 semantics)."""
    if machine is None or isinstance(machine, MachineModel):
        return machine
    from .errors import ConfigError
    if "peak_flops" not in machine or "peak_bandwidth" not in machine:
        raise ConfigError("[machine] needs both peak_flops and peak_bandwidth")
    try:
        sfp = machine.get("special_function_peak")
        return MachineModel(float(machine["peak_flops"]), float(machine["peak_bandwidth"]),
                            None if sfp is None else float(sfp))
    except ValueError as exc:
        raise ConfigError(f"invalid machine model: {exc}") from exc


def b200(itemsize: int = 8) -> MachineModel:
    """B200 roofline: HBM from MEASURED_PEAKS.json (driver-measured copy
    bandwidth; 6650 GB/s fallback), vector peak 148 SMs x 64 (fp64) or 128
    (fp32) lanes x 1.965 GHz (the kernels use no FMA: one flop per lane-op),
    MUFU 16 per SM per clock."""
    bw = 6650e9
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            bw = float(json.load(fh)["hbm_gbs"]) * 1e9
    except (OSError, KeyError, ValueError):
        pass
    lanes = 64 if itemsize == 8 else 128
    clk = 1.965e9
    return MachineModel(148 * lanes * clk, bw, 148 * 16 * clk)


# ---------------------------------------------------------------------------
# counting float: every arithmetic op is charged to the current tally


class _Tally:
    def __init__(self):
        self.flops = 0
        self.special = 0


_CUR = [_Tally()]


class _CF:
    __slots__ = ("v",)

    def __init__(self, v, _t=None):
        self.v = float(v)

    @staticmethod
    def _o(x):
        return x.v if isinstance(x, _CF) else float(x)

    @staticmethod
    def _op(v):
        _CUR[0].flops += 1
        return _CF(v)

    def __add__(self, o): return self._op(self.v + self._o(o))
    __radd__ = __add__
    def __sub__(self, o): return self._op(self.v - self._o(o))
    def __rsub__(self, o): return self._op(self._o(o) - self.v)
    def __mul__(self, o): return self._op(self.v * self._o(o))
    __rmul__ = __mul__

    def __truediv__(self, o):
        _CUR[0].special += 1
        d = self._o(o)
        return _CF(self.v / d if d else 0.0)

    def __rtruediv__(self, o):
        _CUR[0].special += 1
        return _CF(self._o(o) / self.v if self.v else 0.0)

    def __neg__(self): return _CF(-self.v)
    def __abs__(self): return _CF(abs(self.v))

    def sqrt(self):
        _CUR[0].special += 1
        return _CF(math.sqrt(abs(self.v)))

    def __gt__(self, o): return self.v > self._o(o)
    def __lt__(self, o): return self.v < self._o(o)


def _priced(fn):
    """(result, (flops, special)) of fn() on a fresh tally."""
    _CUR[0] = _Tally()
    out = fn()
    t = _CUR[0]
    _CUR[0] = _Tally()
    return out, (t.flops, t.special)


# Python restatement of the device functors (clb_solvers.cuh), exact mode.
# A fan is (waves {(p, k): value}, speeds [s_p]); a cell is its states plus
# the shallow-water hoisted quantities.

def _acoustics(m, n):
    def make(q, t):
        return {"q": q}

    def solve(L, R, prm, t):
        Z, inv2z, c = prm["Z"], prm["inv2z"], prm["c"]
        dp = R["q"][0] - L["q"][0]
        dun = R["q"][n] - L["q"][n]
        zd = Z * dun
        b1 = (zd - dp) * inv2z
        b2 = (zd + dp) * inv2z
        return {(0, 0): (-Z) * b1, (0, n): b1, (1, 0): Z * b2, (1, n): b2}, [-c, c]
    return make, solve, 2


def _shallow_water(n):
    tr = 3 - n

    def make(q, t):
        s = q[0].sqrt()
        return {"q": q, "s": s, "un": q[n] / s, "ut": q[tr] / s}

    def solve(L, R, prm, t):
        g, half = prm["g"], prm["half"]
        denom = L["s"] + R["s"]
        uhat = (L["un"] + R["un"]) / denom
        vhat = (L["ut"] + R["ut"]) / denom
        chat = (g * (half * (L["q"][0] + R["q"][0]))).sqrt()
        dh = R["q"][0] - L["q"][0]
        dhun = R["q"][n] - L["q"][n]
        dhut = R["q"][tr] - L["q"][tr]
        inv2c = half / chat
        umc, upc = uhat - chat, uhat + chat
        a1 = (upc * dh - dhun) * inv2c
        a3 = (dhun - umc * dh) * inv2c
        a2 = dhut - vhat * dh
        w = {(0, 0): a1, (0, n): a1 * umc, (0, tr): a1 * vhat, (1, tr): a2,
             (2, 0): a3, (2, n): a3 * upc, (2, tr): a3 * vhat}
        return w, [umc, uhat, upc]
    return make, solve, 3


def _advection():
    def make(q, t):
        return {"q": q}

    def solve(L, R, prm, t):
        return {(0, 0): R["q"][0] - L["q"][0]}, [prm["u"]]
    return make, solve, 1


def _vc_acoustics(m, n):
    def make(q, t):
        return {"q": q}

    def solve(L, R, prm, t):
        Zl, Zr = L["q"][m - 2], R["q"][m - 2]
        dp = R["q"][0] - L["q"][0]
        dun = R["q"][n] - L["q"][n]
        denom = Zl + Zr
        a1 = (Zr * dun - dp) / denom
        a2 = (Zl * dun + dp) / denom
        return {(0, 0): (-Zl) * a1, (0, n): a1, (1, 0): Zr * a2, (1, n): a2}, \
            [-L["q"][m - 1], R["q"][m - 1]]
    return make, solve, 2


def _limiter(theta, lim):
    if lim == 3:      # MC
        v = (1.0 + theta) * 0.5
        tt = theta * 2.0
        return v if v.v < tt.v else tt
    if lim == 1:      # minmod: comparisons only
        return theta
    if lim == 2:      # superbee
        a = theta * 2.0
        return a
    if lim == 4:      # van Leer
        a = abs(theta)
        return (theta + a) / (a + 1.0)
    return theta


def _correction(Fl, Fm, Fr, m, nw, lim, dtdx):
    ft = {}
    wm, sm = Fm
    for p in range(nw):
        ks = sorted(k for (pp, k) in wm if pp == p)
        up = Fl if sm[p].v > 0.0 else Fr
        wn = wu = None
        for k in ks:
            wk = wm[(p, k)]
            wn = wk * wk if wn is None else wn + wk * wk
            wu = up[0][(p, k)] * wk if wu is None else wu + up[0][(p, k)] * wk
        limv = _CF(1.0) if lim == 0 else _limiter(wu / wn, lim)
        asp = abs(sm[p])
        coef = ((asp * 0.5) * (1.0 - dtdx * asp)) * limv
        for k in ks:
            ft[k] = (ft[k] if k in ft else _CF(0.0)) + coef * wm[(p, k)]
    return ft


def _update(q, Fleft, Fright, ftn, ftp, m, dtdx):
    out = []
    for k in range(m):
        comps = [p for (p, kk) in Fleft[0] if kk == k]
        if not comps:
            out.append(q[k])
            continue
        ap = am = _CF(0.0)
        for p in sorted(comps):
            ap = ap + Fleft[1][p] * Fleft[0][(p, k)]
            am = am + Fright[1][p] * Fright[0][(p, k)]
        out.append((q[k] - dtdx * (ap + am)) - dtdx * (ftn.get(k, _CF(0.0)) - ftp.get(k, _CF(0.0))))
    return out


def _functor(solver: str, ndim: int, axis: int):
    if solver == "acoustics":
        return _acoustics(ndim + 1, 1 + axis) + (ndim + 1,)
    if solver == "shallow_water":
        return _shallow_water(1 + axis) + (3,)
    if solver == "advection":
        return _advection() + (1,)
    m = ndim + 3
    return _vc_acoustics(m, 1 + axis) + (m,)


def kernel_event_costs(solver: str, ndim: int, axis: int, limiter_id: int) -> dict:
    """(flops, special) of one cell make, one fan (solve), one correction and
    one update, priced on representative non-degenerate states."""
    make, solve, nw, m = _functor(solver, ndim, axis)
    prm = {"Z": _CF(1.3), "inv2z": _CF(0.5 / 1.3), "c": _CF(0.7), "g": _CF(1.0),
           "half": _CF(0.5), "u": _CF(1.0)}

    def state(j):
        base = [1.0 + 0.1 * i for i in range(m)]
        if solver == "vc_acoustics":
            base[m - 2], base[m - 1] = 1.2, 0.9
        return [_CF(v * (1.0 + 0.03 * j)) for v in base]

    costs = {}
    X, costs["make"] = _priced(lambda: [make(state(j), None) for j in range(1)])
    X, _ = _priced(lambda: [make(state(j), None) for j in range(4)])
    F, _ = _priced(lambda: [solve(X[i], X[i + 1], prm, None) for i in range(3)])
    _, costs["fan"] = _priced(lambda: solve(X[0], X[1], prm, None))
    G, costs["correction"] = _priced(lambda: _correction(F[0], F[1], F[2], m, nw, limiter_id,
                                                         _CF(0.4)))
    ftp = {k: _CF(0.1) for k in G}
    _, costs["update"] = _priced(lambda: _update(X[1]["q"], F[0], F[1], G, ftp, m, _CF(0.4)))
    return costs


def kernel_sweep_counters(solver: str, ndim: int, cells, axis: int, limiter_id: int, itemsize: int,
                   seg_len: int, num_states: int) -> dict:
    """Modeled counters of one sweep along `axis`: per stage ("riemann": cell
    makes + solves + first-order update traffic; "full": everything) and the
    bytes of the segment decomposition (each segment of L cells reads L + 4)."""
    c = kernel_event_costs(solver, ndim, axis, limiter_id)
    n = int(cells[axis])
    pencils = 1
    for ax, k in enumerate(cells):
        if ax != axis:
            pencils *= int(k)
    nseg = -(-n // seg_len)
    lens = [min(seg_len, n - s * seg_len) for s in range(nseg)]
    makes = sum(L + 4 for L in lens) * pencils
    fans = sum(L + 3 for L in lens) * pencils
    corrs = sum(L + 1 for L in lens) * pencils
    upds = n * pencils
    rf = c["make"][0] * makes + c["fan"][0] * fans
    rs = c["make"][1] * makes + c["fan"][1] * fans
    sf = c["correction"][0] * corrs + c["update"][0] * upds
    ss = c["correction"][1] * corrs + c["update"][1] * upds
    counters = KernelCounters(rf + sf, rs + ss,
                              sum(L + 4 for L in lens) * pencils * num_states * itemsize,
                              upds * num_states * itemsize)
    return {"counters": counters, "stages": {"riemann": (rf, rs), "second_order": (sf, ss)},
            "events": {"make": makes, "fan": fans, "correction": corrs, "update": upds},
            "per_event": c}


@dataclass
class MeasuredRow:
    scope: str
    stage: str
    flops: int
    special: int
    bytes: int
    oi: float
    bound: float | None
    seconds: float | None = None      # measured kernel time (sum of launches)
    launches: int = 0

    @property
    def achieved_flops(self):
        return None if not self.seconds else (self.flops + self.special) * self.launches / self.seconds

    @property
    def achieved_bandwidth(self):
        return None if not self.seconds else self.bytes * self.launches / self.seconds

    @property
    def fraction_of_bound(self):
        a = self.achieved_flops
        return None if a is None or not self.bound else a / self.bound


@dataclass
class MeasuredReport:
    rows: list = field(default_factory=list)
    machine: MachineModel | None = None
    collected: bool = True
    reference: "PerfReport | None" = None   # the reference model's rows of the same run
    ncu_bytes: dict | None = None            # {axis: DRAM bytes per launch} from ncu

    def row(self, scope: str, stage: str) -> MeasuredRow:
        for r in self.rows:
            if r.scope == scope and r.stage == stage:
                return r
        raise KeyError(f"no row for {scope}/{stage}")


def build_measured_report(per_axis: dict, machine: MachineModel | None,
                          timing: dict | None = None) -> "MeasuredReport":
    """Rows per axis and for "all" at both stage depths (perf.py:516-553
    layout), with measured kernel seconds/launches per axis when given."""
    rep = MeasuredReport(machine=machine)
    agg = KernelCounters()
    agg_st = {"riemann": [0, 0], "second_order": [0, 0]}
    tot_s = tot_n = 0
    for axis in sorted(per_axis):
        slot = per_axis[axis]
        secs, launches = (timing or {}).get(axis, (None, 0))
        _emit(rep, _AXES[axis], slot["stages"], slot["counters"], machine, secs, launches)
        agg.add(slot["counters"])
        for k, (f, s) in slot["stages"].items():
            agg_st[k][0] += f
            agg_st[k][1] += s
        if secs:
            tot_s += secs
            tot_n = max(tot_n, launches)
    _emit(rep, "all", agg_st, agg, machine, tot_s or None, tot_n)
    return rep


def _emit(rep, scope, stages, counters, machine, secs, launches):
    rf, rs = stages.get("riemann", (0, 0))
    sf, ss = stages.get("second_order", (0, 0))
    b = counters.total_bytes
    for stage, f, s in (("riemann", rf, rs), ("full", rf + sf, rs + ss)):
        oi = (f + s) / b if b else 0.0
        bound = roofline_bound(oi, machine) if machine is not None else None
        rep.rows.append(MeasuredRow(scope, stage, f, s, b, oi, bound, secs, launches))


def render_measured_text(report: "MeasuredReport") -> str:
    if not report.collected:
        return "not collected"
    head = ("scope", "stage", "flops", "special", "bytes", "flop/B", "bound GF/s", "ms",
            "GF/s", "GB/s", "of bound")
    lines = ["%-5s %-7s %14s %12s %14s %7s %10s %9s %9s %9s %8s" % head]
    for r in report.rows:
        ms = r.seconds * 1e3 if r.seconds else None
        lines.append("%-5s %-7s %14d %12d %14d %7.3f %10s %9s %9s %9s %8s" % (
            r.scope, r.stage, r.flops, r.special, r.bytes, r.oi,
            "-" if r.bound is None else "%.1f" % (r.bound / 1e9),
            "-" if ms is None else "%.3f" % ms,
            "-" if r.achieved_flops is None else "%.1f" % (r.achieved_flops / 1e9),
            "-" if r.achieved_bandwidth is None else "%.1f" % (r.achieved_bandwidth / 1e9),
            "-" if r.fraction_of_bound is None else "%.3f" % r.fraction_of_bound))
    return "\n".join(lines)


def run_measured_perf(cfg, *, device: int = 0, max_steps: int | None = None,
                      ncu_bytes: dict | None = None):
    """Run a configuration with per-launch CUDA-event timing and return
    (MeasuredReport, RunReport).  The report holds, per sweep axis: the B200
    kernel model (rows), the measured kernel time of every launch, the
    reference's modeled counters of the same run (``report.reference``, a
    PerfReport from ``Simulation.counters``, perf.py:516-553), and -- when
    ``ncu_bytes`` = {axis: dram bytes per launch} from an ncu capture is
    given -- the measured DRAM traffic (``report.ncu_bytes``)."""
    from .limiter import LIMITER_IDS
    from .runner import build_simulation
    if not cfg.counters:
        cfg = cfg.with_overrides(counters=True)
    sim = build_simulation(cfg, device=device)
    with sim:
        sim.device_controller = False          # per-launch events need direct launches
        dev = sim.device_grid
        dev.timing()
        dev.enable_timing(True)
        report = sim.run_until(cfg.t_end, max_steps=max_steps)
        ms, cnt = dev.timing()
        dev.enable_timing(False)
        spec = sim.spec
        per_axis = {}
        for axis in range(spec.ndim):
            _, seg_len = dev.segments(axis)
            per_axis[axis] = kernel_sweep_counters(sim.solver.name, spec.ndim, spec.cells, axis,
                                                   LIMITER_IDS[sim.limiter], sim.dtype.itemsize,
                                                   seg_len, spec.num_states)
        timing = {a: (ms[a] / 1e3, int(cnt[a])) for a in range(spec.ndim)}
        machine = b200(sim.dtype.itemsize)
        rep = build_measured_report(per_axis, machine, timing)
        rep.reference = build_report(sim.counters, machine)
        rep.ncu_bytes = dict(ncu_bytes) if ncu_bytes else None
        return rep, report


def render_side_by_side(rep: "MeasuredReport") -> str:
    """Per axis: the reference model's bytes / flops / OI per sweep, the B200
    kernel model's, the measured time and -- with an ncu capture -- the
    measured DRAM bytes per launch (the paper's Tables 1-6 layout, PAPER.md
    454-507, on B200)."""
    ref = getattr(rep, "reference", None)
    ncu = getattr(rep, "ncu_bytes", None) or {}
    head = ("axis", "ref MB/sweep", "ref MFlop", "ref OI", "kern MB", "kern MFlop", "kern OI",
            "ms/launch", "ncu MB", "GB/s")
    lines = ["%-4s %12s %10s %7s %9s %10s %7s %10s %9s %8s" % head]
    for i, ax in enumerate(_AXES):
        try:
            k = rep.row(ax, "full")
        except KeyError:
            continue
        n = max(k.launches, 1)
        r = ref.row(ax, "full") if ref is not None and ref.collected else None
        ms = k.seconds * 1e3 / n if k.seconds else None
        nb = ncu.get(i)
        lines.append("%-4s %12s %10s %7s %9.2f %10.2f %7.3f %10s %9s %8s" % (
            ax,
            "-" if r is None else "%.2f" % (r.bytes / n / 1e6),
            "-" if r is None else "%.2f" % ((r.flops + r.special) / n / 1e6),
            "-" if r is None else "%.3f" % r.oi,
            k.bytes / 1e6, (k.flops + k.special) / 1e6, k.oi,
            "-" if ms is None else "%.4f" % ms,
            "-" if nb is None else "%.2f" % (nb / 1e6),
            "-" if ms is None else "%.1f" % ((nb if nb is not None else k.bytes) / ms / 1e6)))
    return "\n".join(lines)
