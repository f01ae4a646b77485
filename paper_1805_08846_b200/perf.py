"""Modeled work and traffic of the sweeps beside measured kernel times
(§8(f) row 2; the reference's perf model, clawtile/perf.py:35-95,379-588,
re-done for the B200 kernels).

The reference prices one event (a Riemann solve, a fan, a correction, an
update) by shadow-executing its scalar routines on a counting float and
multiplies by event counts from its tile plan.  Here the priced routines are
a Python restatement of what the sm_100a kernels execute
(csrc/clb_solvers.cuh, exact mode: structural zeros elided, per-cell
hoisting of the shallow-water square roots, every division of the
branch-free path counted), and the event counts come from the library's own
segment decomposition (``clb_sweep_segments``), including the 4-cell halo
each segment re-reads.  ``run_perf`` then times every sweep launch with CUDA
events and reports achieved flop/s and bytes/s against the roofline bound of
the B200 (measured HBM bandwidth, fp64/fp32 vector peaks without FMA).

Counting rules (the reference's): +, -, * are flops; / and sqrt are
"special" (one each); comparisons, abs and negation are free.
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, field

_AXES = ("x", "y", "z")


@dataclass
class KernelCounters:
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
    peak_flops: float       # flop/s
    peak_bandwidth: float   # bytes/s
    special_function_peak: float | None = None

    def __post_init__(self):
        if self.peak_flops <= 0.0 or self.peak_bandwidth <= 0.0:
            raise ValueError("machine peaks must be positive")


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


def operational_intensity(c: KernelCounters) -> float:
    if c.total_bytes == 0:
        raise ValueError("operational intensity undefined for zero bytes")
    return c.total_flops / c.total_bytes


def roofline_bound(oi: float, machine: MachineModel) -> float:
    if oi < 0.0:
        raise ValueError("operational intensity cannot be negative")
    return min(machine.peak_flops, oi * machine.peak_bandwidth)


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


def event_costs(solver: str, ndim: int, axis: int, limiter_id: int) -> dict:
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


def sweep_counters(solver: str, ndim: int, cells, axis: int, limiter_id: int, itemsize: int,
                   seg_len: int, num_states: int) -> dict:
    """Modeled counters of one sweep along `axis`: per stage ("riemann": cell
    makes + solves + first-order update traffic; "full": everything) and the
    bytes of the segment decomposition (each segment of L cells reads L + 4)."""
    c = event_costs(solver, ndim, axis, limiter_id)
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
class PerfRow:
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
class PerfReport:
    rows: list = field(default_factory=list)
    machine: MachineModel | None = None
    collected: bool = True

    def row(self, scope: str, stage: str) -> PerfRow:
        for r in self.rows:
            if r.scope == scope and r.stage == stage:
                return r
        raise KeyError(f"no row for {scope}/{stage}")


def build_report(per_axis: dict, machine: MachineModel | None, timing: dict | None = None
                 ) -> PerfReport:
    """Rows per axis and for "all" at both stage depths (perf.py:516-553
    layout), with measured kernel seconds/launches per axis when given."""
    rep = PerfReport(machine=machine)
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
        rep.rows.append(PerfRow(scope, stage, f, s, b, oi, bound, secs, launches))


def render_text(report: PerfReport) -> str:
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


def run_perf(cfg, *, device: int = 0, max_steps: int | None = None):
    """Run a configuration with per-launch CUDA-event timing and return
    (PerfReport, RunReport): modeled counters per sweep launch beside the
    measured kernel time of every launch (runner.py:103-118 contract, with
    measured columns the reference model lacks)."""
    from .limiter import LIMITER_IDS
    from .runner import build_simulation
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
            per_axis[axis] = sweep_counters(sim.solver.name, spec.ndim, spec.cells, axis,
                                            LIMITER_IDS[sim.limiter], sim.dtype.itemsize,
                                            seg_len, spec.num_states)
        timing = {a: (ms[a] / 1e3, int(cnt[a])) for a in range(spec.ndim)}
        return build_report(per_axis, b200(sim.dtype.itemsize), timing), report
