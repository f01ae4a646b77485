"""Host-side handling of the device controller's batch results
(timestep.py Simulation._run_batch) against the per-attempt host loop, on a
scripted engine (TEST INFRASTRUCTURE: no GPU).

The engine returns scripted per-sweep max speeds, so attempt sequences that
are hard to provoke with real data -- two reverts inside one device batch,
the second no better than the first -- can be driven through both paths.
Its run_batch restates the device controller (csrc/clb_controller.cuh
ctl_prepare_next / ctl_finish_dev, i.e. timestep.py:151-243) in Python."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_1805_08846_b200 as P
from paper_1805_08846_b200 import _native as N


class ScriptedEngine:
    def __init__(self, *, ndim, cells, spacing, num_states, dtype, script, **_):
        self.ndim = ndim
        self.shape = (num_states,) + tuple(reversed(cells[:ndim]))
        self.dtype = np.dtype(dtype)
        self.script = list(script)
        self.bufs = [np.zeros(self.shape, self.dtype) for _ in range(3)]

    def upload(self, buf, interior):
        self.bufs[buf][...] = interior

    def download(self, buf, out=None):
        return self.bufs[buf].copy()

    def close(self):
        pass

    def _speeds(self):
        s = self.script.pop(0)
        return [s] * self.ndim, [False] * self.ndim

    def attempt_step(self, dt, src, s0, s1):
        return self._speeds()

    def run_batch(self, b, log_cap=4096):
        recs = []
        while True:
            # ctl_prepare_next
            if b.max_accepted >= 0 and b.n_accepted >= b.max_accepted:
                b.status = N.BATCH_MAXSTEPS
                break
            if not b.t < b.stop:
                b.status = N.BATCH_STOP
                break
            if b.n_attempts >= log_cap:
                b.status = N.BATCH_LOGFULL
                break
            s = b.last_max_speed
            dt = min(b.cfl_target * b.min_spacing / s, b.dt_cap) if s > 0.0 else b.dt_cap
            landed = False
            if dt >= b.stop - b.t:
                dt, landed = b.stop - b.t, True
            # ctl_finish_dev
            speeds, _ = self._speeds()
            step_speed = max([0.0] + speeds)
            nu = dt * step_speed / b.min_spacing
            acc = nu <= b.cfl_max
            r = N.ClbAttempt()
            r.t_start, r.dt, r.max_speed, r.nu = b.t, dt, step_speed, nu
            r.dt_retry = math.nan
            r.accepted, r.landed = int(acc), int(landed and acc)
            if acc:
                b.t = b.stop if landed else b.t + dt
                b.n_accepted += 1
                b.nu_max = max(b.nu_max, nu)
                b.prev_reverted = 0
            else:
                r.dt_retry = b.cfl_target * b.min_spacing / step_speed
                if b.prev_reverted and nu >= b.prev_nu:
                    recs.append(r)
                    b.n_attempts += 1
                    b.status = N.BATCH_UNSTABLE
                    break
                b.prev_reverted = 1
                b.prev_nu = nu
            b.last_max_speed = step_speed
            recs.append(r)
            b.n_attempts += 1
        return recs


def _sim(script, device_controller):
    spec = P.GridSpec((8, 8), (0, 0), (1, 1), 3)
    g = P.create_grid(spec)
    return P.Simulation(
        g, P.get_solver("shallow_water"), P.ShallowWaterParams(1.0),
        P.BoundarySpec.uniform(P.BoundaryKind.PERIODIC, (1, 2)), initial_max_speed=1.0,
        device_controller=device_controller,
        engine=lambda **kw: ScriptedEngine(script=script, **kw))


def _outcome(sim):
    with pytest.raises(P.UnstableStepError) as exc:
        sim.run_until(1.0)
    return (str(exc.value), sim.steps_accepted, sim.steps_reverted,
            float(sim.last_max_speed).hex(), sim._prev_reverted, float(sim._prev_nu).hex(),
            float(sim.t).hex())


@pytest.mark.parametrize("script", [
    # accepted, then revert A (nu 1.8), then retry B no better (nu 1.8)
    [1.0, 2.0, 4.0],
    # revert A at the very first attempt, retry B worse (nu 0.9*8/2 = 3.6)
    [2.0, 8.0],
    # two accepted, revert A, a better revert B, then C no better than B
    [1.0, 1.0, 3.0, 4.0, 16.0],
])
def test_unstable_inside_one_batch_matches_host_loop(script):
    host = _outcome(_sim(script, device_controller=False))
    dev = _outcome(_sim(script, device_controller=True))
    assert dev == host
    assert "->" in host[0]
