// clb_controller.cuh -- the device-resident step controller of clb_run_batch
// (timestep.py:151-243 evaluated in fp64 on one device thread), shared by the
// controller kernels and the sweep kernels that fold it into their last CTA.
#pragma once
#include "../../include/clawb200.h"

namespace clb {

// Per-launch results of the sweeps of one attempt (bit patterns of max |s|
// per sweep slot, non-finite flags, first non-finite cell of the locator).
struct Result {
  unsigned long long smax[4];
  int nonfinite[4];
  unsigned long long first_bad;
};

// ---------------------------------------------------------------------------
// Device-resident controller (clb_run_batch): timestep.py:151-243 in fp64 on
// one device thread.  Every expression keeps the reference's operation order
// (explicit __d*_rn so nothing is contracted); Python's min(a, b) / max(a, b)
// are "b if b < a else a" / "b if b > a else a".

// estimate_dt (timestep.py:151-177) + the run_until loop guards
// (timestep.py:263-270) for the next attempt, or end the batch.
__device__ __forceinline__ void ctl_prepare_next(DevCtl* c) {
  if (c->done) return;
  if (c->max_accepted >= 0 && c->n_accepted >= c->max_accepted) {
    c->status = CLB_BATCH_MAXSTEPS; c->done = 1; return;
  }
  if (!(c->t < c->stop)) { c->status = CLB_BATCH_STOP; c->done = 1; return; }
  if (c->n_attempts >= c->log_cap) { c->status = CLB_BATCH_LOGFULL; c->done = 1; return; }
  const double s = c->last_max_speed;
  double dt;
  if (s > 0.0) {
    dt = __ddiv_rn(__dmul_rn(c->cfl_target, c->min_spacing), s);
    dt = c->dt_cap < dt ? c->dt_cap : dt;
  } else {
    dt = c->dt_cap;
  }
  int landed = 0;
  const double remaining = __dsub_rn(c->stop, c->t);
  if (dt >= remaining) {
    dt = remaining;
    landed = 1;
  }
  if (!isfinite(dt)) { c->status = CLB_BATCH_DTERR; c->done = 1; return; }
  c->dt = dt;
  c->landed = landed;
  // timestep.py:200-206: sweep j reads the previous output, writes scratch[j % 2]
  int cur = c->cur;
  for (int j = 0; j < c->ndim; ++j) {
    const int dst = (j % 2 == 0) ? c->s0 : c->s1;
    c->src[j] = cur;
    c->dst[j] = dst;
    cur = dst;
  }
}

__global__ void ctl_prepare(DevCtl* c);

// The attempt's verdict (timestep.py:207-243), then the next attempt.
__device__ __forceinline__ void ctl_finish_dev(DevCtl* c, Result* r) {
  if (c->done) return;
  double step_speed = 0.0;
  for (int j = 0; j < c->ndim; ++j) {
    if (*reinterpret_cast<volatile int*>(&r->nonfinite[j])) {
      c->status = CLB_BATCH_BLOWUP;
      c->fail_sweep = j;
      c->done = 1;
      return;
    }
    const double sj = __longlong_as_double(
        (long long)*reinterpret_cast<volatile unsigned long long*>(&r->smax[j]));
    step_speed = sj > step_speed ? sj : step_speed;
  }
  for (int j = 0; j < 4; ++j) { r->smax[j] = 0ull; r->nonfinite[j] = 0; }
  const double nu = __ddiv_rn(__dmul_rn(c->dt, step_speed), c->min_spacing);
  const bool accepted = nu <= c->cfl_max;
  clb_attempt rec;
  rec.t_start = c->t;
  rec.dt = c->dt;
  rec.max_speed = step_speed;
  rec.nu = nu;
  rec.dt_retry = __longlong_as_double(0x7ff8000000000000ll);  // None
  rec.accepted = accepted ? 1 : 0;
  rec.landed = (c->landed && accepted) ? 1 : 0;
  clb_attempt* log = (clb_attempt*)c->log;
  if (accepted) {
    const int last = (c->ndim - 1) % 2;
    const int fin = last == 0 ? c->s0 : c->s1;
    const int other = last == 0 ? c->s1 : c->s0;
    c->s0 = c->cur;
    c->s1 = other;
    c->cur = fin;
    c->t = c->landed ? c->stop : __dadd_rn(c->t, c->dt);
    c->n_accepted += 1;
    c->nu_max = nu > c->nu_max ? nu : c->nu_max;
    c->prev_reverted = 0;
  } else {
    rec.dt_retry = __ddiv_rn(__dmul_rn(c->cfl_target, c->min_spacing), step_speed);
    if (c->prev_reverted && nu >= c->prev_nu) {
      // UnstableStepError: logged (the reference counts the revert first),
      // prev_nu kept for the message, last_max_speed not updated
      log[c->n_attempts] = rec;
      c->n_attempts += 1;
      c->status = CLB_BATCH_UNSTABLE;
      c->done = 1;
      return;
    }
    c->prev_reverted = 1;
    c->prev_nu = nu;
  }
  c->last_max_speed = step_speed;
  log[c->n_attempts] = rec;
  c->n_attempts += 1;
  ctl_prepare_next(c);
}

__global__ void ctl_finish(DevCtl* c, Result* r);

}  // namespace clb
