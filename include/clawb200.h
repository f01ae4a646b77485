/* clawb200.h -- C ABI of the B200-native time-step hot path.
 *
 * The reference (clawtile, /root/reference/pkg) has no C ABI: its hot path is
 * the Python operator API below, with numba kernels underneath.
 * specifies a bindings layer ("create/destroy session, evolve, copy-state-out,
 * last-error string") that was never built; this header is
 * that layer, one entry point per reference operation it replaces:
 *
 *   clb_create / clb_destroy   Simulation.__init__ / close          timestep.py:75-132
 *                              (+ StateGrid allocation, grid.py:145-160)
 *   clb_upload / clb_download  fill_initial / StateGrid.interior,   grid.py:174-234
 *                              frame payload order (frames.py:84-99)
 *   clb_sweep                  sweep_axis / sweep_axis_tiled        sweep.py:307-391
 *                              (+ apply_boundary fused, boundary.py:87-122)
 *   clb_sweep_async/clb_fetch  the same, split for multi-GPU halo exchange
 *   clb_attempt_step           the sweep loop of Simulation.attempt_step
 *                              (timestep.py:195-211); the fp64 accept/revert
 *                              arithmetic stays on the host (timestep.py:212-239)
 *   clb_run_batch              Simulation.run_until's attempt loop  timestep.py:245-285
 *                              with estimate_dt / attempt_step      timestep.py:151-243
 *                              evaluated on the device (fp64, same expressions)
 *   clb_write_frame            frames.frame_bytes / write_frame     frames.py:74-104
 *   clb_first_nonfinite        Simulation._check_finite             timestep.py:179-186
 *   clb_solve_pairs            RiemannSolver.solve                  riemann.py:205-223
 *   clb_last_error             (exceptions never cross the ABI)
 *
 * Conventions: every function returns 0 on success and a negative CLB_E*
 * code on failure; clb_last_error(h) (or clb_last_error(NULL) for creation
 * failures) describes it.  One host thread per handle.  Buffers are device-
 * resident padded SoA arrays owned by the handle (3 per handle: the current
 * state plus two sweep scratch buffers, as timestep.py:113).
 */
#ifndef CLAWB200_H
#define CLAWB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Riemann solver ids (riemann.py:256-284 registry names). */
#define CLB_SOLVER_ADVECTION 0     /* "advection"     m=1               */
#define CLB_SOLVER_ACOUSTICS 1     /* "acoustics"     m=ndim+1          */
#define CLB_SOLVER_SHALLOW_WATER 2 /* "shallow_water" m=3, ndim=2       */
#define CLB_SOLVER_VC_ACOUSTICS 3  /* "vc_acoustics"  m=ndim+3 (p,u..,Z,c) builder extension */

/* Limiter ids: limiter.py:33-39 LIMITER_IDS (stable). */
#define CLB_LIMITER_NONE 0
#define CLB_LIMITER_MINMOD 1
#define CLB_LIMITER_SUPERBEE 2
#define CLB_LIMITER_MC 3
#define CLB_LIMITER_VANLEER 4

/* Boundary kinds (boundary.py:20-23) plus HALO: ghost layers read from
 * memory as-is (a neighbouring rank's halo, or caller-filled ghosts). */
#define CLB_BC_OUTFLOW 0
#define CLB_BC_REFLECTIVE 1
#define CLB_BC_PERIODIC 2
#define CLB_BC_HALO 3

/* Error codes. */
#define CLB_OK 0
#define CLB_EINVAL -1     /* ValueError in the reference */
#define CLB_ECUDA -2      /* CUDA runtime failure        */
#define CLB_ENOMEM -3
#define CLB_EUNSUPPORTED -4

typedef struct clb_ctx *clb_handle;

typedef struct clb_desc {
    int32_t ndim;               /* 1..3                                            */
    int32_t num_states;         /* m                                               */
    int32_t itemsize;           /* 4 (float32) | 8 (float64)                       */
    int32_t solver_id;          /* CLB_SOLVER_*                                    */
    int32_t limiter_id;         /* CLB_LIMITER_*                                   */
    int32_t device;             /* CUDA device ordinal                             */
    int64_t cells[3];           /* interior cells per logical axis (x, y, z)       */
    double spacing[3];          /* GridSpec.spacing, fp64 (grid.py:62-66)          */
    double params[8];           /* solver params packed IN THE RUN DTYPE exactly as
                                   RiemannSolver.pack_params (riemann.py:235-253),
                                   then widened to double (exact)                  */
    int32_t bc[3][2];           /* per axis (lo, hi): CLB_BC_*                     */
    int32_t normal_velocity[3]; /* BoundarySpec.normal_velocity; -1 = None         */
} clb_desc;

/* Lifecycle. */
int clb_create(const clb_desc *desc, clb_handle *out);
int clb_destroy(clb_handle h);
const char *clb_last_error(clb_handle h);
int clb_version(void);

/* Optional: run on a caller-owned cudaStream_t (e.g. torch's current stream
 * for NCCL ordering); cudaStreamLegacy ((void*)1) selects the legacy default
 * stream.  NULL restores the handle's own stream. */
int clb_set_stream(clb_handle h, void *cuda_stream);

/* Segment length (cells along the sweep axis per warp/thread) for one
 * axis; 0 = automatic.  Results are bitwise independent of it (segments
 * recompute their shared fans, sweep.py:11-16); exposed for tests/tuning. */
int clb_set_segments(clb_handle h, int axis, int seg_len);

/* x-sweep (contiguous axis) kernel variant of this handle:
 *   CLB_XVAR_AUTO  (0) by solver and grid size (the measured best),
 *   CLB_XVAR_MARCH (1) warp-marching kernel (one lane per cell, shuffles),
 *   CLB_XVAR_TMA   (2) TMA tensor-map transpose kernel (one thread per row),
 *   CLB_XVAR_PAIR  (3) pair warp-march (two cells per lane, 64-cell chunks),
 *   CLB_XVAR_TMA_STREAM (4) TMA transpose with the streaming geometry (64
 *                       rows of 128 bytes; fp64 shallow water only),
 *   CLB_XVAR_TMA_ADAPT  (5) both TMA geometries launched on every x sweep,
 *                       the one the previous strided sweep's share of
 *                       computed (not skipped) cell groups selects does
 *                       the work (fp64 shallow water only; AUTO's choice
 *                       for large grids).
 * Results are bitwise independent of the variant; exposed so every variant
 * can be held to the oracle at any size (tests) and for tuning.  The
 * process-wide default is CLB_CONTIG=tma|shfl|pair|stream|adapt (read
 * once), else AUTO. */
enum {
  CLB_XVAR_AUTO = 0, CLB_XVAR_MARCH = 1, CLB_XVAR_TMA = 2, CLB_XVAR_PAIR = 3,
  CLB_XVAR_TMA_STREAM = 4, CLB_XVAR_TMA_ADAPT = 5
};
int clb_set_x_variant(clb_handle h, int variant);
/* The variant the next x sweep of this handle launches (1 .. 5). */
int clb_x_variant(clb_handle h, int32_t *variant);
/* The geometry pair's selector (CLB_XVAR_TMA_ADAPT only; CLB_EUNSUPPORTED
 * otherwise): the warp groups the strided sweeps computed (not skipped) since
 * the last x sweep, and the count below which the next x sweep runs the
 * streaming twin.  Synchronises the handle's stream (tests / diagnostics). */
int clb_x_activity(clb_handle h, uint64_t *computed, uint64_t *threshold);

/* Interior transfer, frame-payload order: state-major, then z, y, x (x
 * fastest), ghost cells excluded; nbytes must equal m*prod(cells)*itemsize.
 * buf in {0,1,2}. */
int clb_upload(clb_handle h, int buf, const void *interior, size_t nbytes);
int clb_download(clb_handle h, int buf, void *interior, size_t nbytes);

/* Whole padded arrays, exactly the reference StateGrid.data layout
 * (m, [nz+4,] [ny+4,] nx+4), ghosts included (grid.py:145-160).  Used by the
 * per-sweep API, whose ghost cells are caller-filled and read as-is with
 * CLB_BC_HALO on the swept axis (sweep.py:206-212). */
int clb_upload_padded(clb_handle h, int buf, const void *padded, size_t nbytes);
int clb_download_padded(clb_handle h, int buf, void *padded, size_t nbytes);

/* Change the boundary kinds of one axis after creation (CLB_BC_*). */
int clb_set_boundary(clb_handle h, int axis, int lo, int hi);

/* One directional sweep src -> dst (src != dst), BCs fused.  dt > 0 (fp64);
 * dtdx = T(dt / spacing[axis]) is formed exactly as sweep.py:336-337.
 * Outputs: max |s| over every interface solved (widened to double) and a
 * non-finite flag for the dst interior.  Synchronous. */
int clb_sweep(clb_handle h, int axis, double dt, int src, int dst,
              double *max_abs_speed, int32_t *nonfinite);

/* Asynchronous form: results accumulate in result slot `slot` (0..3) until
 * clb_fetch.  `literal`=1 selects the fully literal kernel (no structural-
 * zero elision; used on the blow-up slow path). */
int clb_sweep_async(clb_handle h, int axis, double dt, int src, int dst, int slot,
                    int literal);
int clb_fetch(clb_handle h, int nslots, double *max_abs_speed, int32_t *nonfinite);

/* Segment decomposition of a sweep along its axis (nseg segments of seg_len
 * cells), and a launch of segments [seg_begin, seg_end) only (strided y/z
 * sweeps).  Segment k reads rows
 * [k*seg_len - 2, min(n, (k+1)*seg_len) + 2), so the segments that stay
 * clear of the ghost rows can run while a halo exchange is in flight
 * (multi-GPU overlap); results are bitwise those of one full launch. */
int clb_sweep_segments(clb_handle h, int axis, int32_t *nseg, int32_t *seg_len);
int clb_sweep_async_range(clb_handle h, int axis, double dt, int src, int dst, int slot,
                          int literal, int seg_begin, int seg_end);

/* All ndim sweeps of one step attempt, x then y then z (timestep.py:35-42,
 * 200-211): sweep j reads the previous output and writes scratch[j % 2].
 * One device->host read at the end.  speeds[j], nonfinite[j] per sweep. */
int clb_attempt_step(clb_handle h, double dt, int src, int scratch0, int scratch1,
                     double *speeds, int32_t *nonfinite);

/* First non-finite interior value of `buf` in C order (state, z, y, x);
 * found=0 when the buffer is finite.  cell[] is logical (x, y, z). */
int clb_first_nonfinite(clb_handle h, int buf, int32_t *found, int32_t *state,
                        int64_t cell[3]);

/* Device pointers for halo exchange along the slowest axis (ndim >= 2):
 * for side 0 (lo) / 1 (hi) returns the first byte of the 2 owned boundary
 * rows/planes to SEND and of the 2 ghost rows/planes to RECEIVE into, for
 * state 0; state k is at + k*state_stride_bytes; each block is
 * block_bytes long and contiguous (whole pitched rows/planes, ghost
 * columns included). */
int clb_halo_layout(clb_handle h, int buf, int side, void **send_ptr, void **recv_ptr,
                    size_t *block_bytes, size_t *state_stride_bytes);

/* Host-staged halo transfer (the CPU-transport path of the slab exchange):
 * to_host=1 copies the 2 owned boundary rows/planes of `side` for every
 * state into host (m blocks of block_bytes, state-major); to_host=0 writes
 * host into the ghost rows/planes of `side`.  Synchronous. */
int clb_halo_copy(clb_handle h, int buf, int side, int to_host, void *host);

/* Per-interface solve of n (q_l, q_r) pairs on the device (parity unit for
 * the Riemann plugins).  q arrays are (n, m) row-major in the run dtype;
 * W out (n, nw, m), s out (n, nw). */
int clb_solve_pairs(clb_handle h, int axis, int64_t n, const void *ql, const void *qr,
                    void *W, void *s);

/* Frame writer (frames.py:1-104 CLAWFRM1): header + the interior payload of
 * buffer `buf` (per state, x fastest, ghost cells excluded), written straight
 * into `out` (pinned memory gives a direct device->host copy).  The bytes
 * equal frame_bytes(grid, time, step) of the reference. */
int clb_frame_size(clb_handle h, size_t *nbytes);
int clb_write_frame(clb_handle h, int buf, double time, uint64_t step, void *out, size_t nbytes);

/* Device-resident run loop (timestep.py:245-285 run_until between two stop
 * times).  Attempts run back to back from a CUDA graph: the ndim sweeps read
 * their buffers and dt from a device control block, and a one-thread
 * controller kernel evaluates each attempt with the reference's fp64
 * expressions (timestep.py:151-243: dt = (cfl_target*min_dx)/s capped and
 * clipped to `stop`, nu = (dt*s)/min_dx, accept iff nu <= cfl_max, buffer
 * rotation, t = stop if landed else t + dt, dt_retry, the two-revert
 * instability check) and prepares the next one, so the dt sequence is
 * bit-identical to the host loop.  The batch ends when t reaches `stop`,
 * `max_accepted` attempts were accepted (< 0: no limit), the attempt log is
 * full, or an attempt fails; one device->host read at the end.
 * In: every field up to and including max_accepted.  Out: the controller
 * fields (t .. scratch1) and n_attempts .. fail_dt. */
#define CLB_BATCH_STOP 0      /* t reached stop                                  */
#define CLB_BATCH_MAXSTEPS 1  /* max_accepted attempts accepted                   */
#define CLB_BATCH_LOGFULL 2   /* log_cap attempts recorded; call again            */
#define CLB_BATCH_BLOWUP 3    /* attempt n_attempts produced a non-finite value in
                                 sweep fail_sweep (not logged; buffers untouched)  */
#define CLB_BATCH_UNSTABLE 4  /* the last logged attempt was a second consecutive
                                 revert without improvement (UnstableStepError)   */
#define CLB_BATCH_DTERR 5     /* no finite dt (no wave speed, no cap, no stop)   */

typedef struct clb_batch {
    double t, last_max_speed, prev_nu, nu_max;
    int32_t prev_reverted;
    int32_t cur, scratch0, scratch1;   /* buffer roles (timestep.py:113,216-219) */
    double stop, cfl_target, cfl_max, dt_cap, min_spacing;
    int64_t max_accepted;
    int64_t n_attempts, n_accepted;
    int32_t status, fail_sweep;
    double fail_dt;
} clb_batch;

/* One logged attempt (timestep.py:45-55 StepAttempt). */
typedef struct clb_attempt {
    double t_start, dt, max_speed, nu, dt_retry;
    int32_t accepted, landed;
} clb_attempt;

int clb_run_batch(clb_handle h, clb_batch *b, clb_attempt *log, int64_t log_cap);

/* User device Riemann solvers (the reference's plugin ABI,
 * riemann.py:190-212 RiemannSolver + register_solver, riemann.py:259-262).
 * A user solver is CUDA source for the scalar routine
 *     scalar(q_l, q_r, normal, params, W_out, s_out)
 * compiled at run time (paper_1805_08846_b200/devsolver.py, nvcc with this
 * library's flags and headers) into a separate shared object whose entry
 * points are registered here under an id >= CLB_SOLVER_USER_BASE.  The
 * launch function receives the library's internal per-sweep argument block
 * (`args`, `args_size` bytes, checked at registration) and a cudaStream_t;
 * the pairs function is clb_solve_pairs' kernel.  Each registration fixes
 * the state count and the dimensionality it was compiled for. */
#define CLB_SOLVER_USER_BASE 16
#define CLB_SOLVER_USER_MAX 64
typedef int (*clb_user_launch_fn)(int ndim, int axis, int literal, const void *args,
                                  void *cuda_stream);
typedef int (*clb_user_pairs_fn)(int ndim, int axis, const void *ql, const void *qr, void *W,
                                 void *s, int64_t n, const double *params, void *cuda_stream);
int clb_register_device_solver(int solver_id, int ndim, int num_states, int num_waves,
                               size_t args_size, clb_user_launch_fn launch_f32,
                               clb_user_launch_fn launch_f64, clb_user_pairs_fn pairs_f32,
                               clb_user_pairs_fn pairs_f64);
/* sizeof the per-sweep argument block of this library build. */
size_t clb_sweep_args_size(void);

/* Slab decomposition on the device (slab.py).  Each rank's
 * handle owns its slab of the global grid (slowest axis split); the slow-axis
 * sides with a neighbour are CLB_BC_HALO.  clb_attach_comm creates an NCCL
 * communicator (NCCL is loaded at run time; `id` is the 128-byte
 * ncclUniqueId from clb_nccl_unique_id on one rank, broadcast by the caller)
 * and from then on every attempt -- clb_attempt_step and the attempt graph
 * of clb_run_batch -- exchanges the 2 boundary rows/planes of every state
 * with the neighbours before the slow sweep (pack into fixed staging
 * buffers, ncclSend/ncclRecv on a side stream while the slow sweep's
 * interior segments run, unpack into the ghost layers) and max-allreduces
 * the per-sweep (max |s|, non-finite) results before they are read, so the
 * fp64 controller takes the identical decision on every rank.  lo_nbr /
 * hi_nbr: neighbour ranks (-1 = physical boundary); a rank may be its own
 * neighbour (a periodic axis on one rank).  Collective over the ranks. */
int clb_nccl_unique_id(void *id_out /* 128 bytes */);
int clb_attach_comm(clb_handle h, const void *id, int nranks, int rank, int lo_nbr, int hi_nbr);
/* The exchange alone into buffer `buf`'s ghost layers (blow-up slow path). */
int clb_halo_exchange(clb_handle h, int buf);
/* Max-allreduce of the accumulated per-sweep result slots (no-op without a
 * communicator); clb_fetch then reads the global values. */
int clb_results_allreduce(clb_handle h);

/* Self-test of the branch-free fp64 division / square root used by the
 * sweep kernels (clb_solvers.cuh FastArith) against div.rn.f64 /
 * sqrt.rn.f64 on n host pairs (a[i], b[i]) on device `device`.  out[0] =
 * quotients where the fast path claimed validity but differs bitwise from
 * div.rn, out[1] = same for sqrt(a[i]), out[2] / out[3] = how many
 * quotients / roots fell back to the exact path; out[4..7] the same for the
 * fp32 path on the low 32 bits of a[i], b[i] read as floats; out[8] /
 * out[9] mismatches / fallbacks of the limiter-ratio division (kChkLim: a
 * zero quotient's sign is free), out[10] / out[11] the same for the Roe
 * division (kChkNumNormDen) on the pairs with b in [2^-485, 2^513].  No
 * handle needed. */
int clb_selftest_arith(int device, int64_t n, const double *a, const double *b, int64_t out[12]);

/* Kernel timing (CUDA events on the launch stream) for the bench: when
 * enabled, every sweep launch is bracketed by events; clb_timing returns
 * the summed milliseconds and launch counts per axis and resets them. */
int clb_enable_timing(clb_handle h, int on);
int clb_timing(clb_handle h, double ms_per_axis[3], int64_t launches_per_axis[3]);

/* Pinned host memory for end-to-end transfers. */
void *clb_host_alloc(size_t nbytes);
void clb_host_free(void *p);

/* Device bytes owned by the handle and the pitch (elements) of one row. */
int clb_memory_info(clb_handle h, size_t *device_bytes, int64_t *row_pitch);

#ifdef __cplusplus
}
#endif

#endif /* CLAWB200_H */
