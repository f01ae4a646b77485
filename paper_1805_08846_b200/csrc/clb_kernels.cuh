// clb_kernels.cuh -- the fused directional sweep kernel for sm_100a.
//
// One launch == one directional sweep of the reference (sweep.py:307-377
// sweep_axis_tiled over sweep.py:183-263 sweep_tile) with
//   * the ghost-cell fill of boundary.py:87-122 fused in as a read-side index
//     remap (physical boundaries) or a plain read of memory ghosts (HALO),
//   * the per-sweep max |s| folded by warp shuffle + block reduction + one
//     guarded atomicMax,
//   * the non-finite check of timestep.py:179-186 folded into the store
//     epilogue on the integer pipe.
//
// Thread mapping: one thread per pencil, marching along the sweep axis with
// the reference's three-fan ring (sweep.py:195-200) held in registers.  The
// ring is unrolled by its period (3) so slot rotation costs no moves.
//
// Data movement: a CTA = 4 consumer warps (128 pencils) + 1 producer warp.
// The producer streams the pencils' cells, NC per pencil per stage, into a
// shared-memory ring with cp.async.bulk (TMA engine) tracked by mbarriers
// (full/empty per stage), so HBM latency hides behind NSTAGE-1 stages of
// prefetch while consumers compute:
//   * strided sweeps (y, z): a stage is NC rows of 128 consecutive x-cells
//     per state -- one contiguous bulk copy per row and state; consumer t
//     reads column t (bank-conflict free);
//   * the contiguous sweep (x): a stage is 48 bytes (NC cells) of each of
//     128 rows per state -- one bulk copy per row and state, issued by all
//     32 producer lanes; consumer t reads its own row (a transpose through
//     shared memory, so the x-sweep needs no warp shuffles).
// Segments along the sweep axis recompute the fans they share with their
// neighbour exactly as the reference's tiles do (sweep.py:11-16), so results
// are bitwise independent of the segmentation.
#pragma once
#include <atomic>

#include "clb_async.cuh"
#include "clb_solvers.cuh"

namespace clb {

enum { BC_OUTFLOW = 0, BC_REFLECTIVE = 1, BC_PERIODIC = 2, BC_HALO = 3 };

constexpr unsigned FULL = 0xffffffffu;
constexpr int kConsumers = 128;        // pencils per CTA
#ifndef CLB_INLINE_PRODUCER
#define CLB_INLINE_PRODUCER 0
#endif
#ifndef CLB_X_LEGACY
#define CLB_X_LEGACY 0
#endif
#ifndef CLB_X_ROWS
#define CLB_X_ROWS 128  // rows per CTA of the TMA x sweep (64 or 128)
#endif
// CLB_INLINE_PRODUCER: consumer thread 0 issues the stage copies (no
// producer warp), so a CTA is 4 warps
constexpr bool kInlineProducer = CLB_INLINE_PRODUCER != 0;
constexpr int kThreads = kConsumers + (kInlineProducer ? 0 : 32);
// The TMA x sweep issues its copies from consumer thread 0 by default: its
// shared memory holds 3 CTAs per SM anyway, and without the producer warp
// the same register file gives each thread 168 registers instead of 136
// (the march spills less).  CLB_X_INLINE=0 restores the producer warp.
#ifndef CLB_X_INLINE
#define CLB_X_INLINE 1
#endif
constexpr bool kInlineX = CLB_X_INLINE != 0;
template <bool CONTIG> constexpr bool inline_producer() {
  return (CONTIG && !CLB_X_LEGACY) ? kInlineX : kInlineProducer;
}
constexpr int kXRows = CLB_X_ROWS;
// XS = 1: the streaming geometry of the TMA x sweep (fp64 shallow water):
// 64 rows of 128 bytes per box.  It streams a mostly skipped sweep ~8%
// faster than the default 128 rows x 64 B but leaves fewer warps for active
// flow; the host launches both and each reads the previous strided sweep's
// active-group count to decide which one works (profiles/r2_notes.md r2s).
#ifndef CLB_XS_ROWS
#define CLB_XS_ROWS 64
#endif
#ifndef CLB_XS_ROW
#define CLB_XS_ROW 128
#endif
#ifndef CLB_XS_MINB
#define CLB_XS_MINB 5
#endif
#ifndef CLB_XS_SUB
#define CLB_XS_SUB 1    // boxes side by side along x per stage of the streaming twin
#endif
template <int XS> constexpr int x_rows() { return XS ? CLB_XS_ROWS : kXRows; }
// the solvers whose x sweep has a streaming twin (XS = 1): fp64 shallow
// water; only their strided sweeps count computed groups (SweepArgs::act)
template <typename T, class S> __host__ __device__ constexpr bool has_xs() {
  return sizeof(T) == 8 && S::M == 3 && S::NW >= 3 && !CLB_X_LEGACY;
}
template <bool CONTIG, int XS = 0> constexpr int threads_of() {
  return ((CONTIG && !CLB_X_LEGACY) ? x_rows<XS>() : kConsumers) +
         (inline_producer<CONTIG>() ? 0 : 32);
}
constexpr int kRowStrideContig = 48;   // bytes per row per state in a contig stage

// Device-resident step controller state (clb_capi.cu ctl_* kernels; the
// fp64 controller of timestep.py:151-243 run on the device between the
// sweeps of a batch).  Sweeps launched "indirectly" read their buffers and
// dt from here, so a whole run can be replayed from a CUDA graph without a
// host round trip per attempt.
struct DevCtl {
  double t, last_max_speed, prev_nu, nu_max;
  double stop, cfl_target, cfl_max, dt_cap, min_spacing;
  double dt;                 // current attempt
  long long max_accepted;    // < 0: unlimited
  long long n_attempts, n_accepted, log_cap;
  int prev_reverted, landed;
  int cur, s0, s1;
  int src[3], dst[3];        // buffer roles of the current attempt's sweeps
  int done, status, fail_sweep, ndim;
  void* log;                 // clb_attempt[log_cap]
  unsigned int blocks_done;  // CTAs of the fused final sweep that finished
};

}  // namespace clb
#include "clb_controller.cuh"
namespace clb {

template <typename T> struct SweepArgs {
  const T* qin;     // element (0,0,0) of state 0 (interior origin)
  T* qout;
  int64_t sstride;  // elements between states
  int64_t astride;  // element stride along the sweep axis
  int64_t t1stride; // stride of transverse axis 1 (strided: x = 1; contig: y rows)
  int64_t t2stride; // remaining transverse axis
  int n;            // cells along the sweep axis
  int n1, n2;       // transverse extents
  int seg_len, nseg;
  int seg_base;     // first segment of this launch (segment-range launches)
  int bc_lo, bc_hi, nv;
  int lim_id;
  T dtdx;
  Params<T> P;
  unsigned long long* smax_bits;
  int* nonfinite;
  int tx0, ty0, tz0;  // tensor-map coordinates of interior cell (0,0,0)
  int src, dst;       // buffer indices (select the TMA maps)
  // indirect launch (ctl != nullptr): src, dst and dt come from the
  // controller; bufs are the three buffers' interior origins
  const DevCtl* ctl;
  int axis;
  double spacing;
  const void* bufs[3];
  // the attempt's last sweep: its last CTA runs the controller (no separate
  // controller launch per attempt)
  int fuse_ctl;
  Result* res;
  // x geometry pair (sweep_kernel): non-null on both x launches of a pair;
  // the streaming twin works when *xsel < xsel_thresh.  act: strided sweeps
  // add their computed (not skipped) cell groups, one atomic per warp.
  const unsigned long long* xsel;
  unsigned long long xsel_thresh;
  unsigned long long* act;
};

// TMA descriptors of the three buffers (load: full padded extent; store:
// interior-clipped), passed by value as a __grid_constant__ parameter.
struct TmaMaps {
  alignas(64) unsigned char ld[3][128];
  alignas(64) unsigned char st[3][128];
};

// Per-launch values that an indirect launch reads from the controller:
// buffers (and with them the TMA maps) and dtdx.  Kept out of SweepArgs so
// the kernel never writes into a copy of its by-value parameter (nvcc 12.9
// dropped such stores and kept reading the parameter's original fields).
template <typename T> struct Live {
  const T* qin;
  T* qout;
  T dtdx;
  int src, dst;
};

// Returns false if the controller has finished (graph replays past the end
// of a run are no-ops).
template <typename T> __device__ __forceinline__ bool resolve_live(const SweepArgs<T>& a,
                                                                   Live<T>& L) {
  int src = a.src, dst = a.dst;
  T dtdx = a.dtdx;
  if (a.ctl != nullptr) {
    const DevCtl* c = a.ctl;
    if (c->done) return false;
    src = c->src[a.axis];
    dst = c->dst[a.axis];
    // sweep.py:336-337: dtdx = T(dt / dx[axis]), IEEE fp64 division then rounding
    dtdx = (T)(c->dt / a.spacing);
  }
  // Both launch kinds select the buffers from bufs[] by index.  (Assigning
  // a.qin on the direct path and a selected buffer on the indirect one made
  // nvcc 12.9 fold the pointer back to a.qin for both.)
  L.src = src;
  L.dst = dst;
  L.dtdx = dtdx;
  L.qin = (const T*)(src == 0 ? a.bufs[0] : (src == 1 ? a.bufs[1] : a.bufs[2]));
  L.qout = (T*)const_cast<void*>(dst == 0 ? a.bufs[0] : (dst == 1 ? a.bufs[1] : a.bufs[2]));
  return true;
}

// Conditional IEEE negation (boundary.py:114,122 `*= -1.0`) as a sign-bit
// flip.  Written on the bit pattern so the compiler cannot turn the
// "negate state nv" loop into a dynamically indexed local-memory array.
__device__ __forceinline__ double neg_if(double v, bool f) {
  return __hiloint2double(__double2hiint(v) ^ (f ? (int)0x80000000 : 0), __double2loint(v));
}
__device__ __forceinline__ float neg_if(float v, bool f) {
  return __int_as_float(__float_as_int(v) ^ (f ? (int)0x80000000 : 0));
}

// boundary.py:108-122 as a read-side index map: ghost cell j of a pencil
// reads interior cell remap(j), negating state nv for reflective walls.
__device__ __forceinline__ int remap(int j, int n, int lo, int hi, bool& neg) {
  neg = false;
  if (j < 0) {
    if (lo == BC_OUTFLOW) return 0;
    if (lo == BC_PERIODIC) return n + j;
    if (lo == BC_REFLECTIVE) { neg = true; return -1 - j; }
    return j;  // halo / caller-filled ghosts live in memory
  }
  if (j >= n) {
    if (hi == BC_OUTFLOW) return n - 1;
    if (hi == BC_PERIODIC) return j - n;
    if (hi == BC_REFLECTIVE) { neg = true; return 2 * n - 1 - j; }
    return j;
  }
  return j;
}

// Warp + block reduction of (max |s|, finite key), one guarded atomic per block.
template <typename T>
__device__ __forceinline__ void finish_block(T smax, uint32_t fin, const SweepArgs<T>& a) {
  __shared__ double s_max[32];
  __shared__ uint32_t s_fin[32];
  double v = (double)smax;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    double w = __shfl_xor_sync(FULL, v, o);
    v = w > v ? w : v;
    fin = min(fin, __shfl_xor_sync(FULL, fin, o));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { s_max[wid] = v; s_fin[wid] = fin; }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = 1; i < nw; ++i) {
      v = s_max[i] > v ? s_max[i] : v;
      fin = min(fin, s_fin[i]);
    }
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    if (bits > *((volatile unsigned long long*)a.smax_bits)) atomicMax(a.smax_bits, bits);
    if (fin == 0u) atomicOr(a.nonfinite, 1);
    if (a.fuse_ctl) {
      // last CTA of the attempt's final sweep: every CTA's atomics above are
      // visible (fence + counter), so it evaluates the attempt and prepares
      // the next one exactly as the ctl_finish kernel would
      DevCtl* c = const_cast<DevCtl*>(a.ctl);
      __threadfence();
      const unsigned total = gridDim.x * gridDim.y * gridDim.z;
      if (atomicAdd(&c->blocks_done, 1u) == total - 1u) {
        __threadfence();
        c->blocks_done = 0u;
        ctl_finish_dev(c, a.res);
      }
    }
  }
}

#ifndef CLB_EXACT32
#define CLB_EXACT32 0
#endif
#ifndef CLB_CONTIG_FAST32
#define CLB_CONTIG_FAST32 0
#endif
#ifndef CLB_CONTIG_DEPTH
#define CLB_CONTIG_DEPTH 1
#endif
#ifndef CLB_CONTIG_NSTAGE
#define CLB_CONTIG_NSTAGE 2
#endif
#ifndef CLB_NO_REDO
#define CLB_NO_REDO 0
#endif
#ifndef CLB_CONTIG_MINB
#define CLB_CONTIG_MINB 1  // resident 128-thread CTAs the warp-march register budget targets
#endif
#ifndef CLB_STRIDED_OUT
#define CLB_STRIDED_OUT 2  // strided sweeps stage outputs for row bulk stores (0: per-thread stores)
#endif
#ifndef CLB_STRIDED_NC
#define CLB_STRIDED_NC 3   // rows per strided stage (a multiple of 3)
#endif
#ifndef CLB_F32_MINB
#define CLB_F32_MINB 4
#endif
#ifndef CLB_F64_MINB
#define CLB_F64_MINB 3
#endif
#ifndef CLB_SW_MINB
#define CLB_SW_MINB 3
#endif
#ifndef CLB_SW_MINB_STRIDED
#define CLB_SW_MINB_STRIDED CLB_SW_MINB
#endif
// Resident CTAs per SM the register allocation is sized for: fp64 shallow
// water 3 (128 registers; the march would take ~168 at 2 CTAs, but the extra
// warps win, profiles/r1_notes.md), other fp64 3, fp32 4.
// With the inline producer a CTA is 4 warps, so the same register budget
// fits one more CTA: fp64 shallow water 4 (strided; the TMA x-sweep stays
// at 3, its stages fill the shared memory), other fp64 4, fp32 5.
#ifndef CLB_SW_MINB_INL
#define CLB_SW_MINB_INL 4
#endif
#ifndef CLB_X_MINB
#define CLB_X_MINB 3   // resident CTAs of the TMA x sweep of the other solvers
#endif
#ifndef CLB_SW_MINB_X_INL
#define CLB_SW_MINB_X_INL 3
#endif
template <typename T, class S, bool CONTIG, int XS = 0> constexpr int kMinBlocks() {
  if (XS) return CLB_XS_MINB;
  if (CONTIG && !CLB_X_LEGACY && kInlineX)
    return (sizeof(T) == 8 && S::NW >= 3) ? CLB_SW_MINB_X_INL : CLB_X_MINB;
  if (kInlineProducer)
    return (sizeof(T) == 8 && S::NW >= 3) ? (CONTIG ? CLB_SW_MINB_X_INL : CLB_SW_MINB_INL)
                                          : (sizeof(T) == 4 ? CLB_F32_MINB + 1 : CLB_F64_MINB + 1);
  return (sizeof(T) == 8 && S::NW >= 3) ? (CONTIG ? CLB_SW_MINB : CLB_SW_MINB_STRIDED)
                                        : (sizeof(T) == 4 ? CLB_F32_MINB : CLB_F64_MINB);
}

// (Register budgets come from __launch_bounds__: each SM sub-partition has
// its own 16K-register file, so 3 CTAs of 5 warps -- 4 warps on some
// sub-partitions -- get 128 registers, and an explicit __maxnreg__(136)
// measured a whole CTA less resident per SM.)
template <typename T, class S, bool CONTIG> struct StageGeom {
  static constexpr int NC = CONTIG ? (kRowStrideContig / (int)sizeof(T)) : CLB_STRIDED_NC;  // cells/stage
  static constexpr int BYTES = CONTIG ? S::M * kConsumers * kRowStrideContig
                                      : S::M * NC * kConsumers * (int)sizeof(T);
  // two leading alignment dummies: the prologue cells sit at r = 2..5, so every
  // 3-cell group starts on ring phase 0, and every contig stage box starts
  // 16-byte aligned (TMA requirement) because segments start at multiples of NC.
  static constexpr int A = 2;
  // output staging tiles: TMA stores (contig); row bulk stores for the
  // compute-bound fp64 shallow-water strided sweeps (y 1.88 -> 1.69 ms at
  // 8192^2), per-thread stores elsewhere (acoustics y/z, which need the
  // deeper input ring: 1.45 vs 1.64 ms with staging; fp32 SW 0.83 vs 0.96)
  static constexpr int NOUT = CONTIG ? 2 : ((S::NW >= 3 && sizeof(T) == 8) ? CLB_STRIDED_OUT : 0);
  // strided input ring: as deep as the shared memory of the resident CTAs
  // the register budget targets allows (at most 6 stages)
  static constexpr int BUDGET =
      kInlineProducer ? (225 * 1024 / kMinBlocks<T, S, CONTIG>() - 1024) : 72 * 1024;
  static constexpr int NSTAGE_RAW =
      CONTIG ? (S::M >= 4 ? 2 : CLB_CONTIG_NSTAGE) : (BUDGET / BYTES - NOUT);
  static constexpr int NSTAGE = NSTAGE_RAW < 2 ? 2 : (NSTAGE_RAW > 6 ? 6 : NSTAGE_RAW);
  static constexpr int SMEM = (NSTAGE + NOUT) * BYTES + 2 * NSTAGE * 8;
  static_assert(A % 3 == 2, "prologue phase");
};

// ---------------------------------------------------------------------------
// The ring-march state of one pencil.  Slot p holds interface/cell index
// i with i % 3 == p; P is the slot of the incoming cell.  D is the arithmetic
// policy (clb_solvers.cuh); `bad` collects FastArith domain failures.
#ifndef CLB_UNIFORM_SKIP
#define CLB_UNIFORM_SKIP 1
#endif
#ifndef CLB_STEP_REDO
#define CLB_STEP_REDO 1
#endif
#ifndef CLB_SKIP_BACKOFF
#define CLB_SKIP_BACKOFF 7   // most groups computed unchecked after failed checks
#endif

// Bitwise equality of two cells' states.
template <typename T, int M>
__device__ __forceinline__ bool same_bits(const T (&a)[M], const T (&b)[M]) {
  if constexpr (sizeof(T) == 8) {
    unsigned long long d = 0ull;
#pragma unroll
    for (int k = 0; k < M; ++k)
      d |= (unsigned long long)(__double_as_longlong(a[k]) ^ __double_as_longlong(b[k]));
    return d == 0ull;
  } else {
    uint32_t d = 0u;
#pragma unroll
    for (int k = 0; k < M; ++k) d |= __float_as_uint(a[k]) ^ __float_as_uint(b[k]);
    return d == 0u;
  }
}

template <typename T, class S, int LIM, bool LIT, class D> struct March {
  using Cell = typename S::Cell;
  using Fan = typename S::Fan;
  static constexpr int M = S::M;
  // Uniform-state skip (exact; not in the literal blow-up kernels).  When
  // the incoming cell i and the three before it are bitwise equal, the step
  // is known without arithmetic:
  //   * X[i] = X[i-1] and F[i] = F[i-1]: the same inputs give the same bits
  //     (make / solve are pure), and |s| of F[i] is already in smax;
  //   * every wave of a fan between equal cells is +-0 (all jumps are +0 and
  //     each wave is a product / quotient with a jump factor), so the
  //     correction at interface i-1 is ft = +0 + coef*(+-0) = +0 per state
  //     (wn = +0 gives lim = 1; coef is finite);
  //   * the update of cell i-2 adds only +-0 terms to accumulators started at
  //     +0 and subtracts dtdx*(+0): out = q[i-2] = q[i] bitwise.
  // "Every wave is +-0" needs the fan to be finite (a NaN root of a negative
  // depth would make the reference's outputs NaN), so F[i-1] is tested too.
  // segment_pass skips whole 3-cell groups when every lane of the warp may
  // (a warp-uniform branch); after one skipped group all three ring slots
  // hold the uniform state, so the next skipped groups copy nothing.
  static constexpr bool kSkip = !LIT && CLB_UNIFORM_SKIP != 0 && S::kUniformSkip;
  Cell X[3];
  Fan F[3];
  T G[3][M];
  T smax;
  uint32_t fin;
  bool bad;
  bool idle;  // lane outside the pencil block: never holds a skip back
  bool uni;   // every ring slot holds the uniform state (a group was skipped)
  int run;    // consecutive incoming cells bitwise equal to their predecessor
  int cool, back;  // skip-check back-off (warp-uniform)
  T dtdx;

  __device__ __forceinline__ int lim(const SweepArgs<T>& a) const { return LIM >= 0 ? LIM : a.lim_id; }

  __device__ __forceinline__ static bool fan_finite(Fan f) {
    uint32_t key = 0xffffffffu;
    S::for_regs(f, [&](T& r) { key = min(key, finite_key(r)); });
    return key != 0u;
  }
  // Group skip (cells i, i+1, i+2 arriving; slot PP holds cell i-1): true
  // when the warp skips all three steps; then the ring is made uniform.  The
  // caller emits q0..q2 as the group's outputs.  `run` (consecutive incoming
  // cells bitwise equal to their predecessor) is only maintained here; after
  // a failed check the warp computes the next `cool` groups without checking
  // (exponential back-off up to CLB_SKIP_BACKOFF groups), so flow that is
  // active everywhere pays for about one check in that many groups.
  __device__ __forceinline__ bool check_due() {
    if (cool > 0) {
      --cool;
      run = 0;
      return false;
    }
    return true;
  }
  template <int PP>
  __device__ __forceinline__ bool skip_group(const T (&q0)[M], const T (&q1)[M],
                                             const T (&q2)[M]) {
    const bool e0 = same_bits<T, M>(q0, X[PP].q);
    const bool e1 = same_bits<T, M>(q1, q0), e2 = same_bits<T, M>(q2, q1);
    const bool eq = idle || (e0 && e1 && e2);
    const bool ok = eq && (idle || run >= 2);
    run = e2 ? (e1 ? (e0 ? run + 3 : 2) : 1) : 0;
    if (__all_sync(FULL, ok) && (uni || __all_sync(FULL, idle || fan_finite(F[PP])))) {
      if (!uni) {
        constexpr int Q1 = (PP + 1) % 3, Q2 = (PP + 2) % 3;
        X[Q1] = X[PP];
        X[Q2] = X[PP];
        F[Q1] = F[PP];
        F[Q2] = F[PP];
#pragma unroll
        for (int k = 0; k < M; ++k) {
          G[0][k] = T(0);
          G[1][k] = T(0);
          G[2][k] = T(0);
        }
        uni = true;
      }
      back = 0;
      return true;
    }
    uni = false;
    // a uniform group that only lacked the run-up (run < 2, e.g. after
    // unchecked groups) is checked again at once; anything else backs off
    if (!__all_sync(FULL, eq)) {
      back = min(2 * back + 1, CLB_SKIP_BACKOFF);
      cool = back;
    }
    return false;
  }
  // prologue steps (no output)
  template <int P> __device__ __forceinline__ void first(const T (&q)[M]) {
    X[P] = S::template make<D>(q, bad);
    run = 0;
    cool = 0;
    back = 0;
  }
  // CLB_STEP_REDO (default): a step (fan, correction, update) in which some
  // lane left the FastArith domain is recomputed at once by the warp with
  // ExactArith from the same inputs (the step only writes X[P], F[P], G[P-1]
  // and its output), instead of the CTA re-running its whole segment
  // (SW 8192^2 dam break 39.4 -> 47.2 Gcell-upd/s, profiles/r2_notes.md).
  static constexpr bool kStepRedo = CLB_STEP_REDO && D::template kBranchFree<T>;
  template <int P, class D2> __device__ __forceinline__ void fan_raw(const T (&q)[M],
                                                                     const SweepArgs<T>& a,
                                                                     bool& b) {
    constexpr int P1 = (P + 2) % 3;
    X[P] = S::template make<D2>(q, b);
    F[P] = S::template solve<D2>(X[P1], X[P], a.P, b);
  }
  template <int P, class D2> __device__ __forceinline__ void corr_raw(const SweepArgs<T>& a,
                                                                      bool& b) {
    constexpr int P1 = (P + 2) % 3, P2 = (P + 1) % 3;
    correction<S, LIT, D2, T>(F[P2], F[P1], F[P], a.P, dtdx, lim(a), G[P1], b);
  }
  __device__ __forceinline__ bool redo_due(bool sb) const { return __any_sync(FULL, sb && !idle); }
  template <int P> __device__ __forceinline__ void fan_body(const T (&q)[M],
                                                            const SweepArgs<T>& a, bool fold) {
    if constexpr (kStepRedo) {
      bool sb = false;
      fan_raw<P, D>(q, a, sb);
      if (redo_due(sb)) {
        bool d = false;
        fan_raw<P, ExactArith>(q, a, d);
      }
    } else {
      fan_raw<P, D>(q, a, bad);
    }
    if (fold) fold_speed<S, T>(F[P], a.P, smax);
  }
  template <int P> __device__ __forceinline__ void fan(const T (&q)[M], const SweepArgs<T>& a,
                                                       bool fold) {
    fan_body<P>(q, a, fold);
  }
  template <int P> __device__ __forceinline__ void fan_corr(const T (&q)[M],
                                                            const SweepArgs<T>& a, bool fold) {
    fan<P>(q, a, fold);
    if constexpr (kStepRedo) {
      bool sb = false;
      corr_raw<P, D>(a, sb);
      if (redo_due(sb)) {
        bool d = false;
        corr_raw<P, ExactArith>(a, d);
      }
    } else {
      corr_raw<P, D>(a, bad);
    }
  }
  // steady step: returns the updated cell i-2 in `out`
  template <int P> __device__ __forceinline__ void step(const T (&q)[M], const SweepArgs<T>& a,
                                                        bool fold, T (&out)[M]) {
    constexpr int P1 = (P + 2) % 3, P2 = (P + 1) % 3;
    if constexpr (kStepRedo) {
      bool sb = false;
      fan_raw<P, D>(q, a, sb);
      corr_raw<P, D>(a, sb);
      if (redo_due(sb)) {
        bool d = false;
        fan_raw<P, ExactArith>(q, a, d);
        corr_raw<P, ExactArith>(a, d);
      }
      if (fold) fold_speed<S, T>(F[P], a.P, smax);
    } else {
      fan_body<P>(q, a, fold);
      corr_raw<P, D>(a, bad);
    }
    update<S, LIT, T>(X[P2].q, F[P2], F[P1], G[P1], G[P2], a.P, dtdx, out);
  }
};

// ---------------------------------------------------------------------------
// One pass of a CTA over its segment: the producer warp streams the stages,
// the consumer warps march.  k0 numbers the pass's first stage in the CTA's
// running stage sequence (mbarrier phases continue across passes).  Returns
// the consumer's (smax, fin, bad) in the references.
template <typename T, class S, int LIM, bool LIT, bool CONTIG, class D>
__device__ __forceinline__ void segment_pass(const SweepArgs<T>& a, const Live<T>& L,
                                             const TmaMaps& maps_all,
                                             unsigned char* smem, uint64_t* full, uint64_t* empty,
                                             int k0, T& smax, uint32_t& fin, bool& bad) {
  using G = StageGeom<T, S, CONTIG>;
  constexpr int NC = G::NC, NSTAGE = G::NSTAGE, M = S::M, A = G::A;
  const unsigned char* map_ld = maps_all.ld[L.src];
  const unsigned char* map_st = maps_all.st[L.dst];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int seg = blockIdx.y + a.seg_base;
  const int lo = seg * a.seg_len;
  const int hi = min(a.n, lo + a.seg_len);
  const int ncell = hi - lo + A + 4;
  const int nst = (ncell + NC - 1) / NC;
  // pencil block: strided -> 128 x-columns at transverse index blockIdx.z;
  // contig -> 128 rows (y) of plane z = blockIdx.z
  const int64_t pb = (int64_t)blockIdx.x * kConsumers;
  const int64_t npen = a.n1;
  const int nvalid = (int)(npen - pb < (int64_t)kConsumers ? npen - pb : (int64_t)kConsumers);

  // ------------------------------ producer ------------------------------
  // Issue stage k of this pass into its ring slot (after the slot's previous
  // stage was released by every consumer warp).  Run by the dedicated
  // producer warp's lane 0, or -- CLB_INLINE_PRODUCER -- by consumer thread
  // 0, one stage behind the march (no producer warp: its registers go to a
  // fourth resident CTA).
  auto produce = [&](int k) {
    constexpr int isz = (int)sizeof(T);
    const int kk = k0 + k;
    const int s = kk % NSTAGE;
    if (kk >= NSTAGE) mbar_wait_sleep(&empty[s], ((kk / NSTAGE) - 1) & 1);
    unsigned char* st = smem + s * G::BYTES;
    if (!CONTIG) {
      const uint32_t colbytes = (uint32_t)(((nvalid * isz) + 15) & ~15);
      const T* base = L.qin + pb + (int64_t)blockIdx.z * a.t2stride;
      const int r0 = k * NC, r1 = min(ncell, r0 + NC);
      const int rs = max(r0, A);
      const uint32_t bytes = (r1 > rs ? (uint32_t)(r1 - rs) : 0u) * M * colbytes;
      mbar_arrive_expect_tx(&full[s], bytes);
      for (int r = rs; r < r1; ++r) {
        bool neg;
        const int js = remap(lo - 2 - A + r, a.n, a.bc_lo, a.bc_hi, neg);
        const T* src = base + (int64_t)js * a.astride;
#pragma unroll
        for (int q = 0; q < M; ++q)
          bulk_g2s(st + ((q * NC + (r - r0)) * kConsumers) * isz, src + q * a.sstride,
                   colbytes, &full[s]);
      }
    } else {
      const int cy = a.ty0 + (int)pb, cz = a.tz0 + (int)blockIdx.z;
      mbar_arrive_expect_tx(&full[s], (uint32_t)G::BYTES);
      const int cx = a.tx0 + lo - 2 - A + k * NC;
#pragma unroll
      for (int q = 0; q < M; ++q)
        tma_load_4d(st + q * kConsumers * kRowStrideContig, map_ld, cx, cy, cz, q, &full[s]);
    }
  };
  if (!kInlineProducer && warp == kConsumers / 32) {
    if (lane == 0)
      for (int k = 0; k < nst; ++k) produce(k);
    return;
  }
  int issued = 0;   // inline producer: stages of this pass issued so far
  if (kInlineProducer && tid == 0)
    for (; issued < min(nst, NSTAGE); ++issued) produce(issued);
  // ------------------------------ consumers ------------------------------
  const int t = tid;
  const bool active = t < nvalid;
  March<T, S, LIM, LIT, D> mr;
  mr.smax = T(0);
  mr.fin = 0xffffffffu;
  mr.bad = false;
  mr.idle = !active;
  mr.uni = false;
  mr.run = 0;
  mr.cool = 0;
  mr.back = 0;
  mr.dtdx = L.dtdx;
  unsigned nact = 0;  // computed (not skipped) groups of this warp (a.act)
  const T* pin;
  T* pout;
  if (CONTIG) {
    const int64_t off = (pb + (active ? t : 0)) * a.t1stride + (int64_t)blockIdx.z * a.t2stride;
    pin = L.qin + off;
    pout = L.qout + off;
  } else {
    const int64_t off = pb + (active ? t : 0) + (int64_t)blockIdx.z * a.t2stride;
    pin = L.qin + off;
    pout = L.qout + off;
  }
  const bool halo_lo = a.bc_lo == BC_HALO, halo_hi = a.bc_hi == BC_HALO;
  const bool refl_lo = a.bc_lo == BC_REFLECTIVE, refl_hi = a.bc_hi == BC_REFLECTIVE;
  unsigned char* outs = smem + NSTAGE * G::BYTES;  // output tiles
  // strided output rows go out as bulk copies when a row's bytes are a
  // multiple of 16 (a partial last column block may not be)
  const bool bulk_out = !CONTIG && ((nvalid * (int)sizeof(T)) & 15) == 0;

  // Ghost cells (boundary.py:87-122) are fixed up in the stage itself, once
  // per stage that holds any, by the thread owning the row/column, so the
  // per-cell fetch below is a plain branch-free shared-memory read:
  //   contig: the TMA box read the memory ghosts; physical sides overwrite
  //           them with the remapped interior value (negated for reflective);
  //   strided: the producer already copied the remapped rows; reflective
  //           sides negate the normal-velocity state.
  // The generic-proxy writes are fenced before the stage goes back to the
  // async proxy (the producer's next bulk copy into it).
  auto patch = [&](unsigned char* st, int k) {
    const int r0 = k * NC;
    const int jlo = lo - 2 - A + r0;
    if (CONTIG) {
      const bool any = (jlo < 0 && !halo_lo) || (jlo + NC > a.n && !halo_hi);
      if (!any) return;
#pragma unroll 1
      for (int c = 0; c < NC; ++c) {
        const int j = jlo + c;
        const bool ghost = (j < 0 && !halo_lo) || (j >= a.n && !halo_hi);
        if (!ghost || r0 + c < A) continue;
        bool neg;
        const int js = remap(j, a.n, a.bc_lo, a.bc_hi, neg);
#pragma unroll
        for (int q = 0; q < M; ++q)
          *reinterpret_cast<T*>(st + (q * kConsumers + t) * kRowStrideContig + c * (int)sizeof(T)) =
              neg_if(pin[js + q * a.sstride], neg && q == a.nv);
      }
    } else {
      const bool any = (jlo < 0 && refl_lo) || (jlo + NC > a.n && refl_hi);
      if (!any || a.nv < 0 || a.nv >= M) return;
#pragma unroll 1
      for (int c = 0; c < NC; ++c) {
        const int j = jlo + c;
        if (!((j < 0 && refl_lo) || (j >= a.n && refl_hi)) || r0 + c < A) continue;
        T* e = reinterpret_cast<T*>(st) + (a.nv * NC + c) * kConsumers + t;
        *e = -*e;
      }
    }
    fence_proxy_async_smem();
  };
  auto fetch = [&](const unsigned char* st, int c, T (&q)[M]) {
    if (!CONTIG) {
#pragma unroll
      for (int k = 0; k < M; ++k)
        q[k] = reinterpret_cast<const T*>(st)[(k * NC + c) * kConsumers + t];
    } else {
#pragma unroll
      for (int k = 0; k < M; ++k)
        q[k] = *reinterpret_cast<const T*>(st + (k * kConsumers + t) * kRowStrideContig +
                                           c * (int)sizeof(T));
    }
  };
  // emit the updated cell e = r - A - 4 of the segment (cell lo + e).  Contig
  // sweeps stage it in output tile e / NC (double-buffered) for a TMA store.
  // fold = false: the outputs are known finite (a skipped group)
  auto emit = [&](int r, bool valid, const T (&o)[M], bool fold = true) {
    if (CONTIG) {
      const int e = r - A - 4;
      unsigned char* ob = outs + ((e / NC) & 1) * G::BYTES;
#pragma unroll
      for (int q = 0; q < M; ++q)
        *reinterpret_cast<T*>(ob + (q * kConsumers + t) * kRowStrideContig +
                              (e % NC) * (int)sizeof(T)) = o[q];
      if (fold && valid && active) {
#pragma unroll
        for (int q = 0; q < M; ++q) mr.fin = min(mr.fin, finite_key(o[q]));
      }
    } else if (G::NOUT > 0 && bulk_out) {
      const int e = r - A - 4;
      T* ob = reinterpret_cast<T*>(outs + ((e / NC) & 1) * G::BYTES);
#pragma unroll
      for (int q = 0; q < M; ++q) ob[(q * NC + e % NC) * kConsumers + t] = o[q];
      if (fold && valid && active) {
#pragma unroll
        for (int q = 0; q < M; ++q) mr.fin = min(mr.fin, finite_key(o[q]));
      }
    } else if (valid && active) {
      T* dst = pout + (int64_t)(lo + r - A - 4) * a.astride;
#pragma unroll
      for (int q = 0; q < M; ++q) {
        dst[q * a.sstride] = o[q];
        if (fold) mr.fin = min(mr.fin, finite_key(o[q]));
      }
    }
  };

  // output tile `tile` complete in smem -> one TMA tensor store per state.
  // Before the barrier, thread 0 makes sure the store of tile-2 (issued at
  // the previous flush or earlier) has finished reading the buffer tile+1
  // is about to be written into.
  int flushed = -1;
  auto flush = [&](int tile) {
    fence_proxy_async_smem();
    if (t == 0) bulk_wait_read<0>();
    named_barrier_sync(1, kConsumers);
    if (t == 0) {
      const unsigned char* ob = outs + (tile & 1) * G::BYTES;
      if (CONTIG) {
        const int cx = a.tx0 + lo + tile * NC;
        const int cy = a.ty0 + (int)pb, cz = a.tz0 + (int)blockIdx.z;
#pragma unroll
        for (int q = 0; q < M; ++q)
          tma_store_4d(map_st, ob + q * kConsumers * kRowStrideContig, cx, cy, cz, q);
      } else {
        // strided: each output row of the tile is nvalid contiguous cells
        const uint32_t rowbytes = (uint32_t)nvalid * (uint32_t)sizeof(T);
        T* base = L.qout + pb + (int64_t)blockIdx.z * a.t2stride;
        for (int c = 0; c < NC; ++c) {
          const int e = tile * NC + c;
          if (lo + e >= hi) break;
#pragma unroll
          for (int q = 0; q < M; ++q)
            bulk_s2g(base + (int64_t)(lo + e) * a.astride + q * a.sstride,
                     ob + ((q * NC + c) * kConsumers) * (int)sizeof(T), rowbytes);
        }
      }
      bulk_commit();
    }
    flushed = tile;
  };

  for (int k = 0; k < nst; ++k) {
    const int kk = k0 + k;
    const int s = kk % NSTAGE;
    // inline producer: issue every stage whose slot is already free (a
    // non-blocking probe of its empty barrier), and block only for stage k
    // itself -- thread 0 never waits for the other warps just to prefetch
    if (kInlineProducer && t == 0) {
      while (issued < nst && issued < k + NSTAGE) {
        const int kq = k0 + issued;
        if (issued > k && kq >= NSTAGE &&
            !mbar_test_wait(&empty[kq % NSTAGE], ((kq / NSTAGE) - 1) & 1))
          break;
        produce(issued++);
      }
    }
    mbar_wait(&full[s], (kk / NSTAGE) & 1);
    unsigned char* st = smem + s * G::BYTES;
    patch(st, k);
#pragma unroll 1
    for (int g = 0; g < NC / 3; ++g) {
      const int r0 = k * NC + 3 * g;
      if (r0 >= ncell) break;
      const int c0 = 3 * g;
      T q[M];
      if (r0 >= A + 4) {
        if (decltype(mr)::kSkip && mr.check_due()) {
          T q1[M], q2[M];
          fetch(st, c0, q);
          fetch(st, c0 + 1, q1);
          fetch(st, c0 + 2, q2);
          if (mr.template skip_group<2>(q, q1, q2)) {
            // (finite: a skip needs a finite fan, so no finiteness fold)
            emit(r0, r0 < ncell, q, false);
            emit(r0 + 1, r0 + 1 < ncell, q1, false);
            emit(r0 + 2, r0 + 2 < ncell, q2, false);
            if ((CONTIG || (G::NOUT > 0 && bulk_out)) && (r0 + 2 - A - 4) % NC == NC - 1)
              flush((r0 + 2 - A - 4) / NC);
            continue;
          }
          mr.uni = false;
        }
        if constexpr (has_xs<T, S>()) ++nact;
        T o[M];
        bool v;
        v = r0 < ncell;
        fetch(st, c0, q);
        mr.template step<0>(q, a, v && active, o);
        emit(r0, v, o);
        v = r0 + 1 < ncell;
        fetch(st, c0 + 1, q);
        mr.template step<1>(q, a, v && active, o);
        emit(r0 + 1, v, o);
        v = r0 + 2 < ncell;
        fetch(st, c0 + 2, q);
        mr.template step<2>(q, a, v && active, o);
        emit(r0 + 2, v, o);
        // the group's last cell closes an output tile every NC cells
        if ((CONTIG || (G::NOUT > 0 && bulk_out)) && (r0 + 2 - A - 4) % NC == NC - 1)
          flush((r0 + 2 - A - 4) / NC);
      } else if (r0 == A + 1) {
        fetch(st, c0, q);
        mr.template fan<0>(q, a, active);          // F(lo-1)
        fetch(st, c0 + 1, q);
        mr.template fan<1>(q, a, active);          // F(lo)
        fetch(st, c0 + 2, q);
        mr.template fan_corr<2>(q, a, active);     // F(lo+1), G(lo)
      } else if (r0 == A - 2) {
        fetch(st, c0 + 2, q);
        mr.template first<2>(q);                   // cell lo-2
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (CONTIG || (G::NOUT > 0 && bulk_out)) {
    const int last = (ncell - 1 - A - 4) / NC;  // tile of the segment's last cell
    if (last > flushed) flush(last);
    if (t == 0) bulk_wait<0>();
  }
  if constexpr (!CONTIG && has_xs<T, S>())
    if (a.act && lane == 0 && nact) atomicAdd(a.act, (unsigned long long)nact);
  smax = mr.smax;
  fin = mr.fin;
  bad = mr.bad && active;
}

// ---------------------------------------------------------------------------
// The contiguous-axis (x) pass, TMA transpose with sector-aligned boxes.
//
// A stage is a box of NC = 64 B / itemsize cells of each of the CTA's 128 rows
// per state (64-byte rows: whole 32-byte sectors, so the DRAM traffic is the
// algorithmic traffic), written by the TMA engine with the 64-byte swizzle
// (row t's 16-byte chunks XOR (t >> 1) & 3: two-way instead of four-way bank
// conflicts when thread t reads row t).  Stage k of a segment [lo, hi) holds
// cells lo - NC + k*NC .. lo - 1 + k*NC: stage 0 the prologue (its last four
// cells lo-2 .. lo+1 straddle into stage 1), stage k >= 1 exactly the output
// cells of tile k-1, so every output is written IN PLACE over its own input
// cell (read two steps earlier by the same thread) and each stage >= 1 goes
// back to global memory as one TMA store of the same box.  A stage's ring slot
// is released to the producer when that store has finished reading it.
#ifndef CLB_DIAG_NOSTORE
#define CLB_DIAG_NOSTORE 0
#endif
#if defined(CLB_DEFAULT_LIB) && CLB_DIAG_NOSTORE
#error "CLB_DIAG_NOSTORE is timing-only and not allowed in the default library"
#endif
#ifndef CLB_X_NSTAGE
#define CLB_X_NSTAGE 0   // 0: from CLB_X_BUDGET
#endif
#ifndef CLB_X_ROW
#define CLB_X_ROW 64    // box row bytes of the x stages for m <= 3 states (32, 64, 128)
#endif

#ifndef CLB_X_ROW4
#define CLB_X_ROW4 32   // box row bytes of the x stages for m >= 4 states (32 or 64)
#endif
#ifndef CLB_X_BUDGET
#define CLB_X_BUDGET 0   // stage-ring bytes; 0: the share of the resident CTAs
#endif
// box row bytes of the x stages (host side: clb_capi.cu make_tensor_map)
__host__ __device__ constexpr int x_row_bytes(int m, int xs = 0) {
  return xs ? CLB_XS_ROW : (m >= 4 ? CLB_X_ROW4 : CLB_X_ROW);
}
// cells per stage (x_row_bytes per box, SUB boxes side by side)
__host__ __device__ constexpr int x_stage_bytes(int m, int xs = 0) {
  return x_row_bytes(m, xs) * (xs ? CLB_XS_SUB : 1);
}
template <typename T, class S, int XS = 0> struct XGeom {
  static constexpr int ROWS = x_rows<XS>();             // rows (consumer threads) per CTA
  static constexpr int ROW = x_row_bytes(S::M, XS);     // bytes per row per state and box
  static constexpr int SUB = XS ? CLB_XS_SUB : 1;       // boxes per state and stage
  static constexpr int NCS = ROW / (int)sizeof(T);      // cells per box
  static constexpr int NC = SUB * NCS;                  // cells per stage
  static constexpr int SUBB = ROWS * ROW;               // one box
  static constexpr int SBYTES = SUB * SUBB;             // one state of a stage
  static constexpr int BYTES = S::M * SBYTES;
  // as many stages as the ring budget holds (in-place outputs need >= 3)
  // the resident CTAs' share of the 228 KB (less static + reserved memory)
  static constexpr int BUDGET =
      CLB_X_BUDGET > 0 ? CLB_X_BUDGET : (228 * 1024) / kMinBlocks<T, S, true, XS>() - 3 * 1024;
  static constexpr int NSTAGE_RAW = CLB_X_NSTAGE > 0 ? CLB_X_NSTAGE : BUDGET / BYTES;
  static constexpr int NSTAGE = NSTAGE_RAW < 3 ? 3 : (NSTAGE_RAW > 8 ? 8 : NSTAGE_RAW);
  static constexpr int SMEM = NSTAGE * BYTES + 2 * NSTAGE * 8 + 1024;  // + 1024-B alignment slack
};

template <typename T, class S, int LIM, bool LIT, class D, int XS>
__device__ __forceinline__ void segment_pass_x(const SweepArgs<T>& a, const Live<T>& L,
                                               const TmaMaps& maps_all, unsigned char* ring,
                                               uint64_t* full, uint64_t* empty, int k0,
                                               T& smax, uint32_t& fin, bool& bad) {
  using G = XGeom<T, S, XS>;
  constexpr int NC = G::NC, NSTAGE = G::NSTAGE, M = S::M;
  constexpr int isz = (int)sizeof(T);
  const unsigned char* map_ld = maps_all.ld[L.src];
  const unsigned char* map_st = maps_all.st[L.dst];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int seg = blockIdx.y + a.seg_base;
  const int lo = seg * a.seg_len;
  const int hi = min(a.n, lo + a.seg_len);
  const int len = hi - lo;
  const int nr = len + NC + 2;                 // positions: cells lo-NC .. hi+1
  const int nst = (nr + NC - 1) / NC;
  const int nout = (len + NC - 1) / NC;        // output stages 1 .. nout
  const int64_t pb = (int64_t)blockIdx.x * G::ROWS;
  const int nvalid = (int)(a.n1 - pb < (int64_t)G::ROWS ? a.n1 - pb : (int64_t)G::ROWS);
  const int cy = a.ty0 + (int)pb, cz = a.tz0 + (int)blockIdx.z;
  auto slot = [&](int k) { return (k0 + k) % NSTAGE; };
  auto stage_ptr = [&](int k) { return ring + slot(k) * G::BYTES; };

  auto produce = [&](int k) {
    const int kk = k0 + k;
    const int s = kk % NSTAGE;
    if (kk >= NSTAGE) mbar_wait_sleep(&empty[s], ((kk / NSTAGE) - 1) & 1);
    mbar_arrive_expect_tx(&full[s], (uint32_t)G::BYTES);
    const int cx = a.tx0 + lo - NC + k * NC;
#pragma unroll
    for (int q = 0; q < M; ++q)
#pragma unroll
      for (int u = 0; u < G::SUB; ++u)
        tma_load_4d(ring + s * G::BYTES + q * G::SBYTES + u * G::SUBB, map_ld, cx + u * G::NCS,
                    cy, cz, q, &full[s]);
  };
  if (!kInlineX && warp == G::ROWS / 32) {
    if (lane == 0)
      for (int k = 0; k < nst; ++k) produce(k);
    return;
  }
  if (kInlineX && tid == 0)
    for (int k = 0; k < min(nst, NSTAGE); ++k) produce(k);
  // releases: stage k's slot goes back to the producer exactly once per pass
  int released = 0;                             // stages 0 .. released-1 are released
  auto release_upto = [&](int k) {              // thread 0 only
    for (; released < k; ++released) {
      mbar_arrive(&empty[slot(released)]);
      if (kInlineX && released + NSTAGE < nst) produce(released + NSTAGE);
    }
  };

  // ------------------------------ consumers ------------------------------
  const int t = tid;
  const bool active = t < nvalid;
  const bool halo_lo = a.bc_lo == BC_HALO, halo_hi = a.bc_hi == BC_HALO;
  // swizzled byte offset of (row t, cell c) inside one state's box
  const int rowb = t * G::ROW;
  // 64-byte swizzle: 16-byte chunk ^= (offset >> 7) & 3, i.e. (t >> 1) & 3;
  // 32-byte swizzle: chunk ^= (offset >> 7) & 1, i.e. (t >> 2) & 1
  // (128-byte rows, 128-byte swizzle: chunk ^= t & 7)
  const int xr = G::ROW == 128 ? (t & 7) << 4
                 : G::ROW == 64 ? ((t >> 1) & 3) << 4 : ((t >> 2) & 1) << 4;
  auto cell_off = [&](int c) {
    return (c / G::NCS) * G::SUBB + rowb + (((c % G::NCS) * isz) ^ xr);
  };

  March<T, S, LIM, LIT, D> mr;
  mr.smax = T(0);
  mr.fin = 0xffffffffu;
  mr.bad = false;
  mr.idle = !active;
  mr.uni = false;
  mr.run = 0;
  mr.cool = 0;
  mr.back = 0;
  mr.dtdx = L.dtdx;
  const T* pin = L.qin + (pb + (active ? t : 0)) * a.t1stride + (int64_t)blockIdx.z * a.t2stride;

  // wait for stage k and fix up its physical-boundary ghosts (boundary.py
  // semantics): the box read the memory ghosts, which are overwritten with
  // the remapped interior value (negated for a reflective wall)
  auto enter = [&](int k) {
    mbar_wait(&full[slot(k)], ((k0 + k) / NSTAGE) & 1);
    const int jlo = lo - NC + k * NC;
    const bool any = (jlo < 0 && !halo_lo) || (jlo + NC > a.n && !halo_hi);
    if (!any) return;
    unsigned char* st = stage_ptr(k);
#pragma unroll 1
    for (int c = 0; c < NC; ++c) {
      const int j = jlo + c;
      const bool ghost = (j < 0 && j >= -2 && !halo_lo) || (j >= a.n && j <= a.n + 1 && !halo_hi);
      if (!ghost) continue;
      bool neg;
      const int js = remap(j, a.n, a.bc_lo, a.bc_hi, neg);
#pragma unroll
      for (int q = 0; q < M; ++q)
        *reinterpret_cast<T*>(st + q * G::SBYTES + cell_off(c)) =
            neg_if(pin[js + q * a.sstride], neg && q == a.nv);
    }
    fence_proxy_async_smem();
  };
  // the entered stage and the one before it (a fetch or an output is never
  // older: outputs lag the inputs by two positions)
  int entered = -1;
  unsigned char* cur_st = ring;
  unsigned char* prev_st = ring;
  auto at = [&](int pos) {
    return ((pos / NC) == entered ? cur_st : prev_st) + cell_off(pos & (NC - 1));
  };
  auto fetch = [&](int r, T (&q)[M]) {
    const unsigned char* st = at(r);
#pragma unroll
    for (int k = 0; k < M; ++k) q[k] = *reinterpret_cast<const T*>(st + k * G::SBYTES);
  };
  // output cell e (position NC + e) in place; flush a completed tile
  auto flush = [&](int k) {                     // stage k >= 1 holds tile k-1
    fence_proxy_async_smem();
    named_barrier_sync(1, G::ROWS);
    if (t == 0) {
      const unsigned char* st = stage_ptr(k);
      const int cx = a.tx0 + lo + (k - 1) * NC;
      if (!CLB_DIAG_NOSTORE) {  // timing experiments only: outputs discarded
#pragma unroll
        for (int q = 0; q < M; ++q)
#pragma unroll
          for (int u = 0; u < G::SUB; ++u)
            tma_store_4d(map_st, st + q * G::SBYTES + u * G::SUBB, cx + u * G::NCS, cy, cz, q);
      }
      bulk_commit();
      // every stage before k is consumed; the store of k-1 has read its slot
      // once at most this newest group is still reading
      bulk_wait_read<1>();
      release_upto(k);
    }
  };
  auto emit = [&](int e, const T (&o)[M]) {
    if (e < 0 || e >= len) return;              // (warp-uniform: e is)
    unsigned char* st = at(NC + e);
    // a state no wave touches leaves the update as its input bits (update():
    // out = q), which the in-place slot already holds
#pragma unroll
    for (int q = 0; q < M; ++q)
      if (LIT || !allzero<S>(q)) *reinterpret_cast<T*>(st + q * G::SBYTES) = o[q];
    if (active) {
#pragma unroll
      for (int q = 0; q < M; ++q) mr.fin = min(mr.fin, finite_key(o[q]));
    }
    if (e % NC == NC - 1 || e == len - 1) flush(1 + e / NC);
  };
  // a skipped group's outputs equal its inputs, which already sit in the
  // output slots (in place: slot NC + e still holds cell e's input, equal to
  // the uniform state) and are finite (a skip needs a finite fan, and a
  // non-finite state makes its fans non-finite): nothing to write
  auto emit_same = [&](int e) {
    if (e < 0 || e >= len) return;
    if (e % NC == NC - 1 || e == len - 1) flush(1 + e / NC);
  };
  // stage transitions happen at positions r % NC == 0 (warp-uniform)
  auto need = [&](int r) {
    const int k = r / NC;
    if (k > entered) {
      enter(k);
      entered = k;
      prev_st = cur_st;
      cur_st = stage_ptr(k);
    }
  };

  // prologue: cells lo-2 .. lo+1 at positions NC-2 .. NC+1
  constexpr int PF = (NC - 2) % 3;            // ring phase of position NC-2
  {
    T q[M];
    need(0);
    fetch(NC - 2, q);
    mr.template first<PF>(q);
    fetch(NC - 1, q);
    mr.template fan<(PF + 1) % 3>(q, a, active);
    need(NC);
    fetch(NC, q);
    mr.template fan<(PF + 2) % 3>(q, a, active);
    fetch(NC + 1, q);
    mr.template fan_corr<PF>(q, a, active);
  }
  // steady: position r emits cell e = r - NC - 2, phases (P0, P0+1, P0+2)
  constexpr int P0 = (PF + 1) % 3;
#pragma unroll 1
  for (int r = NC + 2; r < nr; r += 3) {
    const bool v1 = r + 1 < nr, v2 = r + 2 < nr;
    T q[M];
    if constexpr (decltype(mr)::kSkip) {
      if (v2 && mr.check_due()) {
        T q1[M], q2[M];
        need(r);
        fetch(r, q);
        need(r + 1);
        fetch(r + 1, q1);
        need(r + 2);
        fetch(r + 2, q2);
        if (mr.template skip_group<(P0 + 2) % 3>(q, q1, q2)) {
          emit_same(r - NC - 2);
          emit_same(r - NC - 1);
          emit_same(r - NC);
          continue;
        }
        mr.uni = false;
      }
    }
    T o[M];
    need(r);
    fetch(r, q);
    mr.template step<P0>(q, a, active, o);
    emit(r - NC - 2, o);
    if (!v1) break;
    need(r + 1);
    fetch(r + 1, q);
    mr.template step<(P0 + 1) % 3>(q, a, active, o);
    emit(r - NC - 1, o);
    if (!v2) break;
    need(r + 2);
    fetch(r + 2, q);
    mr.template step<(P0 + 2) % 3>(q, a, active, o);
    emit(r - NC, o);
  }
  // every slot of the pass goes back once; the stores have completed before
  // the next pass (or the kernel) ends
  named_barrier_sync(1, G::ROWS);
  if (t == 0) {
    bulk_wait<0>();
    release_upto(nst);
  }
  smax = mr.smax;
  fin = mr.fin;
  bad = mr.bad && active;
  (void)nout;
}

// Number of stages one segment pass streams (same formula as segment_pass).
template <typename T, class S, bool CONTIG>
__device__ __forceinline__ int segment_stages(const SweepArgs<T>& a) {
  using G = StageGeom<T, S, CONTIG>;
  const int lo = (blockIdx.y + a.seg_base) * a.seg_len;
  const int hi = min(a.n, lo + a.seg_len);
  return (hi - lo + G::A + 4 + G::NC - 1) / G::NC;
}

// ---------------------------------------------------------------------------
// The sweep kernel.  Relative cell index r = 0 .. L+A+3 of a segment [lo, hi)
// maps to pencil cell j = lo - 2 - A + r: r < A are alignment dummies, r =
// A..A+3 the prologue (cells lo-2 .. lo+1), r >= A+4 emits cell lo + r - A - 4.
//
// Pass 1 marches with FastArith (branch-free IEEE division / square root).
// If any consumer left the fast-path domain (zero/NaN depths, denormal-scale
// data, overflow), the whole CTA runs pass 2 over the same segment with
// ExactArith: it rewrites every output of the segment (same threads, or the
// same TMA-issuing thread after bulk_wait), and its (smax, fin) replace pass
// 1's.  Literal (blow-up) kernels run one ExactArith pass.
template <typename T, class S, int LIM, bool LIT, bool CONTIG, int XS = 0>
__global__ void __launch_bounds__(threads_of<CONTIG, XS>(), kMinBlocks<T, S, CONTIG, XS>())
    sweep_kernel(const SweepArgs<T> a, const __grid_constant__ TmaMaps maps) {
  // x geometry pair: only the twin the previous strided sweep's activity
  // selects does the work (every CTA reads the same count: it is reset after
  // both x launches and accumulated by the next strided sweep)
  if (CONTIG && a.xsel && ((*(volatile const unsigned long long*)a.xsel < a.xsel_thresh) != (XS == 1)))
    return;
  Live<T> L;
  if (!resolve_live(a, L)) return;
  constexpr bool XNEW = CONTIG && !CLB_X_LEGACY;
  using G = StageGeom<T, S, CONTIG>;
  using XG = XGeom<T, S, XS>;
  constexpr int NSTAGE = XNEW ? XG::NSTAGE : G::NSTAGE;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // the swizzled x stages need 1024-byte aligned buffers
  unsigned char* smem = XNEW ? smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u)
                             : smem_raw;
  uint64_t* full = reinterpret_cast<uint64_t*>(
      smem + (XNEW ? NSTAGE * XG::BYTES : (NSTAGE + G::NOUT) * G::BYTES));
  uint64_t* empty = full + NSTAGE;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      // x stages are released by one thread after their store read them
      mbar_init(&empty[s], XNEW ? 1 : kConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  T smax = T(0);
  uint32_t fin = 0xffffffffu;
  bool bad = false;
  auto pass = [&](auto arith, int k0) {
    using D = decltype(arith);
    if constexpr (XNEW)
      segment_pass_x<T, S, LIM, LIT, D, XS>(a, L, maps, smem, full, empty, k0, smax, fin, bad);
    else
      segment_pass<T, S, LIM, LIT, CONTIG, D>(a, L, maps, smem, full, empty, k0, smax, fin, bad);
  };
  auto stages = [&]() {
    if constexpr (XNEW) {
      const int lo = (blockIdx.y + a.seg_base) * a.seg_len;
      const int len = min(a.n, lo + a.seg_len) - lo;
      constexpr int NC = XG::NC;
      return (len + NC + 2 + NC - 1) / NC;
    } else {
      return segment_stages<T, S, CONTIG>(a);
    }
  };
  // fp32 shallow water: the exact fp32 division (zero numerators short-cut)
  // beats the fp64-pipe fast path (8 divisions per cell; y 0.99 vs 1.33 ms at
  // 8192^2); acoustics' two limiter divisions meet tiny far-field waves that
  // send div.rn.f32 to its slow path, so it keeps the fast path (1.09 vs 1.35)
  if (LIT || (sizeof(T) == 4 && (S::NW >= 3 || CLB_EXACT32))) {
    pass(ExactArith{}, 0);
  } else {
    pass(FastArith{}, 0);
    // CLB_NO_REDO: timing experiments only (results may differ from div.rn)
    if (__syncthreads_or(bad) && !CLB_NO_REDO) {
      smax = T(0);
      fin = 0xffffffffu;
      pass(ExactArith{}, stages());
    }
  }
  finish_block<T>(smax, fin, a);
}

// ---------------------------------------------------------------------------
// Axis 0 (x, unit stride) -- warp-marching variant.  A warp marches along one
// row in 32-cell chunks, lane l owning cell b+l; interface fans, correction
// fluxes and cell updates trail each other by one and two lanes and are
// handed over with __shfl_sync (the two lanes that cross a chunk boundary
// take their neighbours from a per-warp shared-memory carry slot).  Loads
// and stores are fully coalesced.
#ifdef CLB_PLAIN_LD
template <typename T> __device__ __forceinline__ T ld_nc(const T* p) { return *p; }
#else
template <typename T> __device__ __forceinline__ T ld_nc(const T* p) { return __ldg(p); }
#endif

template <typename T, int M>
__device__ __forceinline__ void load_cell(const T* base, int64_t sstride, int64_t astride, int j,
                                          const SweepArgs<T>& a, T (&q)[M]) {
  bool neg;
  const int js = remap(j, a.n, a.bc_lo, a.bc_hi, neg);
  const T* p = base + (int64_t)js * astride;
#pragma unroll
  for (int k = 0; k < M; ++k) q[k] = neg_if(ld_nc(p + k * sstride), neg && k == a.nv);
}

template <typename T, class S> struct CarryLayout {
  static constexpr int kCell = (int)(sizeof(typename S::Cell) / sizeof(T));
  static constexpr int kFan = (int)(sizeof(typename S::Fan) / sizeof(T));
  static constexpr int kAll = kCell + kFan + S::M;
};

// One 32-cell chunk of the warp-marching x sweep under arithmetic policy D:
// lane l owns cell x = b + l.  Pure: reads the loaded cell and the warp's
// carry slots, writes only (c, F, G, o).  In a row's first chunk lanes 0-1
// keep their shuffled (real but unrelated) neighbours instead of the
// not-yet-written carry; their results are never used, and real data cannot
// fake a slow-path flag.
template <typename T, class S, bool LIT, class D>
__device__ __forceinline__ void contig_chunk(
    const SweepArgs<T>& a, T dtdx, int lim_id, const T (&q)[S::M], bool first, int lane,
    T (&carry)[2][CarryLayout<T, S>::kAll], typename S::Cell& c, typename S::Fan& F,
    T (&G)[S::M], T (&o)[S::M], bool& bad) {
  using Cell = typename S::Cell;
  using Fan = typename S::Fan;
  constexpr int M = S::M;
  constexpr int KC = CarryLayout<T, S>::kCell, KF = CarryLayout<T, S>::kFan;
  c = S::template make<D>(q, bad);
  Cell cl = c;
  S::for_cell_regs(cl, [&](T& r) { r = __shfl_sync(FULL, r, (lane + 31) & 31); });
  if (lane == 0 && !first) {
    int i = 0;
    S::for_cell_regs(cl, [&](T& r) { r = carry[1][i++]; });
  }
  F = S::template solve<D>(cl, c, a.P, bad);
  Fan F1 = F, F2 = F;
  S::for_regs(F1, [&](T& r) { r = __shfl_sync(FULL, r, (lane + 31) & 31); });
  S::for_regs(F2, [&](T& r) { r = __shfl_sync(FULL, r, (lane + 30) & 31); });
  if (lane == 0 && !first) {
    int i = KC;
    S::for_regs(F1, [&](T& r) { r = carry[1][i++]; });
  }
  if (lane < 2 && !first) {
    int i = KC;
    S::for_regs(F2, [&](T& r) { r = carry[lane][i++]; });
  }
  correction<S, LIT, D, T>(F2, F1, F, a.P, dtdx, lim_id, G, bad);
  T G1[M], q2[M];
#pragma unroll
  for (int k = 0; k < M; ++k) {
    G1[k] = __shfl_sync(FULL, G[k], (lane + 31) & 31);
    q2[k] = __shfl_sync(FULL, c.q[k], (lane + 30) & 31);
  }
  if (lane == 0 && !first) {
#pragma unroll
    for (int k = 0; k < M; ++k) G1[k] = carry[1][KC + KF + k];
  }
  if (lane < 2 && !first) {
#pragma unroll
    for (int k = 0; k < M; ++k) q2[k] = carry[lane][k];  // Cell starts with q[M]
  }
  update<S, LIT, T>(q2, F2, F1, G, G1, a.P, dtdx, o);
}

// ---------------------------------------------------------------------------
// Axis 0 (contiguous): warp-marching kernel.
template <typename T, class S, int LIM, bool LIT>
__global__ void __launch_bounds__(128, CLB_CONTIG_MINB) sweep_contig(const SweepArgs<T> a) {
  Live<T> L;
  if (!resolve_live(a, L)) return;
  const int lim_id = LIM >= 0 ? LIM : a.lim_id;
  using Cell = typename S::Cell;
  using Fan = typename S::Fan;
  constexpr int M = S::M;
  constexpr int KC = CarryLayout<T, S>::kCell, KF = CarryLayout<T, S>::kFan;
  constexpr int KA = CarryLayout<T, S>::kAll;
  __shared__ T carry[4][2][KA];
  // per-warp double buffer of the next chunk's cells (cp.async, no registers)
  constexpr int kDepth = CLB_CONTIG_DEPTH;  // chunks in flight ahead of the march
  __shared__ T stage[4][kDepth + 1][M][32];

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nrows = (int64_t)a.n1 * a.n2;
  const int64_t row = gw / a.nseg;
  const int seg = (int)(gw - row * a.nseg);

  T smax = T(0);
  uint32_t fin = 0xffffffffu;
  if (row < nrows) {
    const int y = (int)(row % a.n1);
    const int z = (int)(row / a.n1);
    const int64_t off = (int64_t)y * a.t1stride + (int64_t)z * a.t2stride;
    const T* qrow = L.qin + off;
    T* orow = L.qout + off;
    const int lo = seg * a.seg_len;
    const int hi = min(a.n, lo + a.seg_len);

    // chunk cells stream through shared memory with per-thread async copies,
    // one chunk ahead; the ghost remap is applied at issue, the reflective
    // negation at read
    auto issue = [&](int bb, int buf) {
      // chunks clear of both ends need no ghost remap (warp-uniform test)
      int js = min(bb + lane, hi + 1);
      if (!(bb >= 0 && bb + 31 < a.n)) {
        bool neg;
        js = remap(js, a.n, a.bc_lo, a.bc_hi, neg);
      }
      const T* p = qrow + js;
#pragma unroll
      for (int k = 0; k < M; ++k) cp_async<(int)sizeof(T)>(&stage[wib][buf][k][lane], p + k * a.sstride);
      cp_async_commit();
    };
    // prologue: chunks 0 .. kDepth-1 in flight (empty groups past the end
    // keep the group count uniform)
#pragma unroll
    for (int d = 0; d < kDepth; ++d) {
      if (lo - 2 + 32 * d <= hi + 1) issue(lo - 2 + 32 * d, d);
      else cp_async_commit();
    }
    int cur = 0;
    for (int b = lo - 2; b <= hi + 1; b += 32) {
      const int x = b + lane;
      const bool first = b == lo - 2;
      {
        const int nb = b + 32 * kDepth;
        const int slot = (cur + kDepth) % (kDepth + 1);
        if (nb <= hi + 1) issue(nb, slot);
        else cp_async_commit();
        cp_async_wait<kDepth>();
      }
      bool negq = false;
      if (!(b >= 0 && b + 31 < a.n)) remap(min(x, hi + 1), a.n, a.bc_lo, a.bc_hi, negq);
      T q[M];
#pragma unroll
      for (int k = 0; k < M; ++k) q[k] = neg_if(stage[wib][cur][k][lane], negq && k == a.nv);
      cur = cur == kDepth ? 0 : cur + 1;
      Cell c;
      Fan F;
      T G[M], o[M];
      bool bad = false;
      // fp32: the exact branchy division (zero numerators short-cut) measured
      // faster in this kernel than the fp64-pipe fast path
      if (LIT || (sizeof(T) == 4 && !CLB_CONTIG_FAST32)) {
        contig_chunk<T, S, LIT, ExactArith>(a, L.dtdx, lim_id, q, first, lane, carry[wib], c, F, G,
                                            o, bad);
      } else {
        // branch-free IEEE arithmetic; a chunk in which any lane left the
        // fast-path domain is recomputed exactly (its inputs -- loaded cells
        // and the carry -- are untouched until the commit below)
        contig_chunk<T, S, LIT, FastArith>(a, L.dtdx, lim_id, q, first, lane, carry[wib], c, F, G,
                                           o, bad);
        if (__any_sync(FULL, bad)) {
          bad = false;
          contig_chunk<T, S, LIT, ExactArith>(a, L.dtdx, lim_id, q, first, lane, carry[wib], c, F,
                                              G, o, bad);
        }
      }
      // commit: max |s|, outputs, carry
      if (x >= lo - 1 && x <= hi + 1) fold_speed<S, T>(F, a.P, smax);
      if (x >= lo + 2 && x <= hi + 1) {
        T* dst = orow + (x - 2);
#pragma unroll
        for (int k = 0; k < M; ++k) {
          dst[k * a.sstride] = o[k];
          fin = min(fin, finite_key(o[k]));
        }
      }
      __syncwarp();
      if (lane >= 30) {
        T* slot = carry[wib][lane - 30];
        int i = 0;
        S::for_cell_regs(c, [&](T& r) { slot[i++] = r; });
        S::for_regs(F, [&](T& r) { slot[i++] = r; });
#pragma unroll
        for (int k = 0; k < M; ++k) slot[KC + KF + k] = G[k];
      }
      __syncwarp();
    }
  }
  finish_block<T>(smax, fin, a);
}

// ---------------------------------------------------------------------------
// Axis 0 (contiguous): pair warp-march.  A warp marches along one row in
// 64-cell chunks, lane l owning cells x0 = b + 2l and x1 = x0 + 1.  Per lane
// and chunk: the fans F(x0) (left neighbour = lane l-1's second cell) and
// F(x1), the corrections G(x0-1) and G(x0), and the updates of cells x0-2
// and x0-1 (lane l-1's pair).  Lane l-1's second cell, its two fans and its
// G(x0-2) arrive by __shfl_up (lane 0 from the previous chunk's lane 31
// through a per-warp shared-memory carry), and the two output cells' states
// are read from the staged chunk: half the shuffles per cell of
// sweep_contig.  Loads: the next chunk streams into a per-warp shared buffer
// with per-thread cp.async (two consecutive cells per lane per state).
template <typename T, class S> struct PairCarry {
  static constexpr int kCell = (int)(sizeof(typename S::Cell) / sizeof(T));
  static constexpr int kFan = (int)(sizeof(typename S::Fan) / sizeof(T));
  // cell c1, fans Fa, Fb, correction Ga, states q0, q1 of the last lane
  static constexpr int kAll = kCell + 2 * kFan + 3 * S::M;
};

template <typename T, class S, bool LIT, class D>
__device__ __forceinline__ void pair_chunk(const SweepArgs<T>& a, T dtdx, int lim_id,
                                           const T (&q0)[S::M], const T (&q1)[S::M],
                                           bool first, int lane, const T* carry,
                                           typename S::Fan& Fa, typename S::Fan& Fb,
                                           typename S::Cell& c1, T (&Ga)[S::M],
                                           T (&oA)[S::M], T (&oB)[S::M],
                                           const T (&pq0)[S::M], const T (&pq1)[S::M],
                                           bool& bad) {
  using Cell = typename S::Cell;
  using Fan = typename S::Fan;
  constexpr int M = S::M;
  constexpr int KC = PairCarry<T, S>::kCell, KF = PairCarry<T, S>::kFan;
  const Cell c0 = S::template make<D>(q0, bad);
  c1 = S::template make<D>(q1, bad);
  const bool from_carry = lane == 0 && !first;
  Cell cL = c1;
  S::for_cell_regs(cL, [&](T& r) { r = __shfl_up_sync(FULL, r, 1); });
  if (from_carry) {
    int i = 0;
    S::for_cell_regs(cL, [&](T& r) { r = carry[i++]; });
  }
  Fa = S::template solve<D>(cL, c0, a.P, bad);     // F(x0)
  Fb = S::template solve<D>(c0, c1, a.P, bad);     // F(x1)
  Fan Fpa = Fa, Fpb = Fb;                          // lane l-1's F(x0-2), F(x0-1)
  S::for_regs(Fpa, [&](T& r) { r = __shfl_up_sync(FULL, r, 1); });
  S::for_regs(Fpb, [&](T& r) { r = __shfl_up_sync(FULL, r, 1); });
  if (from_carry) {
    int i = KC;
    S::for_regs(Fpa, [&](T& r) { r = carry[i++]; });
    S::for_regs(Fpb, [&](T& r) { r = carry[i++]; });
  }
  T Gm[M];
  correction<S, LIT, D, T>(Fpa, Fpb, Fa, a.P, dtdx, lim_id, Gm, bad);   // G(x0-1)
  correction<S, LIT, D, T>(Fpb, Fa, Fb, a.P, dtdx, lim_id, Ga, bad);    // G(x0)
  T Gl[M];                                                              // G(x0-2)
#pragma unroll
  for (int k = 0; k < M; ++k) Gl[k] = __shfl_up_sync(FULL, Ga[k], 1);
  if (from_carry) {
#pragma unroll
    for (int k = 0; k < M; ++k) Gl[k] = carry[KC + 2 * KF + k];
  }
  update<S, LIT, T>(pq0, Fpa, Fpb, Gm, Gl, a.P, dtdx, oA);   // cell x0-2
  update<S, LIT, T>(pq1, Fpb, Fa, Ga, Gm, a.P, dtdx, oB);    // cell x0-1
}

// every wave component of the fan is +-0 and every register finite
template <class S, class Fan> __device__ __forceinline__ bool pair_zero_fan(Fan f) {
  uint32_t key = 0xffffffffu;
  bool zero = true;
  S::for_regs(f, [&](auto& r) { key = min(key, finite_key(r)); });
#pragma unroll
  for (int p = 0; p < S::NW; ++p) {
#pragma unroll
    for (int k = 0; k < S::M; ++k) {
      if (S::nz(p, k)) {
        const auto w = S::wave(f, p, k);
        zero = zero && (w == decltype(w)(0));
      }
    }
  }
  return zero && key != 0u;
}

#ifndef CLB_PAIR_MINB
#define CLB_PAIR_MINB 2
#endif
template <typename T, class S, int LIM, bool LIT>
__global__ void __launch_bounds__(128, CLB_PAIR_MINB) sweep_pair(const SweepArgs<T> a) {
  Live<T> L;
  if (!resolve_live(a, L)) return;
  const int lim_id = LIM >= 0 ? LIM : a.lim_id;
  using Cell = typename S::Cell;
  using Fan = typename S::Fan;
  constexpr int M = S::M;
  constexpr int KC = PairCarry<T, S>::kCell, KF = PairCarry<T, S>::kFan;
  constexpr int KA = PairCarry<T, S>::kAll;
  __shared__ T carry[4][KA];
  // per warp: the chunk being marched and the next one (64 cells per state)
  __shared__ T stage[4][2][M][64];

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nrows = (int64_t)a.n1 * a.n2;
  const int64_t row = gw / a.nseg;
  const int seg = (int)(gw - row * a.nseg);

  T smax = T(0);
  uint32_t fin = 0xffffffffu;
  if (row < nrows) {
    const int y = (int)(row % a.n1);
    const int z = (int)(row / a.n1);
    const int64_t off = (int64_t)y * a.t1stride + (int64_t)z * a.t2stride;
    const T* qrow = L.qin + off;
    T* orow = L.qout + off;
    const int lo = seg * a.seg_len;
    const int hi = min(a.n, lo + a.seg_len);
    // chunk cells b .. b+63 (cells past hi+1 are never used); ghosts remapped
    // at issue, the reflective negation applied at read
    auto issue = [&](int bb, int buf) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int x = bb + 2 * lane + h;
        int js = min(x, hi + 1);
        if (!(bb >= 0 && bb + 63 < a.n)) {
          bool neg;
          js = remap(js, a.n, a.bc_lo, a.bc_hi, neg);
        }
        const T* p = qrow + js;
#pragma unroll
        for (int k = 0; k < M; ++k)
          cp_async<(int)sizeof(T)>(&stage[wib][buf][k][2 * lane + h], p + k * a.sstride);
      }
      cp_async_commit();
    };
    auto read = [&](int bb, int buf, int idx, T (&q)[M]) {
      bool neg = false;
      if (!(bb >= 0 && bb + 63 < a.n)) remap(min(bb + idx, hi + 1), a.n, a.bc_lo, a.bc_hi, neg);
#pragma unroll
      for (int k = 0; k < M; ++k) q[k] = neg_if(stage[wib][buf][k][idx], neg && k == a.nv);
    };
    const int b0 = lo - 4;
    issue(b0, 0);
    int cur = 0;
    bool uni_pair = false;  // the carry holds a uniform state (warp-uniform)
    for (int b = b0; b - 2 < hi; b += 64) {
      const bool first = b == b0;
      if (b + 64 - 2 < hi) issue(b + 64, cur ^ 1);
      else cp_async_commit();
      cp_async_wait<1>();
      __syncwarp();
      const int x0 = b + 2 * lane;
      T q0[M], q1[M], pq0[M], pq1[M];
      read(b, cur, 2 * lane, q0);
      read(b, cur, 2 * lane + 1, q1);
      // the two output cells (lane l-1's pair): the staged chunk, or the
      // carry for lane 0
      if (lane > 0) {
        read(b, cur, 2 * lane - 2, pq0);
        read(b, cur, 2 * lane - 1, pq1);
      } else {
#pragma unroll
        for (int k = 0; k < M; ++k) {
          pq0[k] = carry[wib][KC + 2 * KF + M + k];
          pq1[k] = carry[wib][KC + 2 * KF + 2 * M + k];
        }
      }
      // Uniform-state skip (exact; see March): when every cell of the chunk
      // equals the carried cells b-2, b-1 and the carried fans F(b-2), F(b-1)
      // are finite with only +-0 waves, every fan of the chunk is that same
      // self-fan, every correction +0, and every output its input: the chunk
      // only streams.  The carry becomes uniform (F(b+62) = F(b+63) = the
      // self-fan, G = +0), so following uniform chunks check the cells alone.
      if constexpr (!LIT && S::kUniformSkip) {
        if (!first) {
          const T* cs = carry[wib];
          T u[M];
#pragma unroll
          for (int k = 0; k < M; ++k) u[k] = cs[KC + 2 * KF + 2 * M + k];  // cell b-1
          bool eq = same_bits<T, M>(q0, u) && same_bits<T, M>(q1, u);
          if (!uni_pair) {
            T u0[M];
#pragma unroll
            for (int k = 0; k < M; ++k) u0[k] = cs[KC + 2 * KF + M + k];     // cell b-2
            Fan ca, cb;
            int i = KC;
            S::for_regs(ca, [&](T& r) { r = cs[i++]; });
            S::for_regs(cb, [&](T& r) { r = cs[i++]; });
            eq = eq && same_bits<T, M>(u0, u) && pair_zero_fan<S>(ca) && pair_zero_fan<S>(cb);
          }
          if (__all_sync(FULL, eq)) {
            if (!uni_pair) {
              __syncwarp();
              if (lane == 31) {
                T* slot = carry[wib];
                for (int i = 0; i < KF; ++i) slot[KC + i] = slot[KC + KF + i];  // Fa := Fb
                for (int k = 0; k < M; ++k) slot[KC + 2 * KF + k] = T(0);       // G := +0
              }
              __syncwarp();
              uni_pair = true;
            }
            // outputs = inputs (finite: a finite self-fan needs a finite state)
            if (x0 - 2 >= lo && x0 - 2 < hi) {
#pragma unroll
              for (int k = 0; k < M; ++k) orow[(x0 - 2) + k * a.sstride] = u[k];
            }
            if (x0 - 1 >= lo && x0 - 1 < hi) {
#pragma unroll
              for (int k = 0; k < M; ++k) orow[(x0 - 1) + k * a.sstride] = u[k];
            }
            __syncwarp();
            cur ^= 1;
            continue;
          }
        }
        uni_pair = false;
      }
      Fan Fa, Fb;
      Cell c1;
      T Ga[M], oA[M], oB[M];
      bool bad = false;
      if (LIT || (sizeof(T) == 4 && !CLB_CONTIG_FAST32)) {
        pair_chunk<T, S, LIT, ExactArith>(a, L.dtdx, lim_id, q0, q1, first, lane, carry[wib], Fa,
                                          Fb, c1, Ga, oA, oB, pq0, pq1, bad);
      } else {
        pair_chunk<T, S, LIT, FastArith>(a, L.dtdx, lim_id, q0, q1, first, lane, carry[wib], Fa,
                                         Fb, c1, Ga, oA, oB, pq0, pq1, bad);
        // the chunk is a pure function of its loads and the carry: recompute
        // it exactly when a real lane left the fast-path domain
        if (__any_sync(FULL, bad && x0 >= lo - 2 && x0 <= hi + 1)) {
          bad = false;
          pair_chunk<T, S, LIT, ExactArith>(a, L.dtdx, lim_id, q0, q1, first, lane, carry[wib],
                                            Fa, Fb, c1, Ga, oA, oB, pq0, pq1, bad);
        }
      }
      // commit: max |s| of the fans in [lo-1, hi+1], the outputs in [lo, hi)
      if (x0 >= lo - 1 && x0 <= hi + 1) fold_speed<S, T>(Fa, a.P, smax);
      if (x0 + 1 >= lo - 1 && x0 + 1 <= hi + 1) fold_speed<S, T>(Fb, a.P, smax);
      if (x0 - 2 >= lo && x0 - 2 < hi) {
        T* dst = orow + (x0 - 2);
#pragma unroll
        for (int k = 0; k < M; ++k) {
          dst[k * a.sstride] = oA[k];
          fin = min(fin, finite_key(oA[k]));
        }
      }
      if (x0 - 1 >= lo && x0 - 1 < hi) {
        T* dst = orow + (x0 - 1);
#pragma unroll
        for (int k = 0; k < M; ++k) {
          dst[k * a.sstride] = oB[k];
          fin = min(fin, finite_key(oB[k]));
        }
      }
      __syncwarp();
      if (lane == 31) {
        T* slot = carry[wib];
        int i = 0;
        S::for_cell_regs(c1, [&](T& r) { slot[i++] = r; });
        S::for_regs(Fa, [&](T& r) { slot[i++] = r; });
        S::for_regs(Fb, [&](T& r) { slot[i++] = r; });
#pragma unroll
        for (int k = 0; k < M; ++k) {
          slot[KC + 2 * KF + k] = Ga[k];
          slot[KC + 2 * KF + M + k] = q0[k];
          slot[KC + 2 * KF + 2 * M + k] = q1[k];
        }
      }
      __syncwarp();
      cur ^= 1;
    }
  }
  finish_block<T>(smax, fin, a);
}

// ---------------------------------------------------------------------------
// Per-interface solve for the Riemann-plugin parity unit (riemann.py:205-223).
template <typename T, class S>
__global__ void solve_pairs(const T* ql, const T* qr, T* W, T* s, int64_t n, Params<T> P) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  constexpr int M = S::M;
  T a[M], b[M];
#pragma unroll
  for (int k = 0; k < M; ++k) { a[k] = ql[i * M + k]; b[k] = qr[i * M + k]; }
  bool bad = false;
  typename S::Cell L = S::template make<ExactArith>(a, bad), R = S::template make<ExactArith>(b, bad);
  typename S::Fan f = S::template solve<ExactArith>(L, R, P, bad);
#pragma unroll
  for (int p = 0; p < S::NW; ++p) {
    s[i * S::NW + p] = S::speed(f, P, p);
#pragma unroll
    for (int k = 0; k < M; ++k) W[(i * S::NW + p) * M + k] = S::wave(f, p, k);
  }
}

// ---------------------------------------------------------------------------
// Launch plumbing shared by the instantiation units.

struct GenericArgs {
  const TmaMaps* maps;  // all three buffers' maps (contig TMA sweep only)
  int src, dst;
  const DevCtl* ctl;    // indirect launch (batch graphs)
  int axis;
  double spacing;
  const void* bufs[3];
  int tx0, ty0, tz0;
  const void* qin;
  void* qout;
  int64_t sstride, astride, t1stride, t2stride;
  int n, n1, n2;
  int bc_lo, bc_hi, nv, lim_id;
  double dtdx;        // already rounded to T by the host
  double params[4];   // already rounded to T by the host
  unsigned long long* smax_bits;
  int* nonfinite;
  int contig;         // 1: axis-0 (x) sweep, warp-marching; 2: axis 0, TMA transpose
  int seg_len, nseg;
  int seg_begin, seg_end;  // segment range of this launch (strided kernels)
  int num_sms;
  int* occ_out;            // non-null: report resident CTAs per SM instead of launching
  int fuse_ctl;
  Result* res;
  int xs;                  // 1: the streaming x geometry (XS = 1 twin)
  const unsigned long long* xsel;
  unsigned long long xsel_thresh;
  unsigned long long* act;
};

template <typename T>
inline SweepArgs<T> to_args(const GenericArgs& g) {
  SweepArgs<T> a;
  a.qin = (const T*)g.qin;
  a.qout = (T*)g.qout;
  a.sstride = g.sstride; a.astride = g.astride; a.t1stride = g.t1stride; a.t2stride = g.t2stride;
  a.n = g.n; a.n1 = g.n1; a.n2 = g.n2;
  a.seg_len = g.seg_len; a.nseg = g.nseg;
  a.seg_base = g.seg_begin;
  a.bc_lo = g.bc_lo; a.bc_hi = g.bc_hi; a.nv = g.nv; a.lim_id = g.lim_id;
  a.dtdx = (T)g.dtdx;
  for (int i = 0; i < 4; ++i) a.P.p[i] = (T)g.params[i];
  a.smax_bits = g.smax_bits;
  a.nonfinite = g.nonfinite;
  a.tx0 = g.tx0; a.ty0 = g.ty0; a.tz0 = g.tz0;
  a.src = g.src; a.dst = g.dst;
  a.ctl = g.ctl;
  a.axis = g.axis;
  a.spacing = g.spacing;
  for (int i = 0; i < 3; ++i) a.bufs[i] = g.bufs[i];
  a.fuse_ctl = g.fuse_ctl;
  a.res = g.res;
  a.xsel = g.xsel;
  a.xsel_thresh = g.xsel_thresh;
  a.act = g.act;
  return a;
}

template <typename T, class S, int LIM, bool LIT>
inline cudaError_t launch_contig_shfl(const GenericArgs& g, cudaStream_t st) {
  if (g.occ_out)
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(g.occ_out, sweep_contig<T, S, LIM, LIT>,
                                                         128, 0);
  SweepArgs<T> a = to_args<T>(g);
  const int64_t warps = (int64_t)g.n1 * g.n2 * g.nseg;
  const int64_t blocks = (warps + 3) / 4;
  sweep_contig<T, S, LIM, LIT><<<(unsigned)blocks, 128, 0, st>>>(a);
  return cudaGetLastError();
}

template <typename T, class S, int LIM, bool LIT>
inline cudaError_t launch_pair(const GenericArgs& g, cudaStream_t st) {
  if (g.occ_out)
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(g.occ_out, sweep_pair<T, S, LIM, LIT>,
                                                         128, 0);
  SweepArgs<T> a = to_args<T>(g);
  const int64_t warps = (int64_t)g.n1 * g.n2 * g.nseg;
  const int64_t blocks = (warps + 3) / 4;
  sweep_pair<T, S, LIM, LIT><<<(unsigned)blocks, 128, 0, st>>>(a);
  return cudaGetLastError();
}

template <typename T, class S, int LIM, bool LIT, bool CONTIG, int XS = 0>
inline cudaError_t launch_kernel(const GenericArgs& g, cudaStream_t st) {
  if (CONTIG && g.contig == 1) return launch_contig_shfl<T, S, LIM, LIT>(g, st);
  if (CONTIG && g.contig == 3) return launch_pair<T, S, LIM, LIT>(g, st);
  constexpr int kSmem = (CONTIG && !CLB_X_LEGACY) ? XGeom<T, S, XS>::SMEM
                                                   : StageGeom<T, S, CONTIG>::SMEM;
  // the dynamic shared-memory opt-in is per device: one bit per device
  // ordinal, set once (atomically: service threads may launch concurrently)
  static std::atomic<unsigned long long> configured{0ull};
  auto fn = sweep_kernel<T, S, LIM, LIT, CONTIG, XS>;
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit, std::memory_order_release);
  }
  if (g.occ_out) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(g.occ_out, fn,
                                                                      threads_of<CONTIG, XS>(),
                                                                      kSmem);
  SweepArgs<T> a = to_args<T>(g);
  static const TmaMaps none{};
  constexpr int rows = (CONTIG && !CLB_X_LEGACY) ? x_rows<XS>() : kConsumers;
  dim3 grid((unsigned)((g.n1 + rows - 1) / rows), (unsigned)(g.seg_end - g.seg_begin),
            (unsigned)g.n2);
  fn<<<grid, threads_of<CONTIG, XS>(), kSmem, st>>>(a, CONTIG ? *g.maps : none);
  return cudaGetLastError();
}

template <typename T, class S, bool CONTIG>
inline cudaError_t launch_lim(const GenericArgs& g, bool literal, cudaStream_t st) {
  if (literal) return launch_kernel<T, S, -1, true, CONTIG>(g, st);
  if constexpr (CONTIG && has_xs<T, S>()) {
    if (g.xs) {
      switch (g.lim_id) {
        case 0: return launch_kernel<T, S, 0, false, true, 1>(g, st);
        case 1: return launch_kernel<T, S, 1, false, true, 1>(g, st);
        case 2: return launch_kernel<T, S, 2, false, true, 1>(g, st);
        case 3: return launch_kernel<T, S, 3, false, true, 1>(g, st);
        default: return launch_kernel<T, S, 4, false, true, 1>(g, st);
      }
    }
  }
  if (g.xs) return cudaErrorInvalidValue;
  switch (g.lim_id) {
    case 0: return launch_kernel<T, S, 0, false, CONTIG>(g, st);
    case 1: return launch_kernel<T, S, 1, false, CONTIG>(g, st);
    case 2: return launch_kernel<T, S, 2, false, CONTIG>(g, st);
    case 3: return launch_kernel<T, S, 3, false, CONTIG>(g, st);
    default: return launch_kernel<T, S, 4, false, CONTIG>(g, st);
  }
}

template <typename T, class S>
inline cudaError_t launch_solver(const GenericArgs& g, bool literal, cudaStream_t st) {
  return g.contig ? launch_lim<T, S, true>(g, literal, st) : launch_lim<T, S, false>(g, literal, st);
}

template <typename T, class S>
inline cudaError_t launch_pairs(const void* ql, const void* qr, void* W, void* s, int64_t n,
                                const double* params, cudaStream_t st) {
  Params<T> P;
  for (int i = 0; i < 4; ++i) P.p[i] = (T)params[i];
  const int64_t blocks = (n + 127) / 128;
  if (blocks > 0)
    solve_pairs<T, S><<<(unsigned)blocks, 128, 0, st>>>((const T*)ql, (const T*)qr, (T*)W, (T*)s,
                                                        n, P);
  return cudaGetLastError();
}

// Entry points defined by the instantiation units (one object per solver
// family and dtype).
#define CLB_DECLARE_FAMILY(fam)                                                               \
  cudaError_t launch_##fam##_f32(int ndim, int axis, bool lit, const GenericArgs& g,          \
                                 cudaStream_t st);                                             \
  cudaError_t launch_##fam##_f64(int ndim, int axis, bool lit, const GenericArgs& g,          \
                                 cudaStream_t st);                                             \
  cudaError_t pairs_##fam##_f32(int ndim, int axis, const void* ql, const void* qr, void* W,  \
                                void* s, int64_t n, const double* p, cudaStream_t st);        \
  cudaError_t pairs_##fam##_f64(int ndim, int axis, const void* ql, const void* qr, void* W,  \
                                void* s, int64_t n, const double* p, cudaStream_t st);
CLB_DECLARE_FAMILY(acoustics)
CLB_DECLARE_FAMILY(shallow_water)
CLB_DECLARE_FAMILY(advection)
CLB_DECLARE_FAMILY(vc_acoustics)
#undef CLB_DECLARE_FAMILY
cudaError_t pairs_dispatch(int solver, int itemsize, int ndim, int axis, const void* ql,
                           const void* qr, void* W, void* s, int64_t n, const double* params,
                           cudaStream_t st);

}  // namespace clb
