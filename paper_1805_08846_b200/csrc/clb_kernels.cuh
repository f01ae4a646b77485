// clb_kernels.cuh -- the fused directional sweep kernels for sm_100a.
//
// One kernel launch == one directional sweep of the reference
// (sweep.py:307-377 sweep_axis_tiled over sweep.py:183-263 sweep_tile),
// with the ghost-cell fill of boundary.py:87-122 fused in as an index remap
// at load time, the per-sweep max |s| folded by warp shuffle + block
// reduction + one guarded atomicMax, and the non-finite check of
// timestep.py:179-186 folded into the store epilogue on the integer pipe.
//
// Two thread mappings, both reading and writing each cell once per segment
// with fully coalesced 128-byte transactions:
//
//  * sweep_contig (axis 0, x, unit stride): a warp marches along one row
//    in 32-cell chunks, lane l owning cell b+l.  Interface fans, correction
//    fluxes and cell updates trail each other by one and two lanes, handed
//    over with __shfl_sync; the two lanes that cross a chunk boundary take
//    their neighbours from a per-warp shared-memory carry slot.
//
//  * sweep_strided (axes 1, 2): one thread per x column marches along the
//    sweep axis with a three-fan register ring (the reference's ring,
//    sweep.py:195-200) and a one-cell register prefetch; a warp covers 32
//    consecutive x, so every load/store is one coalesced row segment.
//
// Rows/columns are split into segments along the sweep axis; each segment
// recomputes the 3 fans it shares with its neighbour exactly as the
// reference's tiles do (sweep.py:11-16), so results are bitwise independent
// of the segmentation.
#pragma once
#include "clb_solvers.cuh"

namespace clb {

enum { BC_OUTFLOW = 0, BC_REFLECTIVE = 1, BC_PERIODIC = 2, BC_HALO = 3 };

constexpr unsigned FULL = 0xffffffffu;

template <typename T> struct SweepArgs {
  const T* qin;     // element (0,0,0) of state 0 (interior origin)
  T* qout;
  int64_t sstride;  // elements between states
  int64_t astride;  // element stride along the sweep axis
  int64_t t1stride; // contig: row stride of transverse axis 1 (y); strided: 1 (x)
  int64_t t2stride; // remaining transverse axis
  int n;            // cells along the sweep axis
  int n1, n2;       // transverse extents
  int seg_len, nseg;
  int bc_lo, bc_hi, nv;
  int lim_id;
  T dtdx;
  Params<T> P;
  unsigned long long* smax_bits;
  int* nonfinite;
};

// boundary.py:108-122 as a read-side index map: ghost cell j of a pencil
// reads interior cell remap(j), negating state nv for reflective walls.
__device__ __forceinline__ int remap(int j, int n, int lo, int hi, bool& neg) {
  neg = false;
  if (j < 0) {
    if (lo == BC_OUTFLOW) return 0;
    if (lo == BC_PERIODIC) return n + j;
    if (lo == BC_REFLECTIVE) { neg = true; return -1 - j; }
    return j;  // halo rows live in memory
  }
  if (j >= n) {
    if (hi == BC_OUTFLOW) return n - 1;
    if (hi == BC_PERIODIC) return j - n;
    if (hi == BC_REFLECTIVE) { neg = true; return 2 * n - 1 - j; }
    return j;
  }
  return j;
}

template <typename T> __device__ __forceinline__ T ld_nc(const T* p) { return __ldg(p); }

template <typename T, int M>
__device__ __forceinline__ void load_cell(const T* base, int64_t sstride, int64_t astride, int j,
                                          const SweepArgs<T>& a, T (&q)[M]) {
  bool neg;
  const int js = remap(j, a.n, a.bc_lo, a.bc_hi, neg);
  const T* p = base + (int64_t)js * astride;
#pragma unroll
  for (int k = 0; k < M; ++k) q[k] = ld_nc(p + k * sstride);
  if (neg) {
#pragma unroll
    for (int k = 0; k < M; ++k)
      if (k == a.nv) q[k] = -q[k];
  }
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
  }
}

template <typename T, class S> struct CarryLayout {
  static constexpr int kCell = (int)(sizeof(typename S::Cell) / sizeof(T));
  static constexpr int kFan = (int)(sizeof(typename S::Fan) / sizeof(T));
  static constexpr int kAll = kCell + kFan + S::M;
};

// ---------------------------------------------------------------------------
// Axis 0 (contiguous): warp-marching kernel.
template <typename T, class S, bool LIT>
__global__ void __launch_bounds__(128) sweep_contig(const SweepArgs<T> a) {
  using Cell = typename S::Cell;
  using Fan = typename S::Fan;
  constexpr int M = S::M;
  constexpr int KC = CarryLayout<T, S>::kCell, KF = CarryLayout<T, S>::kFan;
  constexpr int KA = CarryLayout<T, S>::kAll;
  __shared__ T carry[4][2][KA];

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
    const T* qrow = a.qin + off;
    T* orow = a.qout + off;
    const int lo = seg * a.seg_len;
    const int hi = min(a.n, lo + a.seg_len);

    for (int b = lo - 2; b <= hi + 1; b += 32) {
      const int x = b + lane;
      T q[M];
      load_cell<T, M>(qrow, a.sstride, 1, min(x, hi + 1), a, q);
      Cell c = S::make(q);

      // left neighbour cell (x-1)
      Cell cl = c;
      S::for_cell_regs(cl, [&](T& r) { r = __shfl_sync(FULL, r, (lane + 31) & 31); });
      if (lane == 0) {
        int i = 0;
        S::for_cell_regs(cl, [&](T& r) { r = carry[wib][1][i++]; });
      }
      Fan F = S::solve(cl, c, a.P);
      if (x >= lo - 1 && x <= hi + 1) fold_speed<S, T>(F, a.P, smax);

      Fan F1 = F, F2 = F;
      S::for_regs(F1, [&](T& r) { r = __shfl_sync(FULL, r, (lane + 31) & 31); });
      S::for_regs(F2, [&](T& r) { r = __shfl_sync(FULL, r, (lane + 30) & 31); });
      if (lane == 0) {
        int i = KC;
        S::for_regs(F1, [&](T& r) { r = carry[wib][1][i++]; });
      }
      if (lane < 2) {
        int i = KC;
        S::for_regs(F2, [&](T& r) { r = carry[wib][lane][i++]; });
      }
      T G[M];
      correction<S, LIT, T>(F2, F1, F, a.P, a.dtdx, a.lim_id, G);
      T G1[M], q2[M];
#pragma unroll
      for (int k = 0; k < M; ++k) {
        G1[k] = __shfl_sync(FULL, G[k], (lane + 31) & 31);
        q2[k] = __shfl_sync(FULL, c.q[k], (lane + 30) & 31);
      }
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < M; ++k) G1[k] = carry[wib][1][KC + KF + k];
      }
      if (lane < 2) {
#pragma unroll
        for (int k = 0; k < M; ++k) q2[k] = carry[wib][lane][k];  // Cell starts with q[M]
      }
      if (x >= lo + 2 && x <= hi + 1) {
        T o[M];
        update<S, LIT, T>(q2, F2, F1, G, G1, a.P, a.dtdx, o);
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
// Axes 1 and 2 (strided): thread-per-column marching kernel.
template <typename T, class S, bool LIT>
__global__ void __launch_bounds__(128) sweep_strided(const SweepArgs<T> a) {
  using Cell = typename S::Cell;
  using Fan = typename S::Fan;
  constexpr int M = S::M;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int seg = blockIdx.y;
  const int t2 = blockIdx.z;

  T smax = T(0);
  uint32_t fin = 0xffffffffu;
  if (x < a.n1) {
    const int64_t off = (int64_t)x * a.t1stride + (int64_t)t2 * a.t2stride;
    const T* qc = a.qin + off;
    T* oc = a.qout + off;
    const int lo = seg * a.seg_len;
    const int hi = min(a.n, lo + a.seg_len);
    const int64_t as = a.astride;

    T qa[M];
    load_cell<T, M>(qc, a.sstride, as, lo - 2, a, qa);
    Cell cm1 = S::make(qa);
    load_cell<T, M>(qc, a.sstride, as, lo - 1, a, qa);
    Cell c0 = S::make(qa);
    Fan Fm2 = S::solve(cm1, c0, a.P);  // F(lo-1)
    fold_speed<S, T>(Fm2, a.P, smax);
    load_cell<T, M>(qc, a.sstride, as, lo, a, qa);
    Cell c1 = S::make(qa);
    Fan Fm1 = S::solve(c0, c1, a.P);   // F(lo)
    fold_speed<S, T>(Fm1, a.P, smax);
    load_cell<T, M>(qc, a.sstride, as, lo + 1, a, qa);
    Cell c2 = S::make(qa);
    Fan F = S::solve(c1, c2, a.P);     // F(lo+1)
    fold_speed<S, T>(F, a.P, smax);
    T ftp[M];
    correction<S, LIT, T>(Fm2, Fm1, F, a.P, a.dtdx, a.lim_id, ftp);  // G(lo)
    Fm2 = Fm1;
    Fm1 = F;
    T qm2[M];
#pragma unroll
    for (int k = 0; k < M; ++k) qm2[k] = c1.q[k];
    Cell cm = c2;

    T qn[M];
    load_cell<T, M>(qc, a.sstride, as, min(lo + 2, hi + 1), a, qn);
    for (int i = lo + 2; i <= hi + 1; ++i) {
      T qcur[M];
#pragma unroll
      for (int k = 0; k < M; ++k) qcur[k] = qn[k];
      load_cell<T, M>(qc, a.sstride, as, min(i + 1, hi + 1), a, qn);
      Cell ci = S::make(qcur);
      Fan Fi = S::solve(cm, ci, a.P);
      fold_speed<S, T>(Fi, a.P, smax);
      T ftn[M];
      correction<S, LIT, T>(Fm2, Fm1, Fi, a.P, a.dtdx, a.lim_id, ftn);
      T o[M];
      update<S, LIT, T>(qm2, Fm2, Fm1, ftn, ftp, a.P, a.dtdx, o);
      T* dst = oc + (int64_t)(i - 2) * as;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        dst[k * a.sstride] = o[k];
        fin = min(fin, finite_key(o[k]));
        ftp[k] = ftn[k];
        qm2[k] = cm.q[k];
      }
      Fm2 = Fm1;
      Fm1 = Fi;
      cm = ci;
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
  typename S::Cell L = S::make(a), R = S::make(b);
  typename S::Fan f = S::solve(L, R, P);
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
  const void* qin;
  void* qout;
  int64_t sstride, astride, t1stride, t2stride;
  int n, n1, n2;
  int bc_lo, bc_hi, nv, lim_id;
  double dtdx;        // already rounded to T by the host
  double params[4];   // already rounded to T by the host
  unsigned long long* smax_bits;
  int* nonfinite;
  int contig;         // 1: axis 0 kernel
  int seg_len, nseg;
  int block;          // threads per block
  int num_sms;
};

template <typename T>
inline SweepArgs<T> to_args(const GenericArgs& g) {
  SweepArgs<T> a;
  a.qin = (const T*)g.qin;
  a.qout = (T*)g.qout;
  a.sstride = g.sstride; a.astride = g.astride; a.t1stride = g.t1stride; a.t2stride = g.t2stride;
  a.n = g.n; a.n1 = g.n1; a.n2 = g.n2;
  a.seg_len = g.seg_len; a.nseg = g.nseg;
  a.bc_lo = g.bc_lo; a.bc_hi = g.bc_hi; a.nv = g.nv; a.lim_id = g.lim_id;
  a.dtdx = (T)g.dtdx;
  for (int i = 0; i < 4; ++i) a.P.p[i] = (T)g.params[i];
  a.smax_bits = g.smax_bits;
  a.nonfinite = g.nonfinite;
  return a;
}

template <typename T, class S, bool LIT>
inline cudaError_t launch_one(const GenericArgs& g, cudaStream_t st) {
  SweepArgs<T> a = to_args<T>(g);
  if (g.contig == 1) {
    const int64_t warps = (int64_t)g.n1 * g.n2 * g.nseg;
    const int64_t blocks = (warps + 3) / 4;
    sweep_contig<T, S, LIT><<<(unsigned)blocks, 128, 0, st>>>(a);
  } else {
    dim3 grid((unsigned)((g.n1 + g.block - 1) / g.block), (unsigned)g.nseg, (unsigned)g.n2);
    sweep_strided<T, S, LIT><<<grid, g.block, 0, st>>>(a);
  }
  return cudaGetLastError();
}

template <typename T, class S>
inline cudaError_t launch_solver(const GenericArgs& g, bool literal, cudaStream_t st) {
  return literal ? launch_one<T, S, true>(g, st) : launch_one<T, S, false>(g, st);
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

// Entry points defined by the instantiation units (one per solver family).
cudaError_t launch_acoustics(int itemsize, int ndim, int axis, bool lit, const GenericArgs& g,
                             cudaStream_t st);
cudaError_t launch_shallow_water(int itemsize, int ndim, int axis, bool lit,
                                 const GenericArgs& g, cudaStream_t st);
cudaError_t launch_advection(int itemsize, int ndim, int axis, bool lit, const GenericArgs& g,
                             cudaStream_t st);
cudaError_t launch_vc_acoustics(int itemsize, int ndim, int axis, bool lit,
                                const GenericArgs& g, cudaStream_t st);
cudaError_t pairs_dispatch(int solver, int itemsize, int ndim, int axis, const void* ql,
                           const void* qr, void* W, void* s, int64_t n, const double* params,
                           cudaStream_t st);

}  // namespace clb
