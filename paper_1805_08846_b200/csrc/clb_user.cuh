// clb_user.cuh -- adapter from a user scalar Riemann routine (the
// reference's plugin ABI, riemann.py:190-212: scalar(q_l, q_r, normal,
// params, W_out, s_out)) to the fused sweep kernels, and the entry points a
// run-time compiled user solver exports (paper_1805_08846_b200/devsolver.py
// generates the translation unit; include/clawb200.h
// clb_register_device_solver registers them).
//
// The user writes, in CUDA, the same arithmetic in the same order as the
// Python scalar:
//     template <typename T, int M, int NW>
//     __device__ void scalar(const T (&ql)[M], const T (&qr)[M], int normal,
//                            const T* params, T (&W)[NW][M], T (&s)[NW]);
// Every wave component is carried (no structural-zero elision) and W starts
// at +0 for each interface, so the sweep is the reference's sweep_tile
// literally; with --fmad=false and IEEE division / square root the results
// equal the reference's numba-compiled scalar bit for bit.
#pragma once
#include "clb_kernels.cuh"

namespace clb {

template <typename T, int M_, int N_, int NW_, class U> struct ScalarSolver {
  static constexpr int M = M_, NW = NW_, N = N_;
  static constexpr bool kDataSpeeds = true;
  // a user routine may return nonzero waves for equal states
  static constexpr bool kUniformSkip = false;
  static constexpr bool kSignedSpeeds = false;
  __host__ __device__ static constexpr int speed_sign(int) { return 0; }
  struct Cell { T q[M]; };
  struct Fan { T W[NW][M]; T s[NW]; };
  template <class D = ExactArith>
  __device__ __forceinline__ static Cell make(const T (&q)[M], bool&) {
    Cell c;
#pragma unroll
    for (int k = 0; k < M; ++k) c.q[k] = q[k];
    return c;
  }
  template <class D = ExactArith>
  __device__ __forceinline__ static Fan solve(const Cell& L, const Cell& R, const Params<T>& P,
                                              bool&) {
    Fan f;
#pragma unroll
    for (int p = 0; p < NW; ++p) {
      f.s[p] = T(0);
#pragma unroll
      for (int k = 0; k < M; ++k) f.W[p][k] = T(0);
    }
    U::template scalar<T, M, NW>(L.q, R.q, N, P.p, f.W, f.s);
    return f;
  }
  __device__ __forceinline__ static T speed(const Fan& f, const Params<T>&, int p) { return f.s[p]; }
  __host__ __device__ static constexpr bool nz(int, int) { return true; }
  __device__ __forceinline__ static T wave(const Fan& f, int p, int k) { return f.W[p][k]; }
  template <class F> __device__ __forceinline__ static void for_regs(Fan& f, F&& fn) {
#pragma unroll
    for (int p = 0; p < NW; ++p) {
#pragma unroll
      for (int k = 0; k < M; ++k) fn(f.W[p][k]);
      fn(f.s[p]);
    }
  }
  template <class F> __device__ __forceinline__ static void for_cell_regs(Cell& c, F&& fn) {
#pragma unroll
    for (int k = 0; k < M; ++k) fn(c.q[k]);
  }
};

// All limiters through the run-time limiter id (one kernel per x variant
// instead of five: a user solver compiles in seconds, not minutes).
template <typename T, class S>
inline cudaError_t launch_user(const GenericArgs& g, bool literal, cudaStream_t st) {
  if (g.contig)
    return literal ? launch_kernel<T, S, -1, true, true>(g, st)
                   : launch_kernel<T, S, -1, false, true>(g, st);
  return literal ? launch_kernel<T, S, -1, true, false>(g, st)
                 : launch_kernel<T, S, -1, false, false>(g, st);
}

}  // namespace clb
