// Instantiations: shallow water (riemann.py:136-167), 2-D only (m = 3,
// trans = 3 - normal, riemann.py:140).
// Compiled twice by build.py: -DCLB_DTYPE=4 (float) and -DCLB_DTYPE=8 (double).
#include "clb_kernels.cuh"
#if CLB_DTYPE == 8
#define CLB_T double
#define CLB_SFX(name) name##_f64
#else
#define CLB_T float
#define CLB_SFX(name) name##_f32
#endif

namespace clb {
using T = CLB_T;

cudaError_t CLB_SFX(launch_shallow_water)(int ndim, int axis, bool lit, const GenericArgs& g,
                                          cudaStream_t st) {
  if (ndim != 2) return cudaErrorInvalidValue;
  if (axis == 0) return launch_solver<T, ShallowWater<T, 1>>(g, lit, st);
  return launch_solver<T, ShallowWater<T, 2>>(g, lit, st);
}

cudaError_t CLB_SFX(pairs_shallow_water)(int ndim, int axis, const void* ql, const void* qr,
                                         void* W, void* s, int64_t n, const double* p,
                                         cudaStream_t st) {
  (void)ndim;
  return axis == 0 ? launch_pairs<T, ShallowWater<T, 1>>(ql, qr, W, s, n, p, st)
                   : launch_pairs<T, ShallowWater<T, 2>>(ql, qr, W, s, n, p, st);
}

}  // namespace clb
