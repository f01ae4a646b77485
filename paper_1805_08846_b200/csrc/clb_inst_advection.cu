// Instantiations: scalar advection (riemann.py:170-173), m = 1, any ndim
// (normal_index maps every axis to state 0, riemann.py:280-284).
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

cudaError_t CLB_SFX(launch_advection)(int, int, bool lit, const GenericArgs& g, cudaStream_t st) {
  return launch_solver<T, Advection<T>>(g, lit, st);
}

cudaError_t CLB_SFX(pairs_advection)(int, int, const void* ql, const void* qr, void* W, void* s,
                                     int64_t n, const double* p, cudaStream_t st) {
  return launch_pairs<T, Advection<T>>(ql, qr, W, s, n, p, st);
}

}  // namespace clb
