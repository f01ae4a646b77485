// Instantiations: variable-coefficient acoustics (builder extension,
// SURVEY.md 9.3), m = ndim + 3: (p, u[, v[, w]], Z, c).
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

cudaError_t CLB_SFX(launch_vc_acoustics)(int ndim, int axis, bool lit, const GenericArgs& g,
                                         cudaStream_t st) {
  if (ndim == 1) return launch_solver<T, VcAcoustics<T, 4, 1>>(g, lit, st);
  if (ndim == 2) {
    if (axis == 0) return launch_solver<T, VcAcoustics<T, 5, 1>>(g, lit, st);
    return launch_solver<T, VcAcoustics<T, 5, 2>>(g, lit, st);
  }
  if (axis == 0) return launch_solver<T, VcAcoustics<T, 6, 1>>(g, lit, st);
  if (axis == 1) return launch_solver<T, VcAcoustics<T, 6, 2>>(g, lit, st);
  return launch_solver<T, VcAcoustics<T, 6, 3>>(g, lit, st);
}

cudaError_t CLB_SFX(pairs_vc_acoustics)(int ndim, int axis, const void* ql, const void* qr,
                                        void* W, void* s, int64_t n, const double* p,
                                        cudaStream_t st) {
  if (ndim == 1) return launch_pairs<T, VcAcoustics<T, 4, 1>>(ql, qr, W, s, n, p, st);
  if (ndim == 2)
    return axis == 0 ? launch_pairs<T, VcAcoustics<T, 5, 1>>(ql, qr, W, s, n, p, st)
                     : launch_pairs<T, VcAcoustics<T, 5, 2>>(ql, qr, W, s, n, p, st);
  if (axis == 0) return launch_pairs<T, VcAcoustics<T, 6, 1>>(ql, qr, W, s, n, p, st);
  if (axis == 1) return launch_pairs<T, VcAcoustics<T, 6, 2>>(ql, qr, W, s, n, p, st);
  return launch_pairs<T, VcAcoustics<T, 6, 3>>(ql, qr, W, s, n, p, st);
}

}  // namespace clb
