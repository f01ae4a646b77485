// Instantiations: constant-coefficient acoustics (riemann.py:116-133),
// m = ndim + 1, normal state = 1 + axis.
#include "clb_kernels.cuh"

namespace clb {

template <typename T>
static cudaError_t go(int ndim, int axis, bool lit, const GenericArgs& g, cudaStream_t st) {
  if (ndim == 1) return launch_solver<T, Acoustics<T, 2, 1>>(g, lit, st);
  if (ndim == 2) {
    if (axis == 0) return launch_solver<T, Acoustics<T, 3, 1>>(g, lit, st);
    return launch_solver<T, Acoustics<T, 3, 2>>(g, lit, st);
  }
  if (axis == 0) return launch_solver<T, Acoustics<T, 4, 1>>(g, lit, st);
  if (axis == 1) return launch_solver<T, Acoustics<T, 4, 2>>(g, lit, st);
  return launch_solver<T, Acoustics<T, 4, 3>>(g, lit, st);
}

cudaError_t launch_acoustics(int itemsize, int ndim, int axis, bool lit, const GenericArgs& g,
                             cudaStream_t st) {
  return itemsize == 8 ? go<double>(ndim, axis, lit, g, st) : go<float>(ndim, axis, lit, g, st);
}

template <typename T>
cudaError_t pairs_acoustics(int ndim, int axis, const void* ql, const void* qr, void* W, void* s,
                            int64_t n, const double* p, cudaStream_t st) {
  if (ndim == 1) return launch_pairs<T, Acoustics<T, 2, 1>>(ql, qr, W, s, n, p, st);
  if (ndim == 2)
    return axis == 0 ? launch_pairs<T, Acoustics<T, 3, 1>>(ql, qr, W, s, n, p, st)
                     : launch_pairs<T, Acoustics<T, 3, 2>>(ql, qr, W, s, n, p, st);
  if (axis == 0) return launch_pairs<T, Acoustics<T, 4, 1>>(ql, qr, W, s, n, p, st);
  if (axis == 1) return launch_pairs<T, Acoustics<T, 4, 2>>(ql, qr, W, s, n, p, st);
  return launch_pairs<T, Acoustics<T, 4, 3>>(ql, qr, W, s, n, p, st);
}
template cudaError_t pairs_acoustics<float>(int, int, const void*, const void*, void*, void*,
                                            int64_t, const double*, cudaStream_t);
template cudaError_t pairs_acoustics<double>(int, int, const void*, const void*, void*, void*,
                                             int64_t, const double*, cudaStream_t);

}  // namespace clb
