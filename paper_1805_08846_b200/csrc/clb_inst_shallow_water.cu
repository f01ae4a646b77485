// Instantiations: shallow water (riemann.py:136-167), 2-D only (m = 3,
// trans = 3 - normal, riemann.py:140).
#include "clb_kernels.cuh"

namespace clb {

template <typename T>
static cudaError_t go(int axis, bool lit, const GenericArgs& g, cudaStream_t st) {
  if (axis == 0) return launch_solver<T, ShallowWater<T, 1>>(g, lit, st);
  return launch_solver<T, ShallowWater<T, 2>>(g, lit, st);
}

cudaError_t launch_shallow_water(int itemsize, int ndim, int axis, bool lit,
                                 const GenericArgs& g, cudaStream_t st) {
  if (ndim != 2) return cudaErrorInvalidValue;
  return itemsize == 8 ? go<double>(axis, lit, g, st) : go<float>(axis, lit, g, st);
}

template <typename T>
cudaError_t pairs_shallow_water(int axis, const void* ql, const void* qr, void* W, void* s,
                                int64_t n, const double* p, cudaStream_t st) {
  return axis == 0 ? launch_pairs<T, ShallowWater<T, 1>>(ql, qr, W, s, n, p, st)
                   : launch_pairs<T, ShallowWater<T, 2>>(ql, qr, W, s, n, p, st);
}
template cudaError_t pairs_shallow_water<float>(int, const void*, const void*, void*, void*,
                                                int64_t, const double*, cudaStream_t);
template cudaError_t pairs_shallow_water<double>(int, const void*, const void*, void*, void*,
                                                 int64_t, const double*, cudaStream_t);

}  // namespace clb
