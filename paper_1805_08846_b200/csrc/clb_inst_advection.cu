// Instantiations: scalar advection (riemann.py:170-173), m = 1, any ndim
// (normal_index maps every axis to state 0, riemann.py:280-284).
#include "clb_kernels.cuh"

namespace clb {

cudaError_t launch_advection(int itemsize, int, int, bool lit, const GenericArgs& g,
                             cudaStream_t st) {
  return itemsize == 8 ? launch_solver<double, Advection<double>>(g, lit, st)
                       : launch_solver<float, Advection<float>>(g, lit, st);
}

template <typename T>
cudaError_t pairs_advection(const void* ql, const void* qr, void* W, void* s, int64_t n,
                            const double* p, cudaStream_t st) {
  return launch_pairs<T, Advection<T>>(ql, qr, W, s, n, p, st);
}
template cudaError_t pairs_advection<float>(const void*, const void*, void*, void*, int64_t,
                                            const double*, cudaStream_t);
template cudaError_t pairs_advection<double>(const void*, const void*, void*, void*, int64_t,
                                             const double*, cudaStream_t);

}  // namespace clb
