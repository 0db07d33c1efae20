// device_model_example.cu — a caller-defined objective for PCAL_MODEL_DEVICE_CALLBACK
// (include/pcal_b200.h): f(X) = ½tr(XᵀAX) with the caller's own kernels, the
// device-side counterpart of subclassing orthopt::ObjectiveModel (problems.hpp:24-51).
// The callback only enqueues work on the library's stream, so the solver can
// capture it into its per-iteration CUDA graph.
#include <cuda_runtime.h>

#include <cstdint>

#include "pcal_b200.h"

namespace {

struct QuadraticCtx {
  const double* a;  // n×n column-major, device
  int64_t lda;
  double shift;     // added to every gradient entry (0: exact; the reference's
                    // PerturbedModel fault injection uses 1e-3, test_problems.cpp:27-42)
};

__global__ void k_gradient(const double* __restrict__ a, int64_t lda, const double* __restrict__ x,
                           int64_t ld, int64_t n, int64_t p, double shift, double* __restrict__ g) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * p) return;
  const int64_t i = e % n, j = e / n;
  double s = 0.0;
  for (int64_t k = 0; k < n; ++k) s = fma(a[i + k * lda], x[k + j * ld], s);
  g[i + j * ld] = s + shift;
}

__global__ void k_objective(const double* __restrict__ x, const double* __restrict__ g, int64_t ld,
                            int64_t n, int64_t p, double shift, double* f) {
  __shared__ double sm[256];
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < n * p; e += blockDim.x) s += x[e % n + (e / n) * ld] * (g[e % n + (e / n) * ld] - shift);
  sm[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *f = 0.5 * sm[0];
}

}  // namespace

extern "C" int pcal_example_quadratic_grad(const double* x, int64_t ld, int64_t n, int64_t p,
                                           double* g, double* f, void* stream, void* ctx) {
  const QuadraticCtx* c = static_cast<const QuadraticCtx*>(ctx);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_gradient<<<(unsigned)((n * p + 255) / 256), 256, 0, st>>>(c->a, c->lda, x, ld, n, p, c->shift,
                                                               g);
  k_objective<<<1, 256, 0, st>>>(x, g, ld, n, p, c->shift, f);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
