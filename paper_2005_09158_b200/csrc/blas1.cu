// Deterministic BLAS-1 for the Krylov loop (CGS2 multi-dots, multi-axpy, norms, scaling).
// Fixed grid, fixed per-block ranges and fixed reduction trees: results are bitwise reproducible
// run to run (needed for iteration-count parity, DESIGN.md §3 reading c16).
#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int kBlocks = 148 * 4;
constexpr int kThreads = 256;
constexpr int kMaxK = 32;

struct PtrPack {
  const double* p[kMaxK];
  double c[kMaxK];
};

__global__ void __launch_bounds__(kThreads) multidot_kernel(PtrPack X, int k, const double* __restrict__ y, long long n,
                                                            double* __restrict__ partial) {
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * per, hi = min(n, lo + per);
  double acc[kMaxK];
#pragma unroll
  for (int i = 0; i < kMaxK; ++i) acc[i] = 0.0;
  for (long long t = lo + threadIdx.x; t < hi; t += kThreads) {
    const double yv = y[t];
#pragma unroll
    for (int i = 0; i < kMaxK; ++i)
      if (i < k) acc[i] = fma(X.p[i][t], yv, acc[i]);
  }
  __shared__ double red[kThreads / 32][kMaxK];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < kMaxK; ++i) {
    if (i < k) {
      double v = acc[i];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) red[w][i] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < k) {
    double s = 0.0;
    for (int ww = 0; ww < kThreads / 32; ++ww) s += red[ww][threadIdx.x];
    partial[blockIdx.x * k + threadIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kThreads) reduce_partials_kernel(const double* __restrict__ partial, int nblk, int k,
                                                                   double* __restrict__ out) {
  const int i = blockIdx.x;
  double v = 0.0;
  for (int b = threadIdx.x; b < nblk; b += kThreads) v += partial[(long long)b * k + i];
  __shared__ double red[kThreads / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    out[i] = s;
  }
}

__global__ void __launch_bounds__(kThreads) multiaxpy_kernel(double* __restrict__ y, double alpha, PtrPack X, int k,
                                                             long long n) {
  for (long long t = blockIdx.x * (long long)kThreads + threadIdx.x; t < n; t += (long long)gridDim.x * kThreads) {
    double v = alpha == 0.0 ? 0.0 : alpha * y[t];
    for (int i = 0; i < k; ++i) v = fma(X.c[i], X.p[i][t], v);
    y[t] = v;
  }
}

__global__ void scale_kernel(double* __restrict__ y, const double* __restrict__ x, double a, long long n) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    y[t] = a * x[t];
}
__global__ void axpy_kernel(double* __restrict__ y, const double* __restrict__ x, double a, long long n) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    y[t] = fma(a, x[t], y[t]);
}

}  // namespace

int pd_blas_blocks() { return kBlocks; }

cudaError_t pd_launch_multidot(const double* const* X, int k, const double* y, long long n, double* partial,
                               cudaStream_t st) {
  if (k < 1 || k > kMaxK) return cudaErrorInvalidValue;
  PtrPack pk = {};
  for (int i = 0; i < k; ++i) pk.p[i] = X[i];
  multidot_kernel<<<kBlocks, kThreads, 0, st>>>(pk, k, y, n, partial);
  return cudaGetLastError();
}

cudaError_t pd_launch_reduce_partials(const double* partial, int nblk, int k, double* out, cudaStream_t st) {
  reduce_partials_kernel<<<k, kThreads, 0, st>>>(partial, nblk, k, out);
  return cudaGetLastError();
}

cudaError_t pd_launch_multiaxpy(double* y, double alpha, const double* const* X, const double* coef, int k, long long n,
                                cudaStream_t st) {
  if (k < 0 || k > kMaxK) return cudaErrorInvalidValue;
  PtrPack pk = {};
  for (int i = 0; i < k; ++i) {
    pk.p[i] = X[i];
    pk.c[i] = coef[i];  // host coefficients
  }
  multiaxpy_kernel<<<kBlocks, kThreads, 0, st>>>(y, alpha, pk, k, n);
  return cudaGetLastError();
}

cudaError_t pd_launch_scale(double* y, const double* x, double a, long long n, cudaStream_t st) {
  scale_kernel<<<kBlocks, kThreads, 0, st>>>(y, x, a, n);
  return cudaGetLastError();
}
cudaError_t pd_launch_axpy(double* y, const double* x, double a, long long n, cudaStream_t st) {
  axpy_kernel<<<kBlocks, kThreads, 0, st>>>(y, x, a, n);
  return cudaGetLastError();
}
