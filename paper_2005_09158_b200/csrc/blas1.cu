// Deterministic BLAS-1 for the Krylov loop (classical Gram-Schmidt with one reorthogonalisation, CGS2).
//
// Fused sweeps over the basis V_0..V_{k-1} (each a scaled vector: V_i = s_i * X_i, scales on the host, so
// normalising a new basis vector costs no pass over memory):
//   dots        h_i = <X_i, w>                                      (k+1 vectors read)
//   axpy_dots   w <- a w + sum_i c_i X_i ;  h_i = <X_i, w_new>      (k+1 read, 1 written)
//   axpy_norm   w <- a w + sum_i c_i X_i ;  nrm = <w_new, w_new>    (k+1 read, 1 written)
// Fixed grid, fixed per-block ranges and fixed reduction trees: results are bitwise reproducible run to
// run (iteration-count parity, reading c16).  K is a template parameter (no predicated
// accumulators), loads are 16-byte vectors with four independent accumulator chains per thread.
#include "common.cuh"
#include "kernels.h"

namespace {

#ifndef PD_BLAS_UNROLL
#define PD_BLAS_UNROLL 2
#endif
#ifndef PD_BLAS_BLOCKS_PER_SM
#define PD_BLAS_BLOCKS_PER_SM 16  // measured: 4 -> 8 per SM cut a cfg4 sweep by 25 %, 16 ~1 % more
#endif
constexpr int kBlocks = 148 * PD_BLAS_BLOCKS_PER_SM;
constexpr int kThreads = 256;
constexpr int kMaxK = 32;

struct PtrPack {
  const double* p[kMaxK];
  double c[kMaxK];
};

PD_D double2 ld2_keep(const double* p, long long i) { return __ldg(reinterpret_cast<const double2*>(p) + i); }

// deterministic block reduction of K values per thread -> partial[blockIdx.x * K + i]
template <int K>
PD_D void block_reduce_store(double (&acc)[K], double* partial) {
  __shared__ double red[kThreads / 32][K];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    double v = acc[i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[w][i] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < K; i += kThreads) {
    double s = 0.0;
    for (int ww = 0; ww < kThreads / 32; ++ww) s += red[ww][i];
    partial[blockIdx.x * K + i] = s;
  }
}

// MODE 0: dots h_i = <X_i, y>                                 (y read only)
// MODE 1: y <- a y + sum c_i X_i, then h_i = <X_i, y_new>     (y updated)
// MODE 2: y <- a y + sum c_i X_i, then h_0 = <y_new, y_new>   (y updated; K vectors in, 1 output value)
// MODE 3: y <- sum c_i X_i                                     (y written only, no reduction)
// MODE 4: MODE 3 plus h_i = <X_i, y_new> and h_K = <y_new, y_new>
template <int K, int MODE>
// hsub / hlen (MODE 4): y_new[t] -= hsub[t] for t < hlen before the dots (the GMRES head fix w[head] -= G tail fused
// into the sweep that writes w)
__global__ void __launch_bounds__(kThreads) krylov_kernel(PtrPack X, double a, double* __restrict__ y, long long n2,
                                                          double* __restrict__ partial, const double* __restrict__ hsub,
                                                          long long hlen, long long n) {
  constexpr int NACC = (MODE == 2 || MODE == 3) ? 1 : MODE == 4 ? K + 1 : K;  // mode 4: dots + ||y_new||^2
  constexpr bool YIN = MODE <= 2;  // y is read
  // per-block contiguous range of double2 elements
  const long long per = (n2 + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * per, hi = min(n2, lo + per);
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
  // U elements per thread per trip, all loads issued before the first store (the basis pointers are not
  // __restrict__, so the compiler cannot hoist the next element's loads above a store to y); same per-thread
  // element order as U = 1, so the reductions are bitwise unchanged
  constexpr int U = K <= 8 ? PD_BLAS_UNROLL : 1;
  for (long long t0 = lo + threadIdx.x; t0 < hi; t0 += (long long)U * kThreads) {
    double2 yv[U], xv[U][K];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long t = t0 + (long long)u * kThreads;
      if (t < hi) {
        yv[u] = YIN ? reinterpret_cast<const double2*>(y)[t] : czero();
#pragma unroll
        for (int i = 0; i < K; ++i) xv[u][i] = ld2_keep(X.p[i], t);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long t = t0 + (long long)u * kThreads;
      if (t >= hi) break;
      double2 v = yv[u];
      if constexpr (MODE >= 1) {
        double2 nv = MODE >= 3 ? czero() : make_double2(a * v.x, a * v.y);
#pragma unroll
        for (int i = 0; i < K; ++i) {
          nv.x = fma(X.c[i], xv[u][i].x, nv.x);
          nv.y = fma(X.c[i], xv[u][i].y, nv.y);
        }
        if constexpr (MODE == 4) {
          if (2 * t < hlen) nv.x -= hsub[2 * t];
          if (2 * t + 1 < hlen) nv.y -= hsub[2 * t + 1];
        }
        v = nv;
        __stcs(reinterpret_cast<double2*>(y) + t, v);
      }
      if constexpr (MODE == 2) {
        acc[0] = fma(v.x, v.x, fma(v.y, v.y, acc[0]));
      } else if constexpr (MODE != 3) {
#pragma unroll
        for (int i = 0; i < K; ++i) acc[i] = fma(xv[u][i].x, v.x, fma(xv[u][i].y, v.y, acc[i]));
        if constexpr (MODE == 4) acc[NACC - 1] = fma(v.x, v.x, fma(v.y, v.y, acc[NACC - 1]));
      }
    }
  }
  // odd tail element (n odd): handled by block 0 thread 0
  if (n & 1) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const long long t = n - 1;
      double yv = YIN ? y[t] : 0.0;
      if constexpr (MODE >= 1) {
        double nv = MODE >= 3 ? 0.0 : a * yv;
#pragma unroll
        for (int i = 0; i < K; ++i) nv = fma(X.c[i], X.p[i][t], nv);
        if constexpr (MODE == 4) {
          if (t < hlen) nv -= hsub[t];
        }
        yv = nv;
        y[t] = yv;
      }
      if constexpr (MODE == 2) {
        acc[0] = fma(yv, yv, acc[0]);
      } else if constexpr (MODE != 3) {
#pragma unroll
        for (int i = 0; i < K; ++i) acc[i] = fma(X.p[i][t], yv, acc[i]);
        if constexpr (MODE == 4) acc[NACC - 1] = fma(yv, yv, acc[NACC - 1]);
      }
    }
  }
  if constexpr (MODE != 3) block_reduce_store<NACC>(acc, partial);
}

// y = a*x + b*y elementwise (used for residual copies / scaled updates)
__global__ void __launch_bounds__(kThreads) axpby_kernel(double* __restrict__ y, const double* __restrict__ x, double a,
                                                         double b, long long n) {
  for (long long t = blockIdx.x * (long long)kThreads + threadIdx.x; t < n; t += (long long)gridDim.x * kThreads)
    y[t] = b == 0.0 ? a * x[t] : fma(a, x[t], b * y[t]);
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

template <int MODE>
cudaError_t krylov_launch(const PtrPack& pk, int k, double a, double* y, long long n, double* partial, cudaStream_t st,
                          const double* hsub = nullptr, long long hlen = 0) {
  const long long n2 = n / 2;
  switch (k) {
#define PD_K(K)                                                                              \
  case K:                                                                                    \
    krylov_kernel<K, MODE><<<kBlocks, kThreads, 0, st>>>(pk, a, y, n2, partial, hsub, hlen, n); \
    break;
    PD_K(1) PD_K(2) PD_K(3) PD_K(4) PD_K(5) PD_K(6) PD_K(7) PD_K(8) PD_K(9) PD_K(10) PD_K(11) PD_K(12) PD_K(13)
    PD_K(14) PD_K(15) PD_K(16) PD_K(17) PD_K(18) PD_K(19) PD_K(20) PD_K(21) PD_K(22) PD_K(23) PD_K(24) PD_K(25)
    PD_K(26) PD_K(27) PD_K(28) PD_K(29) PD_K(30) PD_K(31) PD_K(32)
#undef PD_K
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

int pd_blas_blocks() { return kBlocks; }

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

cudaError_t pd_launch_krylov(int mode, const double* const* X, const double* coef, int k, double a, double* y,
                             long long n, double* partial, cudaStream_t st, const double* hsub, long long hlen) {
  if (k < 1 || k > kMaxK) return cudaErrorInvalidValue;
  PtrPack pk = {};
  for (int i = 0; i < k; ++i) {
    pk.p[i] = X[i];
    pk.c[i] = coef ? coef[i] : 0.0;
    if (!aligned16(X[i])) return cudaErrorMisalignedAddress;
  }
  if (!aligned16(y)) return cudaErrorMisalignedAddress;
  if (mode == 0) return krylov_launch<0>(pk, k, a, y, n, partial, st);
  if (mode == 1) return krylov_launch<1>(pk, k, a, y, n, partial, st);
  if (mode == 2) return krylov_launch<2>(pk, k, a, y, n, partial, st);
  if (mode == 4) return krylov_launch<4>(pk, k, a, y, n, partial, st, hsub, hsub ? hlen : 0);
  return krylov_launch<3>(pk, k, a, y, n, partial, st);
}

cudaError_t pd_launch_reduce_partials(const double* partial, int nblk, int k, double* out, cudaStream_t st) {
  reduce_partials_kernel<<<k, kThreads, 0, st>>>(partial, nblk, k, out);
  return cudaGetLastError();
}

cudaError_t pd_launch_axpby(double* y, const double* x, double a, double b, long long n, cudaStream_t st) {
  axpby_kernel<<<kBlocks, kThreads, 0, st>>>(y, x, a, b, n);
  return cudaGetLastError();
}
