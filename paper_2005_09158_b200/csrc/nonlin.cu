// Kernels of the nonlinear ParaDiag-II (simplified Newton, eq 1.4-1.5, P:l.196-227; oracle/nonlinear.py):
//   jac_avg        dbar[x] = (1/Nt) sum_n g'(U_n(x)), g(u) = g3 u^3 + g1 u  (the averaging of P:l.214-216)
//   Step (b) with J = K + diag(dbar) (tridiagonal, not Toeplitz) is the pivoted elimination of gtsv.cu.
#include "common.cuh"
#include "kernels.h"


namespace {

// 64 nodes x 4 time quarters per CTA; each thread keeps 4 independent partial sums, the quarters are combined in a
// fixed order (deterministic)
__global__ void __launch_bounds__(256) jac_avg_kernel(const double* __restrict__ u, double* __restrict__ dbar, int nt,
                                                      long long S, double g3, double g1) {
  __shared__ double part[4][64];
  const int xl = threadIdx.x & 63, q = threadIdx.x >> 6;
  const long long x = (long long)blockIdx.x * 64 + xl;
  const int n0 = q * nt / 4, n1 = (q + 1) * nt / 4;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (x < S) {
    int n = n0;
    for (; n + 4 <= n1; n += 4) {
      const double v0 = u[(long long)n * S + x], v1 = u[(long long)(n + 1) * S + x];
      const double v2 = u[(long long)(n + 2) * S + x], v3 = u[(long long)(n + 3) * S + x];
      s0 = fma(v0, v0, s0);
      s1 = fma(v1, v1, s1);
      s2 = fma(v2, v2, s2);
      s3 = fma(v3, v3, s3);
    }
    for (; n < n1; ++n) {
      const double v = u[(long long)n * S + x];
      s0 = fma(v, v, s0);
    }
  }
  part[q][xl] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (q == 0 && x < S) dbar[x] = 3.0 * g3 * (((part[0][xl] + part[1][xl]) + (part[2][xl] + part[3][xl])) / nt) + g1;
}

}  // namespace

cudaError_t pd_launch_jac_avg(const double* u, double* dbar, int nt, long long S, double g3, double g1, cudaStream_t st) {
  jac_avg_kernel<<<(unsigned)((S + 63) / 64), 256, 0, st>>>(u, dbar, nt, S, g3, g1);
  return cudaGetLastError();
}
