// Kernels of the nonlinear ParaDiag-II (simplified Newton, eq 1.4-1.5, P:l.196-227; oracle/nonlinear.py):
//   jac_avg        dbar[x] = (1/Nt) sum_n g'(U_n(x)), g(u) = g3 u^3 + g1 u  (the averaging of P:l.214-216)
//   thomas_shift   Step (b) with J = K + diag(dbar): lambda_1n I + lambda_2n J is tridiagonal but not Toeplitz,
//                  so the root-factorisation of tridiag.cu does not apply; a Thomas sweep per frequency (one
//                  thread each, forward elimination with the c' coefficients in a scratch row, back substitution
//                  in place).  Diagonally dominant at every shift of the configs (|lambda_1n| + lambda_2n 2nu/h^2
//                  dominates |lambda_2n| (|sub| + |sup|)); the oracle uses pivoted banded LU.
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace {

__global__ void jac_avg_kernel(const double* __restrict__ u, double* __restrict__ dbar, int nt, long long S, double g3,
                               double g1) {
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < S; x += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int n = 0; n < nt; ++n) {
      const double v = u[(long long)n * S + x];
      s = fma(3.0 * g3 * v, v, s);
    }
    dbar[x] = s / nt + g1;
  }
}

__global__ void thomas_shift_kernel(double2* __restrict__ Sh, int N, int F, const double2* __restrict__ lam1,
                                    const double2* __restrict__ lam2, double sub, double dia, double sup,
                                    const double* __restrict__ dbar, double2* __restrict__ cp) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= F) return;
  const double2 l1 = lam1[n], l2 = lam2[n];
  const double2 a = cscale(l2, sub), c = cscale(l2, sup);
  double2* d = Sh + (long long)n * N;
  double2* cr = cp + (long long)n * N;
  // forward: m_i = b_i - a c'_{i-1};  c'_i = c / m_i;  d'_i = (d_i - a d'_{i-1}) / m_i
  double2 cprev = czero(), dprev = czero();
  for (int i = 0; i < N; ++i) {
    const double2 bi = cfma(l2, make_double2(dia + __ldg(dbar + i), 0.0), l1);
    const double2 im = crcp(csub(bi, cmul(a, cprev)));
    cprev = cmul(c, im);
    dprev = cmul(csub(d[i], cmul(a, dprev)), im);
    cr[i] = cprev;
    d[i] = dprev;
  }
  // back substitution: x_{N-1} = d'_{N-1};  x_i = d'_i - c'_i x_{i+1}
  double2 xn = dprev;
  for (int i = N - 2; i >= 0; --i) {
    xn = csub(d[i], cmul(cr[i], xn));
    d[i] = xn;
  }
}

}  // namespace

cudaError_t pd_launch_jac_avg(const double* u, double* dbar, int nt, long long S, double g3, double g1, cudaStream_t st) {
  const unsigned g = (unsigned)std::min<long long>((S + 255) / 256, 148 * 8);
  jac_avg_kernel<<<g, 256, 0, st>>>(u, dbar, nt, S, g3, g1);
  return cudaGetLastError();
}

cudaError_t pd_launch_thomas_shift(double2* Sh, int nx, int nfreq, const double2* lam1, const double2* lam2, double sub,
                                   double dia, double sup, const double* dbar, double2* cp, cudaStream_t st) {
  thomas_shift_kernel<<<(nfreq + 63) / 64, 64, 0, st>>>(Sh, nx, nfreq, lam1, lam2, sub, dia, sup, dbar, cp);
  return cudaGetLastError();
}
