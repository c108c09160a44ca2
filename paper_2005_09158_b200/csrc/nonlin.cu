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

// 32 frequencies per CTA (one warp), lane = frequency.  Rows are walked in tiles of 32: a tile of d (32 rows x 32
// frequencies) is loaded coalesced (one frequency's 32 consecutive rows per instruction) and transposed through
// shared memory, each lane runs the sequential Thomas recurrence over its frequency's 32 rows, and the tile goes
// back the same way.  c' is kept in a scratch row per frequency (tiled the same way).
constexpr int kTT = 32;
__global__ void __launch_bounds__(32) thomas_shift_kernel(double2* __restrict__ Sh, int N, int F,
                                                          const double2* __restrict__ lam1,
                                                          const double2* __restrict__ lam2, double sub, double dia,
                                                          double sup, const double* __restrict__ dbar,
                                                          double2* __restrict__ cp) {
  __shared__ double2 td[kTT][kTT + 1], tc[kTT][kTT + 1];  // [row][frequency]
  const int lane = threadIdx.x;
  const int f0 = blockIdx.x * kTT;
  const int n = f0 + lane;
  const bool on = n < F;
  const double2 l1 = on ? lam1[n] : make_double2(1.0, 0.0), l2 = on ? lam2[n] : czero();
  const double2 a = cscale(l2, sub), c = cscale(l2, sup);
  auto load_tile = [&](double2 (*t)[kTT + 1], const double2* base, int i0) {
    for (int k = 0; k < kTT; ++k) {  // frequency f0 + k, rows i0 + lane
      const bool ok = f0 + k < F && i0 + lane < N;
      t[lane][k] = ok ? base[(long long)(f0 + k) * N + i0 + lane] : czero();
    }
  };
  auto store_tile = [&](double2 (*t)[kTT + 1], double2* base, int i0) {
    for (int k = 0; k < kTT; ++k)
      if (f0 + k < F && i0 + lane < N) base[(long long)(f0 + k) * N + i0 + lane] = t[lane][k];
  };
  // forward elimination: m_i = b_i - a c'_{i-1};  c'_i = c / m_i;  d'_i = (d_i - a d'_{i-1}) / m_i
  double2 cprev = czero(), dprev = czero();
  for (int i0 = 0; i0 < N; i0 += kTT) {
    load_tile(td, Sh, i0);
    __syncwarp();
    const int iend = min(kTT, N - i0);
    for (int r = 0; r < iend; ++r) {
      const double2 bi = cfma(l2, make_double2(dia + __ldg(dbar + i0 + r), 0.0), l1);
      const double2 im = crcp_fast(csub(bi, cmul(a, cprev)));
      cprev = cmul(c, im);
      dprev = cmul(csub(td[r][lane], cmul(a, dprev)), im);
      tc[r][lane] = cprev;
      td[r][lane] = dprev;
    }
    __syncwarp();
    store_tile(td, Sh, i0);
    store_tile(tc, cp, i0);
    __syncwarp();
  }
  // back substitution over the tiles in reverse: x_{N-1} = d'_{N-1};  x_i = d'_i - c'_i x_{i+1}
  double2 xn = czero();
  const int last0 = ((N - 1) / kTT) * kTT;
  for (int i0 = last0; i0 >= 0; i0 -= kTT) {
    load_tile(td, Sh, i0);
    load_tile(tc, cp, i0);
    __syncwarp();
    const int iend = min(kTT, N - i0);
    for (int r = iend - 1; r >= 0; --r) {
      xn = (i0 + r == N - 1) ? td[r][lane] : csub(td[r][lane], cmul(tc[r][lane], xn));
      td[r][lane] = xn;
    }
    __syncwarp();
    store_tile(td, Sh, i0);
    __syncwarp();
  }
}

}  // namespace

cudaError_t pd_launch_jac_avg(const double* u, double* dbar, int nt, long long S, double g3, double g1, cudaStream_t st) {
  jac_avg_kernel<<<(unsigned)((S + 63) / 64), 256, 0, st>>>(u, dbar, nt, S, g3, g1);
  return cudaGetLastError();
}

cudaError_t pd_launch_thomas_shift(double2* Sh, int nx, int nfreq, const double2* lam1, const double2* lam2, double sub,
                                   double dia, double sup, const double* dbar, double2* cp, cudaStream_t st) {
  thomas_shift_kernel<<<(nfreq + kTT - 1) / kTT, kTT, 0, st>>>(Sh, nx, nfreq, lam1, lam2, sub, dia, sup, dbar, cp);
  return cudaGetLastError();
}
