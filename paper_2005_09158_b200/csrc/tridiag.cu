// Step (b), 1D: (lambda_{1,n} I + lambda_{2,n} K) S2_n = S1_n for every frequency n (P:l.182, 816; M = I).
//
// K is the constant-coefficient tridiagonal FD operator (Dirichlet), so every shifted system is a Toeplitz
// tridiagonal  a x_{i-1} + b x_i + c x_{i+1} = d_i  (x_{-1} = x_N = 0) with complex (a, b, c).  With
// r1, r2 the roots of c r^2 + b r + a = 0 (|r2| <= |r1|), the operator factors exactly as
//   w_i - r2 w_{i-1} = d_i,   w_i = c (x_{i+1} - r1 x_i),   w_{-1} = c x_0,
// i.e. a stable forward first-order recurrence (|r2| < 1) followed by a stable backward one
//   x_i = s x_{i+1} - tau w_i,  s = 1/r1, tau = 1/(c r1)   (|s| < 1),
// plus one rank-1 correction for the unknown x_0:  x = x^(d) + (c x_0) q, x_0 = x^(d)_0 / (1 - c q_0), where q
// is the response to w^(1)_i = r2^{i+1}, a geometric sum with the closed form kappa (r2^{i+1} - r2^{N+1} s^{N-i}).  tau = 2/(-b -+ sqrt(b^2-4ac)) stays finite when c -> 0 (lower
// bidiagonal limit) and r2 = a tau, s = c tau.  Setup checks |r2|^N and |s|^N stay bounded (PD_EINVAL).
// Numerically checked against pivoted banded LU on every frequency of configs 0-2.
// First-order recurrences with a *uniform* multiplier parallelise as chunked affine scans: a CTA owns one
// frequency, each thread L consecutive rows in registers, carries cross threads with warp shuffles.
// HBM traffic: 16 B read + 16 B write per complex unknown (the half spectrum, ~8+8 B per real dof).
#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int kL = 16;  // rows per thread

PD_D double2 shfl_up2(double2 v, int d) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
}
PD_D double2 shfl_down2(double2 v, int d) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
}
PD_D double2 cpow_int(double2 m, int e) {
  double2 r = make_double2(1.0, 0.0);
  while (e) {
    if (e & 1) r = cmul(r, m);
    m = cmul(m, m);
    e >>= 1;
  }
  return r;
}

// Exclusive affine scan over the CTA's threads: I_k = M I_{k-1} + e_k, returns I_{k-1} (0 for the first).
// REVERSE scans from the last thread to the first.  tot: smem scratch of NW double2.
template <int NT, bool REVERSE>
PD_D double2 block_affine_scan_excl(double2 e, double2 M, double2* tot) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int vl = REVERSE ? 31 - lane : lane;
  const int vw = REVERSE ? NW - 1 - warp : warp;
  double2 I = e, Md = M;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    double2 o = REVERSE ? shfl_down2(I, d) : shfl_up2(I, d);
    if (vl >= d) I = cfma(Md, o, I);
    Md = cmul(Md, Md);
  }
  // Md == M^32 now
  if (vl == 31) tot[vw] = I;
  __syncthreads();
  double2 P = czero();
  for (int w = 0; w < vw; ++w) P = cfma(Md, P, tot[w]);
  __syncthreads();
  I = cfma(cpow_int(M, vl + 1), P, I);  // global inclusive
  double2 ex = REVERSE ? shfl_down2(I, 1) : shfl_up2(I, 1);
  return vl == 0 ? P : ex;
}

// per-frequency tables in shared memory: R2POW[j] = r2^{j+1}, SPOW[j] = s^j (thread 0; caller synchronises)
PD_D void tri_tables(const pd_tri_coef& cf, double2* R2POW, double2* SPOW) {
  if (threadIdx.x == 0) {
    double2 p = cf.r2, sp = make_double2(1.0, 0.0);
    for (int j = 0; j < kL; ++j) {
      R2POW[j] = p;
      p = cmul(p, cf.r2);
      SPOW[j] = sp;
      sp = cmul(sp, cf.s);
    }
    SPOW[kL] = sp;
  }
}

// Solve the Toeplitz system for the rows this thread holds in registers (d: right-hand side in, x out).
// Thread k owns rows [k*L, k*L + Lk).  All NT threads must call (block scans, barriers).
template <int NT>
PD_D void tri_solve_regs(double2 (&d)[kL], const pd_tri_coef& cf, int Lk, int i0, int N, const double2* R2POW,
                         const double2* SPOW, double2* tot, double2* bc) {
  constexpr int L = kL;
  const int k = threadIdx.x;
  // forward local: w_j = r2 w_{j-1} + d_j (zero carry-in)
  double2 p = czero();
#pragma unroll
  for (int j = 0; j < L; ++j) {
    if (j < Lk) {
      p = cfma(cf.r2, p, d[j]);
      d[j] = p;
    }
  }
  const double2 Vin = block_affine_scan_excl<NT, false>(p, cf.r2L, tot);
#pragma unroll
  for (int j = 0; j < L; ++j)
    if (j < Lk) d[j] = cfma(R2POW[j], Vin, d[j]);

  // backward local: x_j = s x_{j+1} - tau w_j (zero carry-in from the right)
  const double2 mtau = cneg(cf.tau);
  p = czero();
#pragma unroll
  for (int j = L - 1; j >= 0; --j) {
    if (j < Lk) {
      p = cfma(cf.s, p, cmul(mtau, d[j]));
      d[j] = p;
    }
  }
  const double2 Xin = block_affine_scan_excl<NT, true>(p, cf.sL, tot);
  if (k == 0) bc[0] = cfma(SPOW[Lk], Xin, d[0]);  // x^(d)_0 (thread 0 holds row 0)
  __syncthreads();
  const double2 X0 = bc[0];
  // rank-1 boundary correction in closed form (r02ac): the response of the backward recurrence to w_i = r2^{i+1} is
  //   q_i = -tau sum_{k >= i} s^{k-i} r2^{k+1} = kappa (r2^{i+1} - r2^{N+1} s^{N-i}),  kappa = -tau / (1 - s r2),
  // so x_i = x^(d)_i + c x_0 q_i = x^(d)_i + X0 (k1 r2^{i+1} + k2 s^{N-i}), k1 = c kappa / (1 - c q_0), k2 = -k1 r2^{N+1}
  // (host, long double).  The s-term rides on the carry from above (s^{N-i} = s^{N-top} s^{top-i}), the r2-term on the
  // chunk table: no second recurrence and no third block scan.
  const int etop = N - i0 - Lk;
  const double2 Xin2 = cfma(cmul(cf.k2, X0), cpow_int(cf.s, etop > 0 ? etop : 0), Xin);
  const double2 Bg = cmul(cmul(cf.k1, X0), cpow_int(cf.r2, i0));
#pragma unroll
  for (int j = 0; j < L; ++j)
    if (j < Lk) d[j] = cfma(R2POW[j], Bg, cfma(SPOW[Lk - j], Xin2, d[j]));
}

template <int NT>
__global__ void __launch_bounds__(NT) tridiag_kernel(double2* __restrict__ Sh, int N, const pd_tri_coef* __restrict__ coef) {
  constexpr int L = kL;
  extern __shared__ double2 sbuf[];           // staging: NT*L + NT (padded rows)
  __shared__ double2 R2POW[L], SPOW[L + 1], tot[NT / 32], bc[2];
  const int n = blockIdx.x;
  const pd_tri_coef cf = coef[n];
  double2* row = Sh + (long long)n * N;
  tri_tables(cf, R2POW, SPOW);
  // coalesced load into padded staging: element i -> i + i/L (all of a thread's loads in flight first)
  {
    double2 v[L];
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const int i = threadIdx.x + k * NT;
      if (i < N) v[k] = __ldcs(row + i);
    }
#pragma unroll
    for (int k = 0; k < L; ++k) {
      const int i = threadIdx.x + k * NT;
      if (i < N) sbuf[i + i / L] = v[k];
    }
  }
  __syncthreads();

  const int k = threadIdx.x;
  const int i0 = k * L;
  const int Lk = max(0, min(L, N - i0));
  double2 d[L];
#pragma unroll
  for (int j = 0; j < L; ++j) d[j] = (j < Lk) ? sbuf[i0 + j + k] : czero();
  tri_solve_regs<NT>(d, cf, Lk, i0, N, R2POW, SPOW, tot, bc);
  __syncthreads();  // staging buffer reuse
#pragma unroll
  for (int j = 0; j < L; ++j)
    if (j < Lk) sbuf[i0 + j + k] = d[j];
  __syncthreads();
  for (int i = threadIdx.x; i < N; i += NT) __stcs(row + i, sbuf[i + i / L]);
}

// Tail map of the WR tail form (oracle/tail.py tail_map), 1D: for the frequencies
// n = blockIdx.x, blockIdx.x + gridDim.x, ...: right-hand side sum_{t<H} hc[n][t] g_t (the economical Step (a)),
// the Toeplitz solve of Step (b), and the last H rows of Step (c) as weighted sums Re(ow[n][a] x) accumulated in
// registers (ow carries the half-spectrum multiplicity).  Per-CTA partial sums out: part[blockIdx.x][a][N].
template <int NT, int H>
__global__ void __launch_bounds__(NT) tail1d_kernel(const double* __restrict__ g, double* __restrict__ part, int N,
                                                    int F, const pd_tri_coef* __restrict__ coef,
                                                    const double2* __restrict__ hc, const double2* __restrict__ ow) {
  constexpr int L = kL;
  __shared__ double2 R2POW[L], SPOW[L + 1], tot[NT / 32], bc[2];
  const int k = threadIdx.x;
  const int i0 = k * L;
  const int Lk = max(0, min(L, N - i0));
  double acc[H][L];
#pragma unroll
  for (int a = 0; a < H; ++a)
#pragma unroll
    for (int j = 0; j < L; ++j) acc[a][j] = 0.0;
  for (int n = blockIdx.x; n < F; n += gridDim.x) {
    const pd_tri_coef cf = coef[n];
    __syncthreads();  // previous frequency's tables consumed
    tri_tables(cf, R2POW, SPOW);
    __syncthreads();
    double2 hcn[H], own[H];
#pragma unroll
    for (int t = 0; t < H; ++t) {
      hcn[t] = __ldg(hc + (long long)n * H + t);
      own[t] = __ldg(ow + (long long)n * H + t);
    }
    double2 d[L];  // head values re-read per frequency (L1-resident, H*N doubles)
#pragma unroll
    for (int j = 0; j < L; ++j) {
      d[j] = cscale(hcn[0], j < Lk ? __ldg(g + i0 + j) : 0.0);
#pragma unroll
      for (int t = 1; t < H; ++t) d[j] = cfma(hcn[t], make_double2(j < Lk ? __ldg(g + (long long)t * N + i0 + j) : 0.0, 0.0), d[j]);
    }
    tri_solve_regs<NT>(d, cf, Lk, i0, N, R2POW, SPOW, tot, bc);
#pragma unroll
    for (int a = 0; a < H; ++a)
#pragma unroll
      for (int j = 0; j < L; ++j) acc[a][j] += own[a].x * d[j].x - own[a].y * d[j].y;
  }
#pragma unroll
  for (int a = 0; a < H; ++a)
#pragma unroll
    for (int j = 0; j < L; ++j)
      if (j < Lk) part[((long long)blockIdx.x * H + a) * N + i0 + j] = acc[a][j];
}

template <int NT>
cudaError_t launch_nt(double2* Sh, int nx, int nfreq, const pd_tri_coef* coef, cudaStream_t st) {
  const int smem = (NT * kL + NT) * (int)sizeof(double2);
  static int attr = -1;  // device on which the attributes were set
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (attr != dev_) {
    cudaError_t e = cudaFuncSetAttribute(tridiag_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = dev_;
  }
  tridiag_kernel<NT><<<nfreq, NT, smem, st>>>(Sh, nx, coef);
  return cudaGetLastError();
}

template <int NT>
cudaError_t launch_tail_nt(const double* g, double* part, int G, int N, int F, int H, const pd_tri_coef* coef,
                           const double2* hc, const double2* ow, cudaStream_t st) {
  if (H == 2)
    tail1d_kernel<NT, 2><<<G, NT, 0, st>>>(g, part, N, F, coef, hc, ow);
  else
    tail1d_kernel<NT, 1><<<G, NT, 0, st>>>(g, part, N, F, coef, hc, ow);
  return cudaGetLastError();
}

}  // namespace

cudaError_t pd_launch_tail1d(const double* g, double* part, int G, int nx, int nfreq, int H, const pd_tri_coef* coef,
                             const double2* hc, const double2* ow, cudaStream_t st) {
  if (H < 1 || H > 2) return cudaErrorInvalidValue;
  switch (pd_tridiag_threads(nx)) {
    case 32: return launch_tail_nt<32>(g, part, G, nx, nfreq, H, coef, hc, ow, st);
    case 64: return launch_tail_nt<64>(g, part, G, nx, nfreq, H, coef, hc, ow, st);
    case 128: return launch_tail_nt<128>(g, part, G, nx, nfreq, H, coef, hc, ow, st);
    case 256: return launch_tail_nt<256>(g, part, G, nx, nfreq, H, coef, hc, ow, st);
    case 512: return launch_tail_nt<512>(g, part, G, nx, nfreq, H, coef, hc, ow, st);
    case 1024: return launch_tail_nt<1024>(g, part, G, nx, nfreq, H, coef, hc, ow, st);
    default: return cudaErrorInvalidValue;
  }
}

int pd_tridiag_rows_per_thread() { return kL; }

int pd_tridiag_threads(int nx) {
  int t = 32;
  while (t * kL < nx) t <<= 1;
  return t <= 1024 ? t : -1;
}

cudaError_t pd_launch_tridiag(double2* Sh, int nx, int nfreq, const pd_tri_coef* coef, int, cudaStream_t st) {
  switch (pd_tridiag_threads(nx)) {
    case 32: return launch_nt<32>(Sh, nx, nfreq, coef, st);
    case 64: return launch_nt<64>(Sh, nx, nfreq, coef, st);
    case 128: return launch_nt<128>(Sh, nx, nfreq, coef, st);
    case 256: return launch_nt<256>(Sh, nx, nfreq, coef, st);
    case 512: return launch_nt<512>(Sh, nx, nfreq, coef, st);
    case 1024: return launch_nt<1024>(Sh, nx, nfreq, coef, st);
    default: return cudaErrorInvalidValue;
  }
}
