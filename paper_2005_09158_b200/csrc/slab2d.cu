// Step (b), 2D periodic: S2_n = (lambda_{1,n} I + lambda_{2,n} K)^{-1} S1_n for every frequency n
// (P:l.182, 816; 2D periodic ADE P:l.908-918).  K = -nu Lap_h + ax D_x + ay D_y (5-point, centred,
// periodic) is diagonal in the 2D DFT basis with symbol
//   kappa(kx, ky) = (4 nu/h^2)(sin^2(pi kx/N) + sin^2(pi ky/N)) + i (ax sin(2 pi kx/N) + ay sin(2 pi ky/N))/h
// (reading c14), so each slab is solved exactly by   2D FFT -> divide by lambda1 + lambda2 kappa -> 2D IFFT.
//
// The half-spectrum buffer holds F slabs of N x N complex, processed in chunks of slabs (~1 GB: launch
// count, not L2 residency, decides on B200); per chunk three launches run in place:
// (1) row FFTs along x (rows are contiguous), (2) column FFT along y + divide + column IFFT (8 adjacent
// columns per CTA = 128 B row segments), (3) row IFFTs along x.  When the time FFTs already did the x
// transforms (tfx.cu, the default where supported) only launch (2) runs (cols_only).
#include <cstdlib>

#include "fft.cuh"
#include "kernels.h"

// L2 policy of the y-pass tile loads / stores (slab_ytri_kernel, dtri_kernel): 1 = ld.cg / st.cg, 0 = evict-first
// (ld.cs / st.cs).  Measured (r02al/am, cfg4 y-pass): evict-first loads 2.01 ms, ld.cg loads 1.72 ms, the store policy
// makes no difference, ld.lu loads 1.73 ms; so the tiles are loaded with ld.cg and stored evict-first (the inverse time FFT that follows
// wants its L2 for the four-step scratch)
#ifndef PD_SPEC_KEEP_SLAB_LD
#define PD_SPEC_KEEP_SLAB_LD 1
#endif
#ifndef PD_SPEC_KEEP_SLAB_ST
#define PD_SPEC_KEEP_SLAB_ST 0
#endif
#if PD_SPEC_KEEP_SLAB_LD
#define PD_SPEC_LD(p) __ldcg(p)
#else
#define PD_SPEC_LD(p) __ldcs(p)
#endif
#if PD_SPEC_KEEP_SLAB_ST
#define PD_SPEC_ST(p, v) __stcg(p, v)
#else
#define PD_SPEC_ST(p, v) __stcs(p, v)
#endif
using namespace pdfft;

namespace {

constexpr int kBatch = 8;  // rows (launch 1/3) or columns (launch 2) per CTA

template <int N>
struct SlabCfg {
  static constexpr int C = kBatch;
  static constexpr int E = elems_per_thread(N);
  static constexpr int NTH = C * N / E;
#ifndef PD_SLAB_MINB
#define PD_SLAB_MINB 3
#endif
  static constexpr int MINB = NTH <= 256 ? PD_SLAB_MINB : 1;
};

// column kernel: radix cap RM (8 halves the register footprint and doubles the threads per tile)
#ifndef PD_SLAB_COLS_RM
#define PD_SLAB_COLS_RM 8
#endif
#ifndef PD_SLAB_COLS_C
#define PD_SLAB_COLS_C 8
#endif
#ifndef PD_SLAB_COLS_MINB
#define PD_SLAB_COLS_MINB 2
#endif
template <int N>
struct ColCfg {
  static constexpr int C = PD_SLAB_COLS_C;  // columns per CTA (C * 16 B row segments)
  static constexpr int RM = PD_SLAB_COLS_RM;
  static constexpr int E = elems_per_thread(N, RM);
  static constexpr int NTH = C * N / E;
  static constexpr int MINB = NTH <= 512 ? PD_SLAB_COLS_MINB : 1;
};

// rows [blockIdx.x*C, +C) of the flattened chunk (row index over slabs: slab*N + y), FFT along x in place
template <int N, bool INV>
__global__ void __launch_bounds__(SlabCfg<N>::NTH, SlabCfg<N>::MINB)
slab_rows_kernel(double2* __restrict__ base, const double2* __restrict__ tw) {
  using T = SlabCfg<N>;
  constexpr int C = T::C, NTH = T::NTH, R0 = first_radix(N), RL = last_radix(N);
  extern __shared__ double2 sm[];
  __shared__ double2 s_tw[N];
  double2* p = base + (long long)blockIdx.x * C * N;
  load_table(s_tw, tw, N);
  __syncthreads();
  fft_io<N, C, INV, true, NTH, false, false>(
      sm, s_tw,
      [&](int j, auto st, int c, double2* v) {
        const double2* q = p + c * N + j;
#pragma unroll
        for (int m = 0; m < R0; ++m) v[m] = __ldcg(q + m * decltype(st)::value);
      },
      [&](int j, auto st, int c, const double2* w) {
        double2* q = p + c * N + j;
#pragma unroll
        for (int m = 0; m < RL; ++m) __stcg(q + m * decltype(st)::value, w[m]);
      });
}

// columns [c0, c0 + C) of slab (slab0 + blockIdx.y): forward FFT along y, divide, inverse FFT along y.
// FILTER: multiply by tab[ky*N + kx] instead of dividing by lambda1 + lambda2 kappa (the WR tail map, tail.cu).
template <int N, bool FILTER = false>
__global__ void __launch_bounds__(ColCfg<N>::NTH, ColCfg<N>::MINB)
slab_cols_kernel(double2* __restrict__ Sh, int slab0, const double2* __restrict__ lam1,
                 const double2* __restrict__ lam2, const double* __restrict__ sx, const double* __restrict__ sn,
                 pd_slab_params prm, const double2* __restrict__ tw, const double2* __restrict__ tab = nullptr) {
  using T = ColCfg<N>;
  constexpr int C = T::C, NTH = T::NTH, RM = T::RM, R0 = first_radix(N, RM), RL = last_radix(N, RM);
  extern __shared__ double2 sm[];
  __shared__ double2 s_tw[N];
  const int n = slab0 + blockIdx.y;
  const int c0 = blockIdx.x * C;
  double2* slab = Sh + (long long)n * N * N + c0;
  const double2 l1 = FILTER ? czero() : lam1[n], l2 = FILTER ? czero() : lam2[n];
  const double invNN = 1.0 / ((double)N * (double)N);
  load_table(s_tw, tw, N);
  __syncthreads();
  // forward FFT along y; the last pass divides by lambda1 + lambda2 kappa(kx, ky) on its way to smem
  fft_io<N, C, false, false, NTH, false, true, RM>(
      sm, s_tw,
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value;
        const double2* q = slab + (long long)j * N + c;
#pragma unroll
        for (int m = 0; m < R0; ++m) v[m] = __ldcg(q + (long long)m * s * N);
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value;
        const int kx = c0 + c;
        const int a = lin<N, C, false>(j, c);
        if constexpr (FILTER) {
#pragma unroll
          for (int m = 0; m < RL; ++m)
            sm[soff<s * C>(a, m)] = cscale(cmul(w[m], __ldg(tab + (j + m * s) * N + kx)), invNN);
          return;
        }
        const double ax = prm.kd * __ldg(sx + kx), bx = prm.cx * __ldg(sn + kx);
#pragma unroll
        for (int m = 0; m < RL; ++m) {
          const int ky = j + m * s;
          const double2 kap = make_double2(fma(prm.kd, __ldg(sx + ky), ax), fma(prm.cy, __ldg(sn + ky), bx));
          sm[soff<s * C>(a, m)] = cscale(cmul(w[m], crcp_fast(cfma(l2, kap, l1))), invNN);
        }
      });
  __syncthreads();
  fft_io<N, C, true, false, NTH, true, false, RM>(
      sm, s_tw,
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value;
        const int a = lin<N, C, false>(j, c);
#pragma unroll
        for (int m = 0; m < R0; ++m) v[m] = sm[soff<s * C>(a, m)];
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value;
        double2* q = slab + (long long)j * N + c;
#pragma unroll
        for (int m = 0; m < RL; ++m) __stcg(q + (long long)m * s * N, w[m]);
      });
}

template <int N>
int smem_bytes() {
  return smem_elems(kBatch * N) * (int)sizeof(double2);
}
template <int N>
int smem_cols() {
  return smem_elems(ColCfg<N>::C * N) * (int)sizeof(double2);
}

template <int N>
cudaError_t launch_n(double2* Sh, int nfreq, const double2* lam1, const double2* lam2, const double* sx,
                     const double* sn, pd_slab_params prm, const double2* tw, int chunk, int cols_only,
                     cudaStream_t st, int* launches) {
  using T = SlabCfg<N>;
  const int smem = smem_bytes<N>();
  static int attr = -1;  // device on which the attributes were set
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (attr != dev_) {
    cudaError_t e = cudaFuncSetAttribute(slab_rows_kernel<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(slab_rows_kernel<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(slab_cols_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cols<N>());
    if (e != cudaSuccess) return e;
    attr = dev_;
  }
  int nl = 0;
  for (int s0 = 0; s0 < nfreq; s0 += chunk) {
    const int ns = nfreq - s0 < chunk ? nfreq - s0 : chunk;
    double2* base = Sh + (long long)s0 * N * N;
    const unsigned row_ctas = (unsigned)(ns * (N / T::C));
    if (!cols_only) slab_rows_kernel<N, false><<<row_ctas, T::NTH, smem, st>>>(base, tw);
    slab_cols_kernel<N><<<dim3(N / ColCfg<N>::C, ns), ColCfg<N>::NTH, smem_cols<N>(), st>>>(Sh, s0, lam1, lam2, sx, sn, prm, tw);
    if (!cols_only) slab_rows_kernel<N, true><<<row_ctas, T::NTH, smem, st>>>(base, tw);
    nl += cols_only ? 1 : 3;
  }
  if (launches) *launches = nl;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// 2D homogeneous Dirichlet (Table T4A): K = -nu Lap_h is diagonalised by the tensor DST-I, mu_k = (4nu/h^2)
// sin^2(pi k / M), M = 2(N+1).  A DST-I of length N is an FFT of length M of the odd extension
// (0, z_1..z_N, 0, -z_N..-z_1): X[k] = -2i sum_j z_j sin(pi j k/(N+1)); X is itself odd, so after the forward
// transform along y the spectrum is the odd extension of the DST coefficients and the column pass is
// FFT -> divide by lambda1 + lambda2 (mu_kx + mu_ky) -> IFFT, exactly as the periodic pass.  Rows (x) and columns
// (y) hold N values in HBM; the loaders build the extension, the storers keep positions 1..N.  Forward and
// inverse along both directions give M^2 times the solution: the column pass scales by 1/M^2.
PD_D double2 odd_ext(const double2* __restrict__ q, long long stride, int p, int N, int M) {
  if (p == 0 || p == N + 1) return czero();
  return p <= N ? __ldcg(q + (long long)(p - 1) * stride) : cneg(__ldcg(q + (long long)(M - p - 1) * stride));
}

// rows [blockIdx.x*C, +C) of the flattened chunk (total rows nrows = slabs * N), DST along x in place
template <int M, bool INV>
__global__ void __launch_bounds__(SlabCfg<M>::NTH, SlabCfg<M>::MINB)
dst_rows_kernel(double2* __restrict__ base, long long nrows, const double2* __restrict__ tw) {
  using T = SlabCfg<M>;
  constexpr int C = T::C, NTH = T::NTH, N = M / 2 - 1, R0 = first_radix(M), RL = last_radix(M);
  extern __shared__ double2 sm[];
  __shared__ double2 s_tw[M];
  const long long row0 = (long long)blockIdx.x * C;
  load_table(s_tw, tw, M);
  __syncthreads();
  fft_io<M, C, INV, true, NTH, false, false>(
      sm, s_tw,
      [&](int j, auto st, int c, double2* v) {
        const bool ok = row0 + c < nrows;
        const double2* q = base + (row0 + c) * N;
#pragma unroll
        for (int m = 0; m < R0; ++m) v[m] = ok ? odd_ext(q, 1, j + m * decltype(st)::value, N, M) : czero();
      },
      [&](int j, auto st, int c, const double2* w) {
        if (row0 + c >= nrows) return;
        double2* q = base + (row0 + c) * N;
#pragma unroll
        for (int m = 0; m < RL; ++m) {
          const int k = j + m * decltype(st)::value;
          if (k >= 1 && k <= N) __stcg(q + k - 1, w[m]);
        }
      });
}

// columns [c0, c0 + C) of slab (slab0 + blockIdx.y): DST along y, divide, inverse DST along y, x 1/M^2
template <int M>
__global__ void __launch_bounds__(ColCfg<M>::NTH, ColCfg<M>::MINB)
dst_cols_kernel(double2* __restrict__ Sh, int slab0, const double2* __restrict__ lam1, const double2* __restrict__ lam2,
                const double* __restrict__ mu, const double2* __restrict__ tw) {
  using T = ColCfg<M>;
  constexpr int C = T::C, NTH = T::NTH, RM = T::RM, N = M / 2 - 1, R0 = first_radix(M, RM), RL = last_radix(M, RM);
  extern __shared__ double2 sm[];
  __shared__ double2 s_tw[M];
  const int n = slab0 + blockIdx.y;
  const int c0 = blockIdx.x * C;
  double2* slab = Sh + (long long)n * N * N + c0;
  const double2 l1 = lam1[n], l2 = lam2[n];
  const double inv = 1.0 / ((double)M * (double)M);
  load_table(s_tw, tw, M);
  __syncthreads();
  fft_io<M, C, false, false, NTH, false, true, RM>(
      sm, s_tw,
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value;
        const bool ok = c0 + c < N;
#pragma unroll
        for (int m = 0; m < R0; ++m) v[m] = ok ? odd_ext(slab + c, N, j + m * s, N, M) : czero();
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value;
        const double mx = __ldg(mu + c0 + c + 1);  // x-DST index k = element + 1
        const int a = lin<M, C, false>(j, c);
#pragma unroll
        for (int m = 0; m < RL; ++m) {
          const double muy = __ldg(mu + j + m * s);
          sm[soff<s * C>(a, m)] = cscale(cmul(w[m], crcp_fast(cfma(l2, make_double2(mx + muy, 0.0), l1))), inv);
        }
      });
  __syncthreads();
  fft_io<M, C, true, false, NTH, true, false, RM>(
      sm, s_tw,
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value;
        const int a = lin<M, C, false>(j, c);
#pragma unroll
        for (int m = 0; m < R0; ++m) v[m] = sm[soff<s * C>(a, m)];
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value;
        if (c0 + c >= N) return;
#pragma unroll
        for (int m = 0; m < RL; ++m) {
          const int k = j + m * s;
          if (k >= 1 && k <= N) __stcg(slab + c + (long long)(k - 1) * N, w[m]);
        }
      });
}

template <int M>
cudaError_t dst_n(double2* Sh, int nfreq, const double2* lam1, const double2* lam2, const double* mu,
                  const double2* tw, int chunk, cudaStream_t st, int* launches) {
  using T = SlabCfg<M>;
  constexpr int N = M / 2 - 1;
  const int smr = smem_bytes<M>(), smc = smem_cols<M>();
  static int attr = -1;  // device on which the attributes were set
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (attr != dev_) {
    cudaError_t e = cudaFuncSetAttribute(dst_rows_kernel<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smr);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(dst_rows_kernel<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smr);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(dst_cols_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smc);
    if (e != cudaSuccess) return e;
    attr = dev_;
  }
  int nl = 0;
  for (int s0 = 0; s0 < nfreq; s0 += chunk) {
    const int ns = nfreq - s0 < chunk ? nfreq - s0 : chunk;
    double2* base = Sh + (long long)s0 * N * N;
    const long long nrows = (long long)ns * N;
    const unsigned row_ctas = (unsigned)((nrows + T::C - 1) / T::C);
    dst_rows_kernel<M, false><<<row_ctas, T::NTH, smr, st>>>(base, nrows, tw);
    dst_cols_kernel<M><<<dim3((N + ColCfg<M>::C - 1) / ColCfg<M>::C, ns), ColCfg<M>::NTH, smc, st>>>(Sh, s0, lam1, lam2,
                                                                                                    mu, tw);
    dst_rows_kernel<M, true><<<row_ctas, T::NTH, smr, st>>>(base, nrows, tw);
    nl += 3;
  }
  if (launches) *launches = nl;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// y-pass by cyclic Toeplitz tridiagonal solves (see kernels.h pd_ytri_coef).  8 columns per CTA, one warp per
// column, L = N/32 consecutive rows per lane in registers; first-order recurrences carried across lanes by warp
// affine scans, cyclic closures from the scan totals.  ~26 fp64 operations per complex element instead of the
// ~150 of FFT -> divide -> IFFT, so the pass is HBM-bound.  smem: padded column-major tile
// (index c*(N+33) + i + i/L) - conflict-free both for the coalesced row loads and for the lane chunks.
PD_D double2 shfl_up2(double2 v, int d) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
}
PD_D double2 shfl_down2(double2 v, int d) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
}
PD_D double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
PD_D double2 cpow_small(double2 m, int e) {
  double2 r = make_double2(1.0, 0.0);
  while (e) {
    if (e & 1) r = cmul(r, m);
    m = cmul(m, m);
    e >>= 1;
  }
  return r;
}
// exclusive affine scan over the 32 lanes: I_l = M I_{l-1} + e_l; returns I_{l-1} (0 for the first lane);
// *inc_last = the inclusive value at the last lane of the scan order (lane 31 forward, lane 0 reverse)
template <bool REVERSE>
PD_D double2 warp_affine_scan(double2 e, double2 M, double2* inc_last) {
  const int lane = threadIdx.x & 31;
  const int vl = REVERSE ? 31 - lane : lane;
  double2 I = e, Md = M;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double2 o = REVERSE ? shfl_down2(I, d) : shfl_up2(I, d);
    if (vl >= d) I = cfma(Md, o, I);
    Md = cmul(Md, Md);
  }
  *inc_last = shfl2(I, REVERSE ? 0 : 31);
  const double2 ex = REVERSE ? shfl_down2(I, 1) : shfl_up2(I, 1);
  return vl == 0 ? czero() : ex;
}

#ifndef PD_YTRI_C
#define PD_YTRI_C 8  // columns (= warps) per CTA
#endif
#ifndef PD_YTRI_SPLIT
#define PD_YTRI_SPLIT 1  // two interleaved half-length recurrence chains per lane (ILP 2 on the fp64 latency chains)
#endif

// One lane's L rows of a column, both recurrences, with each lane chunk split into halves A (rows 0..H-1) and
// B (rows H..L-1), H = L/2, whose chains run interleaved:
//   forward  a_j = r a_{j-1} + d_j,  b_j = r b_{j-1} + d_{H+j} (zero carry-ins); lane total r^H a_{H-1} + b_{H-1};
//            with the lane carry-in q:  w_j = a_j + r^{j+1} q,  w_{H+j} = b_j + r^{j+1} (r^H q + a_{H-1})
//   backward the mirror image from the top row down with s, -tau w and the carry from above
// (the same sums as the single chain, regrouped).
template <int L>
PD_D void ytri_lane_split(double2* d, const pd_ytri_coef& cf, int lane, double scale) {
  constexpr int H = L / 2;
  double2 rH = cf.r, sH = cf.s;
#pragma unroll
  for (int h = 1; h < H; h <<= 1) {
    rH = cmul(rH, rH);
    sH = cmul(sH, sH);
  }
  double2 a = czero(), b = czero();
#pragma unroll
  for (int j = 0; j < H; ++j) {
    a = cfma(cf.r, a, d[j]);
    d[j] = a;
    b = cfma(cf.r, b, d[H + j]);
    d[H + j] = b;
  }
  double2 tot;
  const double2 cin = warp_affine_scan<false>(cfma(rH, a, b), cf.rL, &tot);
  const double2 W = cmul(tot, cf.ir);
  double2 qa = cfma(cpow_small(cf.rL, lane), W, cin);  // carry + r^{lane L} W
  double2 qb = cfma(rH, qa, a);
#pragma unroll
  for (int j = 0; j < H; ++j) {
    qa = cmul(cf.r, qa);
    d[j] = cadd(d[j], qa);
    qb = cmul(cf.r, qb);
    d[H + j] = cadd(d[H + j], qb);
  }
  const double2 mtau = cneg(cf.tau);
  double2 u = czero(), l = czero();
#pragma unroll
  for (int jj = 0; jj < H; ++jj) {
    u = cfma(cf.s, u, cmul(mtau, d[L - 1 - jj]));
    d[L - 1 - jj] = u;
    l = cfma(cf.s, l, cmul(mtau, d[H - 1 - jj]));
    d[H - 1 - jj] = l;
  }
  const double2 cr = warp_affine_scan<true>(cfma(sH, u, l), cf.sL, &tot);
  const double2 x0 = cmul(tot, cf.is);
  double2 qu = cfma(cpow_small(cf.sL, 31 - lane), x0, cr);  // carry from above the lane
  double2 ql = cfma(sH, qu, u);
#pragma unroll
  for (int jj = 0; jj < H; ++jj) {
    qu = cmul(cf.s, qu);
    d[L - 1 - jj] = cscale(cadd(d[L - 1 - jj], qu), scale);
    ql = cmul(cf.s, ql);
    d[H - 1 - jj] = cscale(cadd(d[H - 1 - jj], ql), scale);
  }
}
#ifndef PD_YTRI_MINB
#define PD_YTRI_MINB 0  // 0: by N (3 / 2 / 1)
#endif
constexpr int kYC = PD_YTRI_C;
template <int N>
__global__ void __launch_bounds__(32 * kYC, PD_YTRI_MINB ? PD_YTRI_MINB : (N <= 256 ? 3 : N <= 512 ? 2 : 1)) slab_ytri_kernel(double2* __restrict__ Sh, int slab0,
                                                                          int fglob0,
                                                                          const pd_ytri_coef* __restrict__ coef,
                                                                          double scale) {
  constexpr int L = N / 32, CS = N + 33;
  extern __shared__ double2 sm[];
  const int n = slab0 + blockIdx.y;
  const int c0 = blockIdx.x * kYC;
  double2* slab = Sh + (long long)n * N * N + c0;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const pd_ytri_coef cf = coef[(long long)(fglob0 + blockIdx.y) * N + c0 + w];  // in flight with the tile
  {
    // all N/32 loads of a thread in flight before the first smem store
    constexpr int PT = N / 32;
    double2 v[PT];
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      const int i = threadIdx.x + k * 32 * kYC, r = i / kYC, c = i % kYC;
      v[k] = PD_SPEC_LD(slab + (long long)r * N + c);
    }
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      const int i = threadIdx.x + k * 32 * kYC, r = i / kYC, c = i % kYC;
      sm[c * CS + r + r / L] = v[k];
    }
  }
  __syncthreads();
  double2* col = sm + w * CS + lane * (L + 1);  // rows lane*L .. lane*L + L - 1 (+ one pad per lane chunk)
  double2 d[L];
#pragma unroll
  for (int j = 0; j < L; ++j) d[j] = col[j];
  if constexpr (PD_YTRI_SPLIT && L >= 4) {
    ytri_lane_split<L>(d, cf, lane, scale);
  } else {
  // forward: w'_i = r w'_{i-1} + d_i (zero carry-in), lane carries by scan, closure W = w_{N-1}
  double2 p = czero();
#pragma unroll
  for (int j = 0; j < L; ++j) {
    p = cfma(cf.r, p, d[j]);
    d[j] = p;
  }
  double2 tot;
  const double2 cin = warp_affine_scan<false>(p, cf.rL, &tot);
  const double2 W = cmul(tot, cf.ir);
  double2 q = cfma(cpow_small(cf.rL, lane), W, cin);  // carry + r^{lane L} W
#pragma unroll
  for (int j = 0; j < L; ++j) {
    q = cmul(cf.r, q);
    d[j] = cadd(d[j], q);
  }
  // backward: x'_i = s x'_{i+1} - tau w_i (zero carry-in from the right), scan from the last lane, closure x_0
  const double2 mtau = cneg(cf.tau);
  p = czero();
#pragma unroll
  for (int j = L - 1; j >= 0; --j) {
    p = cfma(cf.s, p, cmul(mtau, d[j]));
    d[j] = p;
  }
  const double2 cr = warp_affine_scan<true>(p, cf.sL, &tot);
  const double2 x0 = cmul(tot, cf.is);
  q = cfma(cpow_small(cf.sL, 31 - lane), x0, cr);  // carry + s^{N - lane L - L} x_0
#pragma unroll
  for (int j = L - 1; j >= 0; --j) {
    q = cmul(cf.s, q);
    d[j] = cscale(cadd(d[j], q), scale);
  }
  }
#pragma unroll
  for (int j = 0; j < L; ++j) col[j] = d[j];
  __syncthreads();
#pragma unroll 8
  for (int i = threadIdx.x; i < N * kYC; i += 32 * kYC) {
    const int r = i / kYC, c = i % kYC;
    PD_SPEC_ST(slab + (long long)r * N + c, sm[c * CS + r + r / L]);
  }
}

template <int N>
cudaError_t ytri_n(double2* Sh, int nfreq, int f0g, const pd_ytri_coef* coef, double scale, const double2* tw,
                   int chunk, int rows, cudaStream_t st, int* launches) {
  using T = SlabCfg<N>;
  const int smem = kYC * (N + 33) * (int)sizeof(double2), smr = smem_bytes<N>();
  static int attr = -1;  // device on which the attributes were set
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (attr != dev_) {
    cudaError_t e = cudaFuncSetAttribute(slab_ytri_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(slab_rows_kernel<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smr);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(slab_rows_kernel<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smr);
    if (e != cudaSuccess) return e;
    attr = dev_;
  }
  int nl = 0;
  for (int s0 = 0; s0 < nfreq; s0 += chunk) {
    const int ns = nfreq - s0 < chunk ? nfreq - s0 : chunk;
    double2* base = Sh + (long long)s0 * N * N;
    const unsigned row_ctas = (unsigned)(ns * (N / T::C));
    if (rows) slab_rows_kernel<N, false><<<row_ctas, T::NTH, smr, st>>>(base, tw);
    slab_ytri_kernel<N><<<dim3(N / kYC, ns), 32 * kYC, smem, st>>>(Sh, s0, f0g + s0, coef, scale);
    if (rows) slab_rows_kernel<N, true><<<row_ctas, T::NTH, smr, st>>>(base, tw);
    nl += rows ? 3 : 1;
  }
  if (launches) *launches = nl;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// 2D Dirichlet Step (b) with the y-direction solved directly (T4A, PD_WAVE2D_DIRICHLET): after the x-DST row pass
// every (frequency n, x-mode kx) column is the Dirichlet Toeplitz system
//   a x_{y-1} + b x_y + a x_{y+1} = d_y,  x_{-1} = x_N = 0,  a = -lambda2 nu/h^2,  b = lambda1 + lambda2 (mu_kx + 2nu/h^2)
// (K = -nu Lap_h = (mu_x) (x) I + I (x) T_y in the x-DST basis), solved by the characteristic-root recurrences of
// tridiag.cu (forward w_i = r2 w_{i-1} + d_i, backward x_i = s x_{i+1} - tau w_i, rank-1 correction for x_0 with the
// precomputed 1/(1 - c q_0)) on one warp per column, L = (N+1)/32 rows per lane (the last lane one row short), carries
// by warp affine scans.  Replaces the column pass's length-2(N+1) FFT -> divide -> IFFT.  Scale 1/M of the x-DST
// pair (forward and inverse odd-extension FFTs of length M = 2(N+1) multiply by M).
template <int N1>
__global__ void __launch_bounds__(32 * kYC, N1 <= 256 ? 3 : N1 <= 512 ? 2 : 1)
dtri_kernel(double2* __restrict__ Sh, int slab0, int fglob0, const pd_dtri_coef* __restrict__ coef, double scale) {
  constexpr int N = N1 - 1, L = N1 / 32, CS = N1 + 33;
  extern __shared__ double2 sm[];
  const int n = slab0 + blockIdx.y;
  const int c0 = blockIdx.x * kYC;
  double2* slab = Sh + (long long)n * N * N + c0;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool colok = c0 + w < N;
  const pd_dtri_coef cf = coef[(long long)(fglob0 + blockIdx.y) * N + (colok ? c0 + w : 0)];
  {
    constexpr int PT = L;  // ceil(N * kYC / (32 kYC)) = L
    double2 v[PT];
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      const int i = threadIdx.x + k * 32 * kYC, r = i / kYC, c = i % kYC;
      v[k] = (r < N && c0 + c < N) ? PD_SPEC_LD(slab + (long long)r * N + c) : czero();
    }
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      const int i = threadIdx.x + k * 32 * kYC, r = i / kYC, c = i % kYC;
      sm[c * CS + r + r / L] = v[k];
    }
  }
  __syncthreads();
  double2* col = sm + w * CS + lane * (L + 1);
  const int i0 = lane * L;
  const int Lk = lane == 31 ? L - 1 : L;  // row N (= 32 L - 1) does not exist
  double2 d[L];
#pragma unroll
  for (int j = 0; j < L; ++j) d[j] = j < Lk ? col[j] : czero();
  // forward: w_i = r2 w_{i-1} + d_i, carry r2^L across lanes (lanes below 31 are full)
  double2 p = czero();
#pragma unroll
  for (int j = 0; j < L; ++j)
    if (j < Lk) {
      p = cfma(cf.r2, p, d[j]);
      d[j] = p;
    }
  double2 tot;
  const double2 vin = warp_affine_scan<false>(p, cf.r2L, &tot);
  double2 rp = cf.r2;  // r2^{j+1}
#pragma unroll
  for (int j = 0; j < L; ++j)
    if (j < Lk) {
      d[j] = cfma(rp, vin, d[j]);
      rp = cmul(rp, cf.r2);
    }
  // backward: x_i = s x_{i+1} - tau w_i (x_N = 0)
  const double2 mtau = cneg(cf.tau);
  p = czero();
#pragma unroll
  for (int j = L - 1; j >= 0; --j)
    if (j < Lk) {
      p = cfma(cf.s, p, cmul(mtau, d[j]));
      d[j] = p;
    }
  const double2 xin = warp_affine_scan<true>(p, cf.sL, &tot);
  // rank-1 boundary correction in closed form.  The response of the same backward recurrence to w_i = r2^{i+1} is
  //   q_i = -tau sum_{k >= i} s^{k-i} r2^{k+1} = kappa (r2^{i+1} - r2^{N+1} s^{N-i}),  kappa = -tau / (1 - s r2),
  // so x_i = x^(d)_i + (c g x^(d)_0) q_i = x^(d)_i + X0 (k1 r2^{i+1} + k2 s^{N-i}) with the host constants
  // k1 = c g kappa, k2 = -k1 r2^{N+1}: the s-term joins the lane's carry from above (s^{N-i} = s^{N-top} s^{top-i}),
  // the r2-term is one running product - no second recurrence, scan or 16-row table (r02ac)
  const double2 X0 = shfl2(cfma(cf.sL, xin, d[0]), 0);  // x^(d)_0: lane 0 holds L full rows
  const double2 G2 = cmul(cf.k2, X0);
  // s^{N - (i0 + Lk)}: 1 on the last lane, s^{L-1} (s^L)^{30 - lane} below
  const double2 stop = lane == 31 ? make_double2(1.0, 0.0) : cmul(cf.sLm1, cpow_small(cf.sL, 30 - lane));
  const double2 xin2 = cfma(G2, stop, xin);
  double2 sp = make_double2(1.0, 0.0);  // s^{Lk - j}, built from the top row down
#pragma unroll
  for (int j = L - 1; j >= 0; --j)
    if (j < Lk) {
      sp = cmul(sp, cf.s);
      d[j] = cfma(sp, xin2, d[j]);
    }
  double2 rg = cmul(cmul(cf.k1, X0), cmul(cf.r2, cpow_small(cf.r2L, lane)));  // k1 X0 r2^{i0 + 1}
#pragma unroll
  for (int j = 0; j < L; ++j) {
    d[j] = cscale(cadd(d[j], rg), scale);
    rg = cmul(rg, cf.r2);
  }
#pragma unroll
  for (int j = 0; j < L; ++j)
    if (j < Lk) col[j] = d[j];
  __syncthreads();
#pragma unroll 4
  for (int i = threadIdx.x; i < N * kYC; i += 32 * kYC) {
    const int r = i / kYC, c = i % kYC;
    if (c0 + c < N) PD_SPEC_ST(slab + (long long)r * N + c, sm[c * CS + r + r / L]);
  }
}

// ---------------------------------------------------------------------------------------------
// DST-I rows by a HALF-length complex FFT (r02y; replaces the length-2(N+1) odd-extension FFT of dst_rows_kernel in
// the dtri path).  For a row z_1..z_N (N1 = N + 1 a power of two, z_0 = z_N1 = 0) and s_j = sin(pi j / N1):
//   y_j = s_j (z_j + z_{N1-j}) + (z_j - z_{N1-j}) / 2,   W = FFT_N1(y)     (complex-linear in z, so complex rows work)
//   F_{2k}   = (i/2) (W_k - W_{N1-k})                        k = 1 .. N1/2 - 1
//   F_{2k+1} = W_0 / 2 + sum_{i=1..k} (W_i + W_{N1-i}) / 2   k = 0 .. N1/2 - 1   (running sum: one warp scan per row)
// give F_k = sum_j z_j sin(pi j k / N1) (the symmetric part of y transforms to F_{2k+1} - F_{2k-1}, the antisymmetric
// part to F_{2k}).  The transform is its own inverse up to N1/2, so one kernel serves both directions and the y-pass
// between them scales by 2/N1.  Half the FFT length, half the shared memory (two CTAs per SM at N1 = 512 instead of
// one), the mirror loads hit L1.  Rounding: the running sum carries ~N1/2 additions (4e-14 of max|F| at N1 = 512).
template <int N1>
struct DsthCfg {
  static constexpr int C = N1 >= 128 ? kBatch : 1024 / N1;  // rows per CTA (whole warps for the short rows)
  static constexpr int NTH = C * N1 / 16;
  static constexpr int MINB = NTH <= 128 ? 4 : 2;
};

template <int N1>
__global__ void __launch_bounds__(DsthCfg<N1>::NTH, DsthCfg<N1>::MINB)
dsth_rows_kernel(double2* __restrict__ base, long long nrows, const double2* __restrict__ twM) {
  using T = DsthCfg<N1>;
  constexpr int C = T::C, NTH = T::NTH, N = N1 - 1, R0 = first_radix(N1), RL = last_radix(N1);
  extern __shared__ double2 sm[];
  __shared__ double2 s_tws[N1 - 1];     // Stockham-ordered w_N1^k = twM[2k] (twM: the 2 N1-point table): the plain
                                        // table read at the strides m k of the second radix-16 pass is bank conflicted
  __shared__ double s_sin[N1 / 2 + 1];  // sin(pi j / N1) = -Im twM[j]
  const long long row0 = (long long)blockIdx.x * C;
  build_stockham_table<N1, 16>(s_tws, [&](int idx) { return __ldg(twM + 2 * idx); });
  for (int i = threadIdx.x; i <= N1 / 2; i += NTH) s_sin[i] = -__ldg(twM + i).y;
  __syncthreads();
  fft_io<N1, C, false, true, NTH, false, true>(
      sm, TwStockham{s_tws},
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value;
        const bool ok = row0 + c < nrows;
        const double2* q = base + (row0 + c) * N - 1;  // q[p] = z_p, p = 1..N
#pragma unroll
        for (int m = 0; m < R0; ++m) {
          const int p = j + m * s;
          if (ok && p != 0) {
            const double2 a = __ldg(q + p), b = __ldg(q + N1 - p);
            const double sj = s_sin[p <= N1 / 2 ? p : N1 - p];
            v[m] = make_double2(fma(sj, a.x + b.x, 0.5 * (a.x - b.x)), fma(sj, a.y + b.y, 0.5 * (a.y - b.y)));
          } else {
            v[m] = czero();
          }
        }
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value;
#pragma unroll
        for (int m = 0; m < RL; ++m) sm[pad(c * N1 + j + m * s)] = w[m];
      });
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int KB = (N1 / 2 + 31) / 32;
  for (int c = warp; c < C; c += NTH / 32) {
    if (row0 + c >= nrows) continue;  // warp-uniform
    double2* q = base + (row0 + c) * N - 1;  // q[m] = F_m
    double2 carry = czero();
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      const int k = lane + 32 * i;
      const bool act = k < N1 / 2;
      double2 D = czero(), Fe = czero();
      if (act) {
        const double2 Wk = sm[pad(c * N1 + k)], Wm = sm[pad(c * N1 + ((N1 - k) & (N1 - 1)))];
        D = k == 0 ? cscale(Wk, 0.5) : make_double2(0.5 * (Wk.x + Wm.x), 0.5 * (Wk.y + Wm.y));
        Fe = make_double2(-0.5 * (Wk.y - Wm.y), 0.5 * (Wk.x - Wm.x));
      }
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double tx = __shfl_up_sync(0xffffffffu, D.x, o), ty = __shfl_up_sync(0xffffffffu, D.y, o);
        if (lane >= o) D = make_double2(D.x + tx, D.y + ty);
      }
      D = cadd(D, carry);
      carry = make_double2(__shfl_sync(0xffffffffu, D.x, 31), __shfl_sync(0xffffffffu, D.y, 31));
      if (act) {
        if (k >= 1) __stcg(q + 2 * k, Fe);
        __stcg(q + 2 * k + 1, D);
      }
    }
  }
}

template <int N1>
int smem_dsth() {
  return smem_elems(DsthCfg<N1>::C * N1) * (int)sizeof(double2);
}

template <int M>
cudaError_t dst_dtri_n(double2* Sh, int nfreq, int f0g, const pd_dtri_coef* coef, const double2* tw, int chunk,
                       cudaStream_t st, int* launches) {
  using T = SlabCfg<M>;
  constexpr int N = M / 2 - 1, N1 = N + 1;
  const int smr = smem_bytes<M>(), smd = kYC * (N1 + 33) * (int)sizeof(double2);
  static int attr = -1;  // device on which the attributes were set
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (attr != dev_) {
    cudaError_t e = cudaFuncSetAttribute(dst_rows_kernel<M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smr);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(dst_rows_kernel<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smr);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(dtri_kernel<N1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smd);
    if (e != cudaSuccess) return e;
    attr = dev_;
  }
  // PD_DST_FULL=1: the length-M odd-extension FFT rows (the r02j path, kept for A/B and as a second implementation
  // in the tests); PD_DST_CHUNK_MB: slabs per launch triple (default 0 = the caller's ~1 GB chunks: L2-sized chunks,
  // whose three kernels run back to back on L2-resident slabs, measured slower - 16 / 32 / 64 / 128 MB: 3.32 / 2.97 /
  // 2.48 / 2.38 ms vs 2.27 ms per T4A L = 512 Step (b), profiles/r02y_t4a_phases.txt: sub-wave grids)
  const char* ef = getenv("PD_DST_FULL");
  const char* ec = getenv("PD_DST_CHUNK_MB");
  const bool full = ef && atoi(ef) != 0;
  const long long chunk_mb = ec ? atoll(ec) : 0;
  if (!full && chunk_mb > 0) {
    long long cs = (chunk_mb << 20) / ((long long)N * N * (long long)sizeof(double2));
    if (cs < 1) cs = 1;
    if (cs < chunk) chunk = (int)cs;
  }
  using H = DsthCfg<N1>;
  const int smh = smem_dsth<N1>();
  static int attrh = -1;
  if (attrh != dev_) {
    cudaError_t e = cudaFuncSetAttribute(dsth_rows_kernel<N1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smh);
    if (e != cudaSuccess) return e;
    attrh = dev_;
  }
  int nl = 0;
  for (int s0 = 0; s0 < nfreq; s0 += chunk) {
    const int ns = nfreq - s0 < chunk ? nfreq - s0 : chunk;
    double2* base = Sh + (long long)s0 * N * N;
    const long long nrows = (long long)ns * N;
    if (full) {
      const unsigned row_ctas = (unsigned)((nrows + T::C - 1) / T::C);
      dst_rows_kernel<M, false><<<row_ctas, T::NTH, smr, st>>>(base, nrows, tw);
      dtri_kernel<N1><<<dim3((N + kYC - 1) / kYC, ns), 32 * kYC, smd, st>>>(Sh, s0, f0g + s0, coef, 1.0 / M);
      dst_rows_kernel<M, true><<<row_ctas, T::NTH, smr, st>>>(base, nrows, tw);
    } else {
      const unsigned row_ctas = (unsigned)((nrows + H::C - 1) / H::C);
      dsth_rows_kernel<N1><<<row_ctas, H::NTH, smh, st>>>(base, nrows, tw);
      dtri_kernel<N1><<<dim3((N + kYC - 1) / kYC, ns), 32 * kYC, smd, st>>>(Sh, s0, f0g + s0, coef, 2.0 / N1);
      dsth_rows_kernel<N1><<<row_ctas, H::NTH, smh, st>>>(base, nrows, tw);
    }
    nl += 3;
  }
  if (launches) *launches = nl;
  return cudaGetLastError();
}

template <int N>
cudaError_t filter_n(double2* slab, const double2* tab, const double2* tw, cudaStream_t st) {
  using T = SlabCfg<N>;
  const int smem = smem_bytes<N>();
  static int attr = -1;  // device on which the attributes were set
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (attr != dev_) {
    cudaError_t e = cudaFuncSetAttribute(slab_rows_kernel<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(slab_rows_kernel<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(slab_cols_kernel<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cols<N>());
    if (e != cudaSuccess) return e;
    attr = dev_;
  }
  slab_rows_kernel<N, false><<<N / T::C, T::NTH, smem, st>>>(slab, tw);
  slab_cols_kernel<N, true><<<dim3(N / ColCfg<N>::C, 1), ColCfg<N>::NTH, smem_cols<N>(), st>>>(slab, 0, nullptr, nullptr, nullptr,
                                                                           nullptr, pd_slab_params{}, tw, tab);
  slab_rows_kernel<N, true><<<N / T::C, T::NTH, smem, st>>>(slab, tw);
  return cudaGetLastError();
}

}  // namespace

template <int N>
cudaError_t rows_n(double2* base, long long nrows, int inv, const double2* tw, cudaStream_t st) {
  using T = SlabCfg<N>;
  const int smem = smem_bytes<N>();
  cudaError_t e = cudaFuncSetAttribute(slab_rows_kernel<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(slab_rows_kernel<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const unsigned ctas = (unsigned)(nrows / T::C);
  if (inv)
    slab_rows_kernel<N, true><<<ctas, T::NTH, smem, st>>>(base, tw);
  else
    slab_rows_kernel<N, false><<<ctas, T::NTH, smem, st>>>(base, tw);
  return cudaGetLastError();
}

cudaError_t pd_launch_slab2d_rows(double2* base, int n, long long nrows, int inv, const double2* tw, cudaStream_t st) {
  if (nrows % kBatch) return cudaErrorInvalidValue;
  switch (n) {
    case 16: return rows_n<16>(base, nrows, inv, tw, st);
    case 32: return rows_n<32>(base, nrows, inv, tw, st);
    case 64: return rows_n<64>(base, nrows, inv, tw, st);
    case 128: return rows_n<128>(base, nrows, inv, tw, st);
    case 256: return rows_n<256>(base, nrows, inv, tw, st);
    case 512: return rows_n<512>(base, nrows, inv, tw, st);
    case 1024: return rows_n<1024>(base, nrows, inv, tw, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t pd_launch_slab2d_filter(double2* slab, int n, const double2* tab, const double2* tw, cudaStream_t st) {
  switch (n) {
    case 16: return filter_n<16>(slab, tab, tw, st);
    case 32: return filter_n<32>(slab, tab, tw, st);
    case 64: return filter_n<64>(slab, tab, tw, st);
    case 128: return filter_n<128>(slab, tab, tw, st);
    case 256: return filter_n<256>(slab, tab, tw, st);
    case 512: return filter_n<512>(slab, tab, tw, st);
    case 1024: return filter_n<1024>(slab, tab, tw, st);
    default: return cudaErrorInvalidValue;
  }
}

// setup check (host calls once): out[n] = min over (kx, ky) of |l1 + l2 kappa| / (|l1| + |l2| |kappa|)
__global__ void min_den_kernel(const double2* __restrict__ lam1, const double2* __restrict__ lam2,
                               const double* __restrict__ sx, const double* __restrict__ sn, pd_slab_params prm, int N,
                               double* __restrict__ out) {
  __shared__ double red[256];
  const int n = blockIdx.x;
  const double2 l1 = lam1[n], l2 = lam2[n];
  const double a1 = hypot(l1.x, l1.y), a2 = hypot(l2.x, l2.y);
  double m = 1e300;
  const long long NN = (long long)N * N;
  for (long long i = threadIdx.x; i < NN; i += blockDim.x) {
    const int kx = (int)(i % N), ky = (int)(i / N);
    const double2 kap = make_double2(prm.kd * (sx[kx] + sx[ky]), prm.cx * sn[kx] + prm.cy * sn[ky]);
    const double2 d = cfma(l2, kap, l1);
    m = fmin(m, hypot(d.x, d.y) / (a1 + a2 * hypot(kap.x, kap.y) + 1e-300));
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s2 = 128; s2 > 0; s2 >>= 1) {
    if (threadIdx.x < s2) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + s2]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = red[0];
}

cudaError_t pd_launch_min_den(const double2* lam1, const double2* lam2, const double* sx, const double* sn,
                              pd_slab_params prm, int n, int nfreq, double* out, cudaStream_t st) {
  min_den_kernel<<<nfreq, 256, 0, st>>>(lam1, lam2, sx, sn, prm, n, out);
  return cudaGetLastError();
}

int pd_slab2d_dst_supported(int n) {
  return n == 15 || n == 31 || n == 63 || n == 127 || n == 255 || n == 511;
}

cudaError_t pd_launch_slab2d_dst(double2* Sh, int n, int nfreq, const double2* lam1, const double2* lam2,
                                 const double* mu, const double2* tw, int chunk, cudaStream_t st, int* launches) {
  switch (n) {
    case 15: return dst_n<32>(Sh, nfreq, lam1, lam2, mu, tw, chunk, st, launches);
    case 31: return dst_n<64>(Sh, nfreq, lam1, lam2, mu, tw, chunk, st, launches);
    case 63: return dst_n<128>(Sh, nfreq, lam1, lam2, mu, tw, chunk, st, launches);
    case 127: return dst_n<256>(Sh, nfreq, lam1, lam2, mu, tw, chunk, st, launches);
    case 255: return dst_n<512>(Sh, nfreq, lam1, lam2, mu, tw, chunk, st, launches);
    case 511: return dst_n<1024>(Sh, nfreq, lam1, lam2, mu, tw, chunk, st, launches);
    default: return cudaErrorInvalidValue;
  }
}

int pd_slab2d_dtri_supported(int n) { return n == 31 || n == 63 || n == 127 || n == 255 || n == 511; }

cudaError_t pd_launch_slab2d_dtri(double2* Sh, int n, int nfreq, int f0_glob, const pd_dtri_coef* coef,
                                  const double2* tw, int chunk, cudaStream_t st, int* launches) {
  switch (n) {
    case 31: return dst_dtri_n<64>(Sh, nfreq, f0_glob, coef, tw, chunk, st, launches);
    case 63: return dst_dtri_n<128>(Sh, nfreq, f0_glob, coef, tw, chunk, st, launches);
    case 127: return dst_dtri_n<256>(Sh, nfreq, f0_glob, coef, tw, chunk, st, launches);
    case 255: return dst_dtri_n<512>(Sh, nfreq, f0_glob, coef, tw, chunk, st, launches);
    case 511: return dst_dtri_n<1024>(Sh, nfreq, f0_glob, coef, tw, chunk, st, launches);
    default: return cudaErrorInvalidValue;
  }
}

int pd_slab2d_ytri_supported(int n) { return n == 32 || n == 64 || n == 128 || n == 256 || n == 512 || n == 1024; }

cudaError_t pd_launch_slab2d_ytri(double2* Sh, int n, int nfreq, int f0_glob, const pd_ytri_coef* coef, double scale,
                                  const double2* tw, int chunk, int rows, cudaStream_t st, int* launches) {
  switch (n) {
    case 32: return ytri_n<32>(Sh, nfreq, f0_glob, coef, scale, tw, chunk, rows, st, launches);
    case 64: return ytri_n<64>(Sh, nfreq, f0_glob, coef, scale, tw, chunk, rows, st, launches);
    case 128: return ytri_n<128>(Sh, nfreq, f0_glob, coef, scale, tw, chunk, rows, st, launches);
    case 256: return ytri_n<256>(Sh, nfreq, f0_glob, coef, scale, tw, chunk, rows, st, launches);
    case 512: return ytri_n<512>(Sh, nfreq, f0_glob, coef, scale, tw, chunk, rows, st, launches);
    case 1024: return ytri_n<1024>(Sh, nfreq, f0_glob, coef, scale, tw, chunk, rows, st, launches);
    default: return cudaErrorInvalidValue;
  }
}

int pd_slab2d_supported(int n) { return n == 16 || n == 32 || n == 64 || n == 128 || n == 256 || n == 512 || n == 1024; }

int pd_slab2d_chunk(int n, int nfreq) {
  // slabs per chunk: measured on B200 (cfg4) launch-count bound below ~1 GB chunks
  const long long slab = (long long)n * n * 16;
  long long c = (1024LL << 20) / slab;
  if (c < 1) c = 1;
  if (c > nfreq) c = nfreq;
  return (int)c;
}

cudaError_t pd_launch_slab2d(double2* Sh, int n, int nfreq, const double2* lam1, const double2* lam2,
                             const double* sx, const double* sn, pd_slab_params prm, const double2* tw,
                             int chunk, int cols_only, cudaStream_t st, int* launches) {
  switch (n) {
#define PD_CASE(v) \
  case v:          \
    return launch_n<v>(Sh, nfreq, lam1, lam2, sx, sn, prm, tw, chunk, cols_only, st, launches);
    PD_CASE(16) PD_CASE(32) PD_CASE(64) PD_CASE(128) PD_CASE(256) PD_CASE(512) PD_CASE(1024)
#undef PD_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
