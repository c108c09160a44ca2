// Steps (a) and (c) of the ParaDiag-II apply: Gamma-scaled time-axis FFTs of every spatial dof.
//
//   Step (a)  S1 = (F (x) I)(Gamma_alpha (x) I) r            eq 2.12 (P:l.813-815), Matlab fft(Gam.*b.') P:l.866-868
//   Step (c)  z  = (Gamma_alpha^{-1} (x) I)(F^* (x) I) S2     eq 2.12 (P:l.817),    Matlab invGam.*ifft(...) P:l.870-875
//
// r, z: real fp64 [Nt][S] (S spatial dofs, row stride S).  S1, S2: complex128 half spectrum [Nt/2+1][S]
// (r is real, so S_{Nt-n} = conj(S_n); reading c15).  A CTA owns a tile of 2C adjacent spatial columns
// for all Nt time levels; two real columns are packed into one complex sequence (x + i y), transformed
// with one complex FFT and separated again, so the tile is C complex FFTs of length Nt held in shared
// memory (Nt*C*16 B, <= 128 KB).  HBM traffic per apply pass = 8 B/dof read + ~8 B/dof written.
#include <algorithm>

#include "fft.cuh"
#include "kernels.h"

using namespace pdfft;

namespace {

template <int N>
struct TileCfg {
  static constexpr int TILE = N >= 4096 ? 8192 : 4096;                     // complex elements per tile
  static constexpr int C = (TILE / N) < 32 ? (TILE / N) : 32;             // complex sequences per tile
  static constexpr int E = elems_per_thread(N);
  static constexpr int NTH = C * N / E;
  static constexpr int MINB = NTH <= 256 ? 2 : 1;
};

// ---------------------------------------------------------------------------------------------
// Step (a): r (real) -> Gamma r -> FFT over time -> half spectrum.
// ---------------------------------------------------------------------------------------------
template <int N, bool SH>
__global__ void __launch_bounds__(TileCfg<N>::NTH, TileCfg<N>::MINB)
tfft_fwd_kernel(const double* __restrict__ r, const pd_spec sp, long long S,
                const double* __restrict__ gam, const double2* __restrict__ tw) {
  using T = TileCfg<N>;
  constexpr int C = T::C, NTH = T::NTH;
  constexpr bool SMT = N <= 1024;  // stage twiddles and Gamma in shared memory
  extern __shared__ double2 sm[];
  __shared__ double2 s_tw[SMT ? N : 1];
  __shared__ double s_g[SMT ? N : 1];
  const long long s0 = (long long)blockIdx.x * (2 * C);
  const double* rc = r + s0;
  const bool full = s0 + 2 * C <= S;
  if (SMT) {
    load_table(s_tw, tw, N);
    for (int i = threadIdx.x; i < N; i += NTH) s_g[i] = __ldg(gam + i);
    __syncthreads();
  }
  // pass 0 straight from HBM with Gamma fused: sequence c = columns (s0+2c) + i (s0+2c+1)
  constexpr int R0 = first_radix(N), RL = last_radix(N);
  fft_io<N, C, false, false, NTH, false, true>(
      sm, SMT ? s_tw : tw,
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value;
        const double* q = rc + (long long)j * S + 2 * c;
        const long long step = (long long)s * S;
        const bool okx = full || s0 + 2 * c < S, oky = full || s0 + 2 * c + 1 < S;
#pragma unroll
        for (int m = 0; m < R0; ++m) {
          const int t = j + m * s;
          const double g = SMT ? s_g[t] : __ldg(gam + t);
          const double x = okx ? __ldcs(q + m * step) : 0.0;
          const double y = oky ? __ldcs(q + m * step + 1) : 0.0;
          v[m] = make_double2(g * x, g * y);
        }
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value;
        const int a = lin<N, C, false>(j, c);
#pragma unroll
        for (int m = 0; m < RL; ++m) sm[soff<s * C>(a, m)] = w[m];
      });
  __syncthreads();
  // separate the two real columns: X_n = (Z_n + conj Z_{N-n})/2, Y_n = -i (Z_n - conj Z_{N-n})/2
  constexpr int NOUT = (N / 2 + 1) * 2 * C;
#pragma unroll 4
  for (int o = threadIdx.x; o < NOUT; o += NTH) {
    const int col = o % (2 * C), n = o / (2 * C), c = col >> 1;
    const double2 z1 = sm[sidx<N, C, false>(n, c)];
    const double2 z2 = sm[sidx<N, C, false>((N - n) & (N - 1), c)];
    double2 v;
    if (col & 1)
      v = make_double2(0.5 * (z1.y + z2.y), -0.5 * (z1.x - z2.x));
    else
      v = make_double2(0.5 * (z1.x + z2.x), 0.5 * (z1.y - z2.y));
    if (full || s0 + col < S) __stcs(pd_spec_row<SH>(sp, n) + s0 + col, v);
  }
}

// ---------------------------------------------------------------------------------------------
// Step (c): half spectrum -> inverse FFT over time -> Gamma^{-1}/Nt -> real.
// MODE 0: z = result.  MODE 1: z += result (fused stationary update u <- u + P^{-1} r).
// ---------------------------------------------------------------------------------------------
template <int N, int MODE, bool SH>
__global__ void __launch_bounds__(TileCfg<N>::NTH, TileCfg<N>::MINB)
tfft_inv_kernel(const pd_spec sp, double* __restrict__ z, long long S,
                const double* __restrict__ igam, const double2* __restrict__ tw) {
  using T = TileCfg<N>;
  constexpr int C = T::C, NTH = T::NTH;
  constexpr bool SMT = N <= 1024;
  extern __shared__ double2 sm[];
  __shared__ double2 s_tw[SMT ? N : 1];
  __shared__ double s_g[SMT ? N : 1];
  const long long s0 = (long long)blockIdx.x * (2 * C);
  const bool full = s0 + 2 * C <= S;
  if (SMT) {
    load_table(s_tw, tw, N);
    for (int i = threadIdx.x; i < N; i += NTH) s_g[i] = __ldg(igam + i) * (1.0 / N);
  }
  if (MODE) {  // warm L2 with the rows of z this tile will read-modify-write
    for (int t = threadIdx.x; t < N; t += NTH) asm volatile("prefetch.global.L2 [%0];" ::"l"(z + (long long)t * S + s0));
  }
  // stage the half-spectrum tile H[n][col], n = 0..N/2, col = 0..2C-1 (coalesced rows)
  constexpr int NIN = (N / 2 + 1) * 2 * C;
  {
    // all of a thread's loads in flight before the first smem store
    constexpr int PT = (NIN + NTH - 1) / NTH;
    double2 v[PT];
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      const int o = threadIdx.x + k * NTH;
      const int col = o % (2 * C), n = o / (2 * C);
      v[k] = (o < NIN && (full || s0 + col < S)) ? __ldlu(pd_spec_row<SH>(sp, n) + s0 + col) : czero();
    }
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      const int o = threadIdx.x + k * NTH;
      if (o < NIN) sm[pad(o)] = v[k];
    }
  }
  __syncthreads();
  const double invN = 1.0 / N;
  double* zc = z + s0;
  constexpr int R0 = first_radix(N), RL = last_radix(N);
  fft_io<N, C, true, false, NTH, true, false>(
      sm, SMT ? s_tw : tw,
      [&](int j, auto st, int c, double2* v) {  // Z[pos] = X[pos] + i Y[pos], X[N-n] = conj X[n]
        constexpr int s = decltype(st)::value;
#pragma unroll
        for (int m = 0; m < R0; ++m) {
          const int pos = j + m * s;
          const bool lo = pos <= N / 2;
          const int pp = lo ? pos : N - pos;
          const double sg = lo ? 1.0 : -1.0;
          const double2 X = sm[pad(pp * 2 * C + 2 * c)];
          const double2 Y = sm[pad(pp * 2 * C + 2 * c + 1)];
          // conj when pos > N/2: X = (X.x, sg X.y), Y = (Y.x, sg Y.y);  Z = X + i Y
          v[m] = make_double2(fma(-sg, Y.y, X.x), fma(sg, X.y, Y.x));
        }
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value;
        double* q = zc + (long long)j * S + 2 * c;
        const long long step = (long long)s * S;
        const bool okx = full || s0 + 2 * c < S, oky = full || s0 + 2 * c + 1 < S;
#pragma unroll
        for (int m = 0; m < RL; ++m) {
          const int t = j + m * s;
          const double g = SMT ? s_g[t] : __ldg(igam + t) * invN;
          double* row = q + m * step;
          if (MODE) {
            if (okx) row[0] = fma(g, w[m].x, row[0]);
            if (oky) row[1] = fma(g, w[m].y, row[1]);
          } else {
            if (okx) __stcs(row, g * w[m].x);
            if (oky) __stcs(row + 1, g * w[m].y);
          }
        }
      });
}

template <int N>
cudaError_t launch_fwd_n(const double* r, const pd_spec& sp, long long S, const double* gam, const double2* tw,
                         cudaStream_t st) {
  using T = TileCfg<N>;
  const int smem = smem_elems(N * T::C) * (int)sizeof(double2);
  static int attr = -1;  // device on which the attributes were set
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (attr != dev_) {
    cudaError_t e = cudaFuncSetAttribute(tfft_fwd_kernel<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(tfft_fwd_kernel<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = dev_;
  }
  const long long tiles = (S + 2 * T::C - 1) / (2 * T::C);
  if (sp.P > 1)
    tfft_fwd_kernel<N, true><<<(unsigned)tiles, T::NTH, smem, st>>>(r, sp, S, gam, tw);
  else
    tfft_fwd_kernel<N, false><<<(unsigned)tiles, T::NTH, smem, st>>>(r, sp, S, gam, tw);
  return cudaGetLastError();
}

template <int N>
cudaError_t launch_inv_n(const pd_spec& sp, double* z, long long S, const double* igam, const double2* tw,
                         int accumulate, cudaStream_t st) {
  using T = TileCfg<N>;
  const int smem = smem_elems((N / 2 + 1) * 2 * T::C) * (int)sizeof(double2);
  static int attr = -1;  // device on which the attributes were set
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (attr != dev_) {
    cudaError_t e = cudaFuncSetAttribute(tfft_inv_kernel<N, 0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(tfft_inv_kernel<N, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(tfft_inv_kernel<N, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(tfft_inv_kernel<N, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = dev_;
  }
  const long long tiles = (S + 2 * T::C - 1) / (2 * T::C);
  const bool sh = sp.P > 1;
  if (accumulate && sh)
    tfft_inv_kernel<N, 1, true><<<(unsigned)tiles, T::NTH, smem, st>>>(sp, z, S, igam, tw);
  else if (accumulate)
    tfft_inv_kernel<N, 1, false><<<(unsigned)tiles, T::NTH, smem, st>>>(sp, z, S, igam, tw);
  else if (sh)
    tfft_inv_kernel<N, 0, true><<<(unsigned)tiles, T::NTH, smem, st>>>(sp, z, S, igam, tw);
  else
    tfft_inv_kernel<N, 0, false><<<(unsigned)tiles, T::NTH, smem, st>>>(sp, z, S, igam, tw);
  return cudaGetLastError();
}

// Nt = 1 (S:l.89; reading t2): a 1 x 1 alpha-circulant has no wrap entry, Gamma = [1] and the DFT of length 1 is
// the identity, so Steps (a) / (c) only move the real column into / out of the complex spectrum buffer.
__global__ void tfft1_fwd_kernel(const double* __restrict__ r, double2* __restrict__ Sh, long long S) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < S; i += (long long)gridDim.x * blockDim.x)
    Sh[i] = make_double2(r[i], 0.0);
}
__global__ void tfft1_inv_kernel(const double2* __restrict__ Sh, double* __restrict__ z, long long S, int acc) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < S; i += (long long)gridDim.x * blockDim.x)
    z[i] = acc ? z[i] + Sh[i].x : Sh[i].x;
}
unsigned blocks1(long long S) { return (unsigned)std::min<long long>((S + 255) / 256, 148 * 8); }

}  // namespace

int pd_tfft_supported(int nt) { return nt >= 1 && nt <= 8192 && (nt & (nt - 1)) == 0; }

cudaError_t pd_launch_tfft_fwd(int nt, const double* r, const pd_spec& sp, long long S, const double* gam,
                               const double2* tw, cudaStream_t st) {
  if (nt == 1) {
    tfft1_fwd_kernel<<<blocks1(S), 256, 0, st>>>(r, pd_spec_row(sp, 0), S);
    return cudaGetLastError();
  }
  switch (nt) {
#define PD_CASE(n) \
  case n:          \
    return launch_fwd_n<n>(r, sp, S, gam, tw, st);
    PD_CASE(2) PD_CASE(4) PD_CASE(8) PD_CASE(16) PD_CASE(32) PD_CASE(64) PD_CASE(128) PD_CASE(256)
    PD_CASE(512) PD_CASE(1024) PD_CASE(2048) PD_CASE(4096) PD_CASE(8192)
#undef PD_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t pd_launch_tfft_inv(int nt, const pd_spec& sp, double* z, long long S, const double* igam,
                               const double2* tw, int accumulate, cudaStream_t st) {
  if (nt == 1) {
    tfft1_inv_kernel<<<blocks1(S), 256, 0, st>>>(pd_spec_row(sp, 0), z, S, accumulate);
    return cudaGetLastError();
  }
  switch (nt) {
#define PD_CASE(n) \
  case n:          \
    return launch_inv_n<n>(sp, z, S, igam, tw, accumulate, st);
    PD_CASE(2) PD_CASE(4) PD_CASE(8) PD_CASE(16) PD_CASE(32) PD_CASE(64) PD_CASE(128) PD_CASE(256)
    PD_CASE(512) PD_CASE(1024) PD_CASE(2048) PD_CASE(4096) PD_CASE(8192)
#undef PD_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
