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
#include "fft.cuh"
#include "kernels.h"

using namespace pdfft;

namespace {

template <int N>
struct TileCfg {
  static constexpr int C = (8192 / N) < 32 ? (8192 / N) : 32;  // complex sequences per tile
  static constexpr int E = elems_per_thread(N);
  static constexpr int NTH = C * N / E;
  static constexpr int R0 = radix_of(N, 0);
  static constexpr int P = num_passes(N);
};

// ---------------------------------------------------------------------------------------------
// Step (a): r (real) -> Gamma r -> FFT over time -> half spectrum.
// ---------------------------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(TileCfg<N>::NTH)
tfft_fwd_kernel(const double* __restrict__ r, double2* __restrict__ Sh, long long S,
                const double* __restrict__ gam, const double2* __restrict__ tw) {
  using T = TileCfg<N>;
  constexpr int C = T::C, NTH = T::NTH, R0 = T::R0;
  extern __shared__ double2 sm[];
  const long long s0 = (long long)blockIdx.x * (2 * C);

  // pass 0 straight from HBM (LS = 1: no inter-pass twiddles), Gamma fused into the load
  {
    constexpr int BPT = (C * N / R0) / NTH;
    double2 v[BPT][R0];
#pragma unroll
    for (int bi = 0; bi < BPT; ++bi) {
      const int b = threadIdx.x + bi * NTH;
      const int c = b % C, j = b / C;
      const long long col = s0 + 2 * c;
#pragma unroll
      for (int m = 0; m < R0; ++m) {
        const int t = j + m * (N / R0);
        const double g = __ldg(gam + t);
        const double* row = r + (long long)t * S;
        const double x = col < S ? __ldcs(row + col) : 0.0;
        const double y = col + 1 < S ? __ldcs(row + col + 1) : 0.0;
        v[bi][m] = make_double2(g * x, g * y);
      }
    }
#pragma unroll
    for (int bi = 0; bi < BPT; ++bi) {
      const int b = threadIdx.x + bi * NTH;
      const int c = b % C, j = b / C;
      DFT<R0, false>::run(v[bi]);
#pragma unroll
      for (int q = 0; q < R0; ++q) sm[sidx<N, C, false>(j * R0 + q, c)] = v[bi][q];
    }
    __syncthreads();
  }
  Passes<N, C, 1, T::P, false, false, NTH>::run(sm, tw);

  // separate the two real columns: X_n = (Z_n + conj Z_{N-n})/2, Y_n = -i (Z_n - conj Z_{N-n})/2
  constexpr int NOUT = (N / 2 + 1) * 2 * C;
  for (int o = threadIdx.x; o < NOUT; o += NTH) {
    const int col = o % (2 * C), n = o / (2 * C), c = col >> 1;
    const double2 z1 = sm[sidx<N, C, false>(n, c)];
    const double2 z2 = sm[sidx<N, C, false>((N - n) & (N - 1), c)];
    double2 out;
    if (col & 1)
      out = make_double2(0.5 * (z1.y + z2.y), -0.5 * (z1.x - z2.x));
    else
      out = make_double2(0.5 * (z1.x + z2.x), 0.5 * (z1.y - z2.y));
    if (s0 + col < S) Sh[(long long)n * S + s0 + col] = out;
  }
}

// ---------------------------------------------------------------------------------------------
// Step (c): half spectrum -> inverse FFT over time -> Gamma^{-1}/Nt -> real.
// MODE 0: z = result.  MODE 1: z += result (fused stationary update u <- u + P^{-1} r).
// ---------------------------------------------------------------------------------------------
template <int N, int MODE>
__global__ void __launch_bounds__(TileCfg<N>::NTH)
tfft_inv_kernel(const double2* __restrict__ Sh, double* __restrict__ z, long long S,
                const double* __restrict__ igam, const double2* __restrict__ tw) {
  using T = TileCfg<N>;
  constexpr int C = T::C, NTH = T::NTH, R0 = T::R0, P = T::P;
  extern __shared__ double2 sm[];
  const long long s0 = (long long)blockIdx.x * (2 * C);

  // load the half-spectrum tile H[n][col], n = 0..N/2, col = 0..2C-1
  constexpr int NIN = (N / 2 + 1) * 2 * C;
  for (int o = threadIdx.x; o < NIN; o += NTH) {
    const int col = o % (2 * C), n = o / (2 * C);
    sm[pad(o)] = (s0 + col < S) ? __ldcs(Sh + (long long)n * S + s0 + col) : czero();
  }
  __syncthreads();

  constexpr int BPT = (C * N / R0) / NTH;
  double2 v[BPT][R0];
  // pass 0 input: Z[pos] = X[pos] + i Y[pos], with X[N-n] = conj X[n] for n > N/2
#pragma unroll
  for (int bi = 0; bi < BPT; ++bi) {
    const int b = threadIdx.x + bi * NTH;
    const int c = b % C, j = b / C;
#pragma unroll
    for (int m = 0; m < R0; ++m) {
      const int pos = j + m * (N / R0);
      double2 X, Y;
      if (pos <= N / 2) {
        X = sm[pad(pos * 2 * C + 2 * c)];
        Y = sm[pad(pos * 2 * C + 2 * c + 1)];
      } else {
        X = cconj(sm[pad((N - pos) * 2 * C + 2 * c)]);
        Y = cconj(sm[pad((N - pos) * 2 * C + 2 * c + 1)]);
      }
      v[bi][m] = make_double2(X.x - Y.y, X.y + Y.x);
    }
  }
  __syncthreads();
  const double invN = 1.0 / N;
  if constexpr (P == 1) {
    // single pass: output natural order, write HBM directly
#pragma unroll
    for (int bi = 0; bi < BPT; ++bi) {
      const int b = threadIdx.x + bi * NTH;
      const int c = b % C;
      DFT<R0, true>::run(v[bi]);
      const long long col = s0 + 2 * c;
#pragma unroll
      for (int q = 0; q < R0; ++q) {
        const double g = __ldg(igam + q) * invN;
        double* row = z + (long long)q * S;
        if (col < S) row[col] = MODE ? row[col] + g * v[bi][q].x : g * v[bi][q].x;
        if (col + 1 < S) row[col + 1] = MODE ? row[col + 1] + g * v[bi][q].y : g * v[bi][q].y;
      }
    }
    return;
  } else {
#pragma unroll
    for (int bi = 0; bi < BPT; ++bi) {
      const int b = threadIdx.x + bi * NTH;
      const int c = b % C, j = b / C;
      DFT<R0, true>::run(v[bi]);
#pragma unroll
      for (int q = 0; q < R0; ++q) sm[sidx<N, C, false>(j * R0 + q, c)] = v[bi][q];
    }
    __syncthreads();
    Passes<N, C, 1, P - 1, true, false, NTH>::run(sm, tw);

    // last pass: smem -> registers -> HBM (output position j + q*LS, LS = N/R)
    constexpr int RL = radix_of(N, P - 1), LS = ls_of(N, P - 1);
    constexpr int BL = (C * N / RL) / NTH;
    double2 w[BL][RL];
#pragma unroll
    for (int bi = 0; bi < BL; ++bi) {
      const int b = threadIdx.x + bi * NTH;
      const int c = b % C, j = b / C;
#pragma unroll
      for (int m = 0; m < RL; ++m) w[bi][m] = sm[sidx<N, C, false>(j + m * (N / RL), c)];
    }
#pragma unroll
    for (int bi = 0; bi < BL; ++bi) {
      const int b = threadIdx.x + bi * NTH;
      const int c = b % C, j = b / C;
      pass_twiddles<N, RL, LS, true>(w[bi], j, tw);
      DFT<RL, true>::run(w[bi]);
      const long long col = s0 + 2 * c;
#pragma unroll
      for (int q = 0; q < RL; ++q) {
        const int t = j + q * LS;
        const double g = __ldg(igam + t) * invN;
        double* row = z + (long long)t * S;
        if (col < S) row[col] = MODE ? row[col] + g * w[bi][q].x : g * w[bi][q].x;
        if (col + 1 < S) row[col + 1] = MODE ? row[col + 1] + g * w[bi][q].y : g * w[bi][q].y;
      }
    }
  }
}

template <int N>
cudaError_t launch_fwd_n(const double* r, double2* Sh, long long S, const double* gam, const double2* tw,
                         cudaStream_t st) {
  using T = TileCfg<N>;
  const int smem = smem_elems(N * T::C) * (int)sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tfft_fwd_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long tiles = (S + 2 * T::C - 1) / (2 * T::C);
  tfft_fwd_kernel<N><<<(unsigned)tiles, T::NTH, smem, st>>>(r, Sh, S, gam, tw);
  return cudaGetLastError();
}

template <int N>
cudaError_t launch_inv_n(const double2* Sh, double* z, long long S, const double* igam, const double2* tw,
                         int accumulate, cudaStream_t st) {
  using T = TileCfg<N>;
  const int smem = smem_elems((N / 2 + 1) * 2 * T::C) * (int)sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tfft_inv_kernel<N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(tfft_inv_kernel<N, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const long long tiles = (S + 2 * T::C - 1) / (2 * T::C);
  if (accumulate)
    tfft_inv_kernel<N, 1><<<(unsigned)tiles, T::NTH, smem, st>>>(Sh, z, S, igam, tw);
  else
    tfft_inv_kernel<N, 0><<<(unsigned)tiles, T::NTH, smem, st>>>(Sh, z, S, igam, tw);
  return cudaGetLastError();
}

}  // namespace

int pd_tfft_supported(int nt) { return nt >= 2 && nt <= 8192 && (nt & (nt - 1)) == 0; }

cudaError_t pd_launch_tfft_fwd(int nt, const double* r, double2* Sh, long long S, const double* gam,
                               const double2* tw, cudaStream_t st) {
  switch (nt) {
#define PD_CASE(n) \
  case n:          \
    return launch_fwd_n<n>(r, Sh, S, gam, tw, st);
    PD_CASE(2) PD_CASE(4) PD_CASE(8) PD_CASE(16) PD_CASE(32) PD_CASE(64) PD_CASE(128) PD_CASE(256)
    PD_CASE(512) PD_CASE(1024) PD_CASE(2048) PD_CASE(4096) PD_CASE(8192)
#undef PD_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t pd_launch_tfft_inv(int nt, const double2* Sh, double* z, long long S, const double* igam,
                               const double2* tw, int accumulate, cudaStream_t st) {
  switch (nt) {
#define PD_CASE(n) \
  case n:          \
    return launch_inv_n<n>(Sh, z, S, igam, tw, accumulate, st);
    PD_CASE(2) PD_CASE(4) PD_CASE(8) PD_CASE(16) PD_CASE(32) PD_CASE(64) PD_CASE(128) PD_CASE(256)
    PD_CASE(512) PD_CASE(1024) PD_CASE(2048) PD_CASE(4096) PD_CASE(8192)
#undef PD_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
