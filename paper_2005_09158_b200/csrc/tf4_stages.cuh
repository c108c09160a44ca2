// Generic stages of the four-step time FFT (Nt = N1 * N2), shared by tfft4.cu (1D: N2 = 64) and tfx.cu
// (2D with the x-FFT fused into the other stage: N1 = 8).  See tfft4.cu for the index maps.
#pragma once
#include "fft.cuh"

namespace pdfft_tf4 {
using namespace pdfft;

// ---------------------------------------------------------------------------------------------
// forward stage 1 (N2 = stage length, KP pairs per tile): for fixed t1 (blockIdx.y): N2-point FFT over t2 of rows t1 + N1 t2 of P pairs,
// times w_Nt^{t1 n2}; writes Y[t1][n2][pl] (scratch rows of Pc pairs).
// ---------------------------------------------------------------------------------------------
// NORM: also the per-CTA partial sum of r^2 over the tile (npart[part_off + CTA index]; reduced in fixed order by
// the caller) - the GMRES ||b|| fused into the first apply's Step (a) read of b
// tile (bx, by) of the grid ((pairs + KP - 1) / KP, N1); ntx = tiles per t1 (the NORM partial index); a __device__
// body so that the persistent fused kernel (tfx.cu) can run tiles of both stages from one task loop
// PRE() runs in every thread right before its global stores (the persistent kernel's deferred task signal)
template <int NT, int N2, int KP, bool VEC, int RM = 16, bool NORM = false, class PRE = NoHook>
PD_D void tf4_fwd_s1_tile(const double* __restrict__ r, long long S, long long p_begin, long long npairs_chunk,
                          double2* __restrict__ Y, const double* __restrict__ gam, const double2* __restrict__ tw2,
                          const double2* __restrict__ twt, double* __restrict__ npart, long long part_off, int bx, int by,
                          int ntx, PRE pre = PRE()) {
  constexpr int N1 = NT / N2, C = KP, NTH = KP * N2 / RM;
  extern __shared__ double2 sm[];
  __shared__ double2 s_tw2[N2], s_twr[N2];  // 64-point twiddles; w_Nt^{t1 n2}, n2 < 64
  __shared__ double s_g[N2];                 // Gamma of rows t1 + N1 t2
  const int t1 = by;
  const long long pl0 = (long long)bx * KP;  // pair index within the chunk
  const long long p0 = p_begin + pl0;                // global pair index
  const long long Pc = npairs_chunk;
  for (int i = threadIdx.x; i < N2; i += NTH) {
    s_tw2[i] = __ldg(tw2 + i);
    s_twr[i] = __ldg(twt + t1 * i);
    s_g[i] = __ldg(gam + t1 + N1 * i);
  }
  __syncthreads();
  const bool fullp = pl0 + KP <= Pc;
  double nacc = 0.0;
  fft_io<N2, C, false, false, NTH, false, false, RM>(
      sm, s_tw2,
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value, R0 = first_radix(N2, RM);
        const long long col = 2 * (p0 + c);
        const double* q = r + (long long)(t1 + N1 * j) * S + col;
        const long long step = (long long)N1 * s * S;
        const bool ok = fullp || pl0 + c < Pc;
        const bool okx = ok && (VEC || col < S), oky = ok && (VEC || col + 1 < S);
#pragma unroll
        for (int m = 0; m < R0; ++m) {
          const double g = s_g[j + m * s];
          double x = 0.0, y = 0.0;
          if (VEC) {
            if (ok) {
              // read once: ld.lu, 1.7 % faster than ld.cs on the cfg4 forward (r02aq); ld.cg loses 4 %
              const double2 u = __ldlu(reinterpret_cast<const double2*>(q + m * step));
              x = u.x;
              y = u.y;
            }
          } else {
            if (okx) x = __ldcs(q + m * step);
            if (oky) y = __ldcs(q + m * step + 1);
          }
          if (NORM) nacc = fma(x, x, fma(y, y, nacc));
          v[m] = make_double2(g * x, g * y);
        }
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value, RL = last_radix(N2, RM);
        pre();
        if (!(fullp || pl0 + c < Pc)) return;
        double2* q = Y + ((long long)t1 * N2 + j) * Pc + pl0 + c;
#pragma unroll
        for (int m = 0; m < RL; ++m) __stcg(q + (long long)m * s * Pc, cmul(w[m], s_twr[j + m * s]));
      });
  if constexpr (NORM) {  // fixed-order block reduction: warp trees, then warp 0 over the warp sums
    __shared__ double s_red[32];
    for (int o = 16; o > 0; o >>= 1) nacc += __shfl_down_sync(0xffffffffu, nacc, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = nacc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < NTH / 32; ++w) t += s_red[w];
      npart[part_off + (long long)by * ntx + bx] = t;
    }
  }
}

template <int NT, int N2, int KP, bool VEC, int RM = 16, bool NORM = false>
__global__ void __launch_bounds__(KP * N2 / RM) tf4_fwd_s1(const double* __restrict__ r, long long S, long long p_begin,
                                                           long long npairs_chunk, double2* __restrict__ Y,
                                                           const double* __restrict__ gam,
                                                           const double2* __restrict__ tw2,
                                                           const double2* __restrict__ twt,
                                                           double* __restrict__ npart = nullptr,
                                                           long long part_off = 0) {
  tf4_fwd_s1_tile<NT, N2, KP, VEC, RM, NORM>(r, S, p_begin, npairs_chunk, Y, gam, tw2, twt, npart, part_off, blockIdx.x,
                                             blockIdx.y, gridDim.x);
}

// Forward stage 1 reading r = sum_k cb.c[k] cb.x[k] (pd_comb_args, 16-byte aligned vectors, S even): the
// combination of the GMRES final update fused into the time FFT (one read of each basis vector instead of a
// combination sweep that writes r and a stage 1 that reads it back).  Otherwise identical to tf4_fwd_s1<VEC>.
template <int NT, int N2, int KP, int RM = 16>
__global__ void __launch_bounds__(KP * N2 / RM) tf4_fwd_s1_comb(const __grid_constant__ pd_comb_args cb, long long S,
                                                                long long p_begin, long long npairs_chunk,
                                                                double2* __restrict__ Y,
                                                                const double* __restrict__ gam,
                                                                const double2* __restrict__ tw2,
                                                                const double2* __restrict__ twt) {
  constexpr int N1 = NT / N2, C = KP, NTH = KP * N2 / RM;
  extern __shared__ double2 sm[];
  __shared__ double2 s_tw2[N2], s_twr[N2];
  __shared__ double s_g[N2];
  const int t1 = blockIdx.y;
  const long long pl0 = (long long)blockIdx.x * KP;
  const long long p0 = p_begin + pl0;
  const long long Pc = npairs_chunk;
  for (int i = threadIdx.x; i < N2; i += NTH) {
    s_tw2[i] = __ldg(tw2 + i);
    s_twr[i] = __ldg(twt + t1 * i);
    s_g[i] = __ldg(gam + t1 + N1 * i);
  }
  __syncthreads();
  const bool fullp = pl0 + KP <= Pc;
  fft_io<N2, C, false, false, NTH, false, false, RM>(
      sm, s_tw2,
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value, R0 = first_radix(N2, RM);
        const long long off = (long long)(t1 + N1 * j) * S + 2 * (p0 + c);
        const long long step = (long long)N1 * s * S;
        double2 acc[R0];
#pragma unroll
        for (int m = 0; m < R0; ++m) acc[m] = czero();
        if (fullp || pl0 + c < Pc) {
          for (int k = 0; k < cb.k; ++k) {
            const double ck = cb.c[k];
            const double* q = cb.x[k] + off;
            double2 t[R0];
#pragma unroll
            for (int m = 0; m < R0; ++m) t[m] = __ldcs(reinterpret_cast<const double2*>(q + m * step));
#pragma unroll
            for (int m = 0; m < R0; ++m) acc[m] = make_double2(fma(ck, t[m].x, acc[m].x), fma(ck, t[m].y, acc[m].y));
          }
        }
#pragma unroll
        for (int m = 0; m < R0; ++m) {
          const double g = s_g[j + m * s];
          v[m] = make_double2(g * acc[m].x, g * acc[m].y);
        }
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value, RL = last_radix(N2, RM);
        if (!(fullp || pl0 + c < Pc)) return;
        double2* q = Y + ((long long)t1 * N2 + j) * Pc + pl0 + c;
#pragma unroll
        for (int m = 0; m < RL; ++m) __stcg(q + (long long)m * s * Pc, cmul(w[m], s_twr[j + m * s]));
      });
}

// ---------------------------------------------------------------------------------------------
// inverse stage 2: for fixed t1 (blockIdx.y): N2-point inverse FFT over n2 of W[n2][t1][.], outputs
// t = t1 + N1 t2 scaled by Gamma^{-1}_t / Nt into the two real columns of each pair (MODE 1: +=).
// ---------------------------------------------------------------------------------------------
template <int NT, int N2, int KP, bool VEC, int MODE, int RM = 16, class PRE = NoHook>
PD_D void tf4_inv_s2_tile(const double2* __restrict__ W, long long S, long long p_begin, long long npairs_chunk,
                          double* __restrict__ z, const double* __restrict__ igam, const double2* __restrict__ tw2, int bx,
                          int by, PRE pre = PRE()) {
  constexpr int N1 = NT / N2, C = KP, NTH = KP * N2 / RM;
  static_assert(num_passes(N2, RM) >= 2, "the hook-filled tables need pass 0's barrier");
  extern __shared__ double2 sm[];
  __shared__ double2 s_tw2[N2];
  __shared__ double s_g[N2];  // Gamma^{-1} / Nt of rows t1 + N1 t2
  const int t1 = by;
  const long long pl0 = (long long)bx * KP;
  const long long p0 = p_begin + pl0;
  const long long Pc = npairs_chunk;
  auto tables = [&] {  // first read behind pass 0's barrier (twiddles) and in the storer (Gamma)
    for (int i = threadIdx.x; i < N2; i += NTH) {
      s_tw2[i] = __ldg(tw2 + i);
      s_g[i] = __ldg(igam + t1 + N1 * i) * (1.0 / NT);
    }
  };
  const bool fullp = pl0 + KP <= Pc;
  fft_io<N2, C, true, false, NTH, false, false, RM>(
      sm, s_tw2,
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value, R0 = first_radix(N2, RM);
        const bool ok = fullp || pl0 + c < Pc;
        const double2* q = W + ((long long)j * N1 + t1) * Pc + pl0 + c;
#pragma unroll
        for (int m = 0; m < R0; ++m) v[m] = ok ? __ldcg(q + (long long)m * s * N1 * Pc) : czero();
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value, RL = last_radix(N2, RM);
        pre();
        if (!(fullp || pl0 + c < Pc)) return;
        const long long col = 2 * (p0 + c);
        double* q = z + (long long)(t1 + N1 * j) * S + col;
        const long long step = (long long)N1 * s * S;
        const bool okx = VEC || col < S, oky = VEC || col + 1 < S;
        (void)okx;
        (void)oky;
        if constexpr (VEC && MODE) {
          // accumulate: issue all RL loads of the old values before the first store (no aliasing stall)
          double2 o[RL];
#pragma unroll
          for (int m = 0; m < RL; ++m) o[m] = __ldcs(reinterpret_cast<const double2*>(q + m * step));
#pragma unroll
          for (int m = 0; m < RL; ++m) {
            const double g = s_g[j + m * s];
            __stcs(reinterpret_cast<double2*>(q + m * step), make_double2(fma(g, w[m].x, o[m].x), fma(g, w[m].y, o[m].y)));
          }
          return;
        } else if constexpr (!VEC && MODE) {
          const bool a16 = oky && (reinterpret_cast<uintptr_t>(q) & 15) == 0;  // odd S, even t1 S: aligned rows
          if (a16) {
            double2 o[RL];
#pragma unroll
            for (int m = 0; m < RL; ++m) o[m] = __ldcs(reinterpret_cast<const double2*>(q + m * step));
#pragma unroll
            for (int m = 0; m < RL; ++m) {
              const double g = s_g[j + m * s];
              __stcs(reinterpret_cast<double2*>(q + m * step),
                     make_double2(fma(g, w[m].x, o[m].x), fma(g, w[m].y, o[m].y)));
            }
            return;
          }
          double ox[RL], oy[RL];
#pragma unroll
          for (int m = 0; m < RL; ++m) {
            ox[m] = okx ? q[m * step] : 0.0;
            oy[m] = oky ? q[m * step + 1] : 0.0;
          }
#pragma unroll
          for (int m = 0; m < RL; ++m) {
            const double g = s_g[j + m * s];
            if (okx) q[m * step] = fma(g, w[m].x, ox[m]);
            if (oky) q[m * step + 1] = fma(g, w[m].y, oy[m]);
          }
          return;
        } else {
          const bool a16 = VEC || (oky && (reinterpret_cast<uintptr_t>(q) & 15) == 0);
#pragma unroll
          for (int m = 0; m < RL; ++m) {
            const double g = s_g[j + m * s];
            double* row = q + m * step;
            if (a16) {
              __stcs(reinterpret_cast<double2*>(row), make_double2(g * w[m].x, g * w[m].y));
            } else {
              if (okx) row[0] = g * w[m].x;
              if (oky) row[1] = g * w[m].y;
            }
          }
        }
      },
      tables);
}

template <int NT, int N2, int KP, bool VEC, int MODE, int RM = 16>
__global__ void __launch_bounds__(KP * N2 / RM) tf4_inv_s2(const double2* __restrict__ W, long long S, long long p_begin,
                                                           long long npairs_chunk, double* __restrict__ z,
                                                           const double* __restrict__ igam,
                                                           const double2* __restrict__ tw2) {
  tf4_inv_s2_tile<NT, N2, KP, VEC, MODE, RM>(W, S, p_begin, npairs_chunk, z, igam, tw2, blockIdx.x, blockIdx.y);
}

template <int N>
int smem_of(int C) {
  return smem_elems(N * C) * (int)sizeof(double2);
}

}  // namespace pdfft_tf4
