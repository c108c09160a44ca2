// Steps (a)/(c) for the 2D periodic problem with the spatial x-FFT of Step (b) folded in.
//
// Step (b) in 2D solves every slab by 2D FFT -> divide -> 2D IFFT (slab2d.cu, reading c14).  The x-FFT
// of the forward 2D FFT commutes with the time DFT of Step (a), and the x-IFFT with that of Step (c), so
// they are done inside the time-FFT kernels: the spectrum buffer then holds X_n[y][kx] (x already
// transformed) and Step (b) is a single column pass (y-FFT, divide, y-IFFT).  That removes two full
// read+write sweeps of the F x N^2 complex spectrum per apply.
//
// Four-step time FFT with N1 = 8, N2 = Nt/8 (index maps as in tfft4.cu, eq 2.12, P:l.813-817):
//   forward  stage 1 (tf4_stages.cuh): N2-point FFTs over t2, twiddle w_Nt^{t1 n2}      -> Y[t1][n2][pair]
//   forward  stage 2 (here): per (y-row, residue pair n2 / N2-n2): N1-point FFTs over t1 of the 2 x NX/2
//            packed pair sequences (pair p = real columns 2p, 2p+1, reading c15), then NX/2-point FFTs
//            over p of the 16 rows, then the even/odd untangle that yields the x-spectrum directly:
//              A_n = FFT_p(Z_n),  E_n[k] = (A_n[k] + conj A_{Nt-n}[-k]) / 2  (= FFT_p of column 2p of U_n)
//              O_n[k] = (A_n[k] - conj A_{Nt-n}[-k]) / 2i                     (= FFT_p of column 2p+1)
//              X_n[kx] = E_n[kx mod NX/2] + w_NX^kx O_n[kx mod NX/2]           for n <= Nt/2
//   inverse  stage 1 (here): the same maps backwards (E = X[k] + X[k+NX/2], O = (X[k] - X[k+NX/2]) w^-k,
//            A = E + iO; the mirror rows n > Nt/2 from Hermitian symmetry in time), NX/2-point IFFTs over
//            p, N1-point IFFTs over n1, twiddle w_Nt^{-t1 n2}                  -> W[n2][t1][pair]
//   inverse  stage 2 (tf4_stages.cuh): N2-point IFFTs over n2, Gamma^{-1}/Nt, real columns out.
// A stage-2 / inverse stage-1 tile is one full x-row (NX/2 pairs) x 16 rows of length NX/2: 8 NX complex.
// All transforms are unnormalised (the slab column pass scales by 1/N^2, as before).
#include <cstdlib>

#include "kernels.h"
#include "tf4_stages.cuh"

// spectrum rows read once by the inverse stage 1: ld.lu (last use) measured 1 % faster than evict-first ld.cs (r02aq);
// ld.cg loses 3 % (the retained lines push the four-step scratch out of L2)
#define PD_TFX_SPEC_LD(p) __ldlu(p)
using namespace pdfft;
using namespace pdfft_tf4;

namespace {

constexpr int kN1 = 8;
constexpr int kRM = 8;  // the N1 = 8 point DFTs: one radix-8 pass
#ifndef PD_TFX_RM
#define PD_TFX_RM 16    // radix cap of the NX/2-point x-direction FFTs (8: NTH = NX, 16: NTH = NX/2)
#endif
#ifndef PD_TFX_S1_RM
#define PD_TFX_S1_RM 16 // radix cap of the N2-point stage FFTs (tf4_stages.cuh)
#endif
constexpr int kRX = PD_TFX_RM;
#ifndef PD_TFX_MINB
#define PD_TFX_MINB 2   // min resident CTAs per SM (1: 144 regs, one CTA, measured 20 % slower; 3 spills)
#endif
#ifndef PD_TFX_TWX_SMEM
#define PD_TFX_TWX_SMEM 1  // NX-point twiddles staged in smem (0: read through L1)
#endif
#ifndef PD_TFX_XFIRST
#define PD_TFX_XFIRST 1    // x-FFT before the N1-point time DFT (tfx_fwd_s2x / tfx_inv_s1x); 0: the t1-first kernels
#endif
#ifndef PD_TFX_XFIRST_FWD
#define PD_TFX_XFIRST_FWD PD_TFX_XFIRST
#endif
#ifndef PD_TFX_XFIRST_INV
#define PD_TFX_XFIRST_INV PD_TFX_XFIRST
#endif
#ifndef PD_TFX_KPT
#define PD_TFX_KPT 4096  // elements of a stage-1 tile (N2 x KP pairs), Nt >= 1024
#endif
#ifndef PD_TFX_KPT_SMALL
#define PD_TFX_KPT_SMALL 2048  // Nt <= 512 (cfg3: 0.091 / 0.085 ms fwd / inv vs 0.095 / 0.092 with 4096, r02g)
#endif
__host__ __device__ constexpr int tfx_kpt(int nt) { return nt <= 512 ? PD_TFX_KPT_SMALL : PD_TFX_KPT; }
constexpr int kRS = PD_TFX_S1_RM;

template <int NT, int NX>
struct Fx {
  static constexpr int N1 = kN1, N2 = NT / kN1, NP = NX / 2, C = 2 * NP, NTH = 8 * NX / kRX;
  static constexpr int ROWS = 2 * N1;                 // rows (n1, set) of NP values
  static constexpr int SMEM = smem_elems(ROWS * NP);  // complex elements
  static constexpr int KP = tfx_kpt(NT) / N2 < 8 ? 8 : tfx_kpt(NT) / N2;  // stage-1 pairs per tile (N2 * KP = KPT)
};

// ---------------------------------------------------------------------------------------------
// forward stage 2 + x-FFT
// ---------------------------------------------------------------------------------------------
template <int NT, int NX, bool SH>
__global__ void __launch_bounds__(Fx<NT, NX>::NTH, PD_TFX_MINB) tfx_fwd_s2(const double2* __restrict__ Y, long long S,
                                                             long long p_begin, long long Pc,
                                                             const pd_spec sp,
                                                             const double2* __restrict__ twx) {
  using F = Fx<NT, NX>;
  constexpr int N1 = F::N1, N2 = F::N2, NP = F::NP, C = F::C, NTH = F::NTH;
  extern __shared__ double2 sm[];
  __shared__ double2 s_twx[PD_TFX_TWX_SMEM ? NX : 1], s_twp[NP];
  const int n2 = blockIdx.y, n2p = (N2 - n2) % N2;
  const long long pl0 = (long long)blockIdx.x * NP;  // first pair of this x-row within the chunk
  const long long p0 = p_begin + pl0;
  for (int i = threadIdx.x; i < NX; i += NTH) {
    const double2 w = __ldg(twx + i);
    if (PD_TFX_TWX_SMEM) s_twx[i] = w;
    if (!(i & 1)) s_twp[i >> 1] = w;
  }
  // (1) N1-point DFTs over t1 of the sequences c = (set, p); row (n1, set) keeps p contiguous
  fft_io<N1, C, false, false, NTH, false, true, kRM>(
      sm, s_twp,
      [&](int, auto, int c, double2* v) {
        const int rr = c < NP ? n2 : n2p, pc = c & (NP - 1);
        const double2* q = Y + (long long)rr * Pc + pl0 + pc;
#pragma unroll
        for (int m = 0; m < N1; ++m) v[m] = __ldcg(q + (long long)m * N2 * Pc);
      },
      [&](int, auto, int c, const double2* w) {
        const int set = c < NP ? 0 : 1, pc = c & (NP - 1);
#pragma unroll
        for (int m = 0; m < N1; ++m) sm[pad((2 * m + set) * NP + pc)] = w[m];
      });
  __syncthreads();
  // (2) NP-point FFTs over p of the 16 rows, in place
  fft_io<NP, 2 * N1, false, true, NTH, true, true, kRX>(
      sm, s_twp,
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value, R0 = first_radix(NP, kRX);
#pragma unroll
        for (int m = 0; m < R0; ++m) v[m] = sm[pad(c * NP + j + m * s)];
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value, RL = last_radix(NP, kRX);
#pragma unroll
        for (int m = 0; m < RL; ++m) sm[pad(c * NP + j + m * s)] = w[m];
      });
  __syncthreads();
  // (3) untangle the two real columns of each pair and combine the even/odd halves into X_n[kx]
  // row-level index work hoisted out of the element loop (uniform across the CTA)
  const int nsets = n2p == n2 ? 1 : 2;
  for (int rowi = 0; rowi < nsets * N1; ++rowi) {
    const int set = rowi / N1, n1 = rowi % N1;
    const int n = (set ? n2p : n2) + N2 * n1;
    if (n > NT / 2) continue;
    const int m = (NT - n) & (NT - 1);
    const int setp = (m % N2) == n2 ? 0 : 1, n1p = m / N2;
    const int ra = (2 * n1 + set) * NP, rb = (2 * n1p + setp) * NP;
    double2* out = pd_spec_row<SH>(sp, n) + 2 * p0;
#pragma unroll
    for (int kx = threadIdx.x; kx < NX; kx += NTH) {
      const int k = kx & (NP - 1);
      const double2 a = sm[pad(ra + k)];
      const double2 b = sm[pad(rb + ((NP - k) & (NP - 1)))];
      const double2 E = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));     // (a + conj b) / 2
      const double2 O = make_double2(0.5 * (a.y + b.y), -0.5 * (a.x - b.x));    // (a - conj b) / 2i
      __stcs(out + kx, cfma(PD_TFX_TWX_SMEM ? s_twx[kx] : __ldg(twx + kx), O, E));
    }
  }
}

// ---------------------------------------------------------------------------------------------
// x-IFFT + inverse stage 1
// ---------------------------------------------------------------------------------------------
template <int NT, int NX, bool SH>
__global__ void __launch_bounds__(Fx<NT, NX>::NTH, PD_TFX_MINB) tfx_inv_s1(const pd_spec sp, long long S,
                                                             long long p_begin, long long Pc,
                                                             double2* __restrict__ W,
                                                             const double2* __restrict__ twx,
                                                             const double2* __restrict__ twt) {
  using F = Fx<NT, NX>;
  constexpr int N1 = F::N1, N2 = F::N2, NP = F::NP, C = F::C, NTH = F::NTH;
  extern __shared__ double2 sm[];
  __shared__ double2 s_twx[PD_TFX_TWX_SMEM ? NX : 1], s_twp[NP], s_twa[N1], s_twb[N1];
  const int n2 = blockIdx.y, n2p = (N2 - n2) % N2;
  const long long pl0 = (long long)blockIdx.x * NP;
  const long long p0 = p_begin + pl0;
  for (int i = threadIdx.x; i < NX; i += NTH) {
    const double2 w = __ldg(twx + i);
    if (PD_TFX_TWX_SMEM) s_twx[i] = w;
    if (!(i & 1)) s_twp[i >> 1] = w;
  }
  if (threadIdx.x < N1) {
    s_twa[threadIdx.x] = cconj(__ldg(twt + threadIdx.x * n2));
    s_twb[threadIdx.x] = cconj(__ldg(twt + threadIdx.x * n2p));
  }
  __syncthreads();
  // (0) rows n <= Nt/2 of the residue set -> A_n = E_n + i O_n and the mirror row A_{Nt-n}[-k]
  // all of a thread's row loads are issued before any use (up to 2 N1 rows x 2 halves in flight)
  const int nsets = n2p == n2 ? 1 : 2;
  for (int k = threadIdx.x; k < NP; k += NTH) {
    double2 x0[2 * N1], x1[2 * N1];
#pragma unroll
    for (int r = 0; r < 2 * N1; ++r) {
      const int set = r / N1, n1 = r % N1;
      const int n = (set ? n2p : n2) + N2 * n1;
      if (set < nsets && n <= NT / 2) {
        const double2* q = pd_spec_row<SH>(sp, n) + 2 * p0 + k;
        x0[r] = __ldcs(q);
        x1[r] = __ldcs(q + NP);
      }
    }
    const double2 wk = PD_TFX_TWX_SMEM ? s_twx[k] : __ldg(twx + k);
#pragma unroll
    for (int r = 0; r < 2 * N1; ++r) {
      const int set = r / N1, n1 = r % N1;
      const int n = (set ? n2p : n2) + N2 * n1;
      if (!(set < nsets && n <= NT / 2)) continue;
      const double2 E = cadd(x0[r], x1[r]);
      const double2 O = cmulc(csub(x0[r], x1[r]), wk);  // (x0 - x1) w^-k
      sm[pad((2 * n1 + set) * NP + k)] = make_double2(E.x - O.y, E.y + O.x);
      if (n != 0 && n != NT / 2) {
        const int m = NT - n;
        const int setp = (m % N2) == n2 ? 0 : 1, n1p = m / N2;
        sm[pad((2 * n1p + setp) * NP + ((NP - k) & (NP - 1)))] = make_double2(E.x + O.y, O.x - E.y);
      }
    }
  }
  __syncthreads();
  // (1) NP-point inverse FFTs over p of the 16 rows, in place
  fft_io<NP, 2 * N1, true, true, NTH, true, true, kRX>(
      sm, s_twp,
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value, R0 = first_radix(NP, kRX);
#pragma unroll
        for (int m = 0; m < R0; ++m) v[m] = sm[pad(c * NP + j + m * s)];
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value, RL = last_radix(NP, kRX);
#pragma unroll
        for (int m = 0; m < RL; ++m) sm[pad(c * NP + j + m * s)] = w[m];
      });
  __syncthreads();
  // (2) N1-point inverse DFTs over n1 of the sequences (set, p), twiddle, out to W[n2][t1][pair]
  fft_io<N1, C, true, false, NTH, true, false, kRM>(
      sm, s_twp,
      [&](int, auto, int c, double2* v) {
        const int set = c < NP ? 0 : 1, pc = c & (NP - 1);
#pragma unroll
        for (int m = 0; m < N1; ++m) v[m] = sm[pad((2 * m + set) * NP + pc)];
      },
      [&](int, auto, int c, const double2* w) {
        const int set = c < NP ? 0 : 1, pc = c & (NP - 1);
        if (set == 1 && nsets == 1) return;  // duplicate of the self-partnered residue
        const int rr = set ? n2p : n2;
        const double2* tws = set ? s_twb : s_twa;
        double2* q = W + (long long)rr * N1 * Pc + pl0 + pc;
#pragma unroll
        for (int m = 0; m < N1; ++m) __stcg(q + (long long)m * Pc, cmul(w[m], tws[m]));
      });
}

// ---------------------------------------------------------------------------------------------
// x-first variants (PD_TFX_XFIRST): the N1-point DFT over t1 commutes with the NP-point FFT over p
// (the four-step twiddle w_Nt^{t1 n2} is already applied in stage 1 / applied after, per row), so the
// x-FFT runs first and one thread per index k then does the N1-point DFTs of column k of residue set 0
// and of the mirror column NP - k of the partner set, which is exactly what the even/odd untangle pairs
// (row n with row Nt - n at index -k).  The untangle and the N1-point DFTs stay in registers: 2 smem
// writes + 2 reads per element instead of 3 + 3.
// ---------------------------------------------------------------------------------------------
// Mirror rows: n = r + N2 n1 of residue r has Nt - n = (N2 - r) + N2 (N1 - 1 - n1) for r > 0 (the partner
// set) and N2 ((N1 - n1) mod N1) for r = 0 (the same set).
// X_n[i] = E + w^i O, X_n[i + NP] = E - w^i O;  E = (x + conj y) / 2, O = (x - conj y) / 2i, y = A_{Nt-n}[-i]
template <int NP>
PD_D void untangle_store(double2* out, int i, double2 x, double2 y, double2 w) {
  const double2 E = make_double2(0.5 * (x.x + y.x), 0.5 * (x.y - y.y));
  const double2 O = make_double2(0.5 * (x.y + y.y), -0.5 * (x.x - y.x));
  const double2 wO = cmul(w, O);
  __stcs(out + i, cadd(E, wO));
  __stcs(out + i + NP, csub(E, wO));
}

template <int NT, int NX, bool SH, class PRE = NoHook>
PD_D void tfx_fwd_s2x_tile(const double2* __restrict__ Y, long long S, long long p_begin, long long Pc, const pd_spec& sp,
                           const double2* __restrict__ twx, int bx, int by, PRE pre = PRE()) {
  using F = Fx<NT, NX>;
  constexpr int N1 = F::N1, N2 = F::N2, NP = F::NP, NTH = F::NTH;
  extern __shared__ double2 sm[];
  __shared__ double2 s_twx[NP], s_tws[NP - 1];
  const int n2 = by, n2p = (N2 - n2) % N2, nsets = n2p == n2 ? 1 : 2;
  const long long pl0 = (long long)bx * NP;
  const long long p0 = p_begin + pl0;
  // (1) NP-point FFTs over p of the 2 N1 rows c = (set, t1) straight from Y[t1][n2][pair]; the twiddle
  // tables are filled by the hook, after the tile loads are in flight (first used behind pass 0's barrier)
  auto tables = [&] {
    for (int i = threadIdx.x; i < NP; i += NTH) s_twx[i] = __ldg(twx + i);
    build_stockham_table<NP, kRX>(s_tws, [&](int idx) { return __ldg(twx + 2 * idx); });
  };
  fft_io<NP, 2 * N1, false, true, NTH, false, true, kRX>(
      sm, TwStockham{s_tws},
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value, R0 = first_radix(NP, kRX);
        const int set = c / N1, t1 = c % N1;
        const double2* q = Y + ((long long)t1 * N2 + (set ? n2p : n2)) * Pc + pl0 + j;
#pragma unroll
        for (int m = 0; m < R0; ++m) v[m] = __ldcg(q + m * s);
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value, RL = last_radix(NP, kRX);
#pragma unroll
        for (int m = 0; m < RL; ++m) sm[pad(c * NP + j + m * s)] = w[m];
      },
      tables);
  __syncthreads();
  pre();
  // (2) N1-point DFTs over t1 of column k (set 0) and column NP - k (partner set), untangle, store
  const int sb = nsets == 2 ? 1 : 0;
  for (int k = threadIdx.x; k < NP; k += NTH) {
    const int kb = (NP - k) & (NP - 1);
    double2 a[N1], b[N1];
#pragma unroll
    for (int t = 0; t < N1; ++t) {
      a[t] = sm[pad(t * NP + k)];
      b[t] = sm[pad((sb * N1 + t) * NP + kb)];
    }
    DFT<N1, false>::run(a);
    DFT<N1, false>::run(b);
    const double2 wk = s_twx[k], wb = s_twx[kb];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const int n = n2 + N2 * n1;
      if (n <= NT / 2) {
        const double2 y = n2 == 0 ? b[(N1 - n1) & (N1 - 1)] : b[N1 - 1 - n1];
        untangle_store<NP>(pd_spec_row<SH>(sp, n) + 2 * p0, k, a[n1], y, wk);
      }
    }
    if (nsets == 2) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int n = n2p + N2 * n1;
        if (n <= NT / 2) untangle_store<NP>(pd_spec_row<SH>(sp, n) + 2 * p0, kb, b[n1], a[N1 - 1 - n1], wb);
      }
    }
  }
}

template <int NT, int NX, bool SH>
__global__ void __launch_bounds__(Fx<NT, NX>::NTH, PD_TFX_MINB) tfx_fwd_s2x(const double2* __restrict__ Y, long long S,
                                                              long long p_begin, long long Pc,
                                                              const pd_spec sp,
                                                              const double2* __restrict__ twx) {
  tfx_fwd_s2x_tile<NT, NX, SH>(Y, S, p_begin, Pc, sp, twx, blockIdx.x, blockIdx.y);
}

// A_n[i] = E + iO from X_n[i], X_n[i + NP]:  E = x0 + x1, O = (x0 - x1) w^-i;  the mirror row
// A_{Nt-n}[-i] = conj(E - iO)
PD_D double2 a_direct(double2 x0, double2 x1, double2 wi) {
  const double2 E = cadd(x0, x1), O = cmulc(csub(x0, x1), wi);
  return make_double2(E.x - O.y, E.y + O.x);
}
PD_D double2 a_mirror(double2 x0, double2 x1, double2 wi) {
  const double2 E = cadd(x0, x1), O = cmulc(csub(x0, x1), wi);
  return make_double2(E.x + O.y, O.x - E.y);
}

template <int NT, int NX, bool SH, class PRE = NoHook>
PD_D void tfx_inv_s1x_tile(const pd_spec& sp, long long S, long long p_begin, long long Pc, double2* __restrict__ W,
                           const double2* __restrict__ twx, const double2* __restrict__ twt, int bx, int by,
                           PRE pre = PRE()) {
  using F = Fx<NT, NX>;
  constexpr int N1 = F::N1, N2 = F::N2, NP = F::NP, NTH = F::NTH;
  constexpr int NV = N1 / 2 + 1;  // rows n = r + N2 n1 <= Nt/2 have n1 <= N1/2
  static_assert(NTH >= NP, "phase (0) runs one index k per thread");
  extern __shared__ double2 sm[];
  __shared__ double2 s_tws[NP - 1], s_twa[N1], s_twb[N1];
  const int n2 = by, n2p = (N2 - n2) % N2, nsets = n2p == n2 ? 1 : 2;
  const int rb = nsets == 2 ? n2p : n2;  // residue of the partner set (self-partnered: the same set)
  const long long pl0 = (long long)bx * NP;
  const long long p0 = p_begin + pl0;
  if (threadIdx.x < N1) {  // read behind the barrier that ends phase (0)
    s_twa[threadIdx.x] = cconj(__ldg(twt + threadIdx.x * n2));
    s_twb[threadIdx.x] = cconj(__ldg(twt + threadIdx.x * n2p));
  }
  // (0) per k: the stored rows n <= Nt/2 of set 0 at k and of the partner set at NP - k give every row of
  // set 0 at k and of the partner set at NP - k (direct or mirror); N1-point inverse DFTs over n1 -> smem
  for (int k = threadIdx.x; k < NP; k += NTH) {
    const int kb = (NP - k) & (NP - 1);
    double2 x0[NV], x1[NV], y0[NV], y1[NV];
#pragma unroll
    for (int n1 = 0; n1 < NV; ++n1) {
      const int na = n2 + N2 * n1, nb = rb + N2 * n1;
      if (na <= NT / 2) {
        const double2* q = pd_spec_row<SH>(sp, na) + 2 * p0 + k;
        x0[n1] = PD_TFX_SPEC_LD(q);
        x1[n1] = PD_TFX_SPEC_LD(q + NP);
      }
      if (nb <= NT / 2) {
        const double2* q = pd_spec_row<SH>(sp, nb) + 2 * p0 + kb;
        y0[n1] = PD_TFX_SPEC_LD(q);
        y1[n1] = PD_TFX_SPEC_LD(q + NP);
      }
    }
    const double2 wk = __ldg(twx + k), wb = __ldg(twx + kb);
    // NTH >= NP: every thread that fills a table entry passes here exactly once
    build_stockham_table<NP, kRX>(s_tws, [&](int idx) { return __ldg(twx + 2 * idx); });
    double2 a[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      if (n1 < NV && n2 + N2 * n1 <= NT / 2) {
        a[n1] = a_direct(x0[n1 < NV ? n1 : 0], x1[n1 < NV ? n1 : 0], wk);
      } else {  // partner row (N1 - n1) mod N1 for r = 0, N1 - 1 - n1 for r > 0 (compile-time indices)
        const int ma = ((N1 - n1) & (N1 - 1)) < NV ? ((N1 - n1) & (N1 - 1)) : 0;
        const int mb = (N1 - 1 - n1) < NV ? (N1 - 1 - n1) : 0;
        a[n1] = n2 == 0 ? a_mirror(y0[ma], y1[ma], wb) : a_mirror(y0[mb], y1[mb], wb);
      }
    }
    DFT<N1, true>::run(a);
#pragma unroll
    for (int t = 0; t < N1; ++t) sm[pad(t * NP + k)] = a[t];
    if (nsets == 2) {
      double2 b[N1];
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int mb = N1 - 1 - n1;
        if (n1 < NV && rb + N2 * n1 <= NT / 2)
          b[n1] = a_direct(y0[n1 < NV ? n1 : 0], y1[n1 < NV ? n1 : 0], wb);
        else
          b[n1] = a_mirror(x0[mb < NV ? mb : 0], x1[mb < NV ? mb : 0], wk);
      }
      DFT<N1, true>::run(b);
#pragma unroll
      for (int t = 0; t < N1; ++t) sm[pad((N1 + t) * NP + kb)] = b[t];
    }
  }
  __syncthreads();
  // (1) NP-point inverse FFTs over p of the rows (set, t1), twiddle w_Nt^{-t1 n2}, out to W[n2][t1][pair]
  fft_io<NP, 2 * N1, true, true, NTH, true, false, kRX>(
      sm, TwStockham{s_tws},
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value, R0 = first_radix(NP, kRX);
#pragma unroll
        for (int m = 0; m < R0; ++m) v[m] = sm[pad(c * NP + j + m * s)];
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value, RL = last_radix(NP, kRX);
        const int set = c / N1, t1 = c % N1;
        pre();
        if (set == 1 && nsets == 1) return;  // the partner set is the same residue
        const double2 tw = (set ? s_twb : s_twa)[t1];
        double2* q = W + ((long long)(set ? n2p : n2) * N1 + t1) * Pc + pl0 + j;
#pragma unroll
        for (int m = 0; m < RL; ++m) __stcg(q + m * s, cmul(w[m], tw));
      });
}

template <int NT, int NX, bool SH>
__global__ void __launch_bounds__(Fx<NT, NX>::NTH, PD_TFX_MINB) tfx_inv_s1x(const pd_spec sp, long long S,
                                                              long long p_begin, long long Pc,
                                                              double2* __restrict__ W,
                                                              const double2* __restrict__ twx,
                                                              const double2* __restrict__ twt) {
  tfx_inv_s1x_tile<NT, NX, SH>(sp, S, p_begin, Pc, W, twx, twt, blockIdx.x, blockIdx.y);
}

// ---------------------------------------------------------------------------------------------
// Persistent fused time FFT (PD_TFX_PERSIST=1, r02 experiment): ONE launch per call.  Resident CTAs pull tile tasks
// of both stages from a global counter, in an order that keeps stage 2 a fixed lag of kLag x-rows behind stage 1:
//   block k = [stage-1 tiles of x-row k][stage-2 tiles of x-row k - kLag]
// so the stage-1 -> stage-2 scratch is a ring of kRing x-rows (kRing * Nt * NX/2 complex, L2-resident) instead of the
// per-stream chunk buffers, and there are no kernel boundaries (no single-wave launches, no launch gaps).  A
// stage-2 tile of row y waits for done1[y] = all stage-1 tiles of the row (thread 0 polls, then a CTA barrier); a
// stage-1 tile of row y waits for done2[y - kRing] before it overwrites that ring slot.  Tasks are claimed in
// increasing order and a task only ever waits for lower-numbered ones, which running CTAs own: no deadlock, whatever
// the number of resident CTAs.  Tiles are the very device bodies of the per-chunk kernels.
// deferred completion signal of the previous tile: thread 0 fences and bumps the flag right before the CURRENT
// tile's stores, when the previous tile's stores (ordered before by the loop's CTA barriers) have long drained, so
// the fence costs nothing; signalling right after a tile's stores would stall the CTA for their round trip
struct TaskSignal {
  int** pending;  // CTA-uniform, in shared memory
  PD_D void operator()() const {
    if (threadIdx.x == 0 && *pending) {
      __threadfence();
      atomicAdd(*pending, 1);
      *pending = nullptr;
    }
  }
};
// wait until *flag reaches target (thread 0 polls, then a CTA barrier).  Before it blocks, the CTA releases its own
// deferred signal: the tile it waits for may itself be waiting for that one
PD_D void task_wait(const int* flag, int target, const TaskSignal& sig) {
  if (threadIdx.x == 0) {
    const volatile int* f = reinterpret_cast<const volatile int*>(flag);
    if (*f < target) {
      sig();
      while (*f < target) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}
// task t -> (kind 0 = first stage / 1 = second stage, x-row y, tile); NA / NB tiles per row of the two kinds
PD_D void task_decode(int t, int rows, int lag, int NA, int NB, int& kind, int& y, int& tile) {
  const int head = lag * NA, per = NA + NB;
  if (t < head) {
    kind = 0;
    y = t / NA;
    tile = t % NA;
    return;
  }
  const int t1 = t - head, k = lag + t1 / per, rem = t1 % per;
  if (k < rows) {
    kind = rem < NA ? 0 : 1;
    y = kind ? k - lag : k;
    tile = kind ? rem - NA : rem;
    return;
  }
  const int t2 = t - (head + (rows - lag) * per);
  kind = 1;
  y = rows - lag + t2 / NB;
  tile = t2 % NB;
}

// FWD: stage 1 = tf4_fwd_s1 tiles, stage 2 = tfx_fwd_s2x tiles;  !FWD: stage 1 = tfx_inv_s1x, stage 2 = tf4_inv_s2
template <int NT, int NX, bool FWD>
__global__ void __launch_bounds__(Fx<NT, NX>::NTH, PD_TFX_MINB)
tfx_persist(const double* __restrict__ r, double* __restrict__ z, long long S, int rows, int lag, int ring_rows,
            double2* __restrict__ ring, const pd_spec sp, const double* __restrict__ gam,
            const double2* __restrict__ tw2, const double2* __restrict__ twt, const double2* __restrict__ twx,
            int* __restrict__ ctr) {
  using F = Fx<NT, NX>;
  constexpr int N1 = F::N1, N2 = F::N2, NP = F::NP, KP = F::KP, TX = NP / KP;
  constexpr int NT1 = TX * N1, NT2 = N2 / 2 + 1;  // tiles per x-row: N2-point stage / x-FFT stage
  constexpr int NA = FWD ? NT1 : NT2, NB = FWD ? NT2 : NT1;
  static_assert(KP * N2 / kRS == F::NTH, "both tile kinds run on the same thread count");
  __shared__ int s_task;
  __shared__ int* s_pending;
  int* done1 = ctr + 1;
  int* done2 = ctr + 1 + rows;
  const int total = rows * (NA + NB);
  const TaskSignal sig{&s_pending};
  int nxt = 0;
  if (threadIdx.x == 0) {
    s_pending = nullptr;
    nxt = atomicAdd(ctr, 1);
  }
  for (;;) {
    __syncthreads();  // the previous tile's shared-memory reads and global stores are issued
    if (threadIdx.x == 0) s_task = nxt;
    __syncthreads();
    const int t = s_task;
    if (t >= total) break;
    if (threadIdx.x == 0) nxt = atomicAdd(ctr, 1);  // the next task, in flight behind this tile
    int kind, y, tile;
    task_decode(t, rows, lag, NA, NB, kind, y, tile);
    double2* Y = ring + (size_t)(y % ring_rows) * NT * NP;
    int* mine;
    if (kind == 0) {
      if (y >= ring_rows) task_wait(done2 + y - ring_rows, NB, sig);
      if constexpr (FWD)
        tf4_fwd_s1_tile<NT, N2, KP, true, kRS, false>(r, S, (long long)y * NP, NP, Y, gam, tw2, twt, nullptr, 0, tile % TX,
                                                      tile / TX, TX, sig);
      else
        tfx_inv_s1x_tile<NT, NX, false>(sp, S, (long long)y * NP, NP, Y, twx, twt, 0, tile, sig);
      mine = done1 + y;
    } else {
      task_wait(done1 + y, NA, sig);
      if constexpr (FWD)
        tfx_fwd_s2x_tile<NT, NX, false>(Y, S, (long long)y * NP, NP, sp, twx, 0, tile, sig);
      else
        tf4_inv_s2_tile<NT, N2, KP, true, 0, kRS>(Y, S, (long long)y * NP, NP, z, gam, tw2, tile % TX, tile / TX, sig);
      mine = done2 + y;
    }
    if (threadIdx.x == 0) s_pending = mine;  // thread 0 passed its pre-store hook: the older signal is out
  }
  sig();  // s_task >= total: all threads are past the loop barrier; the last tile's stores precede it
}

// workspace of the persistent kernels (experiment: one per process and device, allocated on first use)
struct PersistWs {
  int dev = -1;
  int* ctr = nullptr;
  int nctr = 0;
  double2* ring = nullptr;
  size_t ring_elems = 0;
};
inline cudaError_t persist_ws(PersistWs& w, int nctr, size_t ring_elems) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (w.dev != dev || w.nctr < nctr || w.ring_elems < ring_elems) {
    if (w.dev == dev) {
      cudaFree(w.ctr);
      cudaFree(w.ring);
    }
    w = PersistWs{};
    if (cudaError_t e = cudaMalloc(&w.ctr, (size_t)nctr * sizeof(int))) return e;
    if (cudaError_t e = cudaMalloc(&w.ring, ring_elems * sizeof(double2))) return e;
    w.dev = dev;
    w.nctr = nctr;
    w.ring_elems = ring_elems;
  }
  return cudaSuccess;
}
// lag (x-rows between the stages) so that a stage-2 tile's inputs were claimed ~2.5 grids of tasks earlier, and the ring
// that holds the rows in flight (lag + the rows being written + slack); PD_TFX_LAG overrides
template <int NT, int NX>
inline void persist_plan(int grid, int rows, int* lag, int* ring_rows) {
  using F = Fx<NT, NX>;
  const int per = (F::NP / F::KP) * F::N1 + F::N2 / 2 + 1;
  const char* e = getenv("PD_TFX_LAG");
  int l = e ? atoi(e) : (5 * grid / 2 + per - 1) / per;
  if (l < 2) l = 2;
  if (l > rows - 1) l = rows - 1;
  *lag = l;
  *ring_rows = l + 3 + (grid + per - 1) / per;
}
inline bool persist_enabled() {
  const char* e = getenv("PD_TFX_PERSIST");
  return e && atoi(e) != 0;
}
template <class K>
inline cudaError_t persist_grid(K kernel, int nth, int smem, int* grid) {
  int dev = 0, nsm = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) return e;
  if (cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, nth, smem)) return e;
  if (occ < 1) return cudaErrorLaunchOutOfResources;
  *grid = nsm * occ;
  return cudaSuccess;
}

template <int NT, int NX>
void set_attrs() {
  using F = Fx<NT, NX>;
  static int done = -1;  // device on which the attributes were set
  int dev = 0;
  cudaGetDevice(&dev);
  if (done == dev) return;
  constexpr int N2 = F::N2, KP = F::KP;
  const int sm1 = smem_of<N2>(KP), sm2 = F::SMEM * (int)sizeof(double2);
  cudaFuncSetAttribute(tf4_fwd_s1<NT, N2, KP, true, kRS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
  cudaFuncSetAttribute(tf4_fwd_s1<NT, N2, KP, false, kRS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
  cudaFuncSetAttribute(tf4_fwd_s1<NT, N2, KP, true, kRS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
  cudaFuncSetAttribute(tf4_fwd_s1_comb<NT, N2, KP, kRS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
  cudaFuncSetAttribute(tfx_fwd_s2<NT, NX, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
  cudaFuncSetAttribute(tfx_inv_s1<NT, NX, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
  cudaFuncSetAttribute(tfx_fwd_s2x<NT, NX, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
  cudaFuncSetAttribute(tfx_inv_s1x<NT, NX, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
  cudaFuncSetAttribute(tfx_fwd_s2x<NT, NX, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
  cudaFuncSetAttribute(tfx_inv_s1x<NT, NX, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
  cudaFuncSetAttribute(tf4_inv_s2<NT, N2, KP, true, 0, kRS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
  cudaFuncSetAttribute(tf4_inv_s2<NT, N2, KP, true, 1, kRS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
  cudaFuncSetAttribute(tf4_inv_s2<NT, N2, KP, false, 0, kRS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
  cudaFuncSetAttribute(tf4_inv_s2<NT, N2, KP, false, 1, kRS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
  done = dev;
}

template <int NT, int NX>
cudaError_t fwd(const double* r, const pd_spec& sp, long long S, const double* gam, const pd_tf4_tables& tb,
                const double2* twx, double2* scratch0, long long chunk_pairs, cudaStream_t st0, int* nl,
                const pd_tfx_overlap* ov, const pd_comb_args* comb, double* npart, long long* nparts) {
  using F = Fx<NT, NX>;
  constexpr int N2 = F::N2, KP = F::KP, NP = F::NP;
  set_attrs<NT, NX>();
  const int sm1 = smem_of<N2>(KP), sm2 = F::SMEM * (int)sizeof(double2);
  const bool vec = (reinterpret_cast<uintptr_t>(r) & 15) == 0;
  if (npart && (comb || !vec)) return cudaErrorInvalidValue;  // the norm rides on the 16-byte loader
  long long poff = 0;
  const bool tma = !comb && !npart && pd_tf4_tma_supported(NT, S, r);
  const long long npairs = S / 2;
  int n = 0;
  if constexpr (KP * N2 / kRS == F::NTH && NP % KP == 0) {
    const long long rows = S / NX;
    if (persist_enabled() && !comb && !npart && vec && sp.P == 1 && rows >= 16 && rows * NX == S && rows < (1 << 20)) {
      static PersistWs ws;
      const int nctr = 1 + 2 * (int)rows, smem = sm1 > sm2 ? sm1 : sm2;
      int grid = 0, lag = 0, ring_rows = 0;
      if (cudaError_t e = persist_grid(tfx_persist<NT, NX, true>, F::NTH, smem, &grid)) return e;
      persist_plan<NT, NX>(grid, (int)rows, &lag, &ring_rows);
      if (cudaError_t e = persist_ws(ws, nctr, (size_t)ring_rows * NT * NP)) return e;
      if (cudaError_t e = cudaMemsetAsync(ws.ctr, 0, (size_t)nctr * sizeof(int), st0)) return e;
      tfx_persist<NT, NX, true><<<grid, F::NTH, smem, st0>>>(r, nullptr, S, (int)rows, lag, ring_rows, ws.ring, sp, gam,
                                                            tb.tw2, tb.twt, twx, ws.ctr);
      *nl = 1;
      if (nparts) *nparts = 0;
      return cudaGetLastError();
    }
  }
  if (cudaError_t e = ov_fork(ov, st0)) return e;
  for (long long p = 0, ci = 0; p < npairs; p += chunk_pairs, ++ci) {
    const int lane = ov ? (int)(ci % ov->k) : 0;
    cudaStream_t st = lane ? ov->st[lane] : st0;
    double2* scratch = lane ? ov->scratch[lane] : scratch0;
    const long long pc = npairs - p < chunk_pairs ? npairs - p : chunk_pairs;
    const dim3 g1((unsigned)((pc + KP - 1) / KP), kN1), g2((unsigned)(pc / NP), N2 / 2 + 1);
    if (comb) {
      tf4_fwd_s1_comb<NT, N2, KP, kRS><<<g1, KP * N2 / kRS, sm1, st>>>(*comb, S, p, pc, scratch, gam, tb.tw2, tb.twt);
    } else if (tma) {
      if (cudaError_t e = pd_launch_tf4_fwd_s1_tma(NT, r, S, p, pc, scratch, gam, tb.tw2, tb.twt, st)) return e;
    } else if (npart) {
      tf4_fwd_s1<NT, N2, KP, true, kRS, true><<<g1, KP * N2 / kRS, sm1, st>>>(r, S, p, pc, scratch, gam, tb.tw2, tb.twt,
                                                                            npart, poff);
      poff += (long long)g1.x * g1.y;
    } else if (vec)
      tf4_fwd_s1<NT, N2, KP, true, kRS><<<g1, KP * N2 / kRS, sm1, st>>>(r, S, p, pc, scratch, gam, tb.tw2, tb.twt);
    else
      tf4_fwd_s1<NT, N2, KP, false, kRS><<<g1, KP * N2 / kRS, sm1, st>>>(r, S, p, pc, scratch, gam, tb.tw2, tb.twt);
    if (PD_TFX_XFIRST_FWD && sp.P > 1)
      tfx_fwd_s2x<NT, NX, true><<<g2, F::NTH, sm2, st>>>(scratch, S, p, pc, sp, twx);
    else if (PD_TFX_XFIRST_FWD)
      tfx_fwd_s2x<NT, NX, false><<<g2, F::NTH, sm2, st>>>(scratch, S, p, pc, sp, twx);
    else if (sp.P > 1)
      return cudaErrorInvalidValue;  // the t1-first A/B kernels (PD_TFX_XFIRST=0) are single-GPU only
    else
      tfx_fwd_s2<NT, NX, false><<<g2, F::NTH, sm2, st>>>(scratch, S, p, pc, sp, twx);
    n += 2;
  }
  *nl = n;
  if (nparts) *nparts = poff;
  return ov_join(ov, st0);
}

template <int NT, int NX>
cudaError_t inv(const pd_spec& sp, double* z, long long S, const double* igam, const pd_tf4_tables& tb,
                const double2* twx, double2* scratch0, long long chunk_pairs, int accumulate, cudaStream_t st0,
                int* nl, const pd_tfx_overlap* ov) {
  using F = Fx<NT, NX>;
  constexpr int N2 = F::N2, KP = F::KP, NP = F::NP;
  set_attrs<NT, NX>();
  const int sm1 = smem_of<N2>(KP), sm2 = F::SMEM * (int)sizeof(double2);
  const bool vec = (reinterpret_cast<uintptr_t>(z) & 15) == 0;
  const long long npairs = S / 2;
  int n = 0;
  if constexpr (KP * N2 / kRS == F::NTH && NP % KP == 0) {
    const long long rows = S / NX;
    if (persist_enabled() && !accumulate && vec && sp.P == 1 && rows >= 16 && rows * NX == S && rows < (1 << 20)) {
      static PersistWs ws;
      const int nctr = 1 + 2 * (int)rows, smem = sm1 > sm2 ? sm1 : sm2;
      int grid = 0, lag = 0, ring_rows = 0;
      if (cudaError_t e = persist_grid(tfx_persist<NT, NX, false>, F::NTH, smem, &grid)) return e;
      persist_plan<NT, NX>(grid, (int)rows, &lag, &ring_rows);
      if (cudaError_t e = persist_ws(ws, nctr, (size_t)ring_rows * NT * NP)) return e;
      if (cudaError_t e = cudaMemsetAsync(ws.ctr, 0, (size_t)nctr * sizeof(int), st0)) return e;
      tfx_persist<NT, NX, false><<<grid, F::NTH, smem, st0>>>(nullptr, z, S, (int)rows, lag, ring_rows, ws.ring, sp, igam,
                                                             tb.tw2, tb.twt, twx, ws.ctr);
      *nl = 1;
      return cudaGetLastError();
    }
  }
  if (cudaError_t e = ov_fork(ov, st0)) return e;
  for (long long p = 0, ci = 0; p < npairs; p += chunk_pairs, ++ci) {
    const int lane = ov ? (int)(ci % ov->k) : 0;
    cudaStream_t st = lane ? ov->st[lane] : st0;
    double2* scratch = lane ? ov->scratch[lane] : scratch0;
    const long long pc = npairs - p < chunk_pairs ? npairs - p : chunk_pairs;
    const dim3 g1((unsigned)(pc / NP), N2 / 2 + 1), g2((unsigned)((pc + KP - 1) / KP), kN1);
    if (PD_TFX_XFIRST_INV && sp.P > 1)
      tfx_inv_s1x<NT, NX, true><<<g1, F::NTH, sm2, st>>>(sp, S, p, pc, scratch, twx, tb.twt);
    else if (PD_TFX_XFIRST_INV)
      tfx_inv_s1x<NT, NX, false><<<g1, F::NTH, sm2, st>>>(sp, S, p, pc, scratch, twx, tb.twt);
    else if (sp.P > 1)
      return cudaErrorInvalidValue;
    else
      tfx_inv_s1<NT, NX, false><<<g1, F::NTH, sm2, st>>>(sp, S, p, pc, scratch, twx, tb.twt);
    const int th = KP * N2 / kRS;
    if (vec) {
      if (accumulate)
        tf4_inv_s2<NT, N2, KP, true, 1, kRS><<<g2, th, sm1, st>>>(scratch, S, p, pc, z, igam, tb.tw2);
      else
        tf4_inv_s2<NT, N2, KP, true, 0, kRS><<<g2, th, sm1, st>>>(scratch, S, p, pc, z, igam, tb.tw2);
    } else {
      if (accumulate)
        tf4_inv_s2<NT, N2, KP, false, 1, kRS><<<g2, th, sm1, st>>>(scratch, S, p, pc, z, igam, tb.tw2);
      else
        tf4_inv_s2<NT, N2, KP, false, 0, kRS><<<g2, th, sm1, st>>>(scratch, S, p, pc, z, igam, tb.tw2);
    }
    n += 2;
  }
  *nl = n;
  return ov_join(ov, st0);
}

}  // namespace

// Nt = 256 / 512 too since r02: with the y-pass by cyclic Toeplitz solves the fold wins at cfg3 (apply 0.283 ->
// 0.230 ms: the slab x-FFT row passes leave Step (b)); PD_TFX_SMALL=0 restores the single-tile FFT + row passes.
// NX = 1024 (Nt >= 256 makes it >= 2.7e8 dofs per real vector) takes the single-tile / tf4 + slab route.
int pd_tfx_supported(int nt, int nx) {
  const char* se = getenv("PD_TFX_SMALL");
  const bool small = se == nullptr || atoi(se) != 0;
  const bool t = nt == 1024 || nt == 2048 || nt == 4096 || (small && (nt == 256 || nt == 512));
  const bool x = nx == 32 || nx == 64 || nx == 128 || nx == 256 || nx == 512;
  return t && x;
}
int pd_tfx_n2(int nt) { return nt / kN1; }
long long pd_tfx_chunk_align(int nt, int nx) {
  const long long kp = tfx_kpt(nt) / (nt / kN1) < 8 ? 8 : tfx_kpt(nt) / (nt / kN1);
  const long long np = nx / 2;
  return kp > np ? kp : np;
}

#define PD_TFX_ROW(T, FN, ARGS)                                                                      \
  case T * 10000 + 32: return FN<T, 32> ARGS;                                                       \
  case T * 10000 + 64: return FN<T, 64> ARGS;                                                       \
  case T * 10000 + 128: return FN<T, 128> ARGS;                                                     \
  case T * 10000 + 256: return FN<T, 256> ARGS;                                                     \
  case T * 10000 + 512: return FN<T, 512> ARGS;
#define PD_TFX_SWITCH(FN, ARGS)                                                                      \
  switch (nt * 10000 + nx) {                                                                         \
    PD_TFX_ROW(256, FN, ARGS) PD_TFX_ROW(512, FN, ARGS)                                              \
    PD_TFX_ROW(1024, FN, ARGS) PD_TFX_ROW(2048, FN, ARGS) PD_TFX_ROW(4096, FN, ARGS)                 \
    default: return cudaErrorInvalidValue;                                                           \
  }

cudaError_t pd_launch_tfx_fwd(int nt, int nx, const double* r, const pd_spec& sp, long long S, const double* gam,
                              const pd_tf4_tables& tb, const double2* twx, double2* scratch, long long chunk_pairs,
                              cudaStream_t st, int* nl, const pd_tfx_overlap* ov, const pd_comb_args* comb,
                              double* npart, long long* nparts) {
  PD_TFX_SWITCH(fwd, (r, sp, S, gam, tb, twx, scratch, chunk_pairs, st, nl, ov, comb, npart, nparts))
}

cudaError_t pd_launch_tfx_inv(int nt, int nx, const pd_spec& sp, double* z, long long S, const double* igam,
                              const pd_tf4_tables& tb, const double2* twx, double2* scratch, long long chunk_pairs,
                              int accumulate, cudaStream_t st, int* nl, const pd_tfx_overlap* ov) {
  PD_TFX_SWITCH(inv, (sp, z, S, igam, tb, twx, scratch, chunk_pairs, accumulate, st, nl, ov))
}
