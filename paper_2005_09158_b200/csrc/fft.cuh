// Radix-2/4/8/16 in-register DFTs and Stockham shared-memory passes (complex128).
//
// Used by the time-axis FFTs of Steps (a)/(c) (eq 2.12, P:l.813-819; Matlab fft/ifft pairing
// P:l.864-875) and by the 2D slab FFTs of the periodic Step (b).  Forward = exp(-2 pi i jk/N)
// (unnormalised), inverse = exp(+2 pi i jk/N) (unnormalised; callers scale by 1/N).
//
// A tile holds C independent sequences of length N in shared memory.  Element (pos, c) lives at
//   INTERLEAVED: pad(pos*C + c)      SEQMAJOR: pad(c*N + pos),      pad(i) = i + (i >> 4)
// (one double2 of padding every 16 breaks the power-of-two strides of the first Stockham pass).
// Each thread owns E = 16 elements (min(16, N)) so the register footprint is fixed; a radix-R pass
// runs E/R butterflies per thread.  Radix plan: 16, 16, ..., then the remainder (2, 4 or 8).
#pragma once
#include "common.cuh"

namespace pdfft {

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }
__host__ __device__ constexpr int pad(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int elems_per_thread(int N) { return N < 16 ? N : 16; }
__host__ __device__ constexpr int num_passes(int N) { return N <= 1 ? 0 : (ilog2(N) + 3) / 4; }
// radix of pass p (0-based): 16 for all full passes, the remainder last
__host__ __device__ constexpr int radix_of(int N, int p) {
  return (p < num_passes(N) - 1) ? 16 : (1 << (ilog2(N) - 4 * (num_passes(N) - 1)));
}
__host__ __device__ constexpr int ls_of(int N, int p) { return p == 0 ? 1 : ls_of(N, p - 1) * radix_of(N, p - 1); }
__host__ __device__ constexpr int smem_elems(int n) { return pad(n - 1) + 1; }

// cos(2 pi k / 16), k = 0..15
__device__ constexpr double COS16[16] = {
    1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173,
    0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128675613,
    -1.0, -0.92387953251128675613, -0.70710678118654752440, -0.38268343236508977173,
    0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128675613};

// v * exp(-+ 2 pi i K / R) with compile-time K, R <= 16 (INV: +)
template <int R, int K, bool INV>
PD_D double2 twmul(double2 v) {
  if constexpr (K == 0) {
    return v;
  } else if constexpr (4 * K == R) {
    return cmul_mi<INV>(v);
  } else {
    constexpr int k16 = K * (16 / R);
    constexpr double c = COS16[k16 % 16];
    constexpr double s = COS16[(k16 + 12) % 16];  // sin(2 pi k16 / 16)
    constexpr double sn = INV ? s : -s;            // forward: exp(-i theta) = (c, -s)
    return make_double2(fma(v.x, c, -v.y * sn), fma(v.x, sn, v.y * c));
  }
}

template <int R, int K, bool INV>
struct Combine {
  static PD_D void run(double2* x, const double2* e, const double2* o) {
    if constexpr (K < R / 2) {
      double2 t = twmul<R, K, INV>(o[K]);
      x[K] = cadd(e[K], t);
      x[K + R / 2] = csub(e[K], t);
      Combine<R, K + 1, INV>::run(x, e, o);
    }
  }
};

// In-register DFT of length R (natural order in and out), radix-2 decimation in time.
template <int R, bool INV>
struct DFT {
  static PD_D void run(double2* x) {
    double2 e[R / 2], o[R / 2];
#pragma unroll
    for (int i = 0; i < R / 2; ++i) {
      e[i] = x[2 * i];
      o[i] = x[2 * i + 1];
    }
    DFT<R / 2, INV>::run(e);
    DFT<R / 2, INV>::run(o);
    Combine<R, 0, INV>::run(x, e, o);
  }
};
template <bool INV>
struct DFT<1, INV> {
  static PD_D void run(double2*) {}
};
template <bool INV>
struct DFT<2, INV> {
  static PD_D void run(double2* x) {
    double2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  }
};
template <bool INV>
struct DFT<4, INV> {
  static PD_D void run(double2* x) {
    double2 t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]);
    double2 t2 = cadd(x[1], x[3]), t3 = cmul_mi<INV>(csub(x[1], x[3]));
    x[0] = cadd(t0, t2);
    x[2] = csub(t0, t2);
    x[1] = cadd(t1, t3);
    x[3] = csub(t1, t3);
  }
};

template <int N, int C, bool SEQMAJOR>
PD_D int sidx(int pos, int c) {
  return pad(SEQMAJOR ? c * N + pos : pos * C + c);
}

// inter-pass twiddle exp(-+2 pi i idx / N) from the table tw[idx] = exp(-2 pi i idx / N)
template <bool INV>
PD_D double2 twiddle(const double2* __restrict__ tw, int idx) {
  double2 w = __ldg(tw + idx);
  return INV ? cconj(w) : w;
}

// Apply the inter-pass twiddles of a Stockham pass with stride LS to the R inputs of butterfly j.
template <int N, int R, int LS, bool INV>
PD_D void pass_twiddles(double2* v, int j, const double2* __restrict__ tw) {
  if constexpr (LS > 1) {
    const int k = j & (LS - 1);
    const int step = k * (N / (LS * R));
#pragma unroll
    for (int m = 1; m < R; ++m) v[m] = cmul(v[m], twiddle<INV>(tw, m * step));
  }
}

// One Stockham radix-R pass smem -> smem over C sequences (all NTH threads participate).
template <int N, int C, int R, int LS, bool INV, bool SEQMAJOR, int NTH>
PD_D void stockham_pass(double2* sm, const double2* __restrict__ tw) {
  constexpr int NB = C * N / R;
  constexpr int BPT = NB / NTH;
  static_assert(BPT * NTH == NB, "butterflies must divide evenly");
  double2 v[BPT][R];
#pragma unroll
  for (int bi = 0; bi < BPT; ++bi) {
    const int b = threadIdx.x + bi * NTH;
    const int c = b % C, j = b / C;
#pragma unroll
    for (int m = 0; m < R; ++m) v[bi][m] = sm[sidx<N, C, SEQMAJOR>(j + m * (N / R), c)];
  }
  __syncthreads();
#pragma unroll
  for (int bi = 0; bi < BPT; ++bi) {
    const int b = threadIdx.x + bi * NTH;
    const int c = b % C, j = b / C;
    pass_twiddles<N, R, LS, INV>(v[bi], j, tw);
    DFT<R, INV>::run(v[bi]);
    const int k = j & (LS - 1);
    const int base = (j - k) * R + k;
#pragma unroll
    for (int q = 0; q < R; ++q) sm[sidx<N, C, SEQMAJOR>(base + q * LS, c)] = v[bi][q];
  }
  __syncthreads();
}

// Passes P0..P1-1 (smem -> smem), compile-time recursion.
template <int N, int C, int P, int P1, bool INV, bool SEQMAJOR, int NTH>
struct Passes {
  static PD_D void run(double2* sm, const double2* __restrict__ tw) {
    if constexpr (P < P1) {
      stockham_pass<N, C, radix_of(N, P), ls_of(N, P), INV, SEQMAJOR, NTH>(sm, tw);
      Passes<N, C, P + 1, P1, INV, SEQMAJOR, NTH>::run(sm, tw);
    }
  }
};

// Full in-smem FFT of C sequences (natural order in, natural order out).
template <int N, int C, bool INV, bool SEQMAJOR, int NTH>
PD_D void fft_smem(double2* sm, const double2* __restrict__ tw) {
  Passes<N, C, 0, num_passes(N), INV, SEQMAJOR, NTH>::run(sm, tw);
}

}  // namespace pdfft
