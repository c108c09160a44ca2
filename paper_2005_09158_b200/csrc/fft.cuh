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
#include <type_traits>

#include "common.cuh"

namespace pdfft {

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }
__host__ __device__ constexpr int pad(int i) { return i + (i >> 4); }
// RMAX = largest radix (16 or 8); E = RMAX elements per thread
__host__ __device__ constexpr int elems_per_thread(int N, int RMAX = 16) { return N < RMAX ? N : RMAX; }
__host__ __device__ constexpr int num_passes(int N, int RMAX = 16) {
  return N <= 1 ? 0 : (ilog2(N) + ilog2(RMAX) - 1) / ilog2(RMAX);
}
// radix of pass p (0-based): RMAX for all full passes, the remainder last
__host__ __device__ constexpr int radix_of(int N, int p, int RMAX = 16) {
  return (p < num_passes(N, RMAX) - 1) ? RMAX : (1 << (ilog2(N) - ilog2(RMAX) * (num_passes(N, RMAX) - 1)));
}
__host__ __device__ constexpr int ls_of(int N, int p, int RMAX = 16) {
  return p == 0 ? 1 : ls_of(N, p - 1, RMAX) * radix_of(N, p - 1, RMAX);
}
__host__ __device__ constexpr int smem_elems(int n) { return pad(n - 1) + 1; }
__host__ __device__ constexpr int first_radix(int N, int RMAX = 16) { return radix_of(N, 0, RMAX); }
__host__ __device__ constexpr int last_radix(int N, int RMAX = 16) { return radix_of(N, num_passes(N, RMAX) - 1, RMAX); }

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

// linear (unpadded) index of element (pos, c) and its stride per unit of pos
template <int N, int C, bool SEQMAJOR>
PD_D int lin(int pos, int c) {
  return SEQMAJOR ? c * N + pos : pos * C + c;
}
template <int C, bool SEQMAJOR>
__host__ __device__ constexpr int pos_stride() {
  return SEQMAJOR ? 1 : C;
}
// pad(a + m*K): when K is a multiple of 16 the padding is linear in m, so after unrolling every access of a
// butterfly is the base plus an immediate offset
template <int K>
PD_D int soff(int a, int m) {
  if constexpr (K % 16 == 0)
    return pad(a) + m * (K + K / 16);
  else
    return pad(a + m * K);
}

// butterfly b -> (sequence c, butterfly index j within the sequence); the fastest-varying index follows
// the contiguous smem dimension so that consecutive lanes touch consecutive addresses
template <int N, int C, int R, bool SEQMAJOR>
PD_D void bfly_coords(int b, int& c, int& j) {
  if constexpr (SEQMAJOR) {
    j = b % (N / R);
    c = b / (N / R);
  } else {
    c = b % C;
    j = b / C;
  }
}

// inter-pass twiddle exp(-+2 pi i idx / N) from the table tw[idx] = exp(-2 pi i idx / N).  Kernels stage
// their tables in shared memory (load_table) so the butterfly loops never wait on global loads.
template <bool INV>
PD_D double2 twiddle(const double2* tw, int idx) {
  double2 w = tw[idx];
  return INV ? cconj(w) : w;
}

// copy n table entries global -> shared (all threads; caller synchronises)
PD_D void load_table(double2* dst, const double2* __restrict__ src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldg(src + i);
}

// Apply the inter-pass twiddles of a Stockham pass with stride LS to the R inputs of butterfly j.
template <int N, int R, int LS, bool INV>
PD_D void pass_twiddles(double2* v, int j, const double2* tw) {
  if constexpr (LS > 1) {
    const int k = j & (LS - 1);
    const int step = k * (N / (LS * R));
#pragma unroll
    for (int m = 1; m < R; ++m) v[m] = cmul(v[m], twiddle<INV>(tw, m * step));
  }
}

// Stockham-ordered twiddle table (N - 1 entries): pass p (stride LS, radix R) owns the entries
// LS - 1 + (m - 1) LS + k = w_N^{m k N / (LS R)},  m = 1..R-1, k < LS,
// so the lanes of a pass (consecutive k) read consecutive entries for every m.  A plain N-point table read
// at the strides m k N/(LS R) is up to 8-way bank conflicted (m = 8 in the last pass of N = 256).
struct TwStockham {
  const double2* p;
};
template <int N, int R, int LS, bool INV>
PD_D void pass_twiddles(double2* v, int j, TwStockham tw) {
  if constexpr (LS > 1) {
    const double2* t = tw.p + (LS - 1) + (j & (LS - 1));
#pragma unroll
    for (int m = 1; m < R; ++m) v[m] = cmul(v[m], twiddle<INV>(t, (m - 1) * LS));
  }
}
// fill a TwStockham table for N-point FFTs with radix cap RMAX (all threads; caller synchronises);
// w(idx) returns the forward twiddle w_N^idx
template <int N, int RMAX, int P = 1, class WF>
PD_D void build_stockham_table(double2* dst, WF w) {
  if constexpr (P < num_passes(N, RMAX)) {  // pass 0 has no twiddles: its entries stay unused
    constexpr int LS = ls_of(N, P, RMAX), R = radix_of(N, P, RMAX);
    for (int i = threadIdx.x; i < (R - 1) * LS; i += blockDim.x)
      dst[LS - 1 + i] = w((i / LS + 1) * (i % LS) * (N / (LS * R)));
    build_stockham_table<N, RMAX, P + 1>(dst, w);
  }
}

// read the R inputs (positions j + m*N/R) of butterfly (c, j) from smem
template <int N, int C, int R, bool SEQMAJOR>
PD_D void smem_read_bfly(const double2* sm, int j, int c, double2* v) {
  const int a = lin<N, C, SEQMAJOR>(j, c);
#pragma unroll
  for (int m = 0; m < R; ++m) v[m] = sm[soff<(N / R) * pos_stride<C, SEQMAJOR>()>(a, m)];
}
// write R outputs at positions base + q*LS for sequence c
template <int N, int C, int R, int LS, bool SEQMAJOR>
PD_D void smem_write_out(double2* sm, int base, int c, const double2* v) {
  const int a = lin<N, C, SEQMAJOR>(base, c);
#pragma unroll
  for (int q = 0; q < R; ++q) sm[soff<LS * pos_stride<C, SEQMAJOR>()>(a, q)] = v[q];
}

// One Stockham radix-R pass smem -> smem over C sequences (all NTH threads participate).
template <int N, int C, int R, int LS, bool INV, bool SEQMAJOR, int NTH, class TW>
PD_D void stockham_pass(double2* sm, TW tw) {
  constexpr int NB = C * N / R;
  constexpr int BPT = NB / NTH;
  static_assert(BPT * NTH == NB, "butterflies must divide evenly");
  double2 v[BPT][R];
#pragma unroll
  for (int bi = 0; bi < BPT; ++bi) {
    int c, j;
    bfly_coords<N, C, R, SEQMAJOR>(threadIdx.x + bi * NTH, c, j);
    smem_read_bfly<N, C, R, SEQMAJOR>(sm, j, c, v[bi]);
  }
  __syncthreads();
#pragma unroll
  for (int bi = 0; bi < BPT; ++bi) {
    int c, j;
    bfly_coords<N, C, R, SEQMAJOR>(threadIdx.x + bi * NTH, c, j);
    pass_twiddles<N, R, LS, INV>(v[bi], j, tw);
    DFT<R, INV>::run(v[bi]);
    const int k = j & (LS - 1);
    smem_write_out<N, C, R, LS, SEQMAJOR>(sm, (j - k) * R + k, c, v[bi]);
  }
  __syncthreads();
}

// Passes P0..P1-1 (smem -> smem), compile-time recursion.
template <int N, int C, int P, int P1, bool INV, bool SEQMAJOR, int NTH, int RMAX = 16>
struct Passes {
  template <class TW>
  static PD_D void run(double2* sm, TW tw) {
    if constexpr (P < P1) {
      stockham_pass<N, C, radix_of(N, P, RMAX), ls_of(N, P, RMAX), INV, SEQMAJOR, NTH>(sm, tw);
      Passes<N, C, P + 1, P1, INV, SEQMAJOR, NTH, RMAX>::run(sm, tw);
    }
  }
};

// Full in-smem FFT of C sequences (natural order in, natural order out).
template <int N, int C, bool INV, bool SEQMAJOR, int NTH, class TW>
PD_D void fft_smem(double2* sm, TW tw) {
  Passes<N, C, 0, num_passes(N), INV, SEQMAJOR, NTH>::run(sm, tw);
}

// FFT of C sequences with streaming I/O.
//   ld(j, s, c, v): fill v[m], m < R0, with the inputs at positions j + m*s of sequence c (s = N/R0)
//   st(j, s, c, w): consume w[q], q < RL, the outputs at positions j + q*s of sequence c (s = N/RL)
// s is passed as std::integral_constant so loaders can use it in constant expressions.
// Pass 0 takes its inputs from ld (global memory or a staging buffer), the middle passes run in shared
// memory, the last pass hands its outputs to st straight from registers (natural order).  Loaders and
// storers compute one base address per butterfly and step by the compile-time stride s, so the
// addressing cost is per butterfly, not per element.  LOAD_SMEM / STORE_SMEM: ld reads from / st writes
// into `sm` itself, so barriers separate those accesses from the Stockham passes.  No trailing barrier.
struct NoHook {
  PD_D void operator()() const {}
};

// HOOK() runs (all threads) right after the barrier that follows pass 0's loads: the pipelined kernels use
// it to recycle the stage buffer the loader just consumed.  RMAX: largest radix (16 or 8).
template <int N, int C, bool INV, bool SEQMAJOR, int NTH, bool LOAD_SMEM, bool STORE_SMEM, int RMAX = 16, class LD,
          class ST, class HOOK = NoHook, class TW = const double2*>
PD_D void fft_io(double2* sm, TW tw, LD ld, ST st, HOOK hook = HOOK()) {
  constexpr int P = num_passes(N, RMAX);
  constexpr int R0 = radix_of(N, 0, RMAX);
  constexpr int B0 = (C * N / R0) / NTH;
  static_assert(B0 * NTH == C * N / R0, "pass-0 butterflies must divide evenly");
  double2 v[B0][R0];
#pragma unroll
  for (int bi = 0; bi < B0; ++bi) {
    int c, j;
    bfly_coords<N, C, R0, SEQMAJOR>(threadIdx.x + bi * NTH, c, j);
    ld(j, std::integral_constant<int, N / R0>{}, c, v[bi]);
  }
  if constexpr (P == 1) {
    if constexpr (STORE_SMEM || LOAD_SMEM) __syncthreads();
    hook();
#pragma unroll
    for (int bi = 0; bi < B0; ++bi) {
      int c, j;
      bfly_coords<N, C, R0, SEQMAJOR>(threadIdx.x + bi * NTH, c, j);
      DFT<R0, INV>::run(v[bi]);
      st(j, std::integral_constant<int, 1>{}, c, v[bi]);
    }
  } else {
    if constexpr (LOAD_SMEM) __syncthreads();
    hook();
#pragma unroll
    for (int bi = 0; bi < B0; ++bi) {
      int c, j;
      bfly_coords<N, C, R0, SEQMAJOR>(threadIdx.x + bi * NTH, c, j);
      DFT<R0, INV>::run(v[bi]);
      smem_write_out<N, C, R0, 1, SEQMAJOR>(sm, j * R0, c, v[bi]);
    }
    __syncthreads();
    Passes<N, C, 1, P - 1, INV, SEQMAJOR, NTH, RMAX>::run(sm, tw);
    constexpr int RL = radix_of(N, P - 1, RMAX), LS = ls_of(N, P - 1, RMAX);
    constexpr int BL = (C * N / RL) / NTH;
    double2 w[BL][RL];
#pragma unroll
    for (int bi = 0; bi < BL; ++bi) {
      int c, j;
      bfly_coords<N, C, RL, SEQMAJOR>(threadIdx.x + bi * NTH, c, j);
      smem_read_bfly<N, C, RL, SEQMAJOR>(sm, j, c, w[bi]);
    }
    if constexpr (STORE_SMEM) __syncthreads();
#pragma unroll
    for (int bi = 0; bi < BL; ++bi) {
      int c, j;
      bfly_coords<N, C, RL, SEQMAJOR>(threadIdx.x + bi * NTH, c, j);
      pass_twiddles<N, RL, LS, INV>(w[bi], j, tw);
      DFT<RL, INV>::run(w[bi]);
      st(j, std::integral_constant<int, LS>{}, c, w[bi]);
    }
  }
}

// storer / loader helpers for a natural-order smem tile
template <int N, int C, bool SEQMAJOR, int R>
PD_D void smem_store_strided(double2* sm, int j, int s, int c, const double2* w) {
  const int a = lin<N, C, SEQMAJOR>(j, c);
#pragma unroll
  for (int q = 0; q < R; ++q) sm[pad(a + q * s * pos_stride<C, SEQMAJOR>())] = w[q];
}

}  // namespace pdfft
