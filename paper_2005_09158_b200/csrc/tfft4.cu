// Steps (a)/(c) for long time axes (Nt >= 1024): four-step time FFT, Nt = N1 * N2 (N2 = 64).
//
//   forward:  X[n2 + N2 n1] = sum_t1 w_N1^{t1 n1} [ w_Nt^{t1 n2} sum_t2 x[t1 + N1 t2] w_N2^{t2 n2} ]
//   inverse:  x[t1 + N1 t2] = sum_n2 w_N2^{-t2 n2} [ w_Nt^{-t1 n2} sum_n1 X[n2 + N2 n1] w_N1^{-t1 n1} ]
// (same maps as tfft.cu: Step (a) S1 = F Gamma r, Step (c) z = Gamma^{-1} F^* S2 / Nt, eq 2.12, P:l.813-817;
//  Matlab fft/ifft pairing P:l.864-875).  Two real spatial columns are packed into one complex sequence
// ("pair" p = columns 2p, 2p+1) and separated again on the half spectrum (reading c15).
//
// Why: a single-tile time FFT of Nt = 2048-4096 complex points needs 64-128 KB of shared memory per
// handful of columns, which leaves one CTA per SM (no load/compute overlap) and 32-64 B HBM row
// segments.  Here every stage touches 64 rows x 32 pairs (512 B segments, 32 KB tiles, several CTAs
// per SM); the intermediate Y (complex, Nt x pairs) lives in a scratch buffer processed in column chunks.
// Measured on B200 (cfg4): per-chunk launches of L2-resident chunks (<= 64 MB) are launch/ramp bound
// (~18 us per launch), while chunks of ~1 GB run the two stages at ~6.3 TB/s of actual DRAM traffic with
// the intermediate going through HBM (16 B/dof extra); the default is the latter.  A
// persistent task-queue variant and a cp.async.bulk-pipelined variant were both measured slower.
#include <cstdlib>

#include "fft.cuh"
#include "kernels.h"
#include "tf4_stages.cuh"

using namespace pdfft;
using namespace pdfft_tf4;

namespace {

constexpr int kP = 32;   // pairs (complex sequences) per tile in stage 1
constexpr int kN2 = 64;  // stage-1 FFT length

template <int N>
struct Cfg2 {  // stage FFT of length N over C sequences
  static constexpr int E = elems_per_thread(N);
};

// ---------------------------------------------------------------------------------------------
// forward stage 2: for the pair of residues (n2, N2-n2) (blockIdx.y = n2 in [0, N2/2]): N1-point FFTs over
// t1 of Y[t1][n2][.], then separation of the two real columns on the half spectrum rows n <= Nt/2.
// Sequences c in [0, 2P): c < P -> residue n2, pair c;  c >= P -> residue n2' = (N2-n2)%N2, pair c-P.
// ---------------------------------------------------------------------------------------------
template <int NT, int RM = 16, bool SH = false>
__global__ void __launch_bounds__(2 * kP * (NT / kN2) / elems_per_thread(NT / kN2, RM))
tf4_fwd_s2(const double2* __restrict__ Y, long long S, long long p_begin, long long npairs_chunk,
           const pd_spec sp, const double2* __restrict__ tw1) {
  constexpr int N1 = NT / kN2, C = 2 * kP, NTH = C * N1 / elems_per_thread(N1, RM);
  extern __shared__ double2 sm[];
  __shared__ double2 s_tw1[N1];
  const int n2 = blockIdx.y, n2p = (kN2 - n2) % kN2;
  const long long pl0 = (long long)blockIdx.x * kP;
  const long long p0 = p_begin + pl0;
  const long long Pc = npairs_chunk;
  load_table(s_tw1, tw1, N1);
  __syncthreads();
  const bool fullp = pl0 + kP <= Pc;
  fft_io<N1, C, false, false, NTH, false, true, RM>(
      sm, s_tw1,
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value, R0 = first_radix(N1, RM);
        const int rr = c < kP ? n2 : n2p, pc = c & (kP - 1);
        const bool ok = fullp || pl0 + pc < Pc;
        const double2* q = Y + ((long long)j * kN2 + rr) * Pc + pl0 + pc;
#pragma unroll
        for (int m = 0; m < R0; ++m) v[m] = ok ? __ldcg(q + (long long)m * s * kN2 * Pc) : czero();
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value, RL = last_radix(N1, RM);
        const int a = lin<N1, C, false>(j, c);
#pragma unroll
        for (int m = 0; m < RL; ++m) sm[soff<s * C>(a, m)] = w[m];
      });
  __syncthreads();
  // outputs: rows n = rr + N2 n1 <= Nt/2 for rr in {n2, n2'} (each once), 2P real columns per row
  const int nsets = (n2p == n2) ? 1 : 2;
  const int total = nsets * N1 * 2 * kP;
  for (int o = threadIdx.x; o < total; o += NTH) {
    const int col = o % (2 * kP);
    const int rowi = o / (2 * kP);          // [0, nsets*N1)
    const int set = rowi / N1, n1 = rowi % N1;
    const int rr = set == 0 ? n2 : n2p;
    const int n = rr + kN2 * n1;
    if (n > NT / 2) continue;
    // partner index Nt - n = rr' + N2 n1'
    const int m = (NT - n) & (NT - 1);
    const int rrp = m % kN2, n1p = m / kN2;
    const int pc = col >> 1;
    const int cs = (rr == n2 ? 0 : kP) + pc;
    const int cp = (rrp == n2 ? 0 : kP) + pc;
    const double2 z1 = sm[sidx<N1, C, false>(n1, cs)];
    const double2 z2 = sm[sidx<N1, C, false>(n1p, cp)];
    double2 v;
    if (col & 1)
      v = make_double2(0.5 * (z1.y + z2.y), -0.5 * (z1.x - z2.x));
    else
      v = make_double2(0.5 * (z1.x + z2.x), 0.5 * (z1.y - z2.y));
    const long long gcol = 2 * p0 + col;
    if (pl0 + pc < Pc && gcol < S) __stcs(pd_spec_row<SH>(sp, n) + gcol, v);
  }
}

// ---------------------------------------------------------------------------------------------
// inverse stage 1: for residues (n2, N2-n2): rebuild Z[n] = X[n] + i Y[n] from the half spectrum, N1-point
// inverse FFTs over n1, times w_Nt^{-t1 n2}; writes W[n2][t1][pl].
// ---------------------------------------------------------------------------------------------
template <int NT, int RM = 16, bool SH = false>
__global__ void __launch_bounds__(2 * kP * (NT / kN2) / elems_per_thread(NT / kN2, RM))
tf4_inv_s1(const pd_spec sp, long long S, long long p_begin, long long npairs_chunk,
           double2* __restrict__ W, const double2* __restrict__ tw1, const double2* __restrict__ twt) {
  constexpr int N1 = NT / kN2, C = 2 * kP, NTH = C * N1 / elems_per_thread(N1, RM);
  extern __shared__ double2 sm[];
  __shared__ double2 s_tw1[N1], s_twa[N1], s_twb[N1];  // N1 twiddles; w_Nt^{-t1 n2}, w_Nt^{-t1 n2'}
  const int n2 = blockIdx.y, n2p = (kN2 - n2) % kN2;
  const long long pl0 = (long long)blockIdx.x * kP;
  const long long p0 = p_begin + pl0;
  const long long Pc = npairs_chunk;
  for (int i = threadIdx.x; i < N1; i += NTH) {
    s_tw1[i] = __ldg(tw1 + i);
    s_twa[i] = cconj(__ldg(twt + i * n2));
    s_twb[i] = cconj(__ldg(twt + i * n2p));
  }
  // stage the half-spectrum rows n <= Nt/2 with n % N2 in {n2, n2'}: slot (set, n1) -> 2P complex
  const int nsets = (n2p == n2) ? 1 : 2;
  const int total = nsets * N1 * 2 * kP;
  {
    // all of a thread's loads in flight before the first smem store
    constexpr int PT = (2 * N1 * 2 * kP + NTH - 1) / NTH;
    double2 v[PT];
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      const int o = threadIdx.x + k * NTH;
      const int col = o % (2 * kP);
      const int rowi = o / (2 * kP);
      const int set = rowi / N1, n1 = rowi % N1;
      const int n = (set == 0 ? n2 : n2p) + kN2 * n1;
      const long long gcol = 2 * p0 + col;
      v[k] = czero();
      if (o < total && n <= NT / 2 && pl0 + (col >> 1) < Pc && gcol < S) v[k] = __ldcs(pd_spec_row<SH>(sp, n) + gcol);
    }
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      const int o = threadIdx.x + k * NTH;
      if (o < total) sm[pad(o)] = v[k];
    }
  }
  __syncthreads();
  const bool fullp = pl0 + kP <= Pc;
  fft_io<N1, C, true, false, NTH, true, false, RM>(
      sm, s_tw1,
      [&](int j, auto st, int c, double2* v) {
        constexpr int s = decltype(st)::value, R0 = first_radix(N1, RM);
        const int rr = c < kP ? n2 : n2p, pc = c & (kP - 1);
#pragma unroll
        for (int m = 0; m < R0; ++m) {
          const int n1 = j + m * s;
          const int n = rr + kN2 * n1;
          const bool lo = n <= NT / 2;
          const int mm = lo ? n : NT - n;  // row held in smem (<= Nt/2)
          const int slot = ((mm % kN2) == n2 ? 0 : 1) * N1 + mm / kN2;
          const double sg = lo ? 1.0 : -1.0;
          const int base = slot * 2 * kP + 2 * pc;
          const double2 X = sm[pad(base)], Yv = sm[pad(base + 1)];
          v[m] = make_double2(fma(-sg, Yv.y, X.x), fma(sg, X.y, Yv.x));
        }
      },
      [&](int j, auto st, int c, const double2* w) {
        constexpr int s = decltype(st)::value, RL = last_radix(N1, RM);
        const int rr = c < kP ? n2 : n2p, pc = c & (kP - 1);
        if (c >= kP && nsets == 1) return;  // duplicate of the self-partnered residue
        if (!(fullp || pl0 + pc < Pc)) return;
        const double2* tws = c < kP ? s_twa : s_twb;
        double2* q = W + ((long long)rr * N1 + j) * Pc + pl0 + pc;
#pragma unroll
        for (int m = 0; m < RL; ++m) __stcg(q + (long long)m * s * Pc, cmul(w[m], tws[j + m * s]));
      });
}


// non-persistent grid versions: one CTA per tile
template <int NT, int RM>
void fwd_grid(const double* r, const pd_spec& sp, long long S, const double* gam, const pd_tf4_tables& tb,
              double2* scratch, long long p, long long pc, bool vec, cudaStream_t st) {
  constexpr int N1 = NT / kN2;
  const int sm1 = smem_of<kN2>(kP), sm2 = smem_of<N1>(2 * kP);
  static int attr = -1;  // device on which the attributes were set
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (attr != dev_) {
    cudaFuncSetAttribute(tf4_fwd_s1<NT, kN2, kP, true, RM>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
    cudaFuncSetAttribute(tf4_fwd_s1<NT, kN2, kP, false, RM>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
    cudaFuncSetAttribute(tf4_fwd_s2<NT, RM, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    cudaFuncSetAttribute(tf4_fwd_s2<NT, RM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    attr = dev_;
  }
  const unsigned nt1 = (unsigned)((pc + kP - 1) / kP);
  const dim3 g1(nt1, N1), g2(nt1, kN2 / 2 + 1);
  if (vec)
    tf4_fwd_s1<NT, kN2, kP, true, RM><<<g1, kP * kN2 / RM, sm1, st>>>(r, S, p, pc, scratch, gam, tb.tw2, tb.twt);
  else
    tf4_fwd_s1<NT, kN2, kP, false, RM><<<g1, kP * kN2 / RM, sm1, st>>>(r, S, p, pc, scratch, gam, tb.tw2, tb.twt);
  if (sp.P > 1)
    tf4_fwd_s2<NT, RM, true><<<g2, 2 * kP * N1 / elems_per_thread(N1, RM), sm2, st>>>(scratch, S, p, pc, sp, tb.tw1);
  else
    tf4_fwd_s2<NT, RM, false><<<g2, 2 * kP * N1 / elems_per_thread(N1, RM), sm2, st>>>(scratch, S, p, pc, sp, tb.tw1);
}

template <int NT, int RM>
void inv_grid(const pd_spec& sp, double* z, long long S, const double* igam, const pd_tf4_tables& tb,
              double2* scratch, long long p, long long pc, int accumulate, bool vec, cudaStream_t st) {
  constexpr int N1 = NT / kN2;
  const int sm1 = smem_of<N1>(2 * kP) > smem_elems(2 * N1 * 2 * kP) * (int)sizeof(double2)
                      ? smem_of<N1>(2 * kP)
                      : smem_elems(2 * N1 * 2 * kP) * (int)sizeof(double2);
  const int sm2 = smem_of<kN2>(kP);
  static int attr = -1;  // device on which the attributes were set
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (attr != dev_) {
    cudaFuncSetAttribute(tf4_inv_s1<NT, RM, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
    cudaFuncSetAttribute(tf4_inv_s1<NT, RM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1);
    cudaFuncSetAttribute(tf4_inv_s2<NT, kN2, kP, true, 0, RM>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    cudaFuncSetAttribute(tf4_inv_s2<NT, kN2, kP, true, 1, RM>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    cudaFuncSetAttribute(tf4_inv_s2<NT, kN2, kP, false, 0, RM>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    cudaFuncSetAttribute(tf4_inv_s2<NT, kN2, kP, false, 1, RM>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    attr = dev_;
  }
  const unsigned nt1 = (unsigned)((pc + kP - 1) / kP);
  const dim3 g1(nt1, kN2 / 2 + 1), g2(nt1, N1);
  if (sp.P > 1)
    tf4_inv_s1<NT, RM, true><<<g1, 2 * kP * N1 / elems_per_thread(N1, RM), sm1, st>>>(sp, S, p, pc, scratch, tb.tw1, tb.twt);
  else
    tf4_inv_s1<NT, RM, false><<<g1, 2 * kP * N1 / elems_per_thread(N1, RM), sm1, st>>>(sp, S, p, pc, scratch, tb.tw1, tb.twt);
  const int th2 = kP * kN2 / RM;
  if (vec) {
    if (accumulate)
      tf4_inv_s2<NT, kN2, kP, true, 1, RM><<<g2, th2, sm2, st>>>(scratch, S, p, pc, z, igam, tb.tw2);
    else
      tf4_inv_s2<NT, kN2, kP, true, 0, RM><<<g2, th2, sm2, st>>>(scratch, S, p, pc, z, igam, tb.tw2);
  } else {
    if (accumulate)
      tf4_inv_s2<NT, kN2, kP, false, 1, RM><<<g2, th2, sm2, st>>>(scratch, S, p, pc, z, igam, tb.tw2);
    else
      tf4_inv_s2<NT, kN2, kP, false, 0, RM><<<g2, th2, sm2, st>>>(scratch, S, p, pc, z, igam, tb.tw2);
  }
}

constexpr int kRmaxGrid = 8;  // radix-8 passes: 8 elements per thread, twice the warps of radix 16 (measured faster)

// chunk ci of a call: stream / scratch ci mod K of the optional pipeline (kernels.h pd_tfx_overlap)
template <int NT>
cudaError_t fwd_n(const double* r, const pd_spec& sp, long long S, const double* gam, const pd_tf4_tables& tb,
                  double2* scratch0, long long chunk_pairs, cudaStream_t st0, int* nl, const pd_tfx_overlap* ov) {
  const bool vec = (S % 2 == 0) && ((reinterpret_cast<uintptr_t>(r) & 15) == 0);
  const long long npairs = (S + 1) / 2;
  int n = 0;
  if (cudaError_t e = ov_fork(ov, st0)) return e;
  for (long long p = 0, ci = 0; p < npairs; p += chunk_pairs, ++ci) {
    const int lane = ov ? (int)(ci % ov->k) : 0;
    const long long pc = npairs - p < chunk_pairs ? npairs - p : chunk_pairs;
    fwd_grid<NT, kRmaxGrid>(r, sp, S, gam, tb, lane ? ov->scratch[lane] : scratch0, p, pc, vec,
                            lane ? ov->st[lane] : st0);
    n += 2;
  }
  *nl = n;
  return ov_join(ov, st0);
}

template <int NT>
cudaError_t inv_n(const pd_spec& sp, double* z, long long S, const double* igam, const pd_tf4_tables& tb,
                  double2* scratch0, long long chunk_pairs, int accumulate, cudaStream_t st0, int* nl,
                  const pd_tfx_overlap* ov) {
  const bool vec = (S % 2 == 0) && ((reinterpret_cast<uintptr_t>(z) & 15) == 0);
  const long long npairs = (S + 1) / 2;
  int n = 0;
  if (cudaError_t e = ov_fork(ov, st0)) return e;
  for (long long p = 0, ci = 0; p < npairs; p += chunk_pairs, ++ci) {
    const int lane = ov ? (int)(ci % ov->k) : 0;
    const long long pc = npairs - p < chunk_pairs ? npairs - p : chunk_pairs;
    inv_grid<NT, kRmaxGrid>(sp, z, S, igam, tb, lane ? ov->scratch[lane] : scratch0, p, pc, accumulate, vec,
                            lane ? ov->st[lane] : st0);
    n += 2;
  }
  *nl = n;
  return ov_join(ov, st0);
}

}  // namespace

int pd_tf4_supported(int nt) { return nt == 1024 || nt == 2048 || nt == 4096; }
int pd_tf4_n2() { return kN2; }
int pd_tf4_pairs_per_tile() { return kP; }

cudaError_t pd_launch_tf4_fwd(int nt, const double* r, const pd_spec& sp, long long S, const double* gam,
                              const pd_tf4_tables& tb, double2* scratch, long long chunk_pairs, cudaStream_t st,
                              int* nl, const pd_tfx_overlap* ov) {
  switch (nt) {
    case 1024: return fwd_n<1024>(r, sp, S, gam, tb, scratch, chunk_pairs, st, nl, ov);
    case 2048: return fwd_n<2048>(r, sp, S, gam, tb, scratch, chunk_pairs, st, nl, ov);
    case 4096: return fwd_n<4096>(r, sp, S, gam, tb, scratch, chunk_pairs, st, nl, ov);
    case 8192: return fwd_n<8192>(r, sp, S, gam, tb, scratch, chunk_pairs, st, nl, ov);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t pd_launch_tf4_inv(int nt, const pd_spec& sp, double* z, long long S, const double* igam,
                              const pd_tf4_tables& tb, double2* scratch, long long chunk_pairs, int accumulate,
                              cudaStream_t st, int* nl, const pd_tfx_overlap* ov) {
  switch (nt) {
    case 1024: return inv_n<1024>(sp, z, S, igam, tb, scratch, chunk_pairs, accumulate, st, nl, ov);
    case 2048: return inv_n<2048>(sp, z, S, igam, tb, scratch, chunk_pairs, accumulate, st, nl, ov);
    case 4096: return inv_n<4096>(sp, z, S, igam, tb, scratch, chunk_pairs, accumulate, st, nl, ov);
    case 8192: return inv_n<8192>(sp, z, S, igam, tb, scratch, chunk_pairs, accumulate, st, nl, ov);
    default: return cudaErrorInvalidValue;
  }
}
