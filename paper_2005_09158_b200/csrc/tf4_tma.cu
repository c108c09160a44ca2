// Forward stage 1 of the four-step time FFT (Step (a), eq 2.12, P:l.813-817), TMA-fed and persistent.
//
// Same arithmetic as tf4_fwd_s1 (tf4_stages.cuh): for a tile (t1, pairs [pl0, pl0 + KP)) the N2-point FFTs over t2
// of the Gamma-scaled rows t1 + N1 t2, times w_Nt^{t1 n2}, written to the scratch Y[t1][n2][pair].  The difference is
// how the tile reaches shared memory: one cp.async.bulk.tensor (TMA) box {2 KP doubles, 1, N2 rows} of the 3D view
// r[t2][t1][col] per tile instead of 16 per-thread loads, issued by a producer warp into an NB-deep ring of tile
// buffers guarded by mbarriers (full: TMA bytes landed; empty: the consumer group has read the tile for the last
// time).  NG consumer groups (one tile each at a time, named barriers) keep computing while NB - NG tiles are in
// flight, so the SM always has ~(NB - NG) x 32 KB of loads outstanding instead of alternating load and compute
// phases (the long-scoreboard stalls that bound tf4_fwd_s1).  Columns beyond S come back as zeros
// (TMA out-of-bounds fill).  The FFT runs in place in the tile buffer: 2 radix-R passes with R^2 = N2 (R = 16 for
// N2 = 256); with 8 pairs (128 B) per row every warp access covers whole 128 B rows, so no padding is needed.
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "fft.cuh"
#include "kernels.h"
#include "tma.cuh"

using namespace pdfft;

namespace {

template <int NT, int N2, int KP, int NB, int NG>
struct TmaS1 {
  static constexpr int R = N2 == 256 ? 16 : N2 == 64 ? 8 : 0;
  static_assert(R * R == N2, "two radix-R passes");
  static constexpr int N1 = NT / N2;
  static constexpr int TILE = N2 * KP;  // complex elements per tile
  static constexpr int GT = TILE / R;   // threads per consumer group
  static constexpr int NTH = NG * GT + 32;
  // tile ring + N2-point twiddles + the Nt-point time twiddles and Gamma (every t1 a CTA may visit) + barriers
  static constexpr size_t SMEM = (size_t)NB * TILE * 16 + N2 * 16 + (size_t)NT * 24 + 2 * NB * 8;
  static constexpr int MINB = SMEM * 2 + 2048 <= 232448 ? 2 : 1;  // CTAs per SM the shared memory allows
};

template <int NT, int N2, int KP, int NB, int NG>
__global__ void __launch_bounds__(TmaS1<NT, N2, KP, NB, NG>::NTH, TmaS1<NT, N2, KP, NB, NG>::MINB)
    tf4_fwd_s1_tma(const __grid_constant__ CUtensorMap map, long long p_begin, long long Pc, int ntiles,
                   double2* __restrict__ Y, const double* __restrict__ gam, const double2* __restrict__ tw2,
                   const double2* __restrict__ twt) {
  using T = TmaS1<NT, N2, KP, NB, NG>;
  constexpr int R = T::R, N1 = T::N1, TILE = T::TILE, GT = T::GT;
  extern __shared__ __align__(128) double2 smem[];
  double2* buf = smem;                     // [NB][TILE]
  double2* s_tw2 = smem + NB * TILE;       // [N2]
  double2* s_twt = s_tw2 + N2;             // [NT]  w_Nt^i
  double* s_g = reinterpret_cast<double*>(s_twt + NT);  // [NT]  Gamma
  uint64_t* full = reinterpret_cast<uint64_t*>(s_g + NT);
  uint64_t* empty = full + NB;
  for (int i = threadIdx.x; i < N2; i += blockDim.x) s_tw2[i] = __ldg(tw2 + i);
  for (int i = threadIdx.x; i < NT; i += blockDim.x) {
    s_twt[i] = __ldg(twt + i);
    s_g[i] = __ldg(gam + i);
  }
  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; ++b) {
      pdtma::mbar_init(full + b, 1);
      pdtma::mbar_init(empty + b, GT);
    }
    pdtma::mbar_fence_init();
  }
  __syncthreads();
  const int npt = (int)((Pc + KP - 1) / KP);  // pair tiles in the chunk; tile id = pb * N1 + t1
  if (threadIdx.x >= NG * GT) {             // producer warp
    if (threadIdx.x == NG * GT) {
      for (int k = 0, tile = blockIdx.x; tile < ntiles; ++k, tile += gridDim.x) {
        const int b = k % NB;
        if (k >= NB) pdtma::mbar_wait(empty + b, ((k / NB) - 1) & 1);
        const int t1 = tile % N1, pb = tile / N1;
        pdtma::mbar_arrive_expect_tx(full + b, TILE * 16);
        pdtma::tma_load_3d(buf + (size_t)b * TILE, &map, (int)(2 * (p_begin + (long long)pb * KP)), t1, 0, full + b);
      }
    }
    return;
  }
  const int g = threadIdx.x / GT, lt = threadIdx.x % GT;
  const int c = lt % KP, j = lt / KP;  // pair within the tile, butterfly index (both passes)
  (void)npt;
  for (int k = g, tile = blockIdx.x + g * gridDim.x; tile < ntiles; k += NG, tile += NG * gridDim.x) {
    const int b = k % NB;
    const int t1 = tile % N1, pb = tile / N1;
    double2* tb = buf + (size_t)b * TILE;
    pdtma::mbar_wait(full + b, (k / NB) & 1);
    double2 v[R];
    // pass 0: rows j + R m (m < R), Gamma-scaled; radix-R DFT over m
#pragma unroll
    for (int m = 0; m < R; ++m) {
      const int row = j + R * m;
      const double gm = s_g[t1 + N1 * row];
      const double2 x = tb[row * KP + c];
      v[m] = make_double2(gm * x.x, gm * x.y);
    }
    DFT<R, false>::run(v);
    pdtma::bar_sync(1 + g, GT);  // every thread of the group has read its pass-0 inputs
#pragma unroll
    for (int q = 0; q < R; ++q) tb[(j * R + q) * KP + c] = v[q];
    pdtma::bar_sync(1 + g, GT);
    // pass 1 (stride R): rows j + R m, twiddles w_N2^{m j}, outputs n2 = j + R q
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = tb[(j + R * m) * KP + c];
    pdtma::mbar_arrive(empty + b);  // last read of this tile buffer by this thread
#pragma unroll
    for (int m = 1; m < R; ++m) v[m] = cmul(v[m], s_tw2[m * j]);
    DFT<R, false>::run(v);
    const long long pl = (long long)pb * KP + c;
    if (pl < Pc) {
      double2* q = Y + ((long long)t1 * N2 + j) * Pc + pl;
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int n2 = j + R * m;
        __stcg(q + (long long)m * R * Pc, cmul(v[m], s_twt[t1 * n2]));
      }
    }
  }
}

#ifndef PD_TMA_NB
#define PD_TMA_NB 5  // tile buffers in the ring
#endif
#ifndef PD_TMA_NG
#define PD_TMA_NG 2  // consumer groups (4 warps each)
#endif
constexpr int kKP = 8, kNB = PD_TMA_NB, kNG = PD_TMA_NG;

struct MapKey {
  const void* p;
  long long S;
  int nt;
  bool operator==(const MapKey& o) const { return p == o.p && S == o.S && nt == o.nt; }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.p) ^ (std::hash<long long>()(k.S) * 31) ^ (size_t)k.nt;
  }
};

template <int NT>
cudaError_t launch(const double* r, long long S, long long p_begin, long long pc, double2* Y, const double* gam,
                   const double2* tw2, const double2* twt, cudaStream_t st) {
  constexpr int N2 = 256, N1 = NT / N2;
  using T = TmaS1<NT, N2, kKP, kNB, kNG>;
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> maps;
  static int attr_dev = -1, nsm = 0;
  CUtensorMap map;
  {
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
      cudaFuncSetAttribute(tf4_fwd_s1_tma<NT, N2, kKP, kNB, kNG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)T::SMEM);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      attr_dev = dev;
    }
    const MapKey key{r, S, NT};
    auto it = maps.find(key);
    if (it == maps.end()) {
      if (maps.size() > 256) maps.clear();
      // view r[t][col] as [t2][t1][col]: t = t1 + N1 t2
      const unsigned long long dims[3] = {(unsigned long long)S, (unsigned long long)N1, (unsigned long long)N2};
      const unsigned long long strides[2] = {(unsigned long long)S * 8, (unsigned long long)S * 8 * N1};
      const unsigned box[3] = {2 * kKP, 1, N2};
      if (pd_tma_encode_3d_f64(&map, r, dims, strides, box) != 0) return cudaErrorInvalidValue;
      it = maps.emplace(key, map).first;
    }
    map = it->second;
  }
  const int ntiles = (int)((pc + kKP - 1) / kKP) * N1;
  const int grid = ntiles < nsm * T::MINB ? ntiles : nsm * T::MINB;
  tf4_fwd_s1_tma<NT, N2, kKP, kNB, kNG><<<grid, T::NTH, T::SMEM, st>>>(map, p_begin, pc, ntiles, Y, gam, tw2, twt);
  return cudaGetLastError();
}

}  // namespace

int pd_tma_encode_3d_f64(CUtensorMap* map, const void* base, const unsigned long long dims[3],
                         const unsigned long long strides_bytes[2], const unsigned box[3]) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Fn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return -1;
    fn = reinterpret_cast<Fn>(p);
  }
  const cuuint64_t gd[3] = {dims[0], dims[1], dims[2]};
  const cuuint64_t gs[2] = {strides_bytes[0], strides_bytes[1]};
  const cuuint32_t bd[3] = {box[0], box[1], box[2]};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult e = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), gd, gs, bd, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return e == CUDA_SUCCESS ? 0 : -2;
}

// stage 1 of the forward four-step (N2 = 256) through TMA; r 16-byte aligned with S even (tensor-map strides).
int pd_tf4_tma_supported(int nt, long long S, const void* r) {
  const char* e = getenv("PD_TMA");
  if (!e || atoi(e) == 0) return 0;
  return nt == 2048 && S % 2 == 0 && (reinterpret_cast<uintptr_t>(r) & 15) == 0;
}

cudaError_t pd_launch_tf4_fwd_s1_tma(int nt, const double* r, long long S, long long p_begin, long long pc,
                                     double2* Y, const double* gam, const double2* tw2, const double2* twt,
                                     cudaStream_t st) {
  switch (nt) {
    case 2048: return launch<2048>(r, S, p_begin, pc, Y, gam, tw2, twt, st);
    default: return cudaErrorInvalidValue;
  }
}
