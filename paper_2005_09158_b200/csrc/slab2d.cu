// Step (b), 2D periodic: S2_n = (lambda_{1,n} I + lambda_{2,n} K)^{-1} S1_n for every frequency n
// (P:l.182, 816; 2D periodic ADE P:l.908-918).  K = -nu Lap_h + ax D_x + ay D_y (5-point, centred,
// periodic) is diagonal in the 2D DFT basis with symbol
//   kappa(kx, ky) = (4 nu/h^2)(sin^2(pi kx/N) + sin^2(pi ky/N)) + i (ax sin(2 pi kx/N) + ay sin(2 pi ky/N))/h
// (reading c14), so each slab is solved exactly by   2D FFT -> divide by lambda1 + lambda2 kappa -> 2D IFFT.
//
// One thread-block cluster owns one N x N complex slab at a time and runs three phases with cluster
// barriers in between: (1) row FFTs along x, (2) column FFT along y + divide + column IFFT, (3) row
// IFFTs.  All phases work in place on the slab in global memory; with at most `num_clusters` slabs in
// flight the intermediates stay L2-resident, so HBM sees one read and one write of the slab
// (16+16 B per complex unknown) while the transposes go through L2 (B200: ~12.5 TB/s r+w measured).
#include <cooperative_groups.h>

#include "fft.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;
using namespace pdfft;

namespace {

constexpr int kBatch = 8;  // rows (phase 1/3) or columns (phase 2) per smem tile

template <int N>
struct SlabCfg {
  static constexpr int C = kBatch;
  static constexpr int E = elems_per_thread(N);
  static constexpr int NTH = C * N / E;
};

template <int N>
__global__ void __launch_bounds__(SlabCfg<N>::NTH)
slab2d_kernel(double2* __restrict__ Sh, int nfreq, const double2* __restrict__ lam1, const double2* __restrict__ lam2,
              const double* __restrict__ sx, const double* __restrict__ sn, pd_slab_params prm,
              const double2* __restrict__ tw) {
  using T = SlabCfg<N>;
  constexpr int C = T::C, NTH = T::NTH;
  extern __shared__ double2 sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int cid = blockIdx.x / cs;
  const int ncl = gridDim.x / cs;
  const int per = N / cs;  // rows (or columns) owned by this CTA, multiple of C
  const double invNN = 1.0 / ((double)N * (double)N);

  for (int n = cid; n < nfreq; n += ncl) {
    double2* slab = Sh + (long long)n * N * N;
    // ---- phase 1: forward FFT along x of rows [rank*per, (rank+1)*per) ----
    for (int r0 = rank * per; r0 < (rank + 1) * per; r0 += C) {
      double2* base = slab + (long long)r0 * N;
      for (int o = threadIdx.x; o < C * N; o += NTH) {  // o = c*N + x: contiguous rows
        sm[pad(o)] = __ldcg(base + o);
      }
      __syncthreads();
      fft_smem<N, C, false, true, NTH>(sm, tw);
      for (int o = threadIdx.x; o < C * N; o += NTH) __stcg(base + o, sm[pad(o)]);
      __syncthreads();
    }
    cluster.sync();
    // ---- phase 2: columns [rank*per, (rank+1)*per): FFT along y, divide, inverse FFT along y ----
    const double2 l1 = lam1[n], l2 = lam2[n];
    for (int c0 = rank * per; c0 < (rank + 1) * per; c0 += C) {
      for (int o = threadIdx.x; o < C * N; o += NTH) {  // o = y*C + c: C contiguous columns per row
        const int y = o / C, c = o % C;
        sm[pad(o)] = __ldcg(slab + (long long)y * N + c0 + c);
      }
      __syncthreads();
      fft_smem<N, C, false, false, NTH>(sm, tw);
      for (int o = threadIdx.x; o < C * N; o += NTH) {
        const int ky = o / C, kx = c0 + o % C;
        const double2 kap = make_double2(prm.kd * (sx[kx] + sx[ky]), prm.cx * sn[kx] + prm.cy * sn[ky]);
        const double2 den = cfma(l2, kap, l1);
        sm[pad(o)] = cscale(cdiv(sm[pad(o)], den), invNN);
      }
      __syncthreads();
      fft_smem<N, C, true, false, NTH>(sm, tw);
      for (int o = threadIdx.x; o < C * N; o += NTH) {
        const int y = o / C, c = o % C;
        __stcg(slab + (long long)y * N + c0 + c, sm[pad(o)]);
      }
      __syncthreads();
    }
    cluster.sync();
    // ---- phase 3: inverse FFT along x of the rows ----
    for (int r0 = rank * per; r0 < (rank + 1) * per; r0 += C) {
      double2* base = slab + (long long)r0 * N;
      for (int o = threadIdx.x; o < C * N; o += NTH) sm[pad(o)] = __ldcg(base + o);
      __syncthreads();
      fft_smem<N, C, true, true, NTH>(sm, tw);
      for (int o = threadIdx.x; o < C * N; o += NTH) __stcg(base + o, sm[pad(o)]);
      __syncthreads();
    }
    // no barrier needed before the next slab: it touches a disjoint slab
  }
}

template <int N>
int smem_bytes() {
  return smem_elems(kBatch * N) * (int)sizeof(double2);
}

template <int N>
cudaError_t launch_n(double2* Sh, int nfreq, const double2* lam1, const double2* lam2, const double* sx,
                     const double* sn, pd_slab_params prm, const double2* tw, int ncl, int cs, cudaStream_t st) {
  if (N % (cs * kBatch) != 0) return cudaErrorInvalidValue;
  const int smem = smem_bytes<N>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(slab2d_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess && cs > 8)
      e = cudaFuncSetAttribute(slab2d_kernel<N>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(ncl * cs);
  cfg.blockDim = dim3(SlabCfg<N>::NTH);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, slab2d_kernel<N>, Sh, nfreq, lam1, lam2, sx, sn, prm, tw);
}

template <int N>
int max_clusters_n(int cs) {
  const int smem = smem_bytes<N>();
  cudaFuncSetAttribute(slab2d_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (cs > 8) cudaFuncSetAttribute(slab2d_kernel<N>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(cs * 64);
  cfg.blockDim = dim3(SlabCfg<N>::NTH);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, slab2d_kernel<N>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return ncl;
}

}  // namespace

int pd_slab2d_supported(int n) { return n == 16 || n == 32 || n == 64 || n == 128 || n == 256 || n == 512 || n == 1024; }

int pd_slab2d_max_clusters(int n, int cs) {
  switch (n) {
    case 16: return max_clusters_n<16>(cs);
    case 32: return max_clusters_n<32>(cs);
    case 64: return max_clusters_n<64>(cs);
    case 128: return max_clusters_n<128>(cs);
    case 256: return max_clusters_n<256>(cs);
    case 512: return max_clusters_n<512>(cs);
    case 1024: return max_clusters_n<1024>(cs);
    default: return 0;
  }
}

cudaError_t pd_launch_slab2d(double2* Sh, int n, int nfreq, const double2* lam1, const double2* lam2,
                             const double* sx, const double* sn, pd_slab_params prm, const double2* tw,
                             int num_clusters, int cluster_size, cudaStream_t st) {
  switch (n) {
#define PD_CASE(v) \
  case v:          \
    return launch_n<v>(Sh, nfreq, lam1, lam2, sx, sn, prm, tw, num_clusters, cluster_size, st);
    PD_CASE(16) PD_CASE(32) PD_CASE(64) PD_CASE(128) PD_CASE(256) PD_CASE(512) PD_CASE(1024)
#undef PD_CASE
    default:
      return cudaErrorInvalidValue;
  }
}
