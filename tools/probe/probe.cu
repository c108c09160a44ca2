// Throwaway-style B200 microbenchmarks that decide the kernel architecture
// (HBM segment-width efficiency, L2 bandwidth, fp64 rate, DSMEM bandwidth).
// Not part of the product path. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// tile copy: array [R][S] doubles; CTA copies a W-column x RT-row tile; W in doubles (even)
__global__ void tile_copy_k(const double* __restrict__ a, double* __restrict__ b, int R, int S, int W, int RT) {
  int tiles_x = S / W;
  int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
  int tpr = W / 2;  // threads per row (16 B each)
  int rows_per_pass = blockDim.x / tpr;
  int c = threadIdx.x % tpr, r0 = threadIdx.x / tpr;
  size_t col = (size_t)tx * W + 2 * c;
  for (int r = r0; r < RT; r += rows_per_pass) {
    size_t row = (size_t)ty * RT + r;
    if (row >= (size_t)R) break;
    double2 v = *reinterpret_cast<const double2*>(a + row * S + col);
    *reinterpret_cast<double2*>(b + row * S + col) = v;
  }
}

__global__ void l2_read_k(const double2* __restrict__ a, size_t n, int reps, double* out) {
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(a + i);
      s += v.x + v.y;
    }
  if (s == 12345.678) out[0] = s;
}
__global__ void l2_rw_k(double2* a, size_t n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(a + i);
      v.x += 1.0;
      __stcg(a + i, v);
    }
}

__global__ void dfma_k(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 1.2345) out[0] = s;
}
__global__ void dadd_k(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 += c; a1 += c; a2 += c; a3 += c; a4 += c; a5 += c; a6 += c; a7 += c;
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 1.2345) out[0] = s;
}

// DSMEM: each CTA reads the smem of rank+1 repeatedly
__global__ void dsmem_k(double* out, int reps, int nelem) {
  extern __shared__ double2 sm[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < nelem; i += blockDim.x) sm[i] = make_double2(i, blockIdx.x);
  cl.sync();
  unsigned peer = (cl.block_rank() + 1) % cl.num_blocks();
  double2* ps = cl.map_shared_rank(sm, peer);
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x; i < nelem; i += blockDim.x) { double2 v = ps[i]; s += v.x + v.y; }
  cl.sync();
  if (s == 1.2345) out[0] = s;
}
__global__ void smem_k(double* out, int reps, int nelem) {
  extern __shared__ double2 sm[];
  for (int i = threadIdx.x; i < nelem; i += blockDim.x) sm[i] = make_double2(i, blockIdx.x);
  __syncthreads();
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x; i < nelem; i += blockDim.x) { double2 v = sm[(i + r) % nelem]; s += v.x + v.y; }
  if (s == 1.2345) out[0] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int l2; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  printf("device %s SMs %d L2 %d MB smemOptin %zu clock %d kHz memclk %d kHz bus %d\n", p.name, p.multiProcessorCount,
         l2 >> 20, p.sharedMemPerBlockOptin, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  const size_t NB = (size_t)2 << 30;  // 2 GiB
  double *a, *b, *out;
  CK(cudaMalloc(&a, NB)); CK(cudaMalloc(&b, NB)); CK(cudaMalloc(&out, 64));
  CK(cudaMemset(a, 0, NB)); CK(cudaMemset(b, 0, NB));
  size_t n2 = NB / 16;
  int SMs = p.multiProcessorCount;
  for (int it = 0; it < 2; ++it) copy_k<<<SMs * 8, 256>>>((double2*)a, (double2*)b, n2);
  CK(cudaEventRecord(e0));
  for (int it = 0; it < 5; ++it) copy_k<<<SMs * 8, 256>>>((double2*)a, (double2*)b, n2);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("copy double2 grid-stride: %.1f GB/s (r+w)\n", 5 * 2.0 * NB / (ms * 1e6));

  // tile copies
  int S = 4096;  // row stride 32 KB
  int R = (int)(NB / 8 / S);
  int Ws[] = {2, 4, 8, 16, 32, 64};
  for (int W : Ws) {
    for (int RT : {256, 1024, 4096}) {
      int grid = (S / W) * (R / RT);
      int threads = 256;
      tile_copy_k<<<grid, threads>>>(a, b, R, S, W, RT);
      CK(cudaEventRecord(e0));
      for (int it = 0; it < 3; ++it) tile_copy_k<<<grid, threads>>>(a, b, R, S, W, RT);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("tile copy W=%3d B seg, RT=%4d rows: %.1f GB/s\n", W * 8, RT, 3 * 2.0 * NB / (ms * 1e6));
    }
  }
  // L2-resident
  for (size_t mb : {16, 32, 48, 64}) {
    size_t n = mb * (1 << 20) / 16;
    l2_read_k<<<SMs * 8, 256>>>((double2*)a, n, 2, out);
    CK(cudaEventRecord(e0));
    l2_read_k<<<SMs * 8, 256>>>((double2*)a, n, 50, out);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("L2 read %zu MB: %.1f GB/s\n", mb, 50.0 * mb * (1 << 20) / (ms * 1e6));
    l2_rw_k<<<SMs * 8, 256>>>((double2*)a, n, 2);
    CK(cudaEventRecord(e0));
    l2_rw_k<<<SMs * 8, 256>>>((double2*)a, n, 50);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("L2 read+write %zu MB: %.1f GB/s (r+w)\n", mb, 2 * 50.0 * mb * (1 << 20) / (ms * 1e6));
  }
  // fp64
  {
    int iters = 20000;
    dfma_k<<<SMs * 8, 256>>>(out, 100);
    CK(cudaEventRecord(e0));
    dfma_k<<<SMs * 8, 256>>>(out, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double fl = 2.0 * 8 * iters * (double)SMs * 8 * 256;
    printf("DFMA: %.2f TFLOP/s (%.2f T instr/s)\n", fl / (ms * 1e9), fl / 2 / (ms * 1e9));
    dadd_k<<<SMs * 8, 256>>>(out, 100);
    CK(cudaEventRecord(e0));
    dadd_k<<<SMs * 8, 256>>>(out, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("DADD: %.2f T instr/s\n", 8.0 * iters * SMs * 8 * 256 / (ms * 1e9));
  }
  // smem / DSMEM
  for (int csz : {2, 4, 8, 16}) {
    int smem = 96 * 1024, nelem = smem / 16;
    CK(cudaFuncSetAttribute(dsmem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (csz > 8) CK(cudaFuncSetAttribute(dsmem_k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((SMs / csz) * csz); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
    cfg.attrs = at; cfg.numAttrs = 1;
    int ncl = 0;
    cudaError_t oe = cudaOccupancyMaxActiveClusters(&ncl, dsmem_k, &cfg);
    printf("cluster %d, smem 96KB: max active clusters %d (%s)\n", csz, ncl, cudaGetErrorString(oe));
    {
      int smem2 = 200 * 1024;
      CK(cudaFuncSetAttribute(dsmem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
      cudaLaunchConfig_t c2 = cfg; c2.dynamicSmemBytes = smem2;
      int n2c = 0; cudaError_t e2 = cudaOccupancyMaxActiveClusters(&n2c, dsmem_k, &c2);
      printf("cluster %d, smem 200KB: max active clusters %d (%s)\n", csz, n2c, cudaGetErrorString(e2));
      CK(cudaFuncSetAttribute(dsmem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    if (oe != cudaSuccess || ncl == 0) { cudaGetLastError(); continue; }
    int reps = 200;
    cudaError_t le = cudaLaunchKernelEx(&cfg, dsmem_k, out, 2, nelem);
    if (le != cudaSuccess) { printf("launch fail %s\n", cudaGetErrorString(le)); cudaGetLastError(); continue; }
    CK(cudaEventRecord(e0));
    CK(cudaLaunchKernelEx(&cfg, dsmem_k, out, reps, nelem));
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double bytes = (double)reps * smem * cfg.gridDim.x;
    printf("DSMEM cluster %d: %.1f GB/s total, %.1f B/clk/SM (at %d MHz)\n", csz, bytes / (ms * 1e6),
           bytes / (ms * 1e-3) / cfg.gridDim.x / (p.clockRate * 1e3), p.clockRate / 1000);
  }
  {
    int smem = 96 * 1024, nelem = smem / 16, reps = 200;
    CK(cudaFuncSetAttribute(smem_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    smem_k<<<SMs * 2, 512, smem>>>(out, 2, nelem);
    CK(cudaEventRecord(e0));
    smem_k<<<SMs * 2, 512, smem>>>(out, reps, nelem);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double bytes = (double)reps * smem * SMs * 2;
    printf("local smem: %.1f GB/s total, %.1f B/clk/SM\n", bytes / (ms * 1e6), bytes / (ms * 1e-3) / SMs / (p.clockRate * 1e3));
  }
  CK(cudaDeviceSynchronize());
  printf("probe done\n");
  return 0;
}
