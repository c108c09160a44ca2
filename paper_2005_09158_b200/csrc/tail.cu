// Kernels of the waveform-relaxation tail form (oracle/tail.py is the reference).
//
//   head_G:  (P_alpha - A) restricted to head rows x tail columns,
//            head_a = sum_b (pI[a][b] tail_b + pK[a][b] K tail_b)   (alpha-corner of eq 1.2, P:l.80-84)
//   reduce:  fixed-order sum of the per-CTA partials of the 1D tail map (tridiag.cu tail1d_kernel)
//   tau2d:   2D periodic transfer function of the tail map (H = 1): with K diagonal in the 2D DFT basis
//            (symbol kappa, reading c14), T(g) = Re IFFT2[ tau . FFT2(g) ],
//              tau(kx, ky) = sum_{n < F} ow_n hc_n / (lambda_1n + lambda_2n kappa(kx, ky)),
//            ow_n hc_n = m_n gamma_{Nt-1}^{-1} / Nt exp(2 pi i n (Nt-1) / Nt) (hc_n = gamma_0 = 1; m_n = half-spectrum
//            multiplicity).  Computed once per context (F N^2 complex divisions, fixed order).
//   r2c / take_real: real head <-> complex slab for the 2D filter (slab2d.cu pd_launch_slab2d_filter).
//   2D Dirichlet (leapfrog, H = 2): K = -nu Lap_h is diagonal in the tensor DST-I basis (Y = S X S, S_jk =
//            sin(pi jk/(N+1)), S^-1 = 2/(N+1) S), so tail_a = S^-1 [ sum_t tau_at . (S g_t S) ] S^-1 with the REAL
//              tau_at(kx, ky) = Re sum_{n < F} ow_n[a] hc_n[t] / (lambda_1n + lambda_2n (mu_kx + mu_ky))
//            (the tail map takes Re of the half-spectrum sum and S g S is real).  The DSTs are dense N x N products
//            (N <= 511: 2 N^3 FMAs per transform, microseconds), tiled in shared memory.
#include "common.cuh"
#include "kernels.h"

namespace {

__global__ void head_G_kernel(pd_stencil p, pd_tail_g gc, const double* __restrict__ tail, double* __restrict__ head,
                              long long S) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < S; i += (long long)gridDim.x * blockDim.x) {
    double kt[2] = {0.0, 0.0}, tv[2] = {0.0, 0.0};
    for (int b = 0; b < gc.H; ++b) {
      const double* t = tail + (long long)b * S;
      tv[b] = t[i];
      double k;
      if (p.op == 2) {
        const int nx = p.nx, ny = p.ny;
        const int x = (int)(i % nx), y = (int)(i / nx);
        const int xm = x == 0 ? nx - 1 : x - 1, xp = x == nx - 1 ? 0 : x + 1;
        const int ym = y == 0 ? ny - 1 : y - 1, yp = y == ny - 1 ? 0 : y + 1;
        k = p.k2c * tv[b] + p.k2x_m * t[(long long)y * nx + xm] + p.k2x_p * t[(long long)y * nx + xp] +
            p.k2y_m * t[(long long)ym * nx + x] + p.k2y_p * t[(long long)yp * nx + x];
      } else if (p.op == 3) {  // 2D homogeneous Dirichlet
        const int nx = p.nx, ny = p.ny;
        const int x = (int)(i % nx), y = (int)(i / nx);
        k = p.k2c * tv[b] + (x > 0 ? p.k2x_m * t[i - 1] : 0.0) + (x + 1 < nx ? p.k2x_p * t[i + 1] : 0.0) +
            (y > 0 ? p.k2y_m * t[i - nx] : 0.0) + (y + 1 < ny ? p.k2y_p * t[i + nx] : 0.0);
      } else {
        k = p.dia * tv[b] + (i > 0 ? p.sub * t[i - 1] : 0.0) + (i + 1 < S ? p.sup * t[i + 1] : 0.0);
      }
      kt[b] = k;
    }
    for (int a = 0; a < gc.H; ++a) {
      double v = 0.0;
      for (int b = 0; b < gc.H; ++b) v += gc.pI[a][b] * tv[b] + gc.pK[a][b] * kt[b];
      head[(long long)a * S + i] = v;
    }
  }
}

__global__ void reduce_rows_kernel(const double* __restrict__ part, int G, long long len, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int g = 0; g < G; ++g) s += part[(long long)g * len + i];
    out[i] = s;
  }
}

__global__ void tau2d_kernel(double2* __restrict__ tau, int N, int F, const double2* __restrict__ lam1,
                             const double2* __restrict__ lam2, const double2* __restrict__ w,
                             const double* __restrict__ sx, const double* __restrict__ sn, pd_slab_params prm) {
  const long long NN = (long long)N * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < NN; i += (long long)gridDim.x * blockDim.x) {
    const int kx = (int)(i % N), ky = (int)(i / N);
    const double2 kap = make_double2(prm.kd * (sx[kx] + sx[ky]), prm.cx * sn[kx] + prm.cy * sn[ky]);
    double2 acc = czero();
    for (int n = 0; n < F; ++n) acc = cadd(acc, cdiv(w[n], cfma(lam2[n], kap, lam1[n])));
    tau[i] = acc;
  }
}

__global__ void r2c_kernel(const double* __restrict__ g, double2* __restrict__ z, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    z[i] = make_double2(g[i], 0.0);
}

__global__ void take_real_kernel(const double2* __restrict__ z, double* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = z[i].x;
}

// Step (a) of a head-only vector E_H g: S1_n = sum_{t<H} hc[n][t] gx_t (economical Step (a), P:l.928-931), written
// for every frequency of the half spectrum (gx: the head as complex, x-transformed in the fused 2D layout)
__global__ void head_broadcast_kernel(double2* __restrict__ Sh, int F, long long S, int H, const double2* __restrict__ hc,
                                      const double2* __restrict__ gx) {
  const long long total = (long long)F * S;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(i / S);
    const long long x = i - (long long)n * S;
    double2 v = cmul(__ldg(hc + (long long)n * H), gx[x]);
    if (H == 2) v = cfma(__ldg(hc + (long long)n * H + 1), gx[S + x], v);
    __stcs(Sh + i, v);
  }
}

__global__ void any_nonzero_kernel(const double* __restrict__ x, long long n, int* flag) {
  bool nz = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    nz |= x[i] != 0.0;
  if (__syncthreads_or(nz) && threadIdx.x == 0) *flag = 1;
}

unsigned grid_for(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

namespace {

__global__ void tau_dir_kernel(double* __restrict__ tau, int N, int F, int H, const double2* __restrict__ lam1,
                               const double2* __restrict__ lam2, const double2* __restrict__ w,
                               const double* __restrict__ mu) {
  const long long NN = (long long)N * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < NN; i += (long long)gridDim.x * blockDim.x) {
    const int kx = (int)(i % N), ky = (int)(i / N);
    const double m = mu[kx + 1] + mu[ky + 1];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int n = 0; n < F; ++n) {
      const double2 den = cfma(lam2[n], make_double2(m, 0.0), lam1[n]);
      const double2 inv = crcp(den);
      for (int at = 0; at < H * H; ++at) {
        const double2 wv = w[(long long)at * F + n];
        acc[at] += wv.x * inv.x - wv.y * inv.y;  // Re(w / den)
      }
    }
    for (int at = 0; at < H * H; ++at) tau[(long long)at * NN + i] = acc[at];
  }
}

// out^T = in . S  (in, out: N x N row-major; S symmetric), 32 x 32 output tiles, 32 x 8 threads (4 outputs each)
__global__ void dst_mm_t_kernel(const double* __restrict__ in, const double* __restrict__ S, double* __restrict__ out,
                                int N) {
  __shared__ double a[32][33], b[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k0 = 0; k0 < N; k0 += 32) {
    for (int q = 0; q < 4; ++q) {
      const int r = ty + 8 * q;
      a[r][tx] = (r0 + r < N && k0 + tx < N) ? in[(long long)(r0 + r) * N + k0 + tx] : 0.0;
      b[r][tx] = (k0 + r < N && c0 + tx < N) ? S[(long long)(k0 + r) * N + c0 + tx] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; ++k)
      for (int q = 0; q < 4; ++q) acc[q] = fma(a[ty + 8 * q][k], b[k][tx], acc[q]);
    __syncthreads();
  }
  // out[c][r] = (in S)[r][c]: stage through smem for coalesced stores
  for (int q = 0; q < 4; ++q) a[ty + 8 * q][tx] = acc[q];
  __syncthreads();
  for (int q = 0; q < 4; ++q) {
    const int c = ty + 8 * q;
    if (c0 + c < N && r0 + tx < N) out[(long long)(c0 + c) * N + r0 + tx] = a[tx][c];
  }
}

// out_a = scale * sum_t tau_at . G_t  (a < H)
__global__ void tau_combine_kernel(const double* __restrict__ tau, const double* __restrict__ G, double* __restrict__ out,
                                   long long NN, int H, double scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < NN; i += (long long)gridDim.x * blockDim.x)
    for (int a = 0; a < H; ++a) {
      double v = 0.0;
      for (int t = 0; t < H; ++t) v = fma(tau[(long long)(a * H + t) * NN + i], G[(long long)t * NN + i], v);
      out[(long long)a * NN + i] = scale * v;
    }
}

}  // namespace

cudaError_t pd_launch_tau_dir(double* tau, int n, int nfreq, int H, const double2* lam1, const double2* lam2,
                              const double2* w, const double* mu, cudaStream_t st) {
  tau_dir_kernel<<<grid_for((long long)n * n, 128), 128, 0, st>>>(tau, n, nfreq, H, lam1, lam2, w, mu);
  return cudaGetLastError();
}

// 2D DST-I of H real N x N blocks, both directions (Y = S X S): two transposing products per block via tmp
cudaError_t pd_launch_dst2d_dense(const double* in, double* out, double* tmp, const double* S, int N, int H,
                                  cudaStream_t st) {
  const dim3 grid((N + 31) / 32, (N + 31) / 32), block(32, 8);
  const long long NN = (long long)N * N;
  for (int t = 0; t < H; ++t) {
    dst_mm_t_kernel<<<grid, block, 0, st>>>(in + t * NN, S, tmp, N);
    dst_mm_t_kernel<<<grid, block, 0, st>>>(tmp, S, out + t * NN, N);
  }
  return cudaGetLastError();
}

cudaError_t pd_launch_tau_combine(const double* tau, const double* G, double* out, int N, int H, double scale,
                                  cudaStream_t st) {
  const long long NN = (long long)N * N;
  tau_combine_kernel<<<grid_for(NN, 256), 256, 0, st>>>(tau, G, out, NN, H, scale);
  return cudaGetLastError();
}

cudaError_t pd_launch_head_G(const pd_stencil& p, const pd_tail_g& gc, const double* tail, double* head, long long S,
                             cudaStream_t st) {
  head_G_kernel<<<grid_for(S, 256), 256, 0, st>>>(p, gc, tail, head, S);
  return cudaGetLastError();
}

cudaError_t pd_launch_reduce_rows(const double* part, int G, long long len, double* out, cudaStream_t st) {
  reduce_rows_kernel<<<grid_for(len, 256), 256, 0, st>>>(part, G, len, out);
  return cudaGetLastError();
}

cudaError_t pd_launch_tau2d(double2* tau, int n, int nfreq, const double2* lam1, const double2* lam2, const double2* w,
                            const double* sx, const double* sn, pd_slab_params prm, cudaStream_t st) {
  tau2d_kernel<<<grid_for((long long)n * n, 128), 128, 0, st>>>(tau, n, nfreq, lam1, lam2, w, sx, sn, prm);
  return cudaGetLastError();
}

cudaError_t pd_launch_r2c(const double* g, double2* z, long long n, cudaStream_t st) {
  r2c_kernel<<<grid_for(n, 256), 256, 0, st>>>(g, z, n);
  return cudaGetLastError();
}

cudaError_t pd_launch_take_real(const double2* z, double* out, long long n, cudaStream_t st) {
  take_real_kernel<<<grid_for(n, 256), 256, 0, st>>>(z, out, n);
  return cudaGetLastError();
}

cudaError_t pd_launch_any_nonzero(const double* x, long long n, int* flag, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  any_nonzero_kernel<<<grid_for(n, 256), 256, 0, st>>>(x, n, flag);
  return cudaGetLastError();
}

cudaError_t pd_launch_head_broadcast(double2* Sh, int F, long long S, int H, const double2* hc, const double2* gx,
                                     cudaStream_t st) {
  head_broadcast_kernel<<<148 * 8, 256, 0, st>>>(Sh, F, S, H, hc, gx);
  return cudaGetLastError();
}
