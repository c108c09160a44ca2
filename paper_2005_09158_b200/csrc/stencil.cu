// All-at-once residual r = b - A u and matvec w = A u, A = B1 (x) I + B2 (x) K (eq 1.1, P:l.80-84),
// with the time taps of eq 2.5b (theta-method, P:l.309-319) and eq 3.2b (implicit leapfrog, P:l.1214-1227):
//   (A u)_n = sum_k c1_k u_{n-k} + K ( sum_k c2_k u_{n-k} ),   terms with n-k < 0 dropped (U_0 lives in b).
// One thread per spatial point walks a chunk of time rows, keeping the stencil neighbourhood of the
// previous rows in registers; per-block partial sums of r^2 feed a deterministic fixed-order reduction.
// Also the right-hand side b of A u = b from (U_0, V_0, f) (readings c4, c5).
#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int kTC = 64;     // time rows per thread
constexpr int kBX = 256;    // threads per block

struct Taps {
  double c1[3], c2[3];
  int ntaps;
};

PD_D Taps taps_of(const pd_stencil& p) {
  Taps t;
  if (p.scheme == 2) {
    const double i2 = 1.0 / (p.dt * p.dt);
    t.c1[0] = i2; t.c1[1] = -2.0 * i2; t.c1[2] = i2;
    t.c2[0] = 0.5; t.c2[1] = 0.0; t.c2[2] = 0.5;
    t.ntaps = 3;
  } else {
    t.c1[0] = 1.0 / p.dt; t.c1[1] = -1.0 / p.dt; t.c1[2] = 0.0;
    t.c2[0] = p.theta; t.c2[1] = 1.0 - p.theta; t.c2[2] = 0.0;
    t.ntaps = 2;
  }
  return t;
}

// ---------------- 1D: neighbourhood = (x-1, x, x+1) ----------------
struct N1 { double l, c, r; };

// hl, hr: halo rows (neighbour values for x = -1 and x = nx) or NULL for the Dirichlet zero
PD_D N1 load1(const double* __restrict__ row, int x, int nx, const double* hl, const double* hr) {
  N1 v;
  v.c = row[x];
  v.l = x > 0 ? row[x - 1] : (hl ? *hl : 0.0);
  v.r = x + 1 < nx ? row[x + 1] : (hr ? *hr : 0.0);
  return v;
}

__global__ void __launch_bounds__(kBX) stencil1d_kernel(pd_stencil p, const double* __restrict__ b,
                                                       const double* __restrict__ u, double* __restrict__ out,
                                                       double* __restrict__ partial) {
  const Taps tp = taps_of(p);
  const int x = blockIdx.x * kBX + threadIdx.x;
  const int n0 = blockIdx.y * kTC;
  const int nx = p.nx;
  const bool act = x < nx;
  double acc = 0.0;
  N1 h1 = {0, 0, 0}, h2 = {0, 0, 0};  // rows n-1, n-2
  const double* hl = p.hlo;
  const double* hr = p.hhi;
  if (act) {
    if (n0 - 1 >= 0) h1 = load1(u + (long long)(n0 - 1) * nx, x, nx, hl ? hl + n0 - 1 : nullptr, hr ? hr + n0 - 1 : nullptr);
    if (n0 - 2 >= 0) h2 = load1(u + (long long)(n0 - 2) * nx, x, nx, hl ? hl + n0 - 2 : nullptr, hr ? hr + n0 - 2 : nullptr);
  }
  const int n1 = min(n0 + kTC, p.nt);
#pragma unroll 8
  for (int n = n0; n < n1; ++n) {
    N1 h0 = {0, 0, 0};
    if (act) h0 = load1(u + (long long)n * nx, x, nx, hl ? hl + n : nullptr, hr ? hr + n : nullptr);
    // y = sum_k c2_k u_{n-k}; Au = sum_k c1_k u_{n-k} + K y
    const double yl = tp.c2[0] * h0.l + tp.c2[1] * h1.l + tp.c2[2] * h2.l;
    const double yc = tp.c2[0] * h0.c + tp.c2[1] * h1.c + tp.c2[2] * h2.c;
    const double yr = tp.c2[0] * h0.r + tp.c2[1] * h1.r + tp.c2[2] * h2.r;
    double Au = tp.c1[0] * h0.c + tp.c1[1] * h1.c + tp.c1[2] * h2.c;
    Au += p.sub * yl + p.dia * yc + p.sup * yr;
    if (act) {
      const long long idx = (long long)n * nx + x;
      const double v = b ? b[idx] - Au : Au;
      out[idx] = v;
      acc = fma(v, v, acc);
    }
    h2 = h1;
    h1 = h0;
  }
  // deterministic block reduction
  __shared__ double red[kBX / 32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kBX / 32; ++w) s += red[w];
    partial[blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
}

// ---------------- 2D periodic: neighbourhood = (c, x-1, x+1, y-1, y+1) ----------------
struct N2 { double c, xm, xp, ym, yp; };

// hl, hr: halo rows for y = -1 and y = ny (neighbour ranks) or NULL for the periodic wrap within the slab
PD_D N2 load2(const double* __restrict__ slab, int x, int y, int nx, int ny, const double* hl, const double* hr) {
  N2 v;
  const int xm = x == 0 ? nx - 1 : x - 1, xp = x == nx - 1 ? 0 : x + 1;
  v.c = slab[(long long)y * nx + x];
  v.xm = slab[(long long)y * nx + xm];
  v.xp = slab[(long long)y * nx + xp];
  v.ym = y > 0 ? slab[(long long)(y - 1) * nx + x] : (hl ? hl[x] : slab[(long long)(ny - 1) * nx + x]);
  v.yp = y + 1 < ny ? slab[(long long)(y + 1) * nx + x] : (hr ? hr[x] : slab[x]);
  return v;
}

__global__ void __launch_bounds__(kBX) stencil2d_kernel(pd_stencil p, const double* __restrict__ b,
                                                       const double* __restrict__ u, double* __restrict__ out,
                                                       double* __restrict__ partial) {
  const Taps tp = taps_of(p);
  const int nx = p.nx, ny = p.ny;
  const long long S = (long long)nx * ny;
  const long long s = (long long)blockIdx.x * kBX + threadIdx.x;
  const bool act = s < S;
  const int x = act ? (int)(s % nx) : 0, y = act ? (int)(s / nx) : 0;
  const int n0 = blockIdx.y * kTC;
  double acc = 0.0;
  N2 h1 = {0, 0, 0, 0, 0}, h2 = {0, 0, 0, 0, 0};
  const double* hl = p.hlo;
  const double* hr = p.hhi;
  if (act) {
    if (n0 - 1 >= 0)
      h1 = load2(u + (n0 - 1) * S, x, y, nx, ny, hl ? hl + (long long)(n0 - 1) * nx : nullptr,
                 hr ? hr + (long long)(n0 - 1) * nx : nullptr);
    if (n0 - 2 >= 0)
      h2 = load2(u + (n0 - 2) * S, x, y, nx, ny, hl ? hl + (long long)(n0 - 2) * nx : nullptr,
                 hr ? hr + (long long)(n0 - 2) * nx : nullptr);
  }
  const int n1 = min(n0 + kTC, p.nt);
#pragma unroll 4
  for (int n = n0; n < n1; ++n) {
    N2 h0 = {0, 0, 0, 0, 0};
    if (act)
      h0 = load2(u + n * S, x, y, nx, ny, hl ? hl + (long long)n * nx : nullptr, hr ? hr + (long long)n * nx : nullptr);
    const double yc = tp.c2[0] * h0.c + tp.c2[1] * h1.c + tp.c2[2] * h2.c;
    const double yxm = tp.c2[0] * h0.xm + tp.c2[1] * h1.xm + tp.c2[2] * h2.xm;
    const double yxp = tp.c2[0] * h0.xp + tp.c2[1] * h1.xp + tp.c2[2] * h2.xp;
    const double yym = tp.c2[0] * h0.ym + tp.c2[1] * h1.ym + tp.c2[2] * h2.ym;
    const double yyp = tp.c2[0] * h0.yp + tp.c2[1] * h1.yp + tp.c2[2] * h2.yp;
    double Au = tp.c1[0] * h0.c + tp.c1[1] * h1.c + tp.c1[2] * h2.c;
    Au += p.k2c * yc + p.k2x_m * yxm + p.k2x_p * yxp + p.k2y_m * yym + p.k2y_p * yyp;
    if (act) {
      const long long idx = n * S + s;
      const double v = b ? b[idx] - Au : Au;
      out[idx] = v;
      acc = fma(v, v, acc);
    }
    h2 = h1;
    h1 = h0;
  }
  __shared__ double red[kBX / 32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kBX / 32; ++w) t += red[w];
    partial[blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

// ---------------- right-hand side ----------------
// K v at spatial point s of a single time level (zero Dirichlet / periodic wrap)
PD_D double applyK(const pd_stencil& p, const double* __restrict__ v, long long s, int which) {
  const int hw = p.op == 2 ? p.nx : 1;
  const double* hl = p.hlo ? p.hlo + which * hw : nullptr;
  const double* hr = p.hhi ? p.hhi + which * hw : nullptr;
  if (p.op == 2) {
    const N2 h = load2(v, (int)(s % p.nx), (int)(s / p.nx), p.nx, p.ny, hl, hr);
    return p.k2c * h.c + p.k2x_m * h.xm + p.k2x_p * h.xp + p.k2y_m * h.ym + p.k2y_p * h.yp;
  }
  const N1 h = load1(v, (int)s, p.nx, hl, hr);
  return p.sub * h.l + p.dia * h.c + p.sup * h.r;
}

__global__ void rhs_kernel(pd_stencil p, const double* __restrict__ u0, const double* __restrict__ v0,
                           const double* __restrict__ f, double* __restrict__ b) {
  const long long S = (long long)p.nx * p.ny;
  const long long total = S * p.nt;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(i / S);
    const long long s = i % S;
    double v = 0.0;
    if (p.scheme == 2) {
      // leapfrog (reading c4): b_1 = f_0/2 + U0/dt^2 + V0/dt + dt/2 K V0; b_2 = f_1 - U0/dt^2 - K U0/2; b_n = f_{n-1}
      const double i2 = 1.0 / (p.dt * p.dt);
      if (f) v = (n == 0) ? 0.5 * f[s] : f[(long long)n * S + s];
      if (n == 0) {
        v += u0[s] * i2;
        if (v0) v += v0[s] / p.dt + 0.5 * p.dt * applyK(p, v0, s, 1);
      } else if (n == 1) {
        v += -u0[s] * i2 - 0.5 * applyK(p, u0, s, 0);
      }
    } else {
      // theta-method (P:l.321-323, reading c5): b_n = theta f_n + (1-theta) f_{n-1}; b_1 += (I/dt - (1-theta)K) U0
      if (f) v = p.theta * f[(long long)(n + 1) * S + s] + (1.0 - p.theta) * f[(long long)n * S + s];
      if (n == 0) v += u0[s] / p.dt - (1.0 - p.theta) * applyK(p, u0, s, 0);
    }
    b[i] = v;
  }
}

}  // namespace

cudaError_t pd_launch_stencil(const pd_stencil& p, const double* b, const double* u, double* out, double* partial,
                              int* nblocks_out, cudaStream_t st) {
  const long long S = (long long)p.nx * p.ny;
  dim3 grid((unsigned)((S + kBX - 1) / kBX), (unsigned)((p.nt + kTC - 1) / kTC));
  if (nblocks_out) *nblocks_out = (int)(grid.x * grid.y);
  if (p.op == 2)
    stencil2d_kernel<<<grid, kBX, 0, st>>>(p, b, u, out, partial);
  else
    stencil1d_kernel<<<grid, kBX, 0, st>>>(p, b, u, out, partial);
  return cudaGetLastError();
}

int pd_stencil_num_blocks(const pd_stencil& p) {
  const long long S = (long long)p.nx * p.ny;
  return (int)(((S + kBX - 1) / kBX) * ((p.nt + kTC - 1) / kTC));
}

cudaError_t pd_launch_rhs(const pd_stencil& p, const double* u0, const double* v0, const double* f, double* b,
                          cudaStream_t st) {
  rhs_kernel<<<148 * 8, 256, 0, st>>>(p, u0, v0, f, b);
  return cudaGetLastError();
}
