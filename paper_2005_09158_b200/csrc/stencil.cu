// All-at-once residual r = b - A u and matvec w = A u, A = B1 (x) I + B2 (x) K (eq 1.1, P:l.80-84),
// with the time taps of eq 2.5b (theta-method, P:l.309-319) and eq 3.2b (implicit leapfrog, P:l.1214-1227):
//   (A u)_n = sum_k c1_k u_{n-k} + K ( sum_k c2_k u_{n-k} ),   terms with n-k < 0 dropped (U_0 lives in b).
// One thread per spatial point walks a chunk of time rows, keeping the stencil neighbourhood of the
// previous rows in registers; per-block partial sums of r^2 feed a deterministic fixed-order reduction.
// Also the right-hand side b of A u = b from (U_0, V_0, f) (readings c4, c5).
#include "common.cuh"
#include <cstdlib>

#include "kernels.h"

namespace {

constexpr int kTC = 64;     // time rows per thread
constexpr int kBX = 256;    // threads per block

struct Taps {
  double c1[3], c2[3];
  int ntaps;
};

PD_HD Taps taps_of(const pd_stencil& p) {
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

template <bool NL>
__global__ void __launch_bounds__(kBX, 4) stencil1d_kernel(pd_stencil p, const double* __restrict__ b,
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
    if constexpr (NL) {  // (B2 (x) I) g(u): F(u) = K u + g(u), g pointwise (eq 1.4)
      auto g = [&](double v) { return v * fma(p.g3, v * v, p.g1); };
      Au += tp.c2[0] * g(h0.c) + tp.c2[1] * g(h1.c) + tp.c2[2] * g(h2.c);
    }
    if (act) {
      const long long idx = (long long)n * nx + x;
      const double v = b ? b[idx] - Au : Au;
      if (out) out[idx] = v;  // out == NULL: norm only
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

// Tile of 32 x-points (one warp) by kTY y-rows per block plus two halo warps (rows y0-1 and ylast+1), walking
// kTC time rows.  Each lane loads only its own point per row (one coalesced load); the time combination
// y = sum_k c2_k u_{n-k} of the x-neighbours arrives by warp shuffle (lanes at a tile or domain edge load
// their outside neighbour themselves) and of the y-neighbours through a double-buffered shared row.
constexpr int kTY = 16;
constexpr int kW2 = kTY + 2;
#ifndef PD_STENCIL2D_MINB
#define PD_STENCIL2D_MINB 2
#endif

struct Hist { double h0, h1, h2; };

// NT = number of time taps (2: theta-method, 3: leapfrog); taps read from the parameter bank
template <int NT>
PD_D double comb(const pd_stencil& p, const Hist& h) {
  return NT == 3 ? p.c2[0] * h.h0 + p.c2[1] * h.h1 + p.c2[2] * h.h2 : p.c2[0] * h.h0 + p.c2[1] * h.h1;
}
template <int NT>
PD_D double comb1(const pd_stencil& p, const Hist& h) {
  return NT == 3 ? p.c1[0] * h.h0 + p.c1[1] * h.h1 + p.c1[2] * h.h2 : p.c1[0] * h.h0 + p.c1[1] * h.h1;
}

template <int NT>
__global__ void __launch_bounds__(32 * kW2, PD_STENCIL2D_MINB) stencil2d_kernel(pd_stencil p, const double* __restrict__ b,
                                                             const double* __restrict__ u, double* __restrict__ out,
                                                             double* __restrict__ partial) {
  __shared__ double ysh[2][kW2][32];
  __shared__ double red[kW2];
  const int nx = p.nx, ny = p.ny;
  const long long S = (long long)nx * ny;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * kTY;
  const int ylast = min(y0 + kTY, ny) - 1;
  const int xr = x0 + lane;
  const bool xin = xr < nx;
  const int x = xin ? xr : nx - 1;
  // warp 0..kTY-1: output rows y0+warp; warp kTY: row y0-1; warp kTY+1: row ylast+1
  int srow;  // shared row slot
  int y;
  const double* hsrc = nullptr;  // halo rows of a neighbouring rank ([nt][nx]) replacing the wrap
  if (warp < kTY) {
    y = y0 + warp;
    srow = warp + 1;
  }
  // op 2: periodic wrap within the local rows (or the neighbour rank's halo); op 3: homogeneous Dirichlet
  // (zero outside the domain; the neighbour rank's halo between shards)
  const bool per = p.op == 2;
  bool zrow = false;  // halo warp of a Dirichlet boundary: the row outside the domain is zero
  if (warp == kTY) {
    y = y0 - 1;
    srow = 0;
    if (y < 0) {
      y = ny - 1;
      hsrc = p.hlo;
      zrow = !per && !hsrc;
    }
  } else if (warp > kTY) {
    y = ylast + 1;
    srow = ylast - y0 + 2;
    if (y >= ny) {
      y = 0;
      hsrc = p.hhi;
      zrow = !per && !hsrc;
    }
  }
  const bool outw = warp < kTY && y <= ylast;
  const bool act = outw && xin;
  const bool live = (warp >= kTY && !zrow) || (warp < kTY && y <= ylast);  // rows whose loads are needed
  const bool needL = outw && (lane == 0 || x == 0);
  const bool needR = outw && (lane == 31 || x == nx - 1);
  const int xl = x == 0 ? nx - 1 : x - 1, xp = x == nx - 1 ? 0 : x + 1;
  const double* rowp = hsrc ? hsrc : u + (long long)y * nx;
  const long long rstride = hsrc ? nx : S;  // time stride of this warp's row
  const int n0 = blockIdx.z * kTC;
  const int n1 = min(n0 + kTC, p.nt);
  // per-row pointers advanced by the time stride (row n0); loads of rows < 0 are skipped
  const double* pc = rowp + (long long)n0 * rstride + x;
  const int dl = xl - x, dr = xp - x;
  auto ld = [&](const double* q, int n, int d) -> double { return (n >= 0 && live) ? q[d] : 0.0; };
  Hist c = {0.0, ld(pc - rstride, n0 - 1, 0), NT == 3 ? ld(pc - 2 * rstride, n0 - 2, 0) : 0.0};
  Hist L = {0.0, 0.0, 0.0}, R = {0.0, 0.0, 0.0};
  const bool ldL = needL && (per || x != 0), ldR = needR && (per || x != nx - 1);  // Dirichlet: 0 outside
  if (ldL) { L.h1 = ld(pc - rstride, n0 - 1, dl); if (NT == 3) L.h2 = ld(pc - 2 * rstride, n0 - 2, dl); }
  if (ldR) { R.h1 = ld(pc - rstride, n0 - 1, dr); if (NT == 3) R.h2 = ld(pc - 2 * rstride, n0 - 2, dr); }
  const long long off = (long long)n0 * S + (long long)y * nx + x;
  const double* pb = b ? b + off : nullptr;
  const bool wr = out != nullptr;  // NULL: norm only (no vector written)
  double* po = wr ? out + off : nullptr;
  // one-row prefetch
  double nc = live ? pc[0] : 0.0, nl = ldL ? pc[dl] : 0.0, nr = ldR ? pc[dr] : 0.0;
  double nb = (act && pb) ? pb[0] : 0.0;
  double acc = 0.0;
  int buf = 0;
  for (int n = n0; n < n1; ++n) {
    c.h0 = nc; L.h0 = nl; R.h0 = nr;
    const double bv = nb;
    if (n + 1 < n1) {
      pc += rstride;
      if (live) nc = pc[0];
      if (ldL) nl = pc[dl];
      if (ldR) nr = pc[dr];
      if (act && pb) nb = pb[S];
    }
    const double yc = comb<NT>(p, c);
    if (live || warp >= kTY) ysh[buf][srow][lane] = yc;  // rows past ylast share the slot of the high halo row
    const double up = __shfl_up_sync(0xffffffffu, yc, 1);
    const double dn = __shfl_down_sync(0xffffffffu, yc, 1);
    const double yxm = needL ? comb<NT>(p, L) : up;
    const double yxp = needR ? comb<NT>(p, R) : dn;
    __syncthreads();
    if (act) {
      const double yym = ysh[buf][srow - 1][lane], yyp = ysh[buf][srow + 1][lane];
      double Au = comb1<NT>(p, c);
      Au += p.k2c * yc + p.k2x_m * yxm + p.k2x_p * yxp + p.k2y_m * yym + p.k2y_p * yyp;
      const double v = pb ? bv - Au : Au;
      if (wr) *po = v;
      acc = fma(v, v, acc);
    }
    if (wr) po += S;
    if (pb) pb += S;
    c.h2 = c.h1; c.h1 = c.h0;
    L.h2 = L.h1; L.h1 = L.h0;
    R.h2 = R.h1; R.h1 = R.h0;
    buf ^= 1;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kTY; ++w) t += red[w];
    partial[((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
  }
}

// Two x-points per lane (16-byte loads and stores, 64 x-points per warp tile): the same walk as stencil2d_kernel with
// twice the bytes in flight per lane and half the instructions per point (needs nx % 64 == 0 and 16-byte aligned
// vectors).  Component 0 (x) takes its left neighbour from lane - 1's component 1 and its right one from its own
// component 1; component 1 (x + 1) the mirror image.
template <int NT>
__global__ void __launch_bounds__(32 * kW2, PD_STENCIL2D_MINB) stencil2d_v2_kernel(pd_stencil p, const double* __restrict__ b,
                                                                const double* __restrict__ u, double* __restrict__ out,
                                                                double* __restrict__ partial) {
  __shared__ double2 ysh[2][kW2][32];
  __shared__ double red[kW2];
  const int nx = p.nx, ny = p.ny;
  const long long S = (long long)nx * ny;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x0 = blockIdx.x * 64, y0 = blockIdx.y * kTY;
  const int ylast = min(y0 + kTY, ny) - 1;
  const int x = x0 + 2 * lane;
  int srow = 0, y = 0;
  const double* hsrc = nullptr;
  if (warp < kTY) {
    y = y0 + warp;
    srow = warp + 1;
  }
  const bool per = p.op == 2;
  bool zrow = false;
  if (warp == kTY) {
    y = y0 - 1;
    srow = 0;
    if (y < 0) {
      y = ny - 1;
      hsrc = p.hlo;
      zrow = !per && !hsrc;
    }
  } else if (warp > kTY) {
    y = ylast + 1;
    srow = ylast - y0 + 2;
    if (y >= ny) {
      y = 0;
      hsrc = p.hhi;
      zrow = !per && !hsrc;
    }
  }
  const bool act = warp < kTY && y <= ylast;
  const bool live = (warp >= kTY && !zrow) || (warp < kTY && y <= ylast);
  const bool needL = act && lane == 0, needR = act && lane == 31;
  const int xl = x == 0 ? nx - 1 : x - 1, xr = x + 2 == nx ? 0 : x + 2;
  const double* rowp = hsrc ? hsrc : u + (long long)y * nx;
  const long long rstride = hsrc ? nx : S;
  const int n0 = blockIdx.z * kTC;
  const int n1 = min(n0 + kTC, p.nt);
  const double* pc = rowp + (long long)n0 * rstride + x;
  const int dl = xl - x, dr = xr - x;
  auto ld2 = [&](const double* q, int n) -> double2 {
    return (n >= 0 && live) ? *reinterpret_cast<const double2*>(q) : make_double2(0.0, 0.0);
  };
  auto ld1 = [&](const double* q, int n, int d) -> double { return (n >= 0 && live) ? q[d] : 0.0; };
  double2 c0 = make_double2(0.0, 0.0), c1 = ld2(pc - rstride, n0 - 1),
          c2 = NT == 3 ? ld2(pc - 2 * rstride, n0 - 2) : make_double2(0.0, 0.0);
  Hist L = {0.0, 0.0, 0.0}, R = {0.0, 0.0, 0.0};
  const bool ldL = needL && (per || x != 0), ldR = needR && (per || x + 1 != nx - 1);  // Dirichlet: 0 outside
  if (ldL) { L.h1 = ld1(pc - rstride, n0 - 1, dl); if (NT == 3) L.h2 = ld1(pc - 2 * rstride, n0 - 2, dl); }
  if (ldR) { R.h1 = ld1(pc - rstride, n0 - 1, dr); if (NT == 3) R.h2 = ld1(pc - 2 * rstride, n0 - 2, dr); }
  const long long off = (long long)n0 * S + (long long)y * nx + x;
  const double* pb = b ? b + off : nullptr;
  const bool wr = out != nullptr;
  double* po = wr ? out + off : nullptr;
  double2 nc = live ? *reinterpret_cast<const double2*>(pc) : make_double2(0.0, 0.0);
  double nl = ldL ? pc[dl] : 0.0, nr = ldR ? pc[dr] : 0.0;
  double2 nb = (act && pb) ? *reinterpret_cast<const double2*>(pb) : make_double2(0.0, 0.0);
  double acc = 0.0;
  int buf = 0;
  auto cmb = [&](double h0, double h1, double h2) {
    return NT == 3 ? p.c2[0] * h0 + p.c2[1] * h1 + p.c2[2] * h2 : p.c2[0] * h0 + p.c2[1] * h1;
  };
  auto cmb1 = [&](double h0, double h1, double h2) {
    return NT == 3 ? p.c1[0] * h0 + p.c1[1] * h1 + p.c1[2] * h2 : p.c1[0] * h0 + p.c1[1] * h1;
  };
  for (int n = n0; n < n1; ++n) {
    c0 = nc;
    L.h0 = nl;
    R.h0 = nr;
    const double2 bv = nb;
    if (n + 1 < n1) {
      pc += rstride;
      if (live) nc = *reinterpret_cast<const double2*>(pc);
      if (ldL) nl = pc[dl];
      if (ldR) nr = pc[dr];
      if (act && pb) nb = *reinterpret_cast<const double2*>(pb + S);
    }
    const double2 yc = make_double2(cmb(c0.x, c1.x, c2.x), cmb(c0.y, c1.y, c2.y));
    if (live || warp >= kTY) ysh[buf][srow][lane] = yc;
    const double up = __shfl_up_sync(0xffffffffu, yc.y, 1);
    const double dn = __shfl_down_sync(0xffffffffu, yc.x, 1);
    const double yxm0 = needL ? cmb(L.h0, L.h1, L.h2) : up;
    const double yxp1 = needR ? cmb(R.h0, R.h1, R.h2) : dn;
    __syncthreads();
    if (act) {
      const double2 yym = ysh[buf][srow - 1][lane], yyp = ysh[buf][srow + 1][lane];
      double a0 = cmb1(c0.x, c1.x, c2.x), a1 = cmb1(c0.y, c1.y, c2.y);
      a0 += p.k2c * yc.x + p.k2x_m * yxm0 + p.k2x_p * yc.y + p.k2y_m * yym.x + p.k2y_p * yyp.x;
      a1 += p.k2c * yc.y + p.k2x_m * yc.x + p.k2x_p * yxp1 + p.k2y_m * yym.y + p.k2y_p * yyp.y;
      const double v0 = pb ? bv.x - a0 : a0, v1 = pb ? bv.y - a1 : a1;
      if (wr) *reinterpret_cast<double2*>(po) = make_double2(v0, v1);
      acc = fma(v0, v0, acc);
      acc = fma(v1, v1, acc);
    }
    if (wr) po += S;
    if (pb) pb += S;
    c2 = c1;
    c1 = c0;
    L.h2 = L.h1; L.h1 = L.h0;
    R.h2 = R.h1; R.h1 = R.h0;
    buf ^= 1;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kTY; ++w) t += red[w];
    partial[((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
  }
}

// ---------------- right-hand side ----------------
// K v at spatial point s of a single time level (zero Dirichlet / periodic wrap)
// 2D homogeneous Dirichlet neighbourhood (zero outside; halo rows of neighbour ranks in y)
PD_D N2 load2_dir(const double* __restrict__ slab, int x, int y, int nx, int ny, const double* hl, const double* hr) {
  N2 v;
  v.c = slab[(long long)y * nx + x];
  v.xm = x > 0 ? slab[(long long)y * nx + x - 1] : 0.0;
  v.xp = x + 1 < nx ? slab[(long long)y * nx + x + 1] : 0.0;
  v.ym = y > 0 ? slab[(long long)(y - 1) * nx + x] : (hl ? hl[x] : 0.0);
  v.yp = y + 1 < ny ? slab[(long long)(y + 1) * nx + x] : (hr ? hr[x] : 0.0);
  return v;
}

PD_D double applyK(const pd_stencil& p, const double* __restrict__ v, long long s, int which) {
  const int hw = p.op >= 2 ? p.nx : 1;
  const double* hl = p.hlo ? p.hlo + which * hw : nullptr;
  const double* hr = p.hhi ? p.hhi + which * hw : nullptr;
  if (p.op >= 2) {
    const N2 h = p.op == 2 ? load2(v, (int)(s % p.nx), (int)(s / p.nx), p.nx, p.ny, hl, hr)
                           : load2_dir(v, (int)(s % p.nx), (int)(s / p.nx), p.nx, p.ny, hl, hr);
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
      if (n == 0) {
        v += u0[s] / p.dt - (1.0 - p.theta) * applyK(p, u0, s, 0);
        if (p.g3 != 0.0 || p.g1 != 0.0) v -= (1.0 - p.theta) * u0[s] * fma(p.g3, u0[s] * u0[s], p.g1);  // f(U0)
      }
    }
    b[i] = v;
  }
}

Taps taps_host(const pd_stencil& p) { return taps_of(p); }

}  // namespace

int pd_stencil_num_blocks(const pd_stencil& p) {
  const long long nz = (p.nt + kTC - 1) / kTC;
  if (p.op >= 2) return (int)(((p.nx + 31) / 32) * ((p.ny + kTY - 1) / kTY) * nz);
  return (int)(((p.nx + kBX - 1) / kBX) * nz);
}

cudaError_t pd_launch_stencil(const pd_stencil& p, const double* b, const double* u, double* out, double* partial,
                              int* nblocks_out, cudaStream_t st) {
  if (nblocks_out) *nblocks_out = pd_stencil_num_blocks(p);
  if (p.op >= 2) {
    pd_stencil q = p;
    const Taps t = taps_host(p);
    for (int k = 0; k < 3; ++k) { q.c1[k] = t.c1[k]; q.c2[k] = t.c2[k]; }
    auto al = [](const void* v) { return (reinterpret_cast<uintptr_t>(v) & 15) == 0; };
    static const bool v1_only = getenv("PD_STENCIL_V1") != nullptr;
    const bool v2 = !v1_only && p.nx % 64 == 0 && al(u) && al(b) && al(out) && al(p.hlo) && al(p.hhi);
    const int tw = v2 ? 64 : 32;
    dim3 grid((unsigned)((p.nx + tw - 1) / tw), (unsigned)((p.ny + kTY - 1) / kTY), (unsigned)((p.nt + kTC - 1) / kTC));
    if (nblocks_out) *nblocks_out = (int)(grid.x * grid.y * grid.z);
    if (v2 && t.ntaps == 3)
      stencil2d_v2_kernel<3><<<grid, 32 * kW2, 0, st>>>(q, b, u, out, partial);
    else if (v2)
      stencil2d_v2_kernel<2><<<grid, 32 * kW2, 0, st>>>(q, b, u, out, partial);
    else if (t.ntaps == 3)
      stencil2d_kernel<3><<<grid, 32 * kW2, 0, st>>>(q, b, u, out, partial);
    else
      stencil2d_kernel<2><<<grid, 32 * kW2, 0, st>>>(q, b, u, out, partial);
  } else {
    dim3 grid((unsigned)((p.nx + kBX - 1) / kBX), (unsigned)((p.nt + kTC - 1) / kTC));
    if (p.g3 != 0.0 || p.g1 != 0.0)
      stencil1d_kernel<true><<<grid, kBX, 0, st>>>(p, b, u, out, partial);
    else
      stencil1d_kernel<false><<<grid, kBX, 0, st>>>(p, b, u, out, partial);
  }
  return cudaGetLastError();
}


cudaError_t pd_launch_rhs(const pd_stencil& p, const double* u0, const double* v0, const double* f, double* b,
                          cudaStream_t st) {
  rhs_kernel<<<148 * 8, 256, 0, st>>>(p, u0, v0, f, b);
  return cudaGetLastError();
}
