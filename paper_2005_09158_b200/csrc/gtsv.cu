// Step (b), 1D, by Gaussian elimination with partial pivoting (the LAPACK gtsv scheme): the general solver of the
// shifted systems (lambda_1n I + lambda_2n J) S2_n = S1_n (eq 2.12 Step (b), P:l.182, 816) when the
// characteristic-root recurrences of tridiag.cu do not apply:
//   * J = K + diag(dbar) of the simplified Newton iteration (averaged Jacobian, P:l.214-216; NEXT-4): the rows are
//     no longer Toeplitz, and a strong reaction term (g1 < 0) or a small shift removes diagonal dominance;
//   * constant-coefficient K whose shifted system leaves the recurrence regime (|r2|^N or |s|^N >= 1e8, both
//     characteristic roots on one side of the unit circle): such finite Toeplitz sections are ill-conditioned
//     roughly like |root|^N (reading t4), so the result carries that conditioning, but it is computed by
//     a backward-stable elimination instead of being rejected.
//
// Per row i the incoming raw row (a, b_i, c) is compared with the pending row (d, du) (|re| + |im| magnitudes, as
// LAPACK's CABS1); the larger one becomes the pivot row.  U has at most two super-diagonals: du2_i = c exactly when
// rows i, i+1 were swapped, so only a flag is stored for it.  Factors of row i: 1/d_i, du_i, flag_i; the modified
// right-hand side overwrites Sh in place; back substitution x_i = (y_i - du_i x_{i+1} - [flag_i] c x_{i+2}) / d_i.
//
// Layout: 32 frequencies per CTA (one warp, lane = frequency).  Rows are walked in tiles of 32 loaded coalesced
// (one frequency's 32 consecutive rows per instruction) and transposed through shared memory.  Processing raw row j
// finalises row j - 1, so the tile of raw rows [i0, i0 + 32) is written back as finalised rows [i0 - 1, i0 + 31).
#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int kGT = 32;

PD_D double cabs1(double2 v) { return fabs(v.x) + fabs(v.y); }

__global__ void __launch_bounds__(32) gtsv_shift_kernel(double2* __restrict__ Sh, int N, int F,
                                                        const double2* __restrict__ lam1,
                                                        const double2* __restrict__ lam2, double sub, double dia,
                                                        double sup, const double* __restrict__ dbar,
                                                        double2* __restrict__ f_dinv, double2* __restrict__ f_du,
                                                        unsigned char* __restrict__ f_sw, int* __restrict__ bad) {
  extern __shared__ double2 smem[];  // ty, ti, tu: [row][frequency] tiles; tf: swap flags (dynamic: 51 KB)
  auto ty = reinterpret_cast<double2(*)[kGT + 1]>(smem);
  auto ti = ty + kGT, tu = ti + kGT;
  auto tf = reinterpret_cast<unsigned char(*)[kGT + 1]>(tu + kGT);
  const int lane = threadIdx.x;
  const int f0 = blockIdx.x * kGT;
  const int n = f0 + lane;
  const bool on = n < F;
  const double2 l1 = on ? lam1[n] : make_double2(1.0, 0.0), l2 = on ? lam2[n] : czero();
  const double2 a = cscale(l2, sub), c = cscale(l2, sup);
  auto bdiag = [&](int i) { return cfma(l2, make_double2(dia + (dbar ? __ldg(dbar + i) : 0.0), 0.0), l1); };
  // tile t rows [i0 + off, i0 + off + 32) of frequency f0 + k  <->  t[lane][k]
  auto load = [&](double2 (*t)[kGT + 1], const double2* base, int i0) {
    for (int k = 0; k < kGT; ++k) {
      const int i = i0 + lane;
      t[lane][k] = (f0 + k < F && i >= 0 && i < N) ? base[(long long)(f0 + k) * N + i] : czero();
    }
  };
  auto store = [&](double2 (*t)[kGT + 1], double2* base, int i0) {
    for (int k = 0; k < kGT; ++k) {
      const int i = i0 + lane;
      if (f0 + k < F && i >= 0 && i < N) base[(long long)(f0 + k) * N + i] = t[lane][k];
    }
  };
  bool singular = false;
  // forward elimination; pending row (cd, cdu) with right-hand side cy
  double2 cd = bdiag(0), cdu = N > 1 ? c : czero(), cy = czero();
  for (int i0 = 0; i0 < N; i0 += kGT) {
    load(ty, Sh, i0);
    __syncwarp();
    const int iend = min(kGT, N - i0);
    for (int r = 0; r < iend; ++r) {
      const int j = i0 + r;
      const double2 yj = ty[r][lane];
      if (j == 0) {
        cy = yj;
        continue;
      }
      const double2 nb = bdiag(j), ndu = j < N - 1 ? c : czero();
      double2 dinv, du, y;
      unsigned char sw;
      if (cabs1(cd) >= cabs1(a)) {  // no interchange: pivot on the pending row
        singular |= !(cabs1(cd) > 0.0);
        dinv = crcp(cd);
        const double2 l = cmul(a, dinv);
        du = cdu;
        y = cy;
        sw = 0;
        cd = csub(nb, cmul(l, cdu));
        cdu = ndu;
        cy = csub(yj, cmul(l, cy));
      } else {  // interchange rows j-1 and j: the raw row (a, nb, ndu) becomes U's row j-1
        dinv = crcp(a);
        const double2 l = cmul(cd, dinv);
        du = nb;
        y = yj;
        sw = (j < N - 1) ? 1 : 0;  // du2_{j-1} = ndu = c
        cd = csub(cdu, cmul(l, nb));
        cdu = cneg(cmul(l, ndu));
        cy = csub(cy, cmul(l, yj));
      }
      // finalised row j - 1 -> tile slot r - 1; for r = 0 it is the previous tile's last row (not flushed with
      // that tile): each lane stores its own frequency's entry directly
      if (r > 0) {
        ty[r - 1][lane] = y;
        ti[r - 1][lane] = dinv;
        tu[r - 1][lane] = du;
        tf[r - 1][lane] = sw;
      } else if (on) {
        const long long o = (long long)n * N + j - 1;
        Sh[o] = y;
        f_dinv[o] = dinv;
        f_du[o] = du;
        f_sw[o] = sw;
      }
    }
    if (i0 + iend == N) {  // the last row N - 1 has no successor: finalise it from the pending row
      singular |= !(cabs1(cd) > 0.0);
      ty[iend - 1][lane] = cy;
      ti[iend - 1][lane] = crcp(cd);
      tu[iend - 1][lane] = czero();
      tf[iend - 1][lane] = 0;
    }
    __syncwarp();
    // rows i0 .. i0 + iend - 2 are final (and N - 1 when this is the last tile); row i0 + 31 follows next tile
    const int nrows = (i0 + iend == N) ? iend : iend - 1;
    for (int k = 0; k < kGT; ++k) {
      const int i = i0 + lane;
      if (f0 + k < F && lane < nrows) {
        const long long o = (long long)(f0 + k) * N + i;
        Sh[o] = ty[lane][k];
        f_dinv[o] = ti[lane][k];
        f_du[o] = tu[lane][k];
        f_sw[o] = tf[lane][k];
      }
    }
    __syncwarp();
  }
  if (on && singular) atomicMax(bad, n + 1);
  // back substitution over the tiles in reverse: x_i = (y_i - du_i x_{i+1} - [sw_i] c x_{i+2}) / d_i
  double2 x1 = czero(), x2 = czero();  // x_{i+1}, x_{i+2}
  const int last0 = ((N - 1) / kGT) * kGT;
  for (int i0 = last0; i0 >= 0; i0 -= kGT) {
    load(ty, Sh, i0);
    load(ti, f_dinv, i0);
    load(tu, f_du, i0);
    for (int k = 0; k < kGT; ++k) {
      const int i = i0 + lane;
      tf[lane][k] = (f0 + k < F && i < N) ? f_sw[(long long)(f0 + k) * N + i] : 0;
    }
    __syncwarp();
    const int iend = min(kGT, N - i0);
    for (int r = iend - 1; r >= 0; --r) {
      double2 t = csub(ty[r][lane], cmul(tu[r][lane], x1));
      if (tf[r][lane]) t = csub(t, cmul(c, x2));
      const double2 x = cmul(t, ti[r][lane]);
      ty[r][lane] = x;
      x2 = x1;
      x1 = x;
    }
    __syncwarp();
    store(ty, Sh, i0);
    __syncwarp();
  }
}

}  // namespace

size_t pd_gtsv_scratch_bytes(int nx, int nfreq) {
  return (size_t)nfreq * nx * (2 * sizeof(double2) + 1);
}

cudaError_t pd_launch_gtsv_shift(double2* Sh, int nx, int nfreq, const double2* lam1, const double2* lam2, double sub,
                                 double dia, double sup, const double* dbar, void* scratch, int* bad, cudaStream_t st) {
  double2* dinv = static_cast<double2*>(scratch);
  double2* du = dinv + (size_t)nfreq * nx;
  unsigned char* sw = reinterpret_cast<unsigned char*>(du + (size_t)nfreq * nx);
  constexpr int kSmem = 3 * kGT * (kGT + 1) * sizeof(double2) + kGT * (kGT + 1);
  static int attr = -1;  // device on which the attribute was set
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr != dev) {
    cudaFuncSetAttribute(gtsv_shift_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    attr = dev;
  }
  gtsv_shift_kernel<<<(nfreq + kGT - 1) / kGT, kGT, kSmem, st>>>(Sh, nx, nfreq, lam1, lam2, sub, dia, sup, dbar, dinv, du,
                                                             sw, bad);
  return cudaGetLastError();
}
