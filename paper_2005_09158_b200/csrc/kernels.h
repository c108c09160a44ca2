// Internal launcher prototypes of the ParaDiag-II CUDA kernels (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

// ---- where row n of the half spectrum lives (the output of Step (a), the input of Step (c)) ----
// Single GPU: one owner, base[0] = Sh, pitch = S.  Sharded (dist.cpp): the frequencies [f0[q], f0[q + 1]) belong to
// rank q, whose Step (b) buffer holds them on full spatial rows (pitch = S_glob); base[q] points at this slab's first
// column in it (device memory of this process for virtual ranks, a CUDA-IPC mapping of the peer's buffer over
// NVLink for NCCL ranks).  Step (a)'s stores and Step (c)'s loads then go straight to / from the owner: the
// space -> frequency all-to-all is the time-FFT kernels' own epilogue (and frequency -> space their prologue).
constexpr int kPdMaxRanks = 8;
struct pd_spec {
  double2* base[kPdMaxRanks];
  int f0[kPdMaxRanks];
  int P;
  long long pitch;
};
// SH = false (single GPU): base[0] + n pitch, no owner lookup (the kernels are instantiated for both)
template <bool SH = true>
__host__ __device__ __forceinline__ double2* pd_spec_row(const pd_spec& v, int n) {
  if (!SH) return v.base[0] + (long long)n * v.pitch;
  int q = 0;
#pragma unroll
  for (int i = 1; i < kPdMaxRanks; ++i) q += (i < v.P && n >= v.f0[i]) ? 1 : 0;
  return v.base[q] + (long long)(n - v.f0[q]) * v.pitch;
}
inline pd_spec pd_spec_local(const double2* Sh, long long S) {
  pd_spec v{};
  v.base[0] = const_cast<double2*>(Sh);
  v.P = 1;
  v.pitch = S;
  return v;
}

// ---- Steps (a)/(c): time-axis FFTs (tfft.cu) ----
int pd_tfft_supported(int nt);
// r / z: [Nt][S] real (row stride S), spectrum rows through sp (columns [0, S) of each row)
cudaError_t pd_launch_tfft_fwd(int nt, const double* r, const pd_spec& sp, long long S, const double* gam,
                               const double2* tw, cudaStream_t st);
cudaError_t pd_launch_tfft_inv(int nt, const pd_spec& sp, double* z, long long S, const double* igam,
                               const double2* tw, int accumulate, cudaStream_t st);

// ---- Steps (a)/(c) for Nt >= 1024: four-step time FFT with an L2-resident scratch (tfft4.cu) ----
struct pd_tf4_tables {
  const double2* tw1;  // exp(-2 pi i j / N1), N1 = Nt / 64
  const double2* tw2;  // exp(-2 pi i j / 64)
  const double2* twt;  // exp(-2 pi i j / Nt)
};
int pd_tf4_supported(int nt);
int pd_tf4_n2();
int pd_tf4_pairs_per_tile();
struct pd_tfx_overlap;  // optional K-stream chunk pipeline (below)
// Linear combination sum_i c[i] x[i] of k <= kPdCombMax device vectors (16-byte aligned, S even) read by the
// forward time FFT's stage-1 loader in place of r (the GMRES final update u += P^{-1} (V y), tfx path).
constexpr int kPdCombMax = 32;
struct pd_comb_args {
  const double* x[kPdCombMax];
  double c[kPdCombMax];
  int k;
};
cudaError_t pd_launch_tf4_fwd(int nt, const double* r, const pd_spec& sp, long long S, const double* gam,
                              const pd_tf4_tables& tb, double2* scratch, long long chunk_pairs, cudaStream_t st,
                              int* nl, const pd_tfx_overlap* ov = nullptr);
cudaError_t pd_launch_tf4_inv(int nt, const pd_spec& sp, double* z, long long S, const double* igam,
                              const pd_tf4_tables& tb, double2* scratch, long long chunk_pairs, int accumulate,
                              cudaStream_t st, int* nl, const pd_tfx_overlap* ov = nullptr);

// ---- Step (b), 1D: batched constant-coefficient complex tridiagonal solves (tridiag.cu) ----
// Per frequency n (row n of Sh, nx entries): (a_n x_{i-1} + b_n x_i + c_n x_{i+1}) = d_i with
// a_n = lam2_n*sub, b_n = lam1_n + lam2_n*dia, c_n = lam2_n*sup.  coef[n] holds the host-computed
// per-frequency constants (see struct below).
struct pd_tri_coef {
  double2 r2;    // characteristic root with |r2| <= |r1| of c r^2 + b r + a = 0  (= a tau)
  double2 s;     // 1/r1 (= c tau)
  double2 tau;   // 1/(c r1) = 2/(-b -+ sqrt(b^2 - 4ac)), larger-magnitude denominator
  double2 r2L;   // r2^L (L = rows per thread)
  double2 sL;    // s^L
  double2 k1;    // boundary correction x_i += x^(d)_0 (k1 r2^{i+1} + k2 s^{N-i}): c kappa / (1 - c q_0),
  double2 k2;    //   kappa = -tau / (1 - s r2); k2 = -k1 r2^{N+1}
};
cudaError_t pd_launch_tridiag(double2* Sh, int nx, int nfreq, const pd_tri_coef* coef, int rows_per_thread,
                              cudaStream_t st);
int pd_tridiag_rows_per_thread();
int pd_tridiag_threads(int nx);
// WR tail form (tridiag.cu): per-CTA partial sums part[G][H][nx] of sum_n Re(ow[n][a] x_n), x_n the solve of
// frequency n with right-hand side sum_t hc[n][t] g_t (g: [H][nx] real); G CTAs stride over the nfreq frequencies.
cudaError_t pd_launch_tail1d(const double* g, double* part, int G, int nx, int nfreq, int H, const pd_tri_coef* coef,
                             const double2* hc, const double2* ow, cudaStream_t st);

// ---- Steps (a)/(c), 2D periodic, with the x-FFT of Step (b) folded in (tfx.cu): N1 = 8, N2 = Nt/8 ----
// The spectrum then holds X_n[y][kx]; Step (b) runs only the slab column pass (pd_launch_slab2d cols_only).
// chunk_pairs must be a multiple of pd_tfx_chunk_align (whole x-rows); tables: tw2 = N2-point, twt = Nt-point,
// twx = NX-point twiddles.
int pd_tfx_supported(int nt, int nx);
int pd_tfx_n2(int nt);
long long pd_tfx_chunk_align(int nt, int nx);
// K-stream chunk pipeline (ov != nullptr, PD_TF4_OVERLAP=K): chunk i runs on stream i mod K with scratch
// i mod K (stream 0 / scratch 0 = the caller's), so the stages of consecutive chunks overlap (same-stream order
// protects each scratch); ev_fork orders the extra streams after st on entry, ev_join[k] st after them on exit.
constexpr int kPdMaxOverlap = 4;
struct pd_tfx_overlap {
  int k = 1;
  double2* scratch[kPdMaxOverlap] = {};
  cudaStream_t st[kPdMaxOverlap] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[kPdMaxOverlap] = {};
};
// fork (extra streams wait for st) / join (st waits for the extra streams); no-ops without ov
inline cudaError_t ov_fork(const pd_tfx_overlap* ov, cudaStream_t st) {
  if (!ov) return cudaSuccess;
  cudaError_t e = cudaEventRecord(ov->ev_fork, st);
  for (int k = 1; k < ov->k && e == cudaSuccess; ++k) e = cudaStreamWaitEvent(ov->st[k], ov->ev_fork, 0);
  return e;
}
inline cudaError_t ov_join(const pd_tfx_overlap* ov, cudaStream_t st) {
  if (!ov) return cudaGetLastError();
  cudaError_t e = cudaSuccess;
  for (int k = 1; k < ov->k && e == cudaSuccess; ++k) {
    e = cudaEventRecord(ov->ev_join[k], ov->st[k]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ov->ev_join[k], 0);
  }
  return e == cudaSuccess ? cudaGetLastError() : e;
}
// forward stage 1 through TMA (tf4_tma.cu; PD_TMA=1): same output as tf4_fwd_s1<NT, N2 = 256, ...>
int pd_tf4_tma_supported(int nt, long long S, const void* r);
cudaError_t pd_launch_tf4_fwd_s1_tma(int nt, const double* r, long long S, long long p_begin, long long pc,
                                     double2* Y, const double* gam, const double2* tw2, const double2* twt,
                                     cudaStream_t st);
cudaError_t pd_launch_tfx_fwd(int nt, int nx, const double* r, const pd_spec& sp, long long S, const double* gam,
                              const pd_tf4_tables& tb, const double2* twx, double2* scratch, long long chunk_pairs,
                              cudaStream_t st, int* nl, const pd_tfx_overlap* ov = nullptr,
                              const pd_comb_args* comb = nullptr,  // comb: r unused
                              double* npart = nullptr,            // non-NULL: per-CTA partial sums of r^2 too
                              long long* nparts = nullptr);       // their count (the caller reduces in order)
cudaError_t pd_launch_tfx_inv(int nt, int nx, const pd_spec& sp, double* z, long long S, const double* igam,
                              const pd_tf4_tables& tb, const double2* twx, double2* scratch, long long chunk_pairs,
                              int accumulate, cudaStream_t st, int* nl, const pd_tfx_overlap* ov = nullptr);

// ---- Step (b), 2D periodic: per-frequency slab 2D FFT -> divide -> inverse 2D FFT (slab2d.cu) ----
// denominators lambda1_n + lambda2_n kappa(kx, ky), kappa = kd*(sx[kx]+sx[ky]) + i*(ax sn[kx] + ay sn[ky])/h
struct pd_slab_params {
  double kd;     // 4 nu / h^2
  double cx, cy; // ax / h, ay / h
};
int pd_slab2d_supported(int n);
// Step (b) 2D, y-direction as cyclic Toeplitz tridiagonal solves on x-transformed slabs (slab2d.cu ytri):
// per (frequency n, kx): a x_{y-1} + b x_y + c x_{y+1} = d_y (periodic in y), a = lam2 k2y_m, c = lam2 k2y_p,
// b = lam1 + lam2 (kappa_x(kx) + 2 nu/h^2).  Roots of c r^2 + b r + a: r = a tau (|r| <= 1), s = c tau (|s| <= 1),
// tau = 2/(-b -+ sqrt(b^2 - 4ac)) (larger denominator):  w_y = r w_{y-1} + d_y,  x_y = s x_{y+1} - tau w_y, with
// the cyclic closures w_{N-1} = w'_{N-1}/(1 - r^N), x_0 = x'_0/(1 - s^N).  One table entry per (n, kx).
struct pd_ytri_coef {
  double2 r, s, tau;
  double2 ir;   // 1 / (1 - r^N)
  double2 is;   // 1 / (1 - s^N)
  double2 rL;   // r^L, L = N/32 rows per lane
  double2 sL;   // s^L
};
int pd_slab2d_ytri_supported(int n);
// 2D homogeneous Dirichlet (PD_WAVE2D_DIRICHLET): N = 2^k - 1 interior nodes; tensor DST-I via FFTs of length
// M = 2(N+1) of the odd extension; mu[k] = (4 nu/h^2) sin^2(pi k/M), k < M; tw: M-point twiddles
int pd_slab2d_dst_supported(int n);
// 2D Dirichlet Step (b) as x-DST rows -> y Dirichlet Toeplitz solves per (n, kx) -> inverse x-DST rows (slab2d.cu
// dtri): one table entry per (frequency, kx < N): the roots and their lane powers (L = (N+1)/32 rows per lane) and the
// closed-form boundary correction x_i += x^(d)_0 (k1 r2^{i+1} + k2 s^{N-i}), k1 = c g kappa, k2 = -k1 r2^{N+1},
// g = 1/(1 - c q_0), kappa = -tau/(1 - s r2)
struct pd_dtri_coef {
  double2 r2, s, tau, r2L, sL, sLm1, k1, k2;
};
int pd_slab2d_dtri_supported(int n);
cudaError_t pd_launch_slab2d_dtri(double2* Sh, int n, int nfreq, int f0_glob, const pd_dtri_coef* coef,
                                  const double2* tw, int chunk, cudaStream_t st, int* launches);
// out[n] = min over (kx, ky) of |lam1_n + lam2_n kappa| / (|lam1_n| + |lam2_n| |kappa|)  (setup singularity check)
cudaError_t pd_launch_min_den(const double2* lam1, const double2* lam2, const double* sx, const double* sn,
                              pd_slab_params prm, int n, int nfreq, double* out, cudaStream_t st);
cudaError_t pd_launch_slab2d_dst(double2* Sh, int n, int nfreq, const double2* lam1, const double2* lam2,
                                 const double* mu, const double2* tw, int chunk, cudaStream_t st, int* launches);
int pd_slab2d_chunk(int n, int nfreq);
// chunk = slabs per L2-resident chunk; *launches = kernels launched
// one N x N complex slab in place: 2D FFT, multiply by tab[ky*N + kx] / N^2, inverse 2D FFT (tail map, tail.cu)
cudaError_t pd_launch_slab2d_filter(double2* slab, int n, const double2* tab, const double2* tw, cudaStream_t st);
// nrows (multiple of 8) contiguous complex rows of length n: in-place FFT along the row (inv: inverse), unnormalised
cudaError_t pd_launch_slab2d_rows(double2* base, int n, long long nrows, int inv, const double2* tw, cudaStream_t st);
cudaError_t pd_launch_slab2d(double2* Sh, int n, int nfreq, const double2* lam1, const double2* lam2,
                             const double* sx, const double* sn, pd_slab_params prm, const double2* tw,
                             int chunk, int cols_only, cudaStream_t st, int* launches);
// the y-pass of Step (b) by cyclic Toeplitz solves (x already transformed, by tfx.cu or by the slab row pass when
// rows != 0): frequencies [f0_glob, f0_glob + nfreq) of coef ([F_all][N]); scale applied to the result
cudaError_t pd_launch_slab2d_ytri(double2* Sh, int n, int nfreq, int f0_glob, const pd_ytri_coef* coef, double scale,
                                  const double2* tw, int chunk, int rows, cudaStream_t st, int* launches);

// ---- all-at-once residual / matvec (stencil.cu) ----
struct pd_stencil {
  int op;            // 0 ADE1D, 1 WAVE1D, 2 ADE2D
  int scheme;        // 0 BE, 1 CN, 2 LF
  int nx, ny, nt;    // local sizes (2D: nx = N columns, ny = rows)
  double sub, dia, sup;          // 1D K stencil
  double k2c, k2x_m, k2x_p, k2y_m, k2y_p;  // 2D K stencil: centre, x-1, x+1, y-1, y+1
  double dt;
  double theta;
  // halos of the sharded path (NULL: 1D zero Dirichlet boundary, 2D periodic wrap within the local rows).
  // Stencil: [Nt][hw] (hw = 1 in 1D, N in 2D) = the neighbour's boundary column/row at every time level;
  // rhs: [2][hw] = neighbour values of U_0 (row 0) and V_0 (row 1).
  const double* hlo;
  const double* hhi;
  double c1[3], c2[3];  // time taps (filled by pd_launch_stencil from scheme, dt, theta)
  double g3, g1;        // 1D pointwise reaction g(u) = g3 u^3 + g1 u inside F(u) = K u + g(u) (NEXT-4; 0 = linear)
};
// out = b - A u (b != NULL) or out = A u (b == NULL); per-block partial sums of out^2 into partial[]
cudaError_t pd_launch_stencil(const pd_stencil& p, const double* b, const double* u, double* out, double* partial,
                              int* nblocks_out, cudaStream_t st);
// b of A u = b from u0, v0 (nullable), f (nullable, [Nt+1][S])
cudaError_t pd_launch_rhs(const pd_stencil& p, const double* u0, const double* v0, const double* f, double* b,
                          cudaStream_t st);

// ---- deterministic BLAS-1 for the Krylov loop (blas1.cu) ----
int pd_blas_blocks();
// mode 0: partial <- <X_i, y>;  1: y <- a y + sum c_i X_i, partial <- <X_i, y_new>;
// mode 2: y <- a y + sum c_i X_i, partial <- <y_new, y_new>;  3: y <- sum c_i X_i;
// mode 4: y <- sum c_i X_i (y not read) [- hsub on the first hlen elements], partial <- (<X_i, y_new>, <y_new, y_new>)
// (K' = k + 1).
// partial[blk * K' + i], K' = k (modes 0, 1) or 1 (mode 2); coef on the host.  All vectors 16-byte aligned
// (hsub: any alignment).
cudaError_t pd_launch_krylov(int mode, const double* const* X, const double* coef, int k, double a, double* y,
                             long long n, double* partial, cudaStream_t st, const double* hsub = nullptr,
                             long long hlen = 0);
// sum partials in fixed order: out[i] = sum_blk partial[blk*k + i]  (device out)
cudaError_t pd_launch_reduce_partials(const double* partial, int nblk, int k, double* out, cudaStream_t st);
// y = a x + b y
cudaError_t pd_launch_axpby(double* y, const double* x, double a, double b, long long n, cudaStream_t st);

// WR tail form (tail.cu): (P - A) head-from-tail coefficients, H <= 2 blocks
struct pd_tail_g {
  int H;
  double pI[2][2], pK[2][2];  // head_a = sum_b pI[a][b] tail_b + pK[a][b] K tail_b
};
cudaError_t pd_launch_head_G(const pd_stencil& p, const pd_tail_g& gc, const double* tail, double* head, long long S,
                             cudaStream_t st);
cudaError_t pd_launch_reduce_rows(const double* part, int G, long long len, double* out, cudaStream_t st);
cudaError_t pd_launch_tau2d(double2* tau, int n, int nfreq, const double2* lam1, const double2* lam2, const double2* w,
                            const double* sx, const double* sn, pd_slab_params prm, cudaStream_t st);
// 2D Dirichlet tail map (H blocks): tau[a][t][ky][kx] = Re sum_n w[a*H+t][n] / (lam1_n + lam2_n (mu[kx+1] + mu[ky+1]));
// dense 2D DST-I Y = S X S of H real N x N blocks (S: N x N sine table, tmp: N x N); out_a = scale sum_t tau_at G_t
cudaError_t pd_launch_tau_dir(double* tau, int n, int nfreq, int H, const double2* lam1, const double2* lam2,
                              const double2* w, const double* mu, cudaStream_t st);
cudaError_t pd_launch_dst2d_dense(const double* in, double* out, double* tmp, const double* S, int N, int H,
                                  cudaStream_t st);
cudaError_t pd_launch_tau_combine(const double* tau, const double* G, double* out, int N, int H, double scale,
                                  cudaStream_t st);
cudaError_t pd_launch_r2c(const double* g, double2* z, long long n, cudaStream_t st);
cudaError_t pd_launch_take_real(const double2* z, double* out, long long n, cudaStream_t st);
// Sh[n][x] = sum_{t<H} hc[n][t] gx[t][x] for n < F (Step (a) of a head-only vector)
cudaError_t pd_launch_head_broadcast(double2* Sh, int F, long long S, int H, const double2* hc, const double2* gx,
                                     cudaStream_t st);
// *flag = 1 if any x[i] != 0 (i < n), else unchanged (caller zeroes it)
cudaError_t pd_launch_any_nonzero(const double* x, long long n, int* flag, cudaStream_t st);

// ---- nonlinear ParaDiag-II, simplified Newton (nonlin.cu, oracle/nonlinear.py) ----
// dbar[x] = (1/Nt) sum_n (3 g3 u_n(x)^2 + g1): the time-averaged reaction Jacobian (P:l.214-216)
cudaError_t pd_launch_jac_avg(const double* u, double* dbar, int nt, long long S, double g3, double g1, cudaStream_t st);
// Step (b), 1D, general: per frequency n the tridiagonal (lambda2 sub, lambda1 + lambda2 (dia + dbar_i), lambda2 sup)
// (dbar nullable: 0) by Gaussian elimination with partial pivoting (gtsv.cu), one lane per frequency; scratch of
// pd_gtsv_scratch_bytes; *bad = max (n + 1) over frequencies with a zero / non-finite pivot (caller zeroes it)
size_t pd_gtsv_scratch_bytes(int nx, int nfreq);
cudaError_t pd_launch_gtsv_shift(double2* Sh, int nx, int nfreq, const double2* lam1, const double2* lam2, double sub,
                                 double dia, double sup, const double* dbar, void* scratch, int* bad, cudaStream_t st);
