// Host runtime and C ABI of the B200 ParaDiag-II hot path (see include/paradiag.h for the contract).
//
// pd_setup builds every data-independent quantity once (spectra from closed forms, Gamma tables,
// twiddles, per-frequency tridiagonal constants, 2D symbol tables), checks the shifted systems for
// singularity and allocates the workspace.  The solver loops (eq 5.1 stationary iteration, right-
// preconditioned GMRES(m)) run on the host and enqueue the kernels of csrc/*.cu on the context stream.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "ctx.h"

typedef std::complex<long double> cld;

static thread_local std::string g_setup_err;

pd_status fail(pd_ctx* c, pd_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c)
    c->err = buf;
  else
    g_setup_err = buf;
  return s;
}

template <class T>
static cudaError_t dalloc(T** p, size_t n) {
  return cudaMalloc((void**)p, n * sizeof(T) + 16);
}

// ------------------------------------------------------------------------------------------------
// spectra: closed forms of the DFT of the Gamma-weighted first columns (Lemma 1, P:l.155-174;
// SURVEY §8(c) / DESIGN.md §3): z_n = alpha^{1/Nt} exp(-2 pi i n / Nt) (numpy convention, reading c1)
//   BE: lam1 = (1 - z)/dt, lam2 = 1;  CN: lam1 = (1 - z)/dt, lam2 = (1 + z)/2
//   LF: lam1 = (1 - z)^2/dt^2, lam2 = (1 + z^2)/2
// ------------------------------------------------------------------------------------------------
static void closed_form_spectra(int nt, double alpha, double dt, pd_scheme s, std::vector<cld>& l1,
                                std::vector<cld>& l2) {
  l1.resize(nt);
  l2.resize(nt);
  const long double pi = 3.141592653589793238462643383279502884L;
  const long double a = powl((long double)alpha, 1.0L / nt);
  if (nt == 1) {  // reading t2: the 1 x 1 alpha-circulant is its first-column entry (no wrap, S:l.89)
    const long double d = dt;
    l1[0] = s == PD_LEAPFROG ? 1.0L / (d * d) : 1.0L / d;
    l2[0] = s == PD_BE ? 1.0L : 0.5L;
    return;
  }
  for (int n = 0; n < nt; ++n) {
    // exact argument reduction of n/Nt before the trig call
    const long double th = 2.0L * pi * (long double)n / (long double)nt;
    const cld z = a * cld(cosl(th), -sinl(th));
    const long double d = dt;
    if (s == PD_BE) {
      l1[n] = (1.0L - z) / d;
      l2[n] = 1.0L;
    } else if (s == PD_CN) {
      l1[n] = (1.0L - z) / d;
      l2[n] = (1.0L + z) / 2.0L;
    } else {
      l1[n] = (1.0L - z) * (1.0L - z) / (d * d);
      l2[n] = (1.0L + z * z) / 2.0L;
    }
  }
}

static inline double2 d2(cld v) { return make_double2((double)v.real(), (double)v.imag()); }

// 2D y-pass as cyclic Toeplitz solves (slab2d.cu ytri): per (n, kx) constants; false when any column falls
// outside the stable regime (|r| or |s| > 1, or a closure denominator 1 - r^N near 0): the FFT column pass is
// used instead.
static bool ytri_coefs(const pd_ctx* c, const std::vector<cld>& l1, const std::vector<cld>& l2,
                       std::vector<pd_ytri_coef>& out) {
  const int N = c->g.nx, L = N / 32;
  const long double h = (long double)c->g.length / N, nu = c->g.nu;
  const long double km = -nu / (h * h) - (long double)c->g.ay / (2 * h), kp = -nu / (h * h) + (long double)c->g.ay / (2 * h);
  const long double kd = 4 * nu / (h * h), cx = (long double)c->g.ax / h;
  out.resize((size_t)c->F * N);
  auto cp = [](cld m, int e) {
    cld r = 1.0L;
    while (e) {
      if (e & 1) r *= m;
      m *= m;
      e >>= 1;
    }
    return r;
  };
  for (int n = 0; n < c->F; ++n)
    for (int kx = 0; kx < N; ++kx) {
      const long double pi = 3.141592653589793238462643383279502884L, sk = sinl(pi * kx / N);
      const cld kapx(kd * sk * sk, cx * sinl(2.0L * pi * kx / N));
      const cld A = l2[n] * km, Cc = l2[n] * kp, B = l1[n] + l2[n] * (kapx + 2 * nu / (h * h));
      const cld D = std::sqrt(B * B - 4.0L * A * Cc);
      const cld den1 = -B - D, den2 = -B + D;
      const cld den = std::abs(den1) >= std::abs(den2) ? den1 : den2;
      if (std::abs(den) == 0.0L) return false;
      const cld tau = 2.0L / den, r = A * tau, sv = Cc * tau;
      if (!(std::abs(r) <= 1.0L) || !(std::abs(sv) <= 1.0L)) return false;
      const cld rN = cp(r, N), sN = cp(sv, N);
      if (std::abs(1.0L - rN) < 1e-6L || std::abs(1.0L - sN) < 1e-6L) return false;
      pd_ytri_coef& t = out[(size_t)n * N + kx];
      t.r = d2(r);
      t.s = d2(sv);
      t.tau = d2(tau);
      t.ir = d2(1.0L / (1.0L - rN));
      t.is = d2(1.0L / (1.0L - sN));
      t.rL = d2(cp(r, L));
      t.sL = d2(cp(sv, L));
    }
  return true;
}

// Host check of the pivoted elimination (gtsv.cu) on one constant-coefficient shifted system, in long double: the
// smallest |pivot| relative to the largest matrix entry (0 = singular).  Used when the recurrence solver does not apply.
static long double gtsv_min_pivot(cld A, cld B, cld Cc, int N) {
  auto c1 = [](cld v) { return fabsl(v.real()) + fabsl(v.imag()); };
  const long double scale = std::max(c1(A), std::max(c1(B), c1(Cc)));
  cld cd = B, cdu = N > 1 ? Cc : 0.0L;
  long double mn = INFINITY;
  for (int j = 1; j < N; ++j) {
    const cld ndu = j < N - 1 ? Cc : 0.0L;
    if (c1(cd) >= c1(A)) {
      mn = std::min(mn, c1(cd));
      if (c1(cd) == 0) return 0;
      const cld l = A / cd;
      cd = B - l * cdu;
      cdu = ndu;
    } else {
      mn = std::min(mn, c1(A));
      const cld l = cd / A;
      cd = cdu - l * B;
      cdu = -l * ndu;
    }
  }
  mn = std::min(mn, c1(cd));
  return scale > 0 ? mn / scale : 0;
}

// per-frequency constants of the Toeplitz tridiagonal recurrence solver (tridiag.cu).  When a shifted system leaves
// the recurrence's stable regime (or PD_TRIDIAG_GTSV=1), the context switches to the pivoted elimination (gtsv.cu)
// for every frequency; singular shifts are then detected by the same elimination on the host (reading t4).
static pd_status tri_coefs(pd_ctx* c, const std::vector<cld>& l1, const std::vector<cld>& l2, double sub, double dia,
                           double sup, std::vector<pd_tri_coef>& out) {
  const int N = c->g.nx, L = pd_tridiag_rows_per_thread();
  out.resize(c->F);
  const char* force = getenv("PD_TRIDIAG_GTSV");
  c->use_gtsv = force && atoi(force) != 0;
  for (int n = 0; n < c->F && !c->use_gtsv; ++n) {
    const cld A = l2[n] * (long double)sub, B = l1[n] + l2[n] * (long double)dia, Cc = l2[n] * (long double)sup;
    const cld D = std::sqrt(B * B - 4.0L * A * Cc);
    cld den1 = -B - D, den2 = -B + D;
    const cld den = std::abs(den1) >= std::abs(den2) ? den1 : den2;  // = 2 c r1 (larger root)
    if (std::abs(den) == 0.0L) return fail(c, PD_ESINGULAR, "shifted system n=%d is singular (b = 0, ac = 0)", n);
    const cld tau = 2.0L / den;
    const cld r2 = A * tau, s = Cc * tau;
    // stability of the two first-order recurrences over the N rows; outside it: the pivoted elimination
    const long double g2 = powl(std::abs(r2), (long double)N), gs = powl(std::abs(s), (long double)N);
    if (!(g2 < 1e8L) || !(gs < 1e8L)) {
      c->use_gtsv = true;
      break;
    }
    // singularity: x_0 = x^(d)_0 / (1 - c q_0),  q_0 = -tau sum_{j<N} s^j r2^{j+1}
    cld q0 = 0.0L, sp = 1.0L, rp = r2;
    for (int j = 0; j < N; ++j) {
      q0 += sp * rp;
      sp *= s;
      rp *= r2;
    }
    q0 *= -tau;
    const cld piv = 1.0L - Cc * q0;
    if (std::abs(piv) < 1e-12L)
      return fail(c, PD_ESINGULAR, "shifted system lambda1 I + lambda2 K singular at frequency n=%d (|1-c q0|=%.3Le)",
                  n, std::abs(piv));
    // the closed-form boundary response divides by 1 - s r2 (= 1 - r2/r1: a double root leaves the regime)
    const cld geo = 1.0L - s * r2;
    if (std::abs(geo) < 1e-7L) {
      c->use_gtsv = true;
      break;
    }
    pd_tri_coef t;
    t.r2 = d2(r2);
    t.s = d2(s);
    t.tau = d2(tau);
    cld r2L = 1.0L, sL = 1.0L;
    for (int j = 0; j < L; ++j) {
      r2L *= r2;
      sL *= s;
    }
    t.r2L = d2(r2L);
    t.sL = d2(sL);
    cld r2N1 = r2;
    for (int j = 0; j < N; ++j) r2N1 *= r2;
    const cld k1 = Cc / piv * (-tau / geo);
    t.k1 = d2(k1);
    t.k2 = d2(-k1 * r2N1);
    out[n] = t;
  }
  if (c->use_gtsv) {
    for (int n = 0; n < c->F; ++n) {
      const cld A = l2[n] * (long double)sub, B = l1[n] + l2[n] * (long double)dia, Cc = l2[n] * (long double)sup;
      const long double mp = gtsv_min_pivot(A, B, Cc, N);
      if (!(mp > 1e-15L))
        return fail(c, PD_ESINGULAR,
                    "shifted system lambda1 I + lambda2 K singular at frequency n=%d (pivoted elimination: min "
                    "|pivot| / max |entry| = %.3Le)", n, mp);
      out[n] = pd_tri_coef{};
    }
  }
  return PD_OK;
}

static void free_ctx(pd_ctx* c) {
  if (!c) return;
  pd_tail_free(c);
  if (c->ytri) cudaFree(c->ytri);
  if (c->dtri) cudaFree(c->dtri);
  if (c->mu) cudaFree(c->mu);
  if (c->nl_dbar) cudaFree(c->nl_dbar);
  if (c->gm_head) cudaFree(c->gm_head);
  if (c->gm_full) cudaFree(c->gm_full);
  if (c->npart) cudaFree(c->npart);
  if (c->d2h_st) cudaStreamDestroy(c->d2h_st);
  for (double* p : c->Zs) cudaFree(p);
  if (c->gm_flag) cudaFree(c->gm_flag);
  if (c->ivp_init) cudaFree(c->ivp_init);
  if (c->ivp_f) cudaFree(c->ivp_f);
  if (c->gm_hflag) cudaFreeHost(c->gm_hflag);
  if (c->gtsv_scratch) cudaFree(c->gtsv_scratch);
  if (c->gtsv_bad) cudaFree(c->gtsv_bad);
  if (c->gtsv_hbad) cudaFreeHost(c->gtsv_hbad);
  void* ptrs[] = {c->tw_n1, c->tw_n2, c->tf4_scratch, c->gam, c->igam, c->tw_t, c->lam1, c->lam2, c->tri, c->sx, c->sn, c->tw_s, c->Sh, c->rvec,
                  c->partial, c->dred, c->zvec, c->stage_a, c->stage_b};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (double* p : c->V) cudaFree(p);
  if (c->hred) cudaFreeHost(c->hred);
  for (auto& g : c->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  for (int k = 1; k < kPdMaxOverlap; ++k) {
    if (c->ov.scratch[k]) cudaFree(c->ov.scratch[k]);
    if (c->ov.st[k]) cudaStreamDestroy(c->ov.st[k]);
    if (c->ov.ev_join[k]) cudaEventDestroy(c->ov.ev_join[k]);
  }
  if (c->ov.ev_fork) cudaEventDestroy(c->ov.ev_fork);
  pd_dist_free(c);
  for (auto& e : c->evpool)
    if (e) cudaEventDestroy(e);
  if (c->comm) pd_comm_destroy(c->comm);
  delete c;
}

extern "C" {

const char* pd_last_error(const pd_ctx* c) { return c ? c->err.c_str() : g_setup_err.c_str(); }

pd_status pd_nccl_unique_id(void* out128) {
  if (!out128) return fail(nullptr, PD_EINVAL, "null output");
  return pd_comm_unique_id(out128) == 0 ? PD_OK : fail(nullptr, PD_ENCCL, "%s", pd_comm_last_error());
}

void pd_destroy(pd_ctx* c) {
  if (c && c->st) cudaStreamSynchronize(c->st);
  free_ctx(c);
}

pd_status pd_setup(const pd_grid* g, double dt, int nt, double alpha, pd_scheme s, const pd_dist* dist,
                   void* cuda_stream, pd_ctx** out) {
  if (!out) return fail(nullptr, PD_EINVAL, "out is NULL");
  *out = nullptr;
  if (!g) return fail(nullptr, PD_EINVAL, "grid is NULL");
  if (!(alpha > 0.0 && alpha <= 1.0)) return fail(nullptr, PD_EINVAL, "alpha=%g outside (0,1]", alpha);
  if (!(dt > 0.0)) return fail(nullptr, PD_EINVAL, "dt=%g must be > 0", dt);
  if (!pd_tfft_supported(nt)) return fail(nullptr, PD_EINVAL, "Nt=%d must be a power of two in [1, 8192]", nt);
  if (s != PD_BE && s != PD_CN && s != PD_LEAPFROG) return fail(nullptr, PD_EINVAL, "unknown scheme %d", (int)s);
  if (s == PD_LEAPFROG && nt < 4) return fail(nullptr, PD_EINVAL, "leapfrog needs Nt >= 4");
  if (!(g->length > 0.0)) return fail(nullptr, PD_EINVAL, "length must be > 0");
  if (g->op == PD_ADE1D_DIRICHLET || g->op == PD_WAVE1D_DIRICHLET) {
    if (g->nx < 1 || g->ny != 1) return fail(nullptr, PD_EINVAL, "1D grid needs nx >= 1, ny == 1");
    if (pd_tridiag_threads(g->nx) < 0) return fail(nullptr, PD_EINVAL, "Nx=%d too large (max %d)", g->nx,
                                                   1024 * pd_tridiag_rows_per_thread());
  } else if (g->op == PD_ADE2D_PERIODIC) {
    if (g->nx != g->ny || !pd_slab2d_supported(g->nx))
      return fail(nullptr, PD_EINVAL, "2D grid must be N x N with N a power of two in [16, 1024]");
  } else if (g->op == PD_WAVE2D_DIRICHLET) {
    if (g->nx != g->ny || !pd_slab2d_dst_supported(g->nx))
      return fail(nullptr, PD_EINVAL, "2D Dirichlet grid must be N x N with N + 1 a power of two in [16, 512]");
    if (g->ax != 0.0 || g->ay != 0.0)
      return fail(nullptr, PD_EINVAL, "2D Dirichlet operator is -nu Lap (ax = ay = 0: DST-I diagonalisation)");
  } else {
    return fail(nullptr, PD_EINVAL, "unknown operator %d", (int)g->op);
  }
  const int size = dist ? dist->size : 1, rank = dist ? dist->rank : 0;
  if (size < 1 || rank >= size || (size == 1 && rank != 0)) return fail(nullptr, PD_EINVAL, "bad rank/size %d/%d", rank, size);

  pd_ctx* c = new pd_ctx();
  c->g = *g;
  c->dt = dt;
  c->nt = nt;
  c->F = nt / 2 + 1;
  c->alpha = alpha;
  c->scheme = s;
  c->st = (cudaStream_t)cuda_stream;
  c->rank = rank < 0 ? 0 : rank;
  c->size = size;
  c->Sg = (long long)g->nx * g->ny;

  // ---- distribution: spatial slabs (1D: x-ranges, 2D: y-row ranges) ----
  // dist == NULL or size == 1: single GPU.  rank >= 0: NCCL rank (local slab vectors).  rank < 0: `size`
  // virtual ranks in this process on one GPU (global vectors; the sharded path's test mode).
  c->dist_mode = size > 1 ? (dist->rank < 0 ? 2 : 1) : 0;
  if (c->dist_mode == 1 && !dist->nccl_id && !dist->nccl_comm) {
    free_ctx(c);
    return fail(nullptr, PD_EINVAL, "multi-GPU setup needs an NCCL communicator or unique id (pd_nccl_unique_id)");
  }
  if (c->dist_mode == 1) {
    const pd_plan pl = pd_make_plan(g->op, g->nx, g->ny, nt, size);
    c->off = pl.s_off[rank];
    c->S = pl.s_cnt[rank];
    c->nx_loc = pd_is_2d(g->op) ? g->nx : pl.e_cnt[rank];
    c->ny_loc = pd_is_2d(g->op) ? pl.e_cnt[rank] : 1;
  } else {
    c->nx_loc = g->nx;
    c->ny_loc = g->ny;
    c->off = 0;
    c->S = c->Sg;
  }

  // ---- spectra, Gamma, twiddles ----
  std::vector<cld> l1, l2;
  closed_form_spectra(nt, alpha, dt, s, l1, l2);
  c->lam1_full.resize(nt);
  c->lam2_full.resize(nt);
  for (int n = 0; n < nt; ++n) {
    c->lam1_full[n] = std::complex<double>((double)l1[n].real(), (double)l1[n].imag());
    c->lam2_full[n] = std::complex<double>((double)l2[n].real(), (double)l2[n].imag());
  }
  std::vector<double> hg(nt), hig(nt);
  for (int j = 0; j < nt; ++j) {
    hg[j] = (double)powl((long double)alpha, (long double)j / nt);     // alpha^{j/Nt}  (P:l.163-165)
    hig[j] = (double)powl((long double)alpha, -(long double)j / nt);   // alpha^{-j/Nt} (P:l.877-880)
  }
  auto twiddles = [](int n) {
    std::vector<double2> t(n);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int j = 0; j < n; ++j) {
      const long double th = 2.0L * pi * (long double)j / (long double)n;
      t[j] = make_double2((double)cosl(th), (double)-sinl(th));
    }
    return t;
  };
  std::vector<double2> htw = twiddles(nt), hl1(c->F), hl2(c->F);
  for (int n = 0; n < c->F; ++n) {
    hl1[n] = d2(l1[n]);
    hl2[n] = d2(l2[n]);
  }
  pd_status st = PD_OK;
#define SETUP_CUDA(expr)                                                                   \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      std::string m_ = cudaGetErrorString(e_);                                             \
      free_ctx(c);                                                                         \
      return fail(nullptr, e_ == cudaErrorMemoryAllocation ? PD_ENOMEM : PD_ECUDA, "%s: %s", #expr, m_.c_str()); \
    }                                                                                      \
  } while (0)
  SETUP_CUDA(dalloc(&c->gam, nt));
  SETUP_CUDA(dalloc(&c->igam, nt));
  SETUP_CUDA(dalloc(&c->tw_t, nt));
  SETUP_CUDA(dalloc(&c->lam1, c->F));
  SETUP_CUDA(dalloc(&c->lam2, c->F));
  SETUP_CUDA(cudaMemcpy(c->gam, hg.data(), nt * sizeof(double), cudaMemcpyHostToDevice));
  SETUP_CUDA(cudaMemcpy(c->igam, hig.data(), nt * sizeof(double), cudaMemcpyHostToDevice));
  SETUP_CUDA(cudaMemcpy(c->tw_t, htw.data(), nt * sizeof(double2), cudaMemcpyHostToDevice));
  SETUP_CUDA(cudaMemcpy(c->lam1, hl1.data(), c->F * sizeof(double2), cudaMemcpyHostToDevice));
  SETUP_CUDA(cudaMemcpy(c->lam2, hl2.data(), c->F * sizeof(double2), cudaMemcpyHostToDevice));

  // ---- spatial operator ----
  pd_stencil& sp = c->sten;
  sp.op = g->op == PD_ADE1D_DIRICHLET ? 0 : g->op == PD_WAVE1D_DIRICHLET ? 1 : g->op == PD_ADE2D_PERIODIC ? 2 : 3;
  sp.scheme = s == PD_BE ? 0 : s == PD_CN ? 1 : 2;
  sp.nx = c->nx_loc;
  sp.ny = c->ny_loc;
  sp.nt = nt;
  sp.dt = dt;
  sp.theta = s == PD_BE ? 1.0 : 0.5;
  if (g->op == PD_WAVE2D_DIRICHLET) {
    const int N = g->nx, M = 2 * (N + 1);
    const double h = g->length / (N + 1);
    sp.k2c = 4 * g->nu / (h * h);
    sp.k2x_m = sp.k2x_p = sp.k2y_m = sp.k2y_p = -g->nu / (h * h);
    std::vector<double> hmu(M);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < M; ++k) {
      const long double sk = sinl(pi * k / M);
      hmu[k] = (double)(4.0L * g->nu / ((long double)h * h) * sk * sk);
    }
    // singularity: min |lambda1 + lambda2 (mu_kx + mu_ky)| over the half spectrum and k = 1..N
    long double worst = 1e300L;
    int wn = -1;
    for (int n = 0; n < c->F; ++n)
      for (int kx = 1; kx <= N; ++kx)
        for (int ky = 1; ky <= N; ky += (N > 64 ? 7 : 1)) {
          const long double m = (long double)hmu[kx] + hmu[ky];
          const long double r = std::abs(l1[n] + l2[n] * m) / (std::abs(l1[n]) + std::abs(l2[n]) * m + 1e-300L);
          if (r < worst) {
            worst = r;
            wn = n;
          }
        }
    if (worst < 1e-13L) {
      free_ctx(c);
      return fail(nullptr, PD_ESINGULAR, "shifted system singular at frequency n=%d (relative |den| %.3Le)", wn, worst);
    }
    // y-direction by Dirichlet Toeplitz recurrences per (n, kx) (slab2d.cu dtri) when every column is in their
    // stable regime; otherwise (or PD_NO_DTRI) the DST column pass
    if (pd_slab2d_dtri_supported(N) && getenv("PD_NO_DTRI") == nullptr) {
      const int L = (N + 1) / 32;
      const long double a = -(long double)g->nu / ((long double)h * h), dia2 = 2 * (long double)g->nu / ((long double)h * h);
      std::vector<pd_dtri_coef> dt((size_t)c->F * N);
      bool ok = true;
      auto cp = [](cld m, int e) {
        cld r = 1.0L;
        while (e) {
          if (e & 1) r *= m;
          m *= m;
          e >>= 1;
        }
        return r;
      };
      for (int n = 0; n < c->F && ok; ++n)
        for (int kx = 0; kx < N && ok; ++kx) {
          const cld A = l2[n] * a, Cc = A, B = l1[n] + l2[n] * ((long double)hmu[kx + 1] + dia2);
          const cld D = std::sqrt(B * B - 4.0L * A * Cc);
          const cld den = std::abs(-B - D) >= std::abs(-B + D) ? -B - D : -B + D;
          if (std::abs(den) == 0.0L) {
            ok = false;
            break;
          }
          const cld tau = 2.0L / den, r2 = A * tau, sv = Cc * tau;
          if (!(powl(std::abs(r2), (long double)N) < 1e8L) || !(powl(std::abs(sv), (long double)N) < 1e8L)) {
            ok = false;
            break;
          }
          cld q0 = 0.0L, spw = 1.0L, rpw = r2;
          for (int j = 0; j < N; ++j) {
            q0 += spw * rpw;
            spw *= sv;
            rpw *= r2;
          }
          q0 *= -tau;
          const cld piv = 1.0L - Cc * q0, geo = 1.0L - sv * r2;
          // the closed-form response q_i = kappa (r2^{i+1} - r2^{N+1} s^{N-i}) divides by 1 - s r2
          if (std::abs(piv) < 1e-12L || std::abs(geo) < 1e-7L) {
            ok = false;
            break;
          }
          const cld k1 = Cc / piv * (-tau / geo);
          pd_dtri_coef& t = dt[(size_t)n * N + kx];
          t.r2 = d2(r2);
          t.s = d2(sv);
          t.tau = d2(tau);
          t.r2L = d2(cp(r2, L));
          t.sL = d2(cp(sv, L));
          t.sLm1 = d2(cp(sv, L - 1));
          t.k1 = d2(k1);
          t.k2 = d2(-k1 * cp(r2, N + 1));
        }
      if (ok) {
        SETUP_CUDA(dalloc(&c->dtri, dt.size()));
        SETUP_CUDA(cudaMemcpy(c->dtri, dt.data(), dt.size() * sizeof(pd_dtri_coef), cudaMemcpyHostToDevice));
        c->use_dtri = true;
      }
    }
    std::vector<double2> htw = twiddles(M);
    SETUP_CUDA(dalloc(&c->mu, M));
    SETUP_CUDA(dalloc(&c->tw_s, M));
    SETUP_CUDA(cudaMemcpy(c->mu, hmu.data(), M * sizeof(double), cudaMemcpyHostToDevice));
    SETUP_CUDA(cudaMemcpy(c->tw_s, htw.data(), M * sizeof(double2), cudaMemcpyHostToDevice));
    c->slab_chunk = pd_slab2d_chunk(N, c->F);
  } else if (g->op != PD_ADE2D_PERIODIC) {
    const double h = g->length / (g->nx + 1);
    const double nu = g->nu, a = g->op == PD_ADE1D_DIRICHLET ? g->ax : 0.0;
    sp.sub = -nu / (h * h) - a / (2 * h);
    sp.dia = 2 * nu / (h * h);
    sp.sup = -nu / (h * h) + a / (2 * h);
    std::vector<pd_tri_coef> tc;
    st = tri_coefs(c, l1, l2, sp.sub, sp.dia, sp.sup, tc);
    if (st != PD_OK) {
      std::string m = c->err;
      free_ctx(c);
      return fail(nullptr, st, "%s", m.c_str());
    }
    SETUP_CUDA(dalloc(&c->tri, c->F));
    SETUP_CUDA(cudaMemcpy(c->tri, tc.data(), c->F * sizeof(pd_tri_coef), cudaMemcpyHostToDevice));
  } else {
    const int N = g->nx;
    const double h = g->length / N;
    sp.k2c = 4 * g->nu / (h * h);
    sp.k2x_m = -g->nu / (h * h) - g->ax / (2 * h);
    sp.k2x_p = -g->nu / (h * h) + g->ax / (2 * h);
    sp.k2y_m = -g->nu / (h * h) - g->ay / (2 * h);
    sp.k2y_p = -g->nu / (h * h) + g->ay / (2 * h);
    c->slab.kd = 4 * g->nu / (h * h);
    c->slab.cx = g->ax / h;
    c->slab.cy = g->ay / h;
    std::vector<double> hsx(N), hsn(N);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < N; ++k) {
      const long double sk = sinl(pi * k / N);
      hsx[k] = (double)(sk * sk);
      hsn[k] = (double)sinl(2.0L * pi * k / N);
    }
    // singularity: min |lambda1 + lambda2 kappa| / (|lambda1| + |lambda2| |kappa|) over the half spectrum and all
    // (kx, ky) - an F N^2 reduction, done on the device (min_den_kernel) once the tables are there (below)
    std::vector<double2> htws = twiddles(N);
    SETUP_CUDA(dalloc(&c->sx, N));
    SETUP_CUDA(dalloc(&c->sn, N));
    SETUP_CUDA(dalloc(&c->tw_s, N));
    SETUP_CUDA(cudaMemcpy(c->sx, hsx.data(), N * sizeof(double), cudaMemcpyHostToDevice));
    SETUP_CUDA(cudaMemcpy(c->sn, hsn.data(), N * sizeof(double), cudaMemcpyHostToDevice));
    SETUP_CUDA(cudaMemcpy(c->tw_s, htws.data(), N * sizeof(double2), cudaMemcpyHostToDevice));
    {
      double* dmin = nullptr;
      SETUP_CUDA(dalloc(&dmin, (size_t)c->F));
      SETUP_CUDA(pd_launch_min_den(c->lam1, c->lam2, c->sx, c->sn, c->slab, N, c->F, dmin, c->st));
      std::vector<double> hmin(c->F);
      SETUP_CUDA(cudaMemcpyAsync(hmin.data(), dmin, c->F * sizeof(double), cudaMemcpyDeviceToHost, c->st));
      SETUP_CUDA(cudaStreamSynchronize(c->st));
      cudaFree(dmin);
      int wn = 0;
      for (int n = 1; n < c->F; ++n)
        if (hmin[n] < hmin[wn]) wn = n;
      if (hmin[wn] < 1e-13) {
        free_ctx(c);
        return fail(nullptr, PD_ESINGULAR, "shifted system singular at frequency n=%d (relative |den| %.3e)", wn, hmin[wn]);
      }
    }
    c->slab_chunk = pd_slab2d_chunk(N, c->F);
    // y-pass by cyclic Toeplitz solves where every column is in the stable regime (PD_NO_YTRI: FFT column pass)
    if (pd_slab2d_ytri_supported(N) && getenv("PD_NO_YTRI") == nullptr) {
      std::vector<pd_ytri_coef> yt;
      if (ytri_coefs(c, l1, l2, yt)) {
        SETUP_CUDA(cudaMalloc(reinterpret_cast<void**>(&c->ytri), yt.size() * sizeof(pd_ytri_coef)));
        SETUP_CUDA(cudaMemcpy(c->ytri, yt.data(), yt.size() * sizeof(pd_ytri_coef), cudaMemcpyHostToDevice));
        c->use_ytri = true;
      }
    }
    if (const char* e = getenv("PD_SLAB_CHUNK_MB")) {
      const long long sb = (long long)N * N * 16;
      c->slab_chunk = (int)std::max(1LL, std::min<long long>(c->F, (atoll(e) << 20) / sb));
    }
  }

  // ---- four-step time FFT for long time axes (1D), or with the x-FFT folded in (2D, tfx.cu) ----
  c->use_tfx = g->op == PD_ADE2D_PERIODIC && pd_tfx_supported(nt, g->nx) && getenv("PD_NO_TFX") == nullptr;
  c->use_tf4 = !c->use_tfx && pd_tf4_supported(nt) && getenv("PD_NO_TF4") == nullptr;
  if (const char* ge = getenv("PD_GRAPH")) {
    c->use_graphs = atoi(ge) != 0;
  } else {
    // launch-bound sizes (configs 0 and 1): replay a triple's launch sequence from its second use on (apply -22 %,
    // r02ah).  Not beyond ~2M dofs: at the config-2/3 size the replay gains 2 % per apply and instantiating the ~50-node
    // multi-stream graph costs ~1 ms per triple (r02ai: cfg3 e2e 3.9 -> 5.0 ms over the bench's repetitions)
    c->use_graphs = c->graphs_on_reuse = (long long)nt * c->S <= (1LL << 21);
  }
  if (c->use_tf4 || c->use_tfx) {
    const int n2 = c->use_tfx ? pd_tfx_n2(nt) : pd_tf4_n2(), n1 = nt / n2;
    const long long align = c->use_tfx ? pd_tfx_chunk_align(nt, g->nx) : pd_tf4_pairs_per_tile();
    std::vector<double2> h1 = twiddles(n1), h2 = twiddles(n2);
    SETUP_CUDA(dalloc(&c->tw_n1, n1));
    SETUP_CUDA(dalloc(&c->tw_n2, n2));
    SETUP_CUDA(cudaMemcpy(c->tw_n1, h1.data(), n1 * sizeof(double2), cudaMemcpyHostToDevice));
    SETUP_CUDA(cudaMemcpy(c->tw_n2, h2.data(), n2 * sizeof(double2), cudaMemcpyHostToDevice));
    const long long npairs = (c->S + 1) / 2;
    // column chunk of the stage-1 -> stage-2 scratch; 2D: whole x-rows.  One stream: 1 GB chunks (launch
    // ramp/tail beats L2 residency, §5).  Default: 3 streams of 16 MB chunks (PD_TF4_OVERLAP = 3), so
    // consecutive chunks' stages overlap and the scratch round trip mostly stays in L2 (§5)
    const char* ov_env = getenv("PD_TF4_OVERLAP");
    const int kov = std::min(std::max(ov_env ? atoi(ov_env) : 3, 1), kPdMaxOverlap);
    // the inverse measured best with 4 streams (2.84 vs 2.88 ms on cfg4), the forward with 3 (2.68 vs 2.75)
    const char* ovi_env = getenv("PD_TF4_OVERLAP_INV");
    const int kovi = std::min(std::max(ovi_env ? atoi(ovi_env) : (ov_env ? kov : 4), 1), kPdMaxOverlap);
    const int kmax = std::max(kov, kovi);
    const char* mb_env = getenv("PD_TF4_CHUNK_MB");
    const long long mb = mb_env ? atoll(mb_env) : (kmax > 1 ? 16 : 1024);
    long long chunk = ((mb << 20) / ((long long)nt * 16)) / align * align;
    if (chunk < align) chunk = align;
    if (chunk > npairs) chunk = (npairs + align - 1) / align * align;
    c->tf4_chunk = chunk;
    SETUP_CUDA(dalloc(&c->tf4_scratch, (size_t)nt * chunk));
    c->use_ov = kmax > 1;
    if (c->use_ov) {
      c->ov.k = kmax;
      SETUP_CUDA(cudaEventCreateWithFlags(&c->ov.ev_fork, cudaEventDisableTiming));
      for (int k = 1; k < kmax; ++k) {
        SETUP_CUDA(dalloc(&c->ov.scratch[k], (size_t)nt * chunk));
        SETUP_CUDA(cudaStreamCreateWithFlags(&c->ov.st[k], cudaStreamNonBlocking));
        SETUP_CUDA(cudaEventCreateWithFlags(&c->ov.ev_join[k], cudaEventDisableTiming));
      }
      c->ov_inv = c->ov;
      c->ov.k = kov;
      c->ov_inv.k = kovi;
    }
  }

  // ---- workspace ----
  SETUP_CUDA(dalloc(&c->Sh, (size_t)c->F * c->S));
  SETUP_CUDA(dalloc(&c->rvec, (size_t)nt * c->S));
  {
    pd_stencil tmp = sp;
    const long long Sx = (long long)tmp.nx * tmp.ny;
    const long long nb = ((Sx + 255) / 256) * ((nt + 63) / 64);
    c->npartial = (int)std::max<long long>(nb, (long long)pd_blas_blocks() * 32);
  }
  SETUP_CUDA(dalloc(&c->partial, (size_t)c->npartial));
  SETUP_CUDA(dalloc(&c->dred, 64));
  SETUP_CUDA(cudaMallocHost((void**)&c->hred, 64 * sizeof(double)));
  if (c->dist_mode != 0) {
    // partials of every shard's stencil launch live side by side
    if (c->dist_mode == 2) {
      cudaFree(c->partial);
      c->npartial *= size;
      SETUP_CUDA(dalloc(&c->partial, (size_t)c->npartial));
    }
    const pd_status ds = pd_dist_setup(c, dist->nccl_id, dist->nccl_comm);
    if (ds != PD_OK) {
      std::string m = c->err;
      free_ctx(c);
      return fail(nullptr, ds, "%s", m.c_str());
    }
  }
#undef SETUP_CUDA
  *out = c;
  return PD_OK;
}

pd_status pd_local_shape(const pd_ctx* c, int* nx_local, int* ny_local, long long* offset) {
  if (!c) return PD_EINVAL;
  if (nx_local) *nx_local = c->nx_loc;
  if (ny_local) *ny_local = c->ny_loc;
  if (offset) *offset = c->off;
  return PD_OK;
}

long long pd_local_size(const pd_ctx* c) { return c ? (long long)c->nt * c->S : -1; }

pd_status pd_spectra(const pd_ctx* c, double* l1, double* l2) {
  if (!c || !l1 || !l2) return PD_EINVAL;
  for (int n = 0; n < c->nt; ++n) {
    l1[2 * n] = c->lam1_full[n].real();
    l1[2 * n + 1] = c->lam1_full[n].imag();
    l2[2 * n] = c->lam2_full[n].real();
    l2[2 * n + 1] = c->lam2_full[n].imag();
  }
  return PD_OK;
}

long long pd_kernel_launches(const pd_ctx* c) { return c ? c->launches : -1; }

static void resolve_events(pd_ctx* c) {
  for (auto& pr : c->evrec) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, c->evpool[pr.second], c->evpool[pr.second + 1]) == cudaSuccess) {
      c->phase_ms[pr.first] += ms;
      c->phase_n[pr.first] += 1;
    }
  }
  c->evrec.clear();
}

pd_status pd_enable_phase_timing(pd_ctx* c, int en) {
  if (!c) return PD_EINVAL;
  PD_CUDA(c, cudaStreamSynchronize(c->st));
  c->timing = en != 0;
  c->evrec.clear();
  for (int i = 0; i < 8; ++i) {
    c->phase_ms[i] = 0;
    c->phase_n[i] = 0;
    c->ev_open[i] = -1;
  }
  return PD_OK;
}

pd_status pd_phase_times(pd_ctx* c, double* ms4, long long* n4) {
  if (!c) return PD_EINVAL;
  PD_CUDA(c, cudaStreamSynchronize(c->st));
  resolve_events(c);
  for (int i = 0; i < 8; ++i) {
    if (ms4) ms4[i] = c->phase_ms[i];
    if (n4) n4[i] = c->phase_n[i];
  }
  return PD_OK;
}

}  // extern "C"

// ---- phase timing: CUDA events recorded on the context stream around each kernel, resolved lazily
// (pd_phase_times) so the timed region is not serialised by host syncs ----
// NVTX ranges per kernel slot (nsys / ncu --nvtx timelines; a no-op without a tool attached)
static const char* const kPhaseName[8] = {"step_a_time_fft",  "step_b_spatial_solve", "step_c_inverse_time_fft",
                                          "residual",         "step_c_fused_update",  "matvec",
                                          "krylov_sweep",     "residual_norm"};
static void phase_begin(pd_ctx* c, int ph) {
  nvtxRangePushA(kPhaseName[ph]);
  if (!c->timing) return;
  const int need = (int)(c->evrec.size() + 1) * 2;
  while ((int)c->evpool.size() < need) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    c->evpool.push_back(e);
  }
  const int i = (int)c->evrec.size() * 2;
  cudaEventRecord(c->evpool[i], c->st);
  c->ev_open[ph] = i;
}
static void phase_end(pd_ctx* c, int ph) {
  nvtxRangePop();
  if (!c->timing || c->ev_open[ph] < 0) return;
  const int i = c->ev_open[ph];
  cudaEventRecord(c->evpool[i + 1], c->st);
  c->evrec.emplace_back(ph, i);
  c->ev_open[ph] = -1;
  if (c->evrec.size() >= 2048) {  // bound the pool: resolve (syncs) every 2048 records
    cudaEventSynchronize(c->evpool[i + 1]);
    resolve_events(c);
  }
}

// workspace of the pivoted 1D Step (b) (gtsv.cu), allocated on first use: factors [F][Nx] and the singular flag
pd_status pd_gtsv_ensure(pd_ctx* c) {
  if (!c->gtsv_scratch)
    PD_CUDA(c, cudaMalloc(&c->gtsv_scratch, pd_gtsv_scratch_bytes(c->g.nx, c->F)));
  if (!c->gtsv_bad) {
    PD_CUDA(c, cudaMalloc(reinterpret_cast<void**>(&c->gtsv_bad), sizeof(int)));
    PD_CUDA(c, cudaMemsetAsync(c->gtsv_bad, 0, sizeof(int), c->st));
    PD_CUDA(c, cudaMallocHost(reinterpret_cast<void**>(&c->gtsv_hbad), sizeof(int)));
  }
  return PD_OK;
}

// Step (b) on a spectrum buffer holding frequencies [f0, f0 + nfreq) on full spatial rows
pd_status pd_spatial_solve(pd_ctx* c, double2* Sh, int nfreq, int f0) {
  phase_begin(c, 1);
  if (c->g.op == PD_WAVE2D_DIRICHLET) {
    int nl = 0;
    if (c->use_dtri)
      PD_CUDA(c, pd_launch_slab2d_dtri(Sh, c->g.nx, nfreq, f0, c->dtri, c->tw_s, c->slab_chunk, c->st, &nl));
    else
      PD_CUDA(c, pd_launch_slab2d_dst(Sh, c->g.nx, nfreq, c->lam1 + f0, c->lam2 + f0, c->mu, c->tw_s, c->slab_chunk,
                                      c->st, &nl));
    c->launches += nl;
  } else if (c->g.op == PD_ADE2D_PERIODIC) {
    int nl = 0;
    if (c->use_ytri)
      PD_CUDA(c, pd_launch_slab2d_ytri(Sh, c->g.nx, nfreq, f0, c->ytri, 1.0 / c->g.nx, c->tw_s, c->slab_chunk,
                                       c->use_tfx ? 0 : 1, c->st, &nl));
    else
      PD_CUDA(c, pd_launch_slab2d(Sh, c->g.nx, nfreq, c->lam1 + f0, c->lam2 + f0, c->sx, c->sn, c->slab, c->tw_s,
                                  c->slab_chunk, c->use_tfx ? 1 : 0, c->st, &nl));
    c->launches += nl;
  } else if (c->use_gtsv) {
    if (pd_status s = pd_gtsv_ensure(c); s != PD_OK) return s;
    PD_LAUNCH(c, pd_launch_gtsv_shift(Sh, c->g.nx, nfreq, c->lam1 + f0, c->lam2 + f0, c->sten.sub, c->sten.dia,
                                      c->sten.sup, nullptr, c->gtsv_scratch, c->gtsv_bad, c->st));
  } else {
    PD_LAUNCH(c, pd_launch_tridiag(Sh, c->g.nx, nfreq, c->tri + f0, pd_tridiag_rows_per_thread(), c->st));
  }
  phase_end(c, 1);
  return PD_OK;
}

// Step (a) of a local slab: r [Nt][S] -> Sh [F][S]
pd_status pd_time_fft_fwd(pd_ctx* c, const double* r, const pd_spec& sp, long long S) {
  const pd_tf4_tables tb{c->tw_n1, c->tw_n2, c->tw_t};
  phase_begin(c, 0);
  if (c->use_tfx) {
    int nl = 0;
    PD_CUDA(c, pd_launch_tfx_fwd(c->nt, c->g.nx, r, sp, S, c->gam, tb, c->tw_s, c->tf4_scratch, c->tf4_chunk, c->st, &nl,
                                 c->ov.k > 1 ? &c->ov : nullptr));
    c->launches += nl;
  } else if (c->use_tf4) {
    int nl = 0;
    PD_CUDA(c, pd_launch_tf4_fwd(c->nt, r, sp, S, c->gam, tb, c->tf4_scratch, c->tf4_chunk, c->st, &nl,
                                 c->ov.k > 1 ? &c->ov : nullptr));
    c->launches += nl;
  } else {
    PD_LAUNCH(c, pd_launch_tfft_fwd(c->nt, r, sp, S, c->gam, c->tw_t, c->st));
  }
  phase_end(c, 0);
  return PD_OK;
}

// stream pool view of the inverse time FFT: 4 streams for z = ..., the forward's 3 for the accumulating u += ...
// (which also reads u: 4.02 vs 3.86 ms on cfg4 with 4 streams)
static const pd_tfx_overlap* inv_view(const pd_ctx* c, int accumulate) {
  const pd_tfx_overlap& v = accumulate ? c->ov : c->ov_inv;
  return v.k > 1 ? &v : nullptr;
}

// Step (c) of a local slab: Sh [F][S] -> z [Nt][S] (z += when accumulate)
pd_status pd_time_fft_inv(pd_ctx* c, const pd_spec& sp, double* z, long long S, int accumulate) {
  const pd_tf4_tables tb{c->tw_n1, c->tw_n2, c->tw_t};
  const int ph = accumulate ? 4 : 2;
  phase_begin(c, ph);
  if (c->use_tfx) {
    int nl = 0;
    PD_CUDA(c, pd_launch_tfx_inv(c->nt, c->g.nx, sp, z, S, c->igam, tb, c->tw_s, c->tf4_scratch, c->tf4_chunk,
                                 accumulate, c->st, &nl, inv_view(c, accumulate)));
    c->launches += nl;
  } else if (c->use_tf4) {
    int nl = 0;
    PD_CUDA(c, pd_launch_tf4_inv(c->nt, sp, z, S, c->igam, tb, c->tf4_scratch, c->tf4_chunk, accumulate, c->st, &nl,
                                 inv_view(c, accumulate)));
    c->launches += nl;
  } else {
    PD_LAUNCH(c, pd_launch_tfft_inv(c->nt, sp, z, S, c->igam, c->tw_t, accumulate, c->st));
  }
  phase_end(c, ph);
  return PD_OK;
}

static pd_status apply_direct(pd_ctx* c, const double* r, double* z, int accumulate) {
  if (c->dist_mode != 0) return pd_dist_apply(c, r, z, accumulate);
  const pd_spec sp = pd_spec_local(c->Sh, c->S);
  pd_status s = pd_time_fft_fwd(c, r, sp, c->S);
  if (s != PD_OK) return s;
  s = pd_spatial_solve(c, c->Sh, c->F, 0);
  if (s != PD_OK) return s;
  return pd_time_fft_inv(c, sp, z, c->S, accumulate);
}

// u += P^{-1} (sum_i cb.c[i] cb.x[i]) with the combination read by the forward time FFT's stage-1 loader (tfx path,
// single GPU; the GMRES final update).  The fused forward is timed with the Krylov sweeps (phase 6): it is the
// combination sweep plus a time FFT, so it does not enter the per-call average of the forward time FFT.
static pd_status apply_comb_accumulate(pd_ctx* c, const pd_comb_args* cb, double* u, int accumulate) {
  const pd_tf4_tables tb{c->tw_n1, c->tw_n2, c->tw_t};
  phase_begin(c, 6);
  int nl = 0;
  PD_CUDA(c, pd_launch_tfx_fwd(c->nt, c->g.nx, nullptr, pd_spec_local(c->Sh, c->S), c->S, c->gam, tb, c->tw_s, c->tf4_scratch, c->tf4_chunk,
                               c->st, &nl, c->ov.k > 1 ? &c->ov : nullptr, cb));
  c->launches += nl;
  phase_end(c, 6);
  pd_status s = pd_spatial_solve(c, c->Sh, c->F, 0);
  if (s != PD_OK) return s;
  return pd_time_fft_inv(c, pd_spec_local(c->Sh, c->S), u, c->S, accumulate);
}

// z = P^{-1} r with ||r||^2 taken by the forward time FFT's stage-1 loader (tfx path, single GPU): *rr on the host
// (syncs).  PD_ECUDA-free fallback: returns PD_EINVAL when the fused form does not apply (caller uses dots + apply).
static pd_status apply_with_norm(pd_ctx* c, const double* r, double* z, double* rr) {
  const pd_tf4_tables tb{c->tw_n1, c->tw_n2, c->tw_t};
  if (!c->npart) {  // one partial per stage-1 CTA: <= 8 (npairs / 8 + chunks) (tiles of >= 8 pairs, 8 t1 rows)
    const long long npairs = c->S / 2, chunks = (npairs + c->tf4_chunk - 1) / c->tf4_chunk;
    PD_CUDA(c, dalloc(&c->npart, (size_t)(8 * (npairs / 8 + chunks) + 64)));
  }
  phase_begin(c, 0);
  int nl = 0;
  long long np = 0;
  PD_CUDA(c, pd_launch_tfx_fwd(c->nt, c->g.nx, r, pd_spec_local(c->Sh, c->S), c->S, c->gam, tb, c->tw_s,
                               c->tf4_scratch, c->tf4_chunk, c->st, &nl, c->ov.k > 1 ? &c->ov : nullptr, nullptr,
                               c->npart, &np));
  c->launches += nl;
  PD_LAUNCH(c, pd_launch_reduce_partials(c->npart, (int)np, 1, c->dred, c->st));
  phase_end(c, 0);
  pd_status s = pd_spatial_solve(c, c->Sh, c->F, 0);
  if (s != PD_OK) return s;
  s = pd_time_fft_inv(c, pd_spec_local(c->Sh, c->S), z, c->S, 0);
  if (s != PD_OK) return s;
  PD_CUDA(c, cudaMemcpyAsync(c->hred, c->dred, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  PD_CUDA(c, cudaStreamSynchronize(c->st));
  *rr = c->hred[0];
  return PD_OK;
}

// z = P^{-1} r, or u += P^{-1} r when accumulate.  With graphs enabled (single GPU, phase timing off) the
// launch sequence of each (r, z, accumulate) triple is captured once and replayed as one CUDA graph.
pd_status pd_apply_impl(pd_ctx* c, const double* r, double* z, int accumulate) {
  if (!c->use_graphs || c->dist_mode != 0 || c->timing) return apply_direct(c, r, z, accumulate);
  pd_ctx::GraphEntry* seen = nullptr;
  for (auto& g : c->graphs)
    if (g.r == r && g.z == z && g.acc == accumulate) {
      if (!g.exec) {
        seen = &g;  // second use of the triple: capture now
        break;
      }
      PD_CUDA(c, cudaGraphLaunch(g.exec, c->st));
      c->launches += g.launches;
      return PD_OK;
    }
  if (!seen && c->graphs.size() >= 64) {
    for (auto& g : c->graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
  }
  if (!seen && c->graphs_on_reuse) {  // first use: run directly, remember the triple
    c->graphs.push_back({r, z, accumulate, nullptr, 0});
    return apply_direct(c, r, z, accumulate);
  }
  const long long l0 = c->launches;
  if (!c->cap_stream) PD_CUDA(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  cudaStream_t user = c->st;
  c->st = c->cap_stream;
  PD_CUDA(c, cudaStreamBeginCapture(c->st, cudaStreamCaptureModeRelaxed));
  pd_status s = apply_direct(c, r, z, accumulate);
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(c->st, &graph);
  c->st = user;
  if (s != PD_OK) return s;
  if (e != cudaSuccess) return fail(c, PD_ECUDA, "graph capture: %s", cudaGetErrorString(e));
  cudaGraphExec_t exec = nullptr;
  e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(c, PD_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
  if (seen) {
    seen->exec = exec;
    seen->launches = c->launches - l0;
  } else {
    c->graphs.push_back({r, z, accumulate, exec, c->launches - l0});
  }
  PD_CUDA(c, cudaGraphLaunch(exec, c->st));
  return PD_OK;
}

// out = b - A u (b != NULL) or A u; if norm2 != NULL: deterministic ||out||^2 into *norm2 (host, syncs).
// out == NULL (single GPU, with b and norm2): the norm only, no vector written (timing slot 7, 16 B/dof).
pd_status pd_stencil_impl(pd_ctx* c, const double* b, const double* u, double* out, double* norm2) {
  const int ph = b ? (out ? 3 : 7) : 5;
  phase_begin(c, ph);
  if (c->dist_mode != 0) {
    pd_status s = pd_dist_stencil(c, b, u, out, nullptr);  // local sum of squares -> dred[0]
    if (s != PD_OK) return s;
  } else {
    int nb = 0;
    PD_LAUNCH(c, pd_launch_stencil(c->sten, b, u, out, c->partial, &nb, c->st));
    if (norm2) PD_LAUNCH(c, pd_launch_reduce_partials(c->partial, nb, 1, c->dred, c->st));
  }
  phase_end(c, ph);
  if (norm2) {
    if (c->dist_mode == 1 && pd_comm_allreduce_sum(c->comm, c->dred, 1) != 0)
      return fail(c, PD_ENCCL, "allreduce: %s", pd_comm_last_error());
    PD_CUDA(c, cudaMemcpyAsync(c->hred, c->dred, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    PD_CUDA(c, cudaStreamSynchronize(c->st));
    *norm2 = c->hred[0];
  }
  return PD_OK;
}

// Krylov sweep (blas1.cu) over the local vector; the k (or 1) reduced values all-reduced across ranks and
// copied to host_out (syncs) unless host_out == NULL (mode 3)
pd_status pd_krylov_n(pd_ctx* c, int mode, const double* const* X, const double* coef, int k, double a, double* y,
                      long long n, double* host_out, bool global_sum, const double* hsub, long long hlen) {
  phase_begin(c, 6);
  PD_LAUNCH(c, pd_launch_krylov(mode, X, coef, k, a, y, n, c->partial, c->st, hsub, hlen));
  if (mode != 3) {
    const int kk = mode == 2 ? 1 : mode == 4 ? k + 1 : k;
    PD_LAUNCH(c, pd_launch_reduce_partials(c->partial, pd_blas_blocks(), kk, c->dred, c->st));
    phase_end(c, 6);
    if (global_sum && c->dist_mode == 1 && pd_comm_allreduce_sum(c->comm, c->dred, kk) != 0)
      return fail(c, PD_ENCCL, "allreduce: %s", pd_comm_last_error());
    PD_CUDA(c, cudaMemcpyAsync(c->hred, c->dred, kk * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    PD_CUDA(c, cudaStreamSynchronize(c->st));
    for (int i = 0; i < kk; ++i) host_out[i] = c->hred[i];
  } else {
    phase_end(c, 6);
  }
  return PD_OK;
}

static pd_status krylov_impl(pd_ctx* c, int mode, const double* const* X, const double* coef, int k, double a,
                             double* y, double* host_out) {
  return pd_krylov_n(c, mode, X, coef, k, a, y, (long long)c->nt * c->S, host_out);
}

// dots[i] = <X[i], y>
static pd_status dots_impl(pd_ctx* c, const double* const* X, int k, const double* y, double* host_out) {
  return krylov_impl(c, 0, X, nullptr, k, 0.0, const_cast<double*>(y), host_out);
}

extern "C" {

pd_status pd_apply_precond(pd_ctx* c, const double* r, double* z) {
  if (!c || !r || !z) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  return pd_apply_impl(c, r, z, 0);
}

pd_status pd_residual(pd_ctx* c, const double* b, const double* u, double* r, double* rnorm2_host) {
  if (!c || !b || !u || !r) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  return pd_stencil_impl(c, b, u, r, rnorm2_host);
}

pd_status pd_matvec(pd_ctx* c, const double* u, double* w) {
  if (!c || !u || !w) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  return pd_stencil_impl(c, nullptr, u, w, nullptr);
}

pd_status pd_build_rhs(pd_ctx* c, const double* u0, const double* v0, const double* f, double* b) {
  if (!c || !u0 || !b) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  if (c->dist_mode != 0) return pd_dist_build_rhs(c, u0, v0, f, b);
  PD_LAUNCH(c, pd_launch_rhs(c->sten, u0, v0, f, b, c->st));
  return PD_OK;
}

void pd_report_push(pd_report* rep, double v) {
  if (rep && rep->history && rep->history_len < rep->history_cap) rep->history[rep->history_len] = v;
  if (rep) rep->history_len++;
}

pd_status pd_solve_stationary(pd_ctx* c, const double* b, double* u, double tol, int maxit, pd_report* rep) {
  if (!c || !b || !u) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  if (!(tol > 0) || maxit < 0) return fail(c, PD_EINVAL, "tol must be > 0, maxit >= 0");
  const auto t0 = std::chrono::steady_clock::now();
  if (rep) rep->history_len = 0;
  const double* X[1] = {b};
  double bb = 0;
  pd_status s = dots_impl(c, X, 1, b, &bb);
  if (s != PD_OK) return s;
  const double bnorm = std::sqrt(bb);
  if (bnorm == 0.0) {
    PD_CUDA(c, cudaMemsetAsync(u, 0, sizeof(double) * c->nt * c->S, c->st));
    if (rep) *rep = pd_report{0, 1, 0.0, 0.0, rep->history, rep->history_cap, 0};
    return PD_OK;
  }
  int k = 0;
  double rel = 0;
  for (;;) {
    double rr = 0;
    s = pd_stencil_impl(c, b, u, c->rvec, &rr);  // r = b - A u (eq 5.1)
    if (s != PD_OK) return s;
    rel = std::sqrt(rr) / bnorm;
    if (k > 0) pd_report_push(rep, rel);
    if (rel <= tol || k >= maxit) break;
    s = pd_apply_impl(c, c->rvec, u, 1);  // u += P^{-1} r (fused into Step (c))
    if (s != PD_OK) return s;
    ++k;
  }
  const bool conv = rel <= tol;
  if (rep) {
    rep->iterations = k;
    rep->converged = conv;
    rep->rel_residual = rel;
    rep->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return conv ? PD_OK : PD_NOT_CONVERGED;
}

// head = G tail: the (P_alpha - A) block rows of the corner identity from the last H time blocks of a local vector.
// NCCL ranks: the tails are replicated (zero-padded copy + sum all-reduce of H S_glob doubles), G is applied on the
// global grid (no halos needed) and the local columns are kept.
extern "C++" pd_status pd_corner_head(pd_ctx* c, const pd_tail_g& gc, const double* tail, double* head) {
  if (c->dist_mode != 1) {
    PD_LAUNCH(c, pd_launch_head_G(c->sten, gc, tail, head, c->S, c->st));
    return PD_OK;
  }
  const long long Sg = c->Sg, hn = (long long)gc.H * Sg;
  if (!c->gm_full) PD_CUDA(c, dalloc(&c->gm_full, (size_t)(2 * hn + 2)));
  double *ft = c->gm_full, *fh = c->gm_full + hn;
  PD_CUDA(c, cudaMemsetAsync(ft, 0, sizeof(double) * hn, c->st));
  for (int t = 0; t < gc.H; ++t)
    PD_CUDA(c, cudaMemcpyAsync(ft + t * Sg + c->off, tail + (long long)t * c->S, sizeof(double) * c->S,
                               cudaMemcpyDeviceToDevice, c->st));
  if (pd_comm_allreduce_sum(c->comm, ft, (int)hn) != 0) return fail(c, PD_ENCCL, "allreduce: %s", pd_comm_last_error());
  pd_stencil gs = c->sten;
  gs.nx = c->g.nx;
  gs.ny = c->g.ny;
  gs.hlo = gs.hhi = nullptr;
  PD_LAUNCH(c, pd_launch_head_G(gs, gc, ft, fh, Sg, c->st));
  for (int t = 0; t < gc.H; ++t)
    PD_CUDA(c, cudaMemcpyAsync(head + (long long)t * c->S, fh + t * Sg + c->off, sizeof(double) * c->S,
                               cudaMemcpyDeviceToDevice, c->st));
  return PD_OK;
}

// zero_guess: u is output only (not read; no zero-check sweep); otherwise u is the initial guess
static pd_status gmres_impl(pd_ctx* c, const double* b, double* u, double tol, int m, int maxit, pd_report* rep,
                            bool zero_guess) {
  if (!c || !b || !u) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  if (!(tol > 0) || maxit < 0 || m < 1 || m > 30) return fail(c, PD_EINVAL, "need tol > 0, maxit >= 0, 1 <= m <= 30");
  const auto t0 = std::chrono::steady_clock::now();
  if (rep) rep->history_len = 0;
  const long long n = (long long)c->nt * c->S;
  if (c->gm_m < m) {
    for (double* p : c->V) cudaFree(p);
    c->V.assign(m + 1, nullptr);
    for (auto& p : c->V) {
      cudaError_t e = dalloc(&p, (size_t)n);
      if (e != cudaSuccess) {
        for (double*& q : c->V) {
          if (q) cudaFree(q);
          q = nullptr;
        }
        c->V.clear();
        c->gm_m = 0;
        cudaGetLastError();
        return fail(c, PD_ENOMEM, "GMRES basis (%d vectors of %lld doubles): %s", m + 1, n, cudaGetErrorString(e));
      }
    }
    if (!c->zvec && dalloc(&c->zvec, (size_t)n) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, PD_ENOMEM, "GMRES work vector");
    }
    c->gm_m = m;
  }
  // Z_j = P^{-1} X_j kept for the final assembly u = x0 + sum_j y_j sc_j Z_j (the applies write them anyway), which
  // replaces the final apply P^{-1}(V y) by one combination sweep; only if the m extra vectors fit with 2 GB to spare
  // (PD_GMRES_NO_Z=1: the final apply)
  bool useZ = getenv("PD_GMRES_NO_Z") == nullptr && (reinterpret_cast<uintptr_t>(u) & 15) == 0;
  if (useZ && (int)c->Zs.size() < m) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const size_t need = (size_t)(m - (int)c->Zs.size()) * (size_t)n * sizeof(double) + (2ull << 30);
    if (fr < need) {
      useZ = false;
    } else {
      while ((int)c->Zs.size() < m) {
        double* p = nullptr;
        if (dalloc(&p, (size_t)n) != cudaSuccess) {
          cudaGetLastError();
          useZ = false;
          break;
        }
        c->Zs.push_back(p);
      }
    }
  }
  // Basis kept scaled: V_i = sc[i] * X_i with X_i = c->V[i] in memory, so normalising costs no sweep.
  // Zero initial guess (checked on the device, single GPU): r0 = b exactly, so the first cycle reads X_0 = b in
  // place of a residual sweep; a restart writes the true residual into c->V[0].
  std::vector<const double*> Xv(c->V.begin(), c->V.end());
  double rr = 0;
  bool u_zero = false;
  if (zero_guess && !(c->dist_mode == 0 && (reinterpret_cast<uintptr_t>(b) & 15) == 0)) {
    PD_CUDA(c, cudaMemsetAsync(u, 0, sizeof(double) * n, c->st));  // b not usable in place: the general path
  } else if (zero_guess) {
    u_zero = true;
  } else if (c->dist_mode == 0 && (reinterpret_cast<uintptr_t>(b) & 15) == 0) {  // b read in place by the Krylov kernels
    if (!c->gm_flag) {
      PD_CUDA(c, cudaMalloc(reinterpret_cast<void**>(&c->gm_flag), sizeof(int)));
      PD_CUDA(c, cudaMallocHost(reinterpret_cast<void**>(&c->gm_hflag), sizeof(int)));
    }
    PD_CUDA(c, cudaMemsetAsync(c->gm_flag, 0, sizeof(int), c->st));
    PD_LAUNCH(c, pd_launch_any_nonzero(u, n, c->gm_flag, c->st));
    PD_CUDA(c, cudaMemcpyAsync(c->gm_hflag, c->gm_flag, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    PD_CUDA(c, cudaStreamSynchronize(c->st));
    u_zero = *c->gm_hflag == 0;
  }
  // ||b|| fused into the first apply's Step (a) read of b (zero initial guess, tfx path, single GPU): one sweep over
  // b less per solve; the b = 0 / tol >= 1 exits are then taken after that apply
  const bool fuse_bnorm = u_zero && maxit > 0 && c->dist_mode == 0 && c->use_tfx && !c->use_graphs && c->S % 2 == 0 &&
                          (reinterpret_cast<uintptr_t>(b) & 15) == 0 && getenv("PD_GMRES_NO_FUSED_NORM") == nullptr;
  const double* Xb[1] = {b};
  double bb = 0;
  pd_status s = PD_OK;
  double bnorm = 1.0;  // set by the first apply when fuse_bnorm
  if (!fuse_bnorm) {
    s = dots_impl(c, Xb, 1, b, &bb);
    if (s != PD_OK) return s;
    bnorm = std::sqrt(bb);
    if (bnorm == 0.0) {
      PD_CUDA(c, cudaMemsetAsync(u, 0, sizeof(double) * n, c->st));
      if (rep) *rep = pd_report{0, 1, 0.0, 0.0, rep->history, rep->history_cap, 0};
      return PD_OK;
    }
  }
  if (u_zero) {
    Xv[0] = b;
    rr = bb;
  } else {
    s = pd_stencil_impl(c, b, u, c->V[0], &rr);  // X_0 = r = b - A u
    if (s != PD_OK) return s;
  }
  double beta = std::sqrt(rr);
  int its = 0;
  bool conv = !fuse_bnorm && beta <= tol * bnorm, breakdown = false;
  bool norm_pending = fuse_bnorm;  // u_zero holds (zero_guess with an aligned b): X_0 = b
  std::vector<double> H((m + 1) * m), cs(m), sn(m), gv(m + 1), h(m + 1), h2(m + 2), y(m), coef(m + 1), sc(m + 1);
  auto Hs = [&](int i, int j) -> double& { return H[i * m + j]; };
  const double* const* Xp = Xv.data();
  // corner identity path (single GPU, linear operator); PD_GMRES_MATVEC=1 keeps the explicit matvec
  pd_tail_g gcorner{};
  pd_corner_coefs(c, &gcorner);
  // sharded contexts too: virtual ranks hold global vectors; NCCL ranks replicate the H tail blocks (one all-reduce
  // of H S_glob doubles) and form the head on the global grid (pd_corner_head)
  const bool corner = c->sten.g3 == 0.0 && c->sten.g1 == 0.0 && gcorner.H >= 1 && c->nt >= 2 * gcorner.H &&
                      getenv("PD_GMRES_MATVEC") == nullptr;
  const long long hn_len = (long long)gcorner.H * c->S;
  std::vector<double> eh(m + 2);
  std::vector<const double*> Xh(m + 2);
  const bool lazy_last = getenv("PD_GMRES_NO_LAZY") == nullptr;
  double ww_known = -1.0;                 // ||w||^2 when the second CGS pass is skipped
  const double kReorthSkip = getenv("PD_GMRES_ALWAYS_CGS2") ? -1.0 : 1e-12;
  double* dhead = nullptr;
  if (corner) {
    if (!c->gm_head) PD_CUDA(c, dalloc(&c->gm_head, (size_t)(2 * c->S + 2)));
    dhead = c->gm_head;
  }
  bool u_is_zero = u_zero;  // until the first cycle's update: that update writes u instead of adding to it
  while (!conv && its < maxit) {
    sc[0] = 1.0 / beta;
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int kk = 0;
    for (int j = 0; j < m; ++j) {
      // w_raw = A P^{-1} X_j;  true w = sc[j] * w_raw
      double* zj = useZ ? c->Zs[j] : c->zvec;
      if (norm_pending) {  // first apply of the solve: X_0 = b, ||b||^2 from its Step (a)
        norm_pending = false;
        s = apply_with_norm(c, Xv[0], zj, &bb);
        if (s != PD_OK) return s;
        bnorm = std::sqrt(bb);
        rr = bb;
        beta = bnorm;
        if (bnorm == 0.0 || beta <= tol * bnorm) {  // b = 0, or tol >= 1: u = 0 solves it (no iteration counted)
          PD_CUDA(c, cudaMemsetAsync(u, 0, sizeof(double) * n, c->st));
          if (rep) *rep = pd_report{0, 1, bnorm == 0.0 ? 0.0 : 1.0, 0.0, rep->history, rep->history_cap, 0};
          return PD_OK;
        }
        sc[0] = 1.0 / beta;
        gv[0] = beta;
      } else {
        s = pd_apply_impl(c, Xv[j], zj, 0);
        if (s != PD_OK) return s;
      }
      ++its;
      double* w = c->V[j + 1];
      bool skip_vector = false;  // corner path: the cycle ends at this column, V_{j+1} is not assembled
      if (corner) {
        // A P^{-1} X_j = X_j - E_H G tail(P^{-1} X_j)  ((P - A) touches only head rows x tail columns, the identity
        // behind the tail form): the matvec sweep disappears and, the basis being orthonormal, the first CGS pass is
        // h_i = delta_ij - sc_i sc_j <X_i[head], G tail>: head-only dots.  The second pass measures the true
        // projections of the assembled w as before, so orthogonality is enforced to working precision.
        s = pd_corner_head(c, gcorner, zj + (long long)(c->nt - gcorner.H) * c->S, dhead);
        if (s != PD_OK) return s;
        // <X_i[head], G tail>, and ||G tail||^2 as one more dot of the same launch
        for (int i = 0; i <= j; ++i) Xh[i] = Xp[i];
        Xh[j + 1] = dhead;
        s = pd_krylov_n(c, 0, Xh.data(), nullptr, j + 2, 0.0, dhead, hn_len, eh.data());
        if (s != PD_OK) return s;
        for (int i = 0; i <= j; ++i) {
          h[i] = (i == j ? 1.0 : 0.0) - sc[i] * sc[j] * eh[i];
          coef[i] = -h[i] * sc[i] / sc[j];
        }
        // The new basis vector is only needed by a further iteration of this cycle.  Its norm follows from head-sized
        // numbers: w - sum h_i V_i = -(I - V V^T) E_H c, c = sc_j G tail, so ||.||^2 = sc_j^2 (||G tail||^2 -
        // sum_i sc_i^2 <X_i[head], G tail>^2) for an orthonormal basis.  When that estimate (trusted only while the
        // subtraction keeps 8 digits) says the cycle ends here - converged by the Arnoldi estimate, clear of the
        // threshold, or j = m - 1 - the sweep that would assemble the vector (j + 2 vector moves) is skipped; the true
        // residual at the cycle end still decides (reading c6).  PD_GMRES_NO_LAZY=1 always assembles it.
        if (lazy_last) {
          double pe = 0.0;
          for (int i = 0; i <= j; ++i) pe += sc[i] * sc[i] * eh[i] * eh[i];
          const double dd = eh[j + 1], wwe = dd - pe;
          if (dd > 0.0 && wwe > 1e-8 * dd) {
            const double hne = sc[j] * std::sqrt(wwe);
            std::vector<double> col(h.begin(), h.begin() + j + 1);
            for (int i = 0; i < j; ++i) {
              const double t = cs[i] * col[i] + sn[i] * col[i + 1];
              col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
              col[i] = t;
            }
            const double gn = std::fabs(hne / std::hypot(col[j], hne) * gv[j]);  // |gv[j+1]| after the j-th rotation
            const double thr = tol * bnorm;
            const bool done = gn <= 0.5 * thr, undecided = gn > 0.5 * thr && gn <= 2.0 * thr;
            if (done || (j == m - 1 && !undecided)) {
              ww_known = wwe;
              skip_vector = true;
            }
          }
        }
        if (!skip_vector) {
        coef[j] = sc[j] * sc[j] * eh[j];  // 1 - h_jj without cancellation: w_raw = X_j + E_H delta - sum h_i sc_i/sc_j X_i
        // written fresh, + E_H delta (delta = -G tail) on the head rows inside the same sweep: the dots and ||w||^2
        // are those of the final vector
        s = pd_krylov_n(c, 4, Xp, coef.data(), j + 1, 0.0, w, n, h2.data(), true, dhead, hn_len);
        if (s != PD_OK) return s;
        const double ww1 = h2[j + 1];
        double pmax = 0.0;
        for (int i = 0; i <= j; ++i) {
          h2[i] = sc[i] * sc[j] * h2[i];
          pmax = std::max(pmax, std::fabs(h2[i]));
        }
        if (pmax <= kReorthSkip * sc[j] * std::sqrt(ww1)) {
          // measured projections below 1e-12 of the vector: the second CGS pass would not change it
          ww_known = ww1;
        } else {
          for (int i = 0; i <= j; ++i) {
            coef[i] = -h2[i] * sc[i] / sc[j];
            h[i] += h2[i];
          }
        }
        }  // !skip_vector
      } else {
        s = pd_stencil_impl(c, nullptr, zj, w, nullptr);
        if (s != PD_OK) return s;
        // CGS2: h_i = <V_i, w> = sc_i sc_j <X_i, w_raw>;  w_raw -= sum (h_i sc_i / sc_j) X_i  (fused with 2nd dots)
        s = krylov_impl(c, 0, Xp, nullptr, j + 1, 0.0, w, h.data());
        if (s != PD_OK) return s;
        for (int i = 0; i <= j; ++i) {
          h[i] *= sc[i] * sc[j];
          coef[i] = -h[i] * sc[i] / sc[j];
        }
        s = krylov_impl(c, 1, Xp, coef.data(), j + 1, 1.0, w, h2.data());
        if (s != PD_OK) return s;
        for (int i = 0; i <= j; ++i) {
          h2[i] *= sc[i] * sc[j];
          coef[i] = -h2[i] * sc[i] / sc[j];
          h[i] += h2[i];
        }
      }
      double ww = 0;
      if (ww_known >= 0.0) {
        ww = ww_known;
        ww_known = -1.0;
      } else {
        s = krylov_impl(c, 2, Xp, coef.data(), j + 1, 1.0, w, &ww);
        if (s != PD_OK) return s;
      }
      const double hn = sc[j] * std::sqrt(ww);
      for (int i = 0; i <= j; ++i) Hs(i, j) = h[i];
      Hs(j + 1, j) = hn;
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * Hs(i, j) + sn[i] * Hs(i + 1, j);
        Hs(i + 1, j) = -sn[i] * Hs(i, j) + cs[i] * Hs(i + 1, j);
        Hs(i, j) = t;
      }
      const double den = std::hypot(Hs(j, j), Hs(j + 1, j));
      cs[j] = Hs(j, j) / den;
      sn[j] = Hs(j + 1, j) / den;
      Hs(j, j) = den;
      Hs(j + 1, j) = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      kk = j + 1;
      pd_report_push(rep, std::fabs(gv[j + 1]) / bnorm);
      if (std::fabs(gv[j + 1]) <= tol * bnorm || its >= maxit || skip_vector) break;
      if (hn == 0.0) {
        breakdown = true;
        break;
      }
      sc[j + 1] = sc[j] / hn;  // V_{j+1} = w / hn = (sc_j / hn) X_{j+1}
    }
    // y = H^{-1} g, u += P^{-1} (V y)  (final assembly apply, not counted)
    for (int i = kk - 1; i >= 0; --i) {
      double t = gv[i];
      for (int l = i + 1; l < kk; ++l) t -= Hs(i, l) * y[l];
      y[i] = t / Hs(i, i);
    }
    for (int i = 0; i < kk; ++i) coef[i] = y[i] * sc[i];
    const int acc0 = u_is_zero ? 0 : 1;
    bool streamed = false;  // u's D2H (pd_solve_ivp_host) already issued chunk by chunk behind the assembly
    if (useZ) {  // u (+)= sum_i coef_i Z_i: one sweep over kk + 1 vectors instead of an apply
      u_is_zero = false;
      std::vector<const double*> Zp(c->Zs.begin(), c->Zs.begin() + kk);
      // pd_solve_ivp_host with a converged Arnoldi estimate: assemble u in row chunks and copy each chunk to the
      // host on a second stream right behind it, so the host-link transfer overlaps the rest of the assembly and
      // the true-residual check (the copy is waited for, and redone after the next cycle, if a restart follows)
      const bool stream_d2h = c->ivp_dst && acc0 == 0 && std::fabs(gv[kk]) <= tol * bnorm;
      if (stream_d2h) {
        if (!c->d2h_st) PD_CUDA(c, cudaStreamCreateWithFlags(&c->d2h_st, cudaStreamNonBlocking));
        const int K = 8;
        long long rows = (c->nt + K - 1) / K;
        if (rows % 2) ++rows;  // chunk starts 16-byte aligned for any S
        for (long long r0 = 0; r0 < c->nt; r0 += rows) {
          const long long nr = std::min<long long>(rows, c->nt - r0), off = r0 * c->S;
          std::vector<const double*> Zc(kk);
          for (int i = 0; i < kk; ++i) Zc[i] = Zp[i] + off;
          s = pd_krylov_n(c, 3, Zc.data(), coef.data(), kk, 0.0, u + off, nr * c->S, nullptr);
          if (s != PD_OK) return s;
          cudaEvent_t ev;
          PD_CUDA(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
          PD_CUDA(c, cudaEventRecord(ev, c->st));
          PD_CUDA(c, cudaStreamWaitEvent(c->d2h_st, ev, 0));
          PD_CUDA(c, cudaEventDestroy(ev));  // released once the wait has been satisfied
          PD_CUDA(c, cudaMemcpyAsync(c->ivp_dst + off, u + off, sizeof(double) * nr * c->S, cudaMemcpyDeviceToHost,
                                     c->d2h_st));
        }
        streamed = true;
      } else if (acc0 == 0) {
        s = krylov_impl(c, 3, Zp.data(), coef.data(), kk, 0.0, u, nullptr);
      } else {
        double unused = 0;
        s = krylov_impl(c, 2, Zp.data(), coef.data(), kk, 1.0, u, &unused);
      }
      if (s != PD_OK) return s;
    }
    // fused: the forward time FFT reads the basis combination itself (tfx path, single GPU, no graphs)
    bool fused = !useZ && c->use_tfx && c->dist_mode == 0 && !c->use_graphs && kk <= kPdCombMax && c->S % 2 == 0 &&
                 getenv("PD_GMRES_NO_FUSED_UPDATE") == nullptr;
    pd_comb_args cb{};
    for (int i = 0; fused && i < kk; ++i) {
      fused = (reinterpret_cast<uintptr_t>(Xp[i]) & 15) == 0;
      cb.x[i] = Xp[i];
      cb.c[i] = coef[i];
    }
    cb.k = kk;
    const int acc = u_is_zero ? 0 : 1;  // u = 0: u + x == x exactly, so write x (no read of u)
    u_is_zero = false;
    if (useZ) {
      // assembled above
    } else if (fused) {
      s = apply_comb_accumulate(c, &cb, u, acc);
      if (s != PD_OK) return s;
    } else {
      s = krylov_impl(c, 3, Xp, coef.data(), kk, 0.0, c->zvec, nullptr);
      if (s != PD_OK) return s;
      s = pd_apply_impl(c, c->zvec, u, acc);
      if (s != PD_OK) return s;
    }
    // true residual norm; the residual vector (the restart vector X_0) is written only when a restart follows
    // (single GPU: the norm-only stencil writes nothing)
    const bool norm_only = c->dist_mode == 0;
    s = pd_stencil_impl(c, b, u, norm_only ? nullptr : c->V[0], &rr);
    if (s != PD_OK) return s;
    if (norm_only && !(std::sqrt(rr) <= tol * bnorm) && its < maxit && !breakdown) {
      s = pd_stencil_impl(c, b, u, c->V[0], &rr);
      if (s != PD_OK) return s;
    }
    if (streamed) {
      if (std::sqrt(rr) <= tol * bnorm || its >= maxit || breakdown) {
        c->ivp_done = true;  // this u is final: its copy is in flight (pd_solve_ivp_host synchronises)
      } else {
        PD_CUDA(c, cudaStreamSynchronize(c->d2h_st));  // a restart rewrites u: finish the stale copy first
      }
    }
    Xv[0] = c->V[0];
    beta = std::sqrt(rr);
    conv = beta <= tol * bnorm;
    if (breakdown) break;
  }
  if (u_is_zero && zero_guess) PD_CUDA(c, cudaMemsetAsync(u, 0, sizeof(double) * n, c->st));  // no cycle ran
  if (rep) {
    rep->iterations = its;
    rep->converged = conv;
    rep->rel_residual = beta / bnorm;
    rep->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  if (conv) return PD_OK;
  if (breakdown) return fail(c, PD_EBREAKDOWN, "GMRES breakdown at iteration %d, residual %.3e", its, beta / bnorm);
  return PD_NOT_CONVERGED;
}

pd_status pd_solve_gmres(pd_ctx* c, const double* b, double* u, double tol, int m, int maxit, pd_report* rep) {
  return gmres_impl(c, b, u, tol, m, maxit, rep, false);
}

pd_status pd_solve(pd_ctx* c, int solver, const double* b, double* u, double tol, int m, int maxit, pd_report* rep) {
  if (!c) return PD_EINVAL;
  const bool zero = (solver & PD_SOLVE_ZERO_GUESS) != 0;
  solver &= ~PD_SOLVE_ZERO_GUESS;
  if (solver == 1) return gmres_impl(c, b, u, tol, m, maxit, rep, zero);
  if (solver != 0) return fail(c, PD_EINVAL, "pd_solve: solver %d not in {0 stationary, 1 gmres}", solver);
  if (zero && u) PD_CUDA(c, cudaMemsetAsync(u, 0, sizeof(double) * c->nt * c->S, c->st));
  return pd_solve_stationary(c, b, u, tol, maxit, rep);
}

// ---- host-buffer variants ----
static pd_status ensure_stage(pd_ctx* c) {
  const size_t n = (size_t)c->nt * c->S;
  if (!c->stage_a && dalloc(&c->stage_a, n) != cudaSuccess) return fail(c, PD_ENOMEM, "staging buffer");
  if (!c->stage_b && dalloc(&c->stage_b, n) != cudaSuccess) return fail(c, PD_ENOMEM, "staging buffer");
  return PD_OK;
}

pd_status pd_apply_precond_host(pd_ctx* c, const double* rh, double* zh) {
  if (!c || !rh || !zh) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  pd_status s = ensure_stage(c);
  if (s != PD_OK) return s;
  const size_t bytes = sizeof(double) * c->nt * c->S;
  PD_CUDA(c, cudaMemcpyAsync(c->stage_a, rh, bytes, cudaMemcpyHostToDevice, c->st));
  s = pd_apply_impl(c, c->stage_a, c->stage_b, 0);
  if (s != PD_OK) return s;
  PD_CUDA(c, cudaMemcpyAsync(zh, c->stage_b, bytes, cudaMemcpyDeviceToHost, c->st));
  PD_CUDA(c, cudaStreamSynchronize(c->st));
  return PD_OK;
}

pd_status pd_solve_host(pd_ctx* c, int solver, const double* bh, double* uh, double tol, int m, int maxit,
                        pd_report* rep) {
  if (!c || !bh || !uh) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  const bool zero = (solver & PD_SOLVE_ZERO_GUESS) != 0;
  solver &= ~PD_SOLVE_ZERO_GUESS;
  if (solver != 0 && solver != 1)
    return fail(c, PD_EINVAL, "pd_solve_host: solver %d not in {0 stationary, 1 gmres} (| PD_SOLVE_ZERO_GUESS)", solver);
  pd_status s = ensure_stage(c);
  if (s != PD_OK) return s;
  const size_t bytes = sizeof(double) * c->nt * c->S;
  PD_CUDA(c, cudaMemcpyAsync(c->stage_a, bh, bytes, cudaMemcpyHostToDevice, c->st));
  if (!zero)
    PD_CUDA(c, cudaMemcpyAsync(c->stage_b, uh, bytes, cudaMemcpyHostToDevice, c->st));
  else if (solver == 0)
    PD_CUDA(c, cudaMemsetAsync(c->stage_b, 0, bytes, c->st));
  s = solver == 0 ? pd_solve_stationary(c, c->stage_a, c->stage_b, tol, maxit, rep)
                  : gmres_impl(c, c->stage_a, c->stage_b, tol, m, maxit, rep, zero);
  c->ivp_dst = nullptr;
  if (c->d2h_st) PD_CUDA(c, cudaStreamSynchronize(c->d2h_st));
  if (s < 0) return s;
  if (!c->ivp_done) PD_CUDA(c, cudaMemcpyAsync(uh, c->stage_b, bytes, cudaMemcpyDeviceToHost, c->st));
  c->ivp_done = false;
  PD_CUDA(c, cudaStreamSynchronize(c->st));
  return s;
}

pd_status pd_solve_ivp_host(pd_ctx* c, int solver, const double* u0h, const double* v0h, const double* fh, double* uh,
                            double tol, int m, int maxit, pd_report* rep) {
  if (!c || !u0h || !uh) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  if (solver < 0 || solver > 4) return fail(c, PD_EINVAL, "solver %d not in 0..4", solver);
  pd_status s = ensure_stage(c);
  if (s != PD_OK) return s;
  const size_t Sb = sizeof(double) * c->S, bytes = Sb * c->nt;
  if (!c->ivp_init && dalloc(&c->ivp_init, (size_t)2 * c->S + 2) != cudaSuccess) return fail(c, PD_ENOMEM, "ivp buffers");
  double *du0 = c->ivp_init, *dv0 = c->ivp_init + c->S;
  PD_CUDA(c, cudaMemcpyAsync(du0, u0h, Sb, cudaMemcpyHostToDevice, c->st));
  if (v0h) PD_CUDA(c, cudaMemcpyAsync(dv0, v0h, Sb, cudaMemcpyHostToDevice, c->st));
  double* df = nullptr;
  if (fh) {
    if (!c->ivp_f && dalloc(&c->ivp_f, (size_t)(c->nt + 1) * c->S) != cudaSuccess) return fail(c, PD_ENOMEM, "ivp f");
    df = c->ivp_f;
    PD_CUDA(c, cudaMemcpyAsync(df, fh, Sb * (c->nt + 1), cudaMemcpyHostToDevice, c->st));
  }
  s = pd_build_rhs(c, du0, v0h ? dv0 : nullptr, df, c->stage_a);
  if (s != PD_OK) return s;
  // from u = 0: GMRES takes the zero-guess path (u output only), the others start from a zeroed u
  if (solver != 1) PD_CUDA(c, cudaMemsetAsync(c->stage_b, 0, bytes, c->st));
  c->ivp_dst = solver == 1 ? uh : nullptr;  // GMRES streams u to the host behind its final assembly
  c->ivp_done = false;
  switch (solver) {
    case 0: s = pd_solve_stationary(c, c->stage_a, c->stage_b, tol, maxit, rep); break;
    case 1: s = gmres_impl(c, c->stage_a, c->stage_b, tol, m, maxit, rep, true); break;
    case 2: s = pd_solve_stationary_tail(c, c->stage_a, c->stage_b, tol, maxit, rep); break;
    case 3: s = pd_solve_gmres_tail(c, c->stage_a, c->stage_b, tol, m, maxit, rep); break;
    default: s = pd_solve_newton(c, c->stage_a, c->stage_b, tol, maxit, rep); break;
  }
  c->ivp_dst = nullptr;
  if (c->d2h_st) PD_CUDA(c, cudaStreamSynchronize(c->d2h_st));
  if (s < 0) return s;
  if (!c->ivp_done) PD_CUDA(c, cudaMemcpyAsync(uh, c->stage_b, bytes, cudaMemcpyDeviceToHost, c->st));
  c->ivp_done = false;
  PD_CUDA(c, cudaStreamSynchronize(c->st));
  return s;
}

}  // extern "C"

