// Waveform-relaxation "tail" form of the stationary iteration and of GMRES.
// Reference implementation and derivation: oracle/tail.py (O3).  In brief (P:l.120-124, 762-773, 928-931):
//   P_alpha - A touches only the first H time blocks (rows) and the last H blocks (columns), H = 1 for the
//   theta-method and 2 for leapfrog:  (P - A) u = E_H G U_tail.  Hence
//     stationary:  t^{k+1} = tail(P^{-1} b) + T(G t^k),  ||b - A u^k|| = ||G (t^k - t^{k-1})||,
//                  u^k = P^{-1}(b + E_H G t^{k-1}) assembled once at exit;
//     GMRES:       every Krylov vector is a r0 + E_H h, A P^{-1}(a r0 + E_H h) = a (r0 - E_H q0) + E_H (h - G T(h)),
//                  q0 = G tail(P^{-1} r0); the basis is carried as (a_j on the host, h_j on the device).
//   T(g) = tail(P^{-1}(E_H g)) is the tail map: the economical Step (a) (an H-term sum), the shifted solves of
//   Step (b) for every frequency and only the last H rows of Step (c) - tridiag.cu tail1d_kernel in 1D, the
//   transfer function tau in 2D (tail.cu).  Per iteration the work is O(H S) memory traffic plus the per-
//   frequency solves (1D) instead of three full passes over Nt S dofs.
// Sharded contexts (SURVEY 8(f) NEXT-1 at P > 1): heads and tails (H x S_global values) are replicated on every
// rank, so all O(H S) work is redundant and reduction-free; the 1D tail map splits the frequency range over the
// ranks and sums with one H S all-reduce (instead of the two all-to-alls of a full apply), the 2D tail map (a
// slab FFT filter, microseconds) runs on every rank; only the full applies at start and exit are distributed.
// The virtual-rank executor runs the same per-shard frequency split on one GPU.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstring>
#include <vector>

#include "ctx.h"

namespace {

constexpr int kScr = 10;  // head-sized scratch vectors

cudaError_t dalloc_d(double** p, size_t n) { return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 2) * sizeof(double)); }
cudaError_t dalloc_c(double2** p, size_t n) { return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(double2)); }

long long hs(const pd_ctx* c) { return (long long)c->tail.H * c->Sg; }   // replicated head / tail size

}  // namespace

// (P_alpha - A) = E_H G U_tail: H and the coefficients of G from the alpha-corner of the time first columns
void pd_corner_coefs(const pd_ctx* c, pd_tail_g* gc) {
  const int H = c->scheme == PD_LEAPFROG ? 2 : 1;
  const int nt = c->nt;
  const double dt = c->dt, al = c->alpha;
  pd_tail_g T{};
  T.H = H;
  double c1[3] = {0, 0, 0}, c2[3] = {0, 0, 0};
  if (c->scheme == PD_LEAPFROG) {
    c1[0] = 1.0 / (dt * dt); c1[1] = -2.0 / (dt * dt); c1[2] = 1.0 / (dt * dt);
    c2[0] = 0.5; c2[2] = 0.5;
  } else {
    const double th = c->scheme == PD_BE ? 1.0 : 0.5;
    c1[0] = 1.0 / dt; c1[1] = -1.0 / dt;
    c2[0] = th; c2[1] = 1.0 - th;
  }
  // alpha-corner of the alpha-circulants: entry (a, j) with a < j, j = Nt-H+b, tap k = a - j + Nt = a - b + H
  for (int a = 0; a < H; ++a)
    for (int b = 0; b < H; ++b) {
      const int j = nt - H + b, k = a - b + H;
      if (a < j && k >= 1 && k <= 2) {
        T.pI[a][b] = al * c1[k];
        T.pK[a][b] = al * c2[k];
      }
    }
  *gc = T;
}

namespace {

pd_status tail_setup(pd_ctx* c) {
  auto& T = c->tail;
  if (T.ready) return PD_OK;
  if (c->use_gtsv)
    return fail(c, PD_EINVAL, "tail form: the 1D tail map needs the recurrence Step (b) (context uses pivoted elimination)");
  const int H = c->scheme == PD_LEAPFROG ? 2 : 1;
  if (c->nt < 2 * H) return fail(c, PD_EINVAL, "tail form needs Nt >= %d", 2 * H);
  const int nt = c->nt, F = c->F;
  const double al = c->alpha;
  pd_corner_coefs(c, &T.gc);
  // global-grid stencil for the head-from-tail product on the replicated tails
  T.gsten = c->sten;
  if (c->dist_mode == 1) {
    T.gsten.nx = c->g.nx;
    T.gsten.ny = c->g.ny;
  }
  T.gsten.hlo = T.gsten.hhi = nullptr;
  // economical Step (a) coefficients and last-H-row Step (c) weights (long double, closed form)
  typedef std::complex<long double> cld;
  const long double pi = 3.141592653589793238462643383279502884L;
  std::vector<double2> hc((size_t)F * H), ow((size_t)F * H), w2((size_t)F);
  for (int n = 0; n < F; ++n) {
    const long double mult = (n == 0 || 2 * n == nt) ? 1.0L : 2.0L;
    for (int t = 0; t < H; ++t) {
      const long double g = powl((long double)al, (long double)t / nt);
      const cld v = g * std::exp(cld(0.0L, -2.0L * pi * n * t / nt));
      hc[(size_t)n * H + t] = make_double2((double)v.real(), (double)v.imag());
    }
    for (int a = 0; a < H; ++a) {
      const int t = nt - H + a;
      const long double ig = powl((long double)al, -(long double)t / nt);
      const cld v = mult * ig / (long double)nt * std::exp(cld(0.0L, 2.0L * pi * n * t / nt));
      ow[(size_t)n * H + a] = make_double2((double)v.real(), (double)v.imag());
    }
    const cld wv = cld(ow[(size_t)n * H].x, ow[(size_t)n * H].y) * cld(hc[(size_t)n * H].x, hc[(size_t)n * H].y);
    w2[n] = make_double2((double)wv.real(), (double)wv.imag());
  }
  const long long Sg = c->Sg;
  if (c->g.op == PD_ADE2D_PERIODIC) {
    const int N = c->g.nx;
    double2* wd = nullptr;
    PD_CUDA(c, dalloc_c(&wd, F));
    PD_CUDA(c, cudaMemcpy(wd, w2.data(), F * sizeof(double2), cudaMemcpyHostToDevice));
    PD_CUDA(c, dalloc_c(&T.tau, (size_t)N * N));
    PD_CUDA(c, dalloc_c(&T.work, (size_t)N * N));
    PD_LAUNCH(c, pd_launch_tau2d(T.tau, N, F, c->lam1, c->lam2, wd, c->sx, c->sn, c->slab, c->st));
    PD_CUDA(c, cudaStreamSynchronize(c->st));
    cudaFree(wd);
  } else if (c->g.op == PD_WAVE2D_DIRICHLET) {
    // tensor DST-I basis: real transfer tables tau[a][t][ky][kx] (tail.cu tau_dir), the N x N sine table
    const int N = c->g.nx;
    const long long NN = (long long)N * N;
    std::vector<double2> wat((size_t)H * H * F);
    for (int a = 0; a < H; ++a)
      for (int t = 0; t < H; ++t)
        for (int n = 0; n < F; ++n) {
          const cld v = cld(ow[(size_t)n * H + a].x, ow[(size_t)n * H + a].y) * cld(hc[(size_t)n * H + t].x,
                                                                                  hc[(size_t)n * H + t].y);
          wat[((size_t)a * H + t) * F + n] = make_double2((double)v.real(), (double)v.imag());
        }
    double2* wd = nullptr;
    PD_CUDA(c, dalloc_c(&wd, wat.size()));
    PD_CUDA(c, cudaMemcpy(wd, wat.data(), wat.size() * sizeof(double2), cudaMemcpyHostToDevice));
    PD_CUDA(c, dalloc_d(&T.taud, (size_t)H * H * NN));
    PD_LAUNCH(c, pd_launch_tau_dir(T.taud, N, F, H, c->lam1, c->lam2, wd, c->mu, c->st));
    PD_CUDA(c, cudaStreamSynchronize(c->st));
    cudaFree(wd);
    std::vector<double> sn((size_t)NN);
    for (int j = 0; j < N; ++j)
      for (int k = 0; k < N; ++k)
        sn[(size_t)j * N + k] = (double)sinl(pi * (long double)((j + 1) * (long long)(k + 1) % (2 * (N + 1))) / (N + 1));
    PD_CUDA(c, dalloc_d(&T.dsin, (size_t)NN));
    PD_CUDA(c, cudaMemcpy(T.dsin, sn.data(), sn.size() * sizeof(double), cudaMemcpyHostToDevice));
    PD_CUDA(c, dalloc_d(&T.dwork, (size_t)(2 * H + 1) * NN));
  } else {
    PD_CUDA(c, dalloc_c(&T.ow, (size_t)F * H));
    PD_CUDA(c, cudaMemcpy(T.ow, ow.data(), ow.size() * sizeof(double2), cudaMemcpyHostToDevice));
    T.G = std::min(F, 4 * 148);
    PD_CUDA(c, dalloc_d(&T.part, (size_t)T.G * H * Sg));
    if (c->dist_mode == 2) PD_CUDA(c, dalloc_d(&T.acc, (size_t)H * Sg));
  }
  PD_CUDA(c, dalloc_c(&T.hc, (size_t)F * H));
  PD_CUDA(c, cudaMemcpy(T.hc, hc.data(), hc.size() * sizeof(double2), cudaMemcpyHostToDevice));
  PD_CUDA(c, dalloc_c(&T.gx, (size_t)H * Sg));
  T.scr.assign(kScr, nullptr);
  for (auto& p : T.scr) PD_CUDA(c, dalloc_d(&p, (size_t)H * Sg));
  PD_CUDA(c, cudaMalloc(reinterpret_cast<void**>(&T.flag), sizeof(int)));
  PD_CUDA(c, cudaMallocHost(reinterpret_cast<void**>(&T.hflag), sizeof(int)));
  T.H = H;
  T.ready = true;
  return PD_OK;
}

pd_status allreduce(pd_ctx* c, double* d, long long n) {
  if (c->dist_mode != 1) return PD_OK;
  if (pd_comm_allreduce_sum(c->comm, d, (int)n) != 0) return fail(c, PD_ENCCL, "allreduce: %s", pd_comm_last_error());
  return PD_OK;
}

// full [H][Sg] (replicated) <- the H blocks starting at `rows` of a local [Nt][S] vector
pd_status gather_full(pd_ctx* c, const double* rows, double* full) {
  const int H = c->tail.H;
  if (c->dist_mode != 1) {
    PD_CUDA(c, cudaMemcpyAsync(full, rows, sizeof(double) * H * c->Sg, cudaMemcpyDeviceToDevice, c->st));
    return PD_OK;
  }
  PD_CUDA(c, cudaMemsetAsync(full, 0, sizeof(double) * H * c->Sg, c->st));
  for (int t = 0; t < H; ++t)
    PD_CUDA(c, cudaMemcpyAsync(full + (long long)t * c->Sg + c->off, rows + (long long)t * c->S, sizeof(double) * c->S,
                               cudaMemcpyDeviceToDevice, c->st));
  return allreduce(c, full, (long long)H * c->Sg);
}

// the H blocks starting at `rows` of a local vector <- this rank's part of full [H][Sg]
pd_status local_of(pd_ctx* c, const double* full, double* rows) {
  const int H = c->tail.H;
  for (int t = 0; t < H; ++t)
    PD_CUDA(c, cudaMemcpyAsync(rows + (long long)t * c->S, full + (long long)t * c->Sg + (c->dist_mode == 1 ? c->off : 0),
                               sizeof(double) * c->S, cudaMemcpyDeviceToDevice, c->st));
  return PD_OK;
}

pd_status comb(pd_ctx* c, std::vector<const double*> X, std::vector<double> coef, double* y, long long n) {
  return pd_krylov_n(c, 3, X.data(), coef.data(), (int)X.size(), 0.0, y, n, nullptr, false);
}

// out = T(g): last H blocks of P^{-1}(E_H g)   (g, out: replicated [H][Sg], out must not alias g)
pd_status tail_map(pd_ctx* c, const double* g, double* out) {
  auto& T = c->tail;
  const long long Sg = c->Sg, Hn = (long long)T.H * Sg;
  if (c->g.op == PD_WAVE2D_DIRICHLET) {  // every rank: S^-1 [sum_t tau_at . (S g_t S)] S^-1 on the whole head
    const int N = c->g.nx;
    const long long NN = (long long)N * N;
    double *G = T.dwork, *Ta = T.dwork + T.H * NN, *tmp = T.dwork + 2 * T.H * NN;
    PD_CUDA(c, pd_launch_dst2d_dense(g, G, tmp, T.dsin, N, T.H, c->st));
    const double sc = 2.0 / (N + 1);
    PD_CUDA(c, pd_launch_tau_combine(T.taud, G, Ta, N, T.H, sc * sc, c->st));
    PD_CUDA(c, pd_launch_dst2d_dense(Ta, out, tmp, T.dsin, N, T.H, c->st));
    c->launches += 4 * T.H + 1;
    return PD_OK;
  }
  if (c->g.op == PD_ADE2D_PERIODIC) {  // every rank: one slab FFT filter of the whole head
    PD_LAUNCH(c, pd_launch_r2c(g, T.work, Sg, c->st));
    PD_CUDA(c, pd_launch_slab2d_filter(T.work, c->g.nx, T.tau, c->tw_s, c->st));
    c->launches += 3;
    PD_LAUNCH(c, pd_launch_take_real(T.work, out, Sg, c->st));
    return PD_OK;
  }
  auto range = [&](int f0, int fc, double* dst) -> pd_status {
    const int G = std::max(1, std::min(fc, T.G));
    PD_LAUNCH(c, pd_launch_tail1d(g, T.part, G, c->g.nx, fc, T.H, c->tri + f0, T.hc + (long long)f0 * T.H,
                                  T.ow + (long long)f0 * T.H, c->st));
    PD_LAUNCH(c, pd_launch_reduce_rows(T.part, G, Hn, dst, c->st));
    return PD_OK;
  };
  if (c->dist_mode == 0) return range(0, c->F, out);
  if (c->dist_mode == 1) {  // this rank's frequencies, summed over the ranks
    pd_status s = range(c->plan.f_off[c->rank], c->plan.f_cnt[c->rank], out);
    return s != PD_OK ? s : allreduce(c, out, Hn);
  }
  // virtual ranks: the same split, summed on the device in shard order
  for (size_t i = 0; i < c->shards.size(); ++i) {
    const int f0 = c->plan.f_off[i], fc = c->plan.f_cnt[i];
    if (fc == 0) continue;
    pd_status s = range(f0, fc, i == 0 ? out : T.acc);
    if (s != PD_OK) return s;
    if (i > 0) {
      s = comb(c, {out, T.acc}, {1.0, 1.0}, out, Hn);
      if (s != PD_OK) return s;
    }
  }
  return PD_OK;
}

pd_status head_G(pd_ctx* c, const double* tail, double* head) {
  PD_LAUNCH(c, pd_launch_head_G(c->tail.gsten, c->tail.gc, tail, head, c->Sg, c->st));
  return PD_OK;
}

// true if any of x[0..n) is non-zero on any rank (syncs)
pd_status any_nonzero(pd_ctx* c, const double* x, long long n, bool* out) {
  auto& T = c->tail;
  PD_CUDA(c, cudaMemsetAsync(T.flag, 0, sizeof(int), c->st));
  PD_LAUNCH(c, pd_launch_any_nonzero(x, n, T.flag, c->st));
  PD_CUDA(c, cudaMemcpyAsync(T.hflag, T.flag, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  PD_CUDA(c, cudaStreamSynchronize(c->st));
  double v = *T.hflag != 0 ? 1.0 : 0.0;
  if (c->dist_mode == 1) {
    c->hred[0] = v;
    PD_CUDA(c, cudaMemcpyAsync(c->dred, c->hred, sizeof(double), cudaMemcpyHostToDevice, c->st));
    pd_status s = allreduce(c, c->dred, 1);
    if (s != PD_OK) return s;
    PD_CUDA(c, cudaMemcpyAsync(c->hred, c->dred, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    PD_CUDA(c, cudaStreamSynchronize(c->st));
    v = c->hred[0];
  }
  *out = v != 0.0;
  return PD_OK;
}

// dots of replicated vectors (no cross-rank sum)
pd_status dots(pd_ctx* c, std::vector<const double*> X, const double* y, long long n, double* out) {
  return pd_krylov_n(c, 0, X.data(), nullptr, (int)X.size(), 0.0, const_cast<double*>(y), n, out, false);
}

// u = P^{-1}(E_H g) (u += when acc), g replicated [H][Sg].  Single GPU: Step (a) of a head-only vector is the
// weighted broadcast sum_t hc[n][t] g_t (of the x-transformed head in the fused 2D layout), so the forward time FFT
// and the full-size right-hand side are skipped; sharded: the distributed apply of the embedded vector.
pd_status apply_head(pd_ctx* c, const double* g, double* u, int acc) {
  auto& T = c->tail;
  const long long n = (long long)c->nt * c->S;
  if (c->dist_mode != 0) {
    PD_CUDA(c, cudaMemsetAsync(c->rvec, 0, sizeof(double) * n, c->st));
    pd_status s = local_of(c, g, c->rvec);
    return s != PD_OK ? s : pd_apply_impl(c, c->rvec, u, acc);
  }
  const long long Hn = (long long)T.H * c->S;
  PD_LAUNCH(c, pd_launch_r2c(g, T.gx, Hn, c->st));
  if (c->use_tfx) PD_LAUNCH(c, pd_launch_slab2d_rows(T.gx, c->g.nx, (long long)T.H * c->g.ny, 0, c->tw_s, c->st));
  PD_LAUNCH(c, pd_launch_head_broadcast(c->Sh, c->F, c->S, T.H, T.hc, T.gx, c->st));
  pd_status s = pd_spatial_solve(c, c->Sh, c->F, 0);
  return s != PD_OK ? s : pd_time_fft_inv(c, pd_spec_local(c->Sh, c->S), u, c->S, acc);
}

pd_status zero_report(pd_ctx* c, double* u, pd_report* rep) {
  PD_CUDA(c, cudaMemsetAsync(u, 0, sizeof(double) * c->nt * c->S, c->st));
  if (rep) *rep = pd_report{0, 1, 0.0, 0.0, rep->history, rep->history_cap, 0};
  return PD_OK;
}

#define PD_TRY(expr)              \
  do {                            \
    pd_status s_ = (expr);        \
    if (s_ != PD_OK) return s_;   \
  } while (0)

}  // namespace

void pd_tail_free(pd_ctx* c) {
  auto& T = c->tail;
  for (void* p : {(void*)T.hc, (void*)T.ow, (void*)T.part, (void*)T.tau, (void*)T.work, (void*)T.flag, (void*)T.acc,
                  (void*)T.gx, (void*)T.taud, (void*)T.dsin, (void*)T.dwork})
    if (p) cudaFree(p);
  for (double* p : T.scr) cudaFree(p);
  for (double* p : T.Vh) cudaFree(p);
  if (T.hflag) cudaFreeHost(T.hflag);
  T = pd_ctx::TailState{};
}

extern "C" {

pd_status pd_tail_map(pd_ctx* c, const double* head, double* tail) {
  if (!c || !head || !tail) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  PD_TRY(tail_setup(c));
  if (c->dist_mode != 1) return tail_map(c, head, tail);
  // NCCL ranks: local head slab in, local tail slab out
  auto& T = c->tail;
  PD_TRY(gather_full(c, head, T.scr[8]));
  PD_TRY(tail_map(c, T.scr[8], T.scr[9]));
  return local_of(c, T.scr[9], tail);
}

pd_status pd_solve_stationary_tail(pd_ctx* c, const double* b, double* u, double tol, int maxit, pd_report* rep) {
  if (!c || !b || !u) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  if (!(tol > 0) || maxit < 0) return fail(c, PD_EINVAL, "tol must be > 0, maxit >= 0");
  PD_TRY(tail_setup(c));
  const auto t0 = std::chrono::steady_clock::now();
  if (rep) rep->history_len = 0;
  auto& T = c->tail;
  const long long n = (long long)c->nt * c->S, Hn = hs(c), Hl = (long long)T.H * c->S;
  double bb = 0;
  PD_TRY(pd_krylov_n(c, 0, &b, nullptr, 1, 0.0, const_cast<double*>(b), n, &bb));
  const double bnorm = std::sqrt(bb);
  if (bnorm == 0.0) return zero_report(c, u, rep);
  bool u_nz = true;
  PD_TRY(any_nonzero(c, u, n, &u_nz));
  double rr = bb;  // zero initial guess: r^0 = b
  if (u_nz) PD_TRY(pd_stencil_impl(c, b, u, c->rvec, &rr));  // r^0 = b - A u^0
  double rel = std::sqrt(rr) / bnorm;
  int k = 0;
  if (rel > tol && maxit > 0) {
    double *tp = T.scr[0], *tc = T.scr[1], *yt = T.scr[2], *hd = T.scr[3], *dd = T.scr[4], *bh = T.scr[5];
    const long long tail_off = (long long)(c->nt - T.H) * c->S;
    if (u_nz)
      PD_TRY(gather_full(c, u + tail_off, tp));  // t^0
    else
      PD_CUDA(c, cudaMemsetAsync(tp, 0, sizeof(double) * Hn, c->st));
    bool nonhead = true;
    PD_TRY(any_nonzero(c, b + Hl, n - Hl, &nonhead));
    if (nonhead) {
      PD_TRY(pd_apply_impl(c, b, u, 0));  // u = y = P^{-1} b
      PD_TRY(gather_full(c, u + tail_off, yt));
    } else {
      PD_TRY(gather_full(c, b, bh));
      PD_TRY(tail_map(c, bh, yt));  // b supported on the head: tail(P^{-1} b) = T(b_head)
    }
    for (;;) {
      PD_TRY(head_G(c, tp, hd));
      PD_TRY(tail_map(c, hd, tc));
      PD_TRY(comb(c, {tc, yt}, {1.0, 1.0}, tc, Hn));  // t^{k+1} = y_tail + T(G t^k)
      ++k;
      PD_TRY(comb(c, {tc, tp}, {1.0, -1.0}, dd, Hn));
      PD_TRY(head_G(c, dd, hd));  // r^{k+1} = E_H G (t^{k+1} - t^k)
      double h2 = 0;
      PD_TRY(dots(c, {hd}, hd, Hn, &h2));
      rel = std::sqrt(h2) / bnorm;
      pd_report_push(rep, rel);
      if (rel <= tol || k >= maxit) break;
      std::swap(tp, tc);
    }
    // u^k = P^{-1}(b + E_H G t^{k-1})
    PD_TRY(head_G(c, tp, hd));
    if (nonhead) {
      PD_TRY(apply_head(c, hd, u, 1));  // u = y + P^{-1}(E_H G t^{k-1})
    } else {
      PD_TRY(comb(c, {bh, hd}, {1.0, 1.0}, hd, Hn));
      PD_TRY(apply_head(c, hd, u, 0));
    }
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

pd_status pd_solve_gmres_tail(pd_ctx* c, const double* b, double* u, double tol, int m, int maxit, pd_report* rep) {
  if (!c || !b || !u) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  if (!(tol > 0) || maxit < 0 || m < 1 || m > 30) return fail(c, PD_EINVAL, "need tol > 0, maxit >= 0, 1 <= m <= 30");
  PD_TRY(tail_setup(c));
  const auto t0 = std::chrono::steady_clock::now();
  if (rep) rep->history_len = 0;
  auto& T = c->tail;
  const long long n = (long long)c->nt * c->S, Hn = hs(c), Hl = (long long)T.H * c->S;
  const long long tail_off = (long long)(c->nt - T.H) * c->S;
  if ((int)T.Vh.size() < m + 1) {
    for (double* p : T.Vh) cudaFree(p);
    T.Vh.assign(m + 1, nullptr);
    for (auto& p : T.Vh) PD_CUDA(c, dalloc_d(&p, (size_t)Hn));
  }
  if (!c->zvec) PD_CUDA(c, dalloc_d(&c->zvec, (size_t)n));
  double bb = 0;
  PD_TRY(pd_krylov_n(c, 0, &b, nullptr, 1, 0.0, const_cast<double*>(b), n, &bb));
  const double bnorm = std::sqrt(bb);
  if (bnorm == 0.0) return zero_report(c, u, rep);
  bool u_nz = true;
  PD_TRY(any_nonzero(c, u, n, &u_nz));
  double rr = bb;
  const double* anchor = b;  // zero initial guess: r0 = b, read in place
  if (u_nz) {
    PD_TRY(pd_stencil_impl(c, b, u, c->rvec, &rr));  // anchor r0 = b - A u0 (kept in rvec)
    anchor = c->rvec;
  }
  double beta = std::sqrt(rr);
  int its = 0;
  bool conv = beta <= tol * bnorm, breakdown = false;
  double *q0 = T.scr[0], *tq = T.scr[1], *gt = T.scr[2], *w = T.scr[3], *ch = T.scr[4], *r0h = T.scr[5];
  std::vector<double> H((m + 1) * m), cs(m), sn(m), gv(m + 1), y(m), A(m + 1), Sd(m + 1), d(m + 2), d2(m + 2);
  auto Hs = [&](int i, int j) -> double& { return H[i * m + j]; };
  while (!conv && its < maxit) {
    bool nonhead = true;
    PD_TRY(gather_full(c, anchor, r0h));  // replicated head of the anchor
    PD_TRY(any_nonzero(c, anchor + Hl, n - Hl, &nonhead));
    if (nonhead) {
      if (anchor != c->rvec) {  // the final right-hand side scales the anchor in place
        PD_CUDA(c, cudaMemcpyAsync(c->rvec, anchor, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->st));
        anchor = c->rvec;
      }
      PD_TRY(pd_apply_impl(c, c->rvec, c->zvec, 0));  // q0 = G tail(P^{-1} r0)
      PD_TRY(gather_full(c, c->zvec + tail_off, tq));
      PD_TRY(head_G(c, tq, q0));
      A[0] = 1.0 / beta;
      PD_CUDA(c, cudaMemsetAsync(T.Vh[0], 0, sizeof(double) * Hn, c->st));
      Sd[0] = 0.0;
    } else {
      A[0] = 0.0;  // anchor supported on the head: carry it in h
      PD_TRY(comb(c, {r0h}, {1.0 / beta}, T.Vh[0], Hn));
      Sd[0] = beta;  // <h_0, r0h> = ||r0||^2 / beta
    }
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int kk = 0;
    for (int j = 0; j < m; ++j) {
      // w = A P^{-1} v_j = (a_j, h_j - G T(h_j) - a_j q0)
      PD_TRY(tail_map(c, T.Vh[j], tq));
      PD_TRY(head_G(c, tq, gt));
      if (nonhead)
        PD_TRY(comb(c, {T.Vh[j], gt, q0}, {1.0, -1.0, -A[j]}, w, Hn));
      else
        PD_TRY(comb(c, {T.Vh[j], gt}, {1.0, -1.0}, w, Hn));
      double wa = A[j];
      ++its;
      // CGS2 in the (a, h) representation: <x, y> = xa ya rr + xa <r0h, yh> + ya <xh, r0h> + <xh, yh>
      std::vector<const double*> X(T.Vh.begin(), T.Vh.begin() + j + 1);
      X.push_back(r0h);
      std::vector<double> hsum(j + 1, 0.0);
      PD_TRY(dots(c, X, w, Hn, d.data()));
      for (int pass = 0; pass < 2; ++pass) {
        const double e = d[j + 1];  // <r0h, w>
        std::vector<double> coef(j + 2, 0.0);
        double da = 0.0;
        for (int i = 0; i <= j; ++i) {
          const double hij = wa * A[i] * rr + wa * Sd[i] + A[i] * e + d[i];
          hsum[i] += hij;
          coef[i] = -hij;
          da += hij * A[i];
        }
        wa -= da;
        // w <- w - sum h_i h_i-vectors; partial dots of the updated w with X (next pass / norm)
        PD_TRY(pd_krylov_n(c, 1, X.data(), coef.data(), j + 2, 1.0, w, Hn, d.data(), false));
      }
      double ww = 0;
      PD_TRY(dots(c, {w}, w, Hn, &ww));
      const double e = d[j + 1];
      const double hn = std::sqrt(std::max(0.0, wa * wa * rr + 2.0 * wa * e + ww));
      for (int i = 0; i <= j; ++i) Hs(i, j) = hsum[i];
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
      if (std::fabs(gv[j + 1]) <= tol * bnorm || its >= maxit) break;
      if (hn == 0.0) {
        breakdown = true;
        break;
      }
      PD_TRY(comb(c, {w}, {1.0 / hn}, T.Vh[j + 1], Hn));
      A[j + 1] = wa / hn;
      Sd[j + 1] = e / hn;
    }
    for (int i = kk - 1; i >= 0; --i) {
      double t = gv[i];
      for (int l = i + 1; l < kk; ++l) t -= Hs(i, l) * y[l];
      y[i] = t / Hs(i, i);
    }
    double ca = 0.0;
    for (int i = 0; i < kk; ++i) ca += y[i] * A[i];
    std::vector<const double*> Xc(T.Vh.begin(), T.Vh.begin() + kk);
    PD_TRY(comb(c, Xc, std::vector<double>(y.begin(), y.begin() + kk), ch, Hn));
    if (!nonhead) {
      // anchor supported on the head: u += P^{-1}(E_H (ca r0h + ch)) without a full-size right-hand side
      PD_TRY(comb(c, {r0h, ch}, {ca, 1.0}, ch, Hn));
      PD_TRY(apply_head(c, ch, u, 1));
    } else {
      // u += P^{-1}(ca r0 + E_H ch): the anchor buffer becomes the right-hand side (this rank's part of ch)
      PD_LAUNCH(c, pd_launch_axpby(c->rvec, c->rvec, ca, 0.0, n, c->st));
      PD_TRY(local_of(c, ch, gt));
      PD_TRY(comb(c, {c->rvec, gt}, {1.0, 1.0}, c->rvec, Hl));
      PD_TRY(pd_apply_impl(c, c->rvec, u, 1));
    }
    PD_TRY(pd_stencil_impl(c, b, u, c->rvec, &rr));  // true residual; the next cycle's anchor
    anchor = c->rvec;
    beta = std::sqrt(rr);
    conv = beta <= tol * bnorm;
    if (breakdown) break;
  }
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

}  // extern "C"
