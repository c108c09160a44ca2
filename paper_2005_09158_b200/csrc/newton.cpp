// Nonlinear ParaDiag-II by simplified Newton (eq 1.4-1.5, P:l.196-227; oracle/nonlinear.py).
//   pd_set_reaction: F(u) = K u + g(u), g(u) = g3 u^3 + g1 u pointwise; from then on pd_residual / pd_matvec /
//   pd_build_rhs are those of the nonlinear all-at-once system eq 1.4 (1D operators, theta-method).
//   pd_solve_newton: r = b - ((B1 (x) I) u + (B2 (x) I) F(u));  dbar = time average of g'(U_n);
//   du = P_alpha(u)^{-1} r with J = K + diag(dbar) (Steps (a), (b) by pivoted elimination per frequency (gtsv.cu),
//   (c) fused with u += du); stop when ||r|| <= tol ||b||.  A zero / non-finite pivot in Step (b) (a singular
//   averaged-Jacobian system, or a diverging iterate) ends the solve with PD_ESINGULAR naming the frequency.
#include <chrono>
#include <cmath>

#include "ctx.h"

extern "C" {

pd_status pd_set_reaction(pd_ctx* c, double g3, double g1) {
  if (!c) return PD_EINVAL;
  if (pd_is_2d(c->g.op) || c->scheme == PD_LEAPFROG)
    return fail(c, PD_EINVAL, "reaction terms: 1D operators with the theta-method only");
  c->sten.g3 = g3;
  c->sten.g1 = g1;
  for (auto& gr : c->graphs)
    if (gr.exec) cudaGraphExecDestroy(gr.exec);  // captured applies baked in the old operator
  c->graphs.clear();
  return PD_OK;
}

pd_status pd_solve_newton(pd_ctx* c, const double* b, double* u, double tol, int maxit, pd_report* rep) {
  if (!c || !b || !u) return c ? fail(c, PD_EINVAL, "null vector") : PD_EINVAL;
  if (!(tol > 0) || maxit < 0) return fail(c, PD_EINVAL, "tol must be > 0, maxit >= 0");
  if (c->dist_mode != 0 || pd_is_2d(c->g.op) || c->scheme == PD_LEAPFROG)
    return fail(c, PD_EINVAL, "simplified Newton: single-GPU 1D theta-method contexts only");
  const auto t0 = std::chrono::steady_clock::now();
  if (rep) rep->history_len = 0;
  const long long n = (long long)c->nt * c->S;
  if (!c->nl_dbar) PD_CUDA(c, cudaMalloc(reinterpret_cast<void**>(&c->nl_dbar), sizeof(double) * (c->S + 2)));
  if (pd_status e = pd_gtsv_ensure(c); e != PD_OK) return e;
  PD_CUDA(c, cudaMemsetAsync(c->gtsv_bad, 0, sizeof(int), c->st));
  double bb = 0;
  pd_status s = pd_krylov_n(c, 0, &b, nullptr, 1, 0.0, const_cast<double*>(b), n, &bb);
  if (s != PD_OK) return s;
  const double bnorm = std::sqrt(bb);
  if (bnorm == 0.0) {
    PD_CUDA(c, cudaMemsetAsync(u, 0, sizeof(double) * n, c->st));
    if (rep) *rep = pd_report{0, 1, 0.0, 0.0, rep->history, rep->history_cap, 0};
    return PD_OK;
  }
  int k = 0;
  double rel = 0;
  for (;;) {
    double rr = 0;
    s = pd_stencil_impl(c, b, u, c->rvec, &rr);  // r = b - (B1 u + B2 F(u))  (eq 1.5 right-hand side)
    if (s != PD_OK) return s;
    rel = std::sqrt(rr) / bnorm;
    if (k > 0) {  // the previous Step (b)'s pivot flag (the residual's norm read above synchronised the stream)
      PD_CUDA(c, cudaMemcpy(c->gtsv_hbad, c->gtsv_bad, sizeof(int), cudaMemcpyDeviceToHost));
      if (*c->gtsv_hbad)
        return fail(c, PD_ESINGULAR, "Newton iteration %d: shifted system lambda1 I + lambda2 (K + diag(dbar)) has a "
                    "zero or non-finite pivot at frequency n=%d", k, *c->gtsv_hbad - 1);
      pd_report_push(rep, rel);
    }
    if (rel <= tol || k >= maxit) break;
    PD_LAUNCH(c, pd_launch_jac_avg(u, c->nl_dbar, c->nt, c->S, c->sten.g3, c->sten.g1, c->st));
    s = pd_time_fft_fwd(c, c->rvec, pd_spec_local(c->Sh, c->S), c->S);  // Step (a)
    if (s != PD_OK) return s;
    PD_LAUNCH(c, pd_launch_gtsv_shift(c->Sh, c->g.nx, c->F, c->lam1, c->lam2, c->sten.sub, c->sten.dia, c->sten.sup,
                                      c->nl_dbar, c->gtsv_scratch, c->gtsv_bad, c->st));  // Step (b), J = K + diag(dbar)
    s = pd_time_fft_inv(c, pd_spec_local(c->Sh, c->S), u, c->S, 1);  // Step (c) fused with u += du
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

}  // extern "C"
