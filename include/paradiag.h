/*
 * paradiag.h — C ABI of the B200 ParaDiag-II hot path (arXiv 2005.09158).
 *
 * What it computes (P:l.N = /root/reference/PAPER.md line N):
 *   all-at-once system      A = B1 (x) M + B2 (x) K              (P:l.80-84, eq 1.1), M = I (P:l.74-76)
 *   preconditioner          P_alpha = C1 (x) M + C2 (x) K         (P:l.114-116, eq 1.2; corners eq 2.11b, 3.4)
 *   apply z = P_alpha^{-1} r in three steps                       (P:l.179-185 eq 1.3; P:l.813-819 eq 2.12)
 *     (a) S1 = (F (x) I)(Gamma_alpha (x) I) r       time FFT of every spatial dof, Gamma fused
 *     (b) S2_n = (lambda_{1,n} I + lambda_{2,n} K)^{-1} S1_n     batched complex-shifted spatial solves
 *     (c) z = (Gamma_alpha^{-1} (x) I)(F^* (x) I) S2             inverse time FFT, Gamma^{-1} fused
 *   residual r = b - A u                                          (P:l.1563-1565, eq 5.1)
 *   stationary iteration u <- u + P_alpha^{-1}(b - A u)           (P:l.120-124, eq 5.1)
 *   right-preconditioned GMRES(m) on A P_alpha^{-1}               (P:l.125-132; stop rule P:l.1315-1317)
 *
 * Vectors.  Unless a function says HOST, every vector argument is a DEVICE pointer to fp64 data owned
 * by the caller, laid out time-major: 1D [Nt][Nx], 2D [Nt][Ny][Nx] with x fastest; block n holds time
 * level t_{n+1} = (n+1) dt (U_1 .. U_Nt of eq 1.1).  Work is enqueued on the context's CUDA stream
 * (pd_setup argument); calls return once the work is enqueued unless stated otherwise.
 *
 * Errors.  Every entry point returns a pd_status and never aborts or throws across the ABI.
 * pd_last_error() returns a description of the last failure on that context (or of the last failed
 * pd_setup when given NULL).
 *
 * Threading.  One context per (device, stream); a context is not reentrant.
 */
#ifndef PARADIAG_H
#define PARADIAG_H

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define PD_API __attribute__((visibility("default")))
#else
#define PD_API
#endif

typedef struct pd_ctx pd_ctx; /* opaque: owns workspace, tables, streams, NCCL communicator */

typedef enum {
  PD_OK = 0,
  PD_NOT_CONVERGED = 1, /* non-fatal: maxit exhausted, report filled, last iterate in u */
  PD_EINVAL = -1,       /* bad argument (alpha outside (0,1], Nt not a power of two, ...) */
  PD_ESINGULAR = -2,    /* a shifted system lambda_1 I + lambda_2 K is singular (message names n) */
  PD_ECUDA = -3,        /* a CUDA runtime error (message holds cudaGetErrorString) */
  PD_ENCCL = -4,        /* an NCCL error (multi-GPU) */
  PD_ENOMEM = -5,       /* device allocation failed */
  PD_EBREAKDOWN = -6    /* GMRES breakdown above tolerance */
} pd_status;

typedef enum { PD_BE = 0, PD_CN = 1, PD_LEAPFROG = 2 } pd_scheme;

typedef enum {
  PD_ADE1D_DIRICHLET = 0,  /* u_t = nu u_xx - ax u_x on (0,L), u=0 at both ends, Nx interior nodes, h = L/(Nx+1) */
  PD_WAVE1D_DIRICHLET = 1, /* u_tt = nu u_xx on (0,L), Dirichlet (nu = c^2; use PD_LEAPFROG)                  */
  PD_ADE2D_PERIODIC = 2,   /* u_t = nu Lap u - (ax, ay).grad u on [0,L)^2 periodic, N x N, h = L/N (5-point)  */
  PD_WAVE2D_DIRICHLET = 3  /* u_tt = nu Lap u on (0,L)^2, u = 0 on the boundary, N x N interior nodes,
                              h = L/(N+1), N + 1 a power of two in [16, 512]; ax = ay = 0 (Table T4A,
                              P:l.1309-1349; use PD_LEAPFROG).  Step (b) by the tensor DST-I (exact). */
} pd_operator;

typedef struct {
  pd_operator op;
  int nx, ny;       /* 1D: nx = Nx, ny = 1.  2D: nx = ny = N (periodic: power of two; Dirichlet: 2^k - 1) */
  double length;    /* domain length L (1 for the 1D configs, 2*pi for the 2D configs) */
  double nu, ax, ay;
} pd_grid;

/* Distribution: rank p owns the spatial slab of pd_partition() for all Nt levels (1D: an
 * x-range, 2D: a range of y-rows); Step (b) runs on frequency shards after an all-to-all over NCCL.
 *   size == 1              single GPU (rank must be 0, nccl_id ignored)
 *   size > 1, rank >= 0    NCCL rank `rank` of `size`; vectors passed to the context are the LOCAL slab
 *                          [Nt][S_local] (pd_local_shape).  Communicator: nccl_comm when non-NULL (an existing
 *                          ncclComm_t of exactly these ranks, e.g. torch's ProcessGroupNCCL._comm_ptr(); borrowed,
 *                          never destroyed by the library), else a new one from nccl_id (pd_nccl_unique_id on one
 *                          rank, shared by all; owned and destroyed by pd_destroy)
 *   size > 1, rank < 0     `size` virtual ranks inside this process on one GPU: vectors are GLOBAL, every
 *                          exchange of the plan is executed with device copies (test mode of the sharded
 *                          path; same plan, partition and kernels as the NCCL mode) */
typedef struct {
  int rank, size;
  const void* nccl_id;          /* 128-byte ncclUniqueId shared by all ranks (used when nccl_comm is NULL) */
  void* nccl_comm;              /* borrowed ncclComm_t of the caller's process group, or NULL */
} pd_dist;

typedef struct {
  int iterations;       /* P_alpha^{-1} applications inside the loop (GMRES final assembly not counted) */
  int converged;        /* 1 if ||b - A u|| <= tol ||b|| at exit */
  double rel_residual;  /* true ||b - A u||_2 / ||b||_2 at exit */
  double wall_ms;       /* host wall time of the call */
  double* history;      /* HOST, caller-owned, capacity history_cap (may be NULL): per-iteration relative
                           residuals (true residual for stationary, Arnoldi estimate for GMRES) */
  int history_cap;
  int history_len;
} pd_report;

/* Create a context: validate, build the spectra lambda_{1,n}, lambda_{2,n} (Lemma 1, P:l.155-174; closed
 * forms DESIGN.md §3), Gamma tables, twiddles; allocate the workspace; check every shifted system for
 * singularity.  alpha in (0,1]; Nt a power of two in [1, 8192] (>= 4 for PD_LEAPFROG; Nt = 1 is one plain solve
 * (c1 I + c2 K) z = r, S:l.89, reading t2); dt > 0.
 * cuda_stream: a cudaStream_t (NULL = legacy default stream).  dist may be NULL (single GPU).
 * For Nt >= 1024 the context also owns up to three internal non-blocking streams and their scratch chunks (the time-FFT
 * chunk pipeline); every call still behaves as if ordered on cuda_stream (event fork / join).
 * Tuning environment (read here, at setup): PD_TF4_OVERLAP / PD_TF4_OVERLAP_INV (streams of the forward /
 * inverse time FFT, default 3 / 4), PD_TF4_CHUNK_MB, PD_GRAPH (CUDA-graph replay of the apply: unset = for Nt * S <= 2^21
 * from the second use of an (r, z) pair, 1 = always, 0 = never; a replay bakes in the pointers and the launch path of
 * the capture).  Read per call (A/B switches of measured alternatives; the defaults are the measured
 * best): PD_GMRES_NO_LAZY, PD_GMRES_NO_Z, PD_GMRES_MATVEC (GMRES variants), PD_DST_FULL, PD_DST_CHUNK_MB (2D Dirichlet
 * x-DST rows), PD_TFX_PERSIST, PD_TFX_LAG (persistent fused time FFT; experimental: its scratch ring is one per
 * process and device, so run one context at a time with it).
 * Returns PD_EINVAL / PD_ESINGULAR / PD_ENOMEM / PD_ECUDA / PD_ENCCL on failure (*out = NULL). */
PD_API pd_status pd_setup(const pd_grid* g, double dt, int nt, double alpha, pd_scheme s, const pd_dist* dist,
                   void* cuda_stream, pd_ctx** out);
PD_API void pd_destroy(pd_ctx* ctx);
PD_API const char* pd_last_error(const pd_ctx* ctx);

/* The 128-byte NCCL unique id for a multi-GPU setup (rank 0 creates it and broadcasts it). */
PD_API pd_status pd_nccl_unique_id(void* out128);

/* Partition plan (pure host, no GPU): for each of `size` ranks the spatial slab [s_off, s_off + s_cnt) in
 * dofs and the half-spectrum frequency range [f_off, f_off + f_cnt).  Arrays of length size (nullable). */
PD_API pd_status pd_partition(int op, int nx, int ny, int nt, int size, long long* s_off, long long* s_cnt,
                              int* f_off, int* f_cnt);

/* Local slab of this rank: 1D x-range [offset, offset+nx_local), 2D y-rows [offset/nx, ...). */
PD_API pd_status pd_local_shape(const pd_ctx* ctx, int* nx_local, int* ny_local, long long* offset);
/* Elements of one local all-at-once vector (Nt * local spatial dofs). */
PD_API long long pd_local_size(const pd_ctx* ctx);

/* Copy the spectra (numpy convention, n = 0..Nt-1) to HOST arrays lam1[2*Nt], lam2[2*Nt] (re, im). */
PD_API pd_status pd_spectra(const pd_ctx* ctx, double* lam1_host, double* lam2_host);

/* z = P_alpha^{-1} r (Steps (a)-(c)).  r, z: device [Nt][local spatial dofs]; r == z allowed. */
PD_API pd_status pd_apply_precond(pd_ctx* ctx, const double* r, double* z);

/* r = b - A u (all three device vectors; r may alias neither b nor u).  If rnorm2_host != NULL the call
 * synchronises the stream and stores ||r||_2^2 (deterministic fixed-order reduction). */
PD_API pd_status pd_residual(pd_ctx* ctx, const double* b, const double* u, double* r, double* rnorm2_host);
/* w = A u. */
PD_API pd_status pd_matvec(pd_ctx* ctx, const double* u, double* w);

/* b of A u = b from the initial data and the source (DESIGN.md §3 readings c4, c5):
 *   u0, v0: device [local spatial dofs] (v0 may be NULL = 0; used by PD_LEAPFROG only)
 *   f: device [(Nt+1)][local spatial dofs] sampled at t_n = n dt, n = 0..Nt, or NULL for f = 0. */
PD_API pd_status pd_build_rhs(pd_ctx* ctx, const double* u0, const double* v0, const double* f, double* b);

/* Stationary ParaDiag-II iteration (eq 5.1) from the initial guess in u until ||b-Au|| <= tol ||b||. */
PD_API pd_status pd_solve_stationary(pd_ctx* ctx, const double* b, double* u, double tol, int maxit, pd_report* rep);
/* Right-preconditioned restarted GMRES(m), CGS2 orthogonalisation, deterministic reductions.
 * Workspace for the basis ((m+1) vectors) is allocated on first use and kept by the context. */
PD_API pd_status pd_solve_gmres(pd_ctx* ctx, const double* b, double* u, double tol, int m, int maxit, pd_report* rep);
/* Either solver with flags: solver 0 stationary, 1 GMRES, OR-ed with PD_SOLVE_ZERO_GUESS = start from u = 0 with u
 * output only (not read, may hold anything on entry: GMRES then skips the zero-guess check sweep and writes the
 * first cycle's update instead of adding it).  Otherwise identical to pd_solve_stationary / pd_solve_gmres. */
PD_API pd_status pd_solve(pd_ctx* ctx, int solver, const double* b, double* u, double tol, int m, int maxit,
                          pd_report* rep);

/* ---- waveform-relaxation tail form (oracle/tail.py) ----
 * P_alpha - A is non-zero only between the first H time blocks (rows) and the last H blocks (columns),
 * H = 1 for PD_BE / PD_CN and 2 for PD_LEAPFROG (alpha-corner of eq 1.2, P:l.80-84), so the iterations can
 * carry only the "tail" of u between iterations (head-tail coupling of WR, P:l.762-773; economical Step (a),
 * P:l.928-931).  Same iterates, iteration counts and stopping rule (||b - A u|| <= tol ||b||) as the
 * residual-form solvers above; per iteration the work is the tail map below plus O(H S) vector operations
 * instead of full passes over Nt x S.  Sharded contexts (NCCL or virtual ranks) replicate the H head / tail blocks
 * on every rank: the 1D tail map splits its frequencies over the ranks and all-reduces the H x S tail, the 2D one
 * runs replicated (tailform.cpp).  PD_EINVAL when Nt < 2H, and for 1D contexts whose Step (b) uses the pivoted
 * fallback (the tail map needs the recurrence solver).  Per-context tables (1D: F x H coefficients; 2D periodic: the
 * N x N transfer function tau, F N^2 divisions; 2D Dirichlet: H x H real transfer tables in the DST-I basis and the
 * N x N sine table, the map then being two dense 2D DSTs per head block) are built on the first call and kept.
 *
 * pd_tail_map: tail = last H blocks of P_alpha^{-1} (E_H head), head and tail device [H][local dofs]
 *   (must not alias).  Economical Step (a), Step (b) for every frequency, last H rows of Step (c). */
PD_API pd_status pd_tail_map(pd_ctx* ctx, const double* head, double* tail);
/* Stationary iteration (eq 5.1) in tail form; u: initial guess in, solution out (device [Nt][S]).
 * rep->rel_residual = ||G (t^k - t^{k-1})|| / ||b|| = ||b - A u^k|| / ||b|| (P - A only touches the head). */
PD_API pd_status pd_solve_stationary_tail(pd_ctx* ctx, const double* b, double* u, double tol, int maxit, pd_report* rep);
/* Right-preconditioned restarted GMRES(m) in tail form: basis vectors a_j r0 + E_H h_j (a_j host, h_j device).
 * Reports the true residual of the returned u (recomputed by the stencil at exit, as pd_solve_gmres). */
PD_API pd_status pd_solve_gmres_tail(pd_ctx* ctx, const double* b, double* u, double tol, int m, int maxit, pd_report* rep);

/* ---- nonlinear problems by simplified Newton (eq 1.4-1.5, P:l.196-227; oracle/nonlinear.py) ----
 * pd_set_reaction: M U' + f(U) = 0 with f(U) = K U + g(U), g(u) = g3 u^3 + g1 u pointwise.  Afterwards pd_residual,
 *   pd_matvec and pd_build_rhs are those of the nonlinear all-at-once system (B1 (x) I) u + (B2 (x) I) F(u) = b
 *   (b_1 = U_0/dt - (1-theta) f(U_0)); (0, 0) restores the linear problem.  1D operators, PD_BE / PD_CN only
 *   (PD_EINVAL otherwise).
 * pd_solve_newton: u^{k+1} = u^k + P_alpha(u^k)^{-1} (b - (B1 u^k + B2 F(u^k))) with
 *   P_alpha(u) = C1 (x) I + C2 (x) (K + diag((1/Nt) sum_n g'(U_n))) (the averaged Jacobian of P:l.214-216; its
 *   shifted systems are tridiagonal but not Toeplitz: Thomas per frequency), until ||r|| <= tol ||b||.
 *   u: initial guess in, solution out.  Single-GPU 1D theta-method contexts only. */
PD_API pd_status pd_set_reaction(pd_ctx* ctx, double g3, double g1);
PD_API pd_status pd_solve_newton(pd_ctx* ctx, const double* b, double* u, double tol, int maxit, pd_report* rep);

/* HOST-buffer variants for end-to-end use: copy the HOST input(s) to device workspace on the context
 * stream (pinned memory recommended), run, copy the HOST output back, synchronise.  Every HOST vector holds
 * exactly Nt * (local spatial dofs) doubles (pd_local_size); the library cannot check host extents, so a shorter
 * buffer is an out-of-bounds access (the Python binding checks dtype, device, contiguity and element count).
 * pd_solve_host: solver 0 stationary, 1 GMRES; OR-ing PD_SOLVE_ZERO_GUESS starts from u = 0 without copying
 * u_host in (u_host is then output only: one host->device copy per solve instead of two).  Any other solver code
 * is PD_EINVAL. */
#define PD_SOLVE_ZERO_GUESS 16
PD_API pd_status pd_apply_precond_host(pd_ctx* ctx, const double* r_host, double* z_host);
PD_API pd_status pd_solve_host(pd_ctx* ctx, int solver /*0 stationary, 1 gmres*/, const double* b_host,
                        double* u_host, double tol, int m, int maxit, pd_report* rep);

/* End-to-end solve of the initial-value problem from HOST initial data: copy u0 [S] (v0 [S] for leapfrog, may
 * be NULL = 0; f [(Nt+1)][S] sampled at t_n = n dt, may be NULL = 0) to the device, build b there
 * (pd_build_rhs), solve from u = 0, copy the space-time solution [Nt][S] to u_host, synchronise.
 * solver: 0 stationary, 1 GMRES, 2 stationary tail form, 3 GMRES tail form, 4 simplified Newton (needs
 * pd_set_reaction).  Host->device traffic is the initial data only. */
PD_API pd_status pd_solve_ivp_host(pd_ctx* ctx, int solver, const double* u0_host, const double* v0_host,
                                   const double* f_host, double* u_host, double tol, int m, int maxit, pd_report* rep);

/* Number of kernels this context has launched so far (for the bench's gpu_launches claim). */
PD_API long long pd_kernel_launches(const pd_ctx* ctx);

/* Per-kernel timing: when enabled, the library records CUDA events on the context stream around every
 * kernel of the path, without host synchronisation, and pd_phase_times (which synchronises) returns the
 * accumulated device milliseconds and launch counts per slot:
 *   0 Step (a) time FFT, 1 Step (b) spatial solve, 2 Step (c) inverse time FFT, 3 residual b - A u,
 *   4 Step (c) fused with the update u += z, 5 matvec A u, 6 Krylov sweeps (and the GMRES final update whose
 *   combination the forward time FFT reads), 7 norm-only residual ||b - A u|| (no vector written; GMRES cycle ends).
 *   ms8, count8: HOST arrays of 8. */
PD_API pd_status pd_enable_phase_timing(pd_ctx* ctx, int enable);
PD_API pd_status pd_phase_times(pd_ctx* ctx, double* ms8, long long* count8);

#ifdef __cplusplus
}
#endif
#endif /* PARADIAG_H */
