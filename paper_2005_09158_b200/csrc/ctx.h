// Context of the ParaDiag-II library (shared by paradiag.cpp and dist.cpp; not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include <complex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/paradiag.h"
#include "comm.h"
#include "kernels.h"

// partition plan: spatial slabs (1D x-ranges, 2D y-row ranges, in dofs) and frequency ranges per rank
inline bool pd_is_2d(int op) { return op == PD_ADE2D_PERIODIC || op == PD_WAVE2D_DIRICHLET; }

struct pd_plan {
  int P = 1;
  std::vector<long long> s_off, s_cnt;  // spatial dofs
  std::vector<int> f_off, f_cnt;        // half-spectrum frequencies
  std::vector<int> e_off, e_cnt;        // extent units (1D: x, 2D: y rows)
};
pd_plan pd_make_plan(int op, int nx, int ny, int nt, int P);

// per-rank state of the sharded path
struct pd_shard {
  int rank = 0;
  long long S = 0, off = 0;   // local spatial dofs and first global dof
  int ext = 0, ext_off = 0;   // local extent (1D: x points, 2D: y rows) and its global start
  int F = 0, f0 = 0;          // local frequencies
  double2* Sh_loc = nullptr;  // [F_all][S]  all frequencies of the local slab
  double2* Sg = nullptr;      // [F][S_glob] local frequencies of every spatial dof
  double2* stage = nullptr;   // NCCL receive/send staging (fallback exchange when peer mappings are unavailable)
  double2* peer[kPdMaxRanks] = {};  // NCCL ranks with P2P: rank q's Sg mapped into this process (CUDA IPC)
  double* hlo = nullptr;      // halos [Nt][hw]
  double* hhi = nullptr;
  double* h1lo = nullptr;     // single-level halos for the rhs (u0, v0): [2][hw]
  double* h1hi = nullptr;
  double* sendlo = nullptr;   // NCCL halo send buffers [Nt][hw]
  double* sendhi = nullptr;
  double* r_loc = nullptr;    // mode 2: local copies of in/out vectors [Nt][S]
  double* z_loc = nullptr;
  double* b_loc = nullptr;
  pd_stencil sten{};          // local stencil parameters
};

struct pd_ctx {
  // problem
  pd_grid g{};
  double dt = 0, alpha = 0;
  int nt = 0, F = 0;
  pd_scheme scheme = PD_BE;
  cudaStream_t st = nullptr;
  // distribution: mode 0 single GPU; 1 NCCL rank of `size` (local vectors); 2 `size` virtual ranks in this
  // process on one GPU (global vectors, exchanges by device copies; test mode for the sharded path)
  int rank = 0, size = 1, dist_mode = 0;
  pd_comm* comm = nullptr;
  bool p2p = false;              // mode 1: Step (a) / (c) read and write the owners' Sg through NVLink peer mappings
  std::vector<pd_shard> shards;  // modes 1 (one entry: this rank) and 2 (all virtual ranks)
  pd_plan plan;
  int nx_loc = 0, ny_loc = 0;    // local spatial extent (1D: x-range, 2D: y-rows)
  long long off = 0;             // first local spatial dof (global index)
  long long S = 0;               // local spatial dofs
  long long Sg = 0;              // global spatial dofs
  // tables (device)
  double* gam = nullptr;
  double* igam = nullptr;
  double2* tw_t = nullptr;       // exp(-2 pi i j / Nt)
  double2* tw_n1 = nullptr;      // four-step tables (Nt >= 1024)
  double2* tw_n2 = nullptr;
  double2* tf4_scratch = nullptr;
  // PD_TF4_OVERLAP: second scratch chunk + stream for the two-stream four-step pipeline (tfx path)
  bool use_ov = false;
  pd_tfx_overlap ov{};      // forward time FFT view (owns the streams / scratches / events, up to the larger count)
  pd_tfx_overlap ov_inv{};  // inverse view of the same pool (its own stream count)
  long long tf4_chunk = 0;
  bool use_tf4 = false;
  bool use_tfx = false;           // 2D: four-step time FFT with the x-FFT folded in (tfx.cu)
  double2* lam1 = nullptr;       // half spectrum, F entries
  double2* lam2 = nullptr;
  pd_tri_coef* tri = nullptr;    // 1D
  double* sx = nullptr;          // 2D: sin^2(pi k / N)
  double* sn = nullptr;          // 2D: sin(2 pi k / N)
  double2* tw_s = nullptr;       // 2D: exp(-2 pi i j / N)
  pd_ytri_coef* ytri = nullptr;  // 2D: [F][N] cyclic Toeplitz y-pass constants (slab2d.cu ytri)
  double* nl_dbar = nullptr;     // NEXT-4: time-averaged reaction Jacobian [S]
  bool use_gtsv = false;         // 1D Step (b) by pivoted elimination (gtsv.cu) instead of the recurrences
  void* gtsv_scratch = nullptr;  // gtsv factors [F][Nx] (1/d, du, swap flags), allocated on first use
  int* gtsv_bad = nullptr;       // device: max (frequency + 1) with a zero / non-finite pivot (0: none)
  int* gtsv_hbad = nullptr;      // pinned host copy
  double* mu = nullptr;          // 2D Dirichlet: [M] DST eigenvalues (4 nu/h^2) sin^2(pi k / M), M = 2(N+1)
  pd_dtri_coef* dtri = nullptr;  // 2D Dirichlet: [F][N] y-direction recurrence constants (slab2d.cu dtri)
  bool use_dtri = false;
  bool use_ytri = false;
  pd_slab_params slab{};
  int slab_chunk = 1;
  pd_stencil sten{};
  // host copies
  std::vector<std::complex<double>> lam1_full, lam2_full;
  // workspace
  double2* Sh = nullptr;         // half spectrum [F][S] complex (frequency-sharded layout when size > 1)
  double* rvec = nullptr;        // residual / temp vector
  double* partial = nullptr;     // reduction partials
  double* npart = nullptr;       // per-CTA partial sums of ||b||^2 fused into the first GMRES apply
  int npartial = 0;
  double* dred = nullptr;        // reduced scalars (device)
  double* hred = nullptr;        // pinned host scalars
  // GMRES
  int gm_m = 0;
  std::vector<double*> V;
  double* zvec = nullptr;
  std::vector<double*> Zs;       // GMRES: Z_j = P^{-1} X_j of the current cycle (final assembly by one sweep)
  double* gm_head = nullptr;     // head-sized work vector of the corner-identity GMRES path
  double* gm_full = nullptr;     // NCCL ranks: replicated [H][S_glob] tail and head of the corner identity
  int* gm_flag = nullptr;        // zero-initial-guess check
  double* ivp_init = nullptr;    // pd_solve_ivp_host: u0, v0 on the device
  double* ivp_f = nullptr;       // pd_solve_ivp_host: source samples
  double* ivp_dst = nullptr;     // pd_solve_ivp_host (GMRES): host destination of u, streamed behind the assembly
  bool ivp_done = false;         // that copy was issued for the final u
  cudaStream_t d2h_st = nullptr; // its copy stream
  int* gm_hflag = nullptr;
  // host-buffer staging
  double* stage_a = nullptr;
  double* stage_b = nullptr;
  // CUDA graphs of the apply, keyed by (r, z, accumulate).  PD_GRAPH=1: captured at the first use of a triple;
  // default for launch-bound sizes (Nt S <= 2^21: configs 0 and 1): captured at its SECOND use (exec == nullptr marks a
  // triple seen once), so a one-off solve never pays for an instantiation; PD_GRAPH=0: never
  struct GraphEntry {
    const double* r;
    double* z;
    int acc;
    cudaGraphExec_t exec;
    long long launches;
  };
  std::vector<GraphEntry> graphs;
  bool use_graphs = false;
  bool graphs_on_reuse = false;
  cudaStream_t cap_stream = nullptr;  // private stream for capture (the legacy stream cannot capture)
  // WR tail form (tailform.cpp), built on first use
  struct TailState {
    bool ready = false;
    int H = 0, G = 0;
    pd_tail_g gc{};
    double2* hc = nullptr;    // 1D: [F][H] economical Step (a) coefficients
    double2* ow = nullptr;    // 1D: [F][H] Step (c) weights of the last H rows (with multiplicity)
    double* part = nullptr;   // 1D: [G][H][S] per-CTA partial sums
    double* acc = nullptr;    // [H][Sg] per-shard tail accumulation (virtual ranks)
    double2* gx = nullptr;    // [H][Sg] complex head for the head-only apply
    pd_stencil gsten{};       // stencil of the GLOBAL grid (heads and tails are replicated on every rank)
    double2* tau = nullptr;   // 2D: [N][N] transfer function
    double2* work = nullptr;  // 2D: [N][N] complex slab
    double* taud = nullptr;   // 2D Dirichlet: [H][H][N][N] real transfer tables
    double* dsin = nullptr;   // 2D Dirichlet: [N][N] DST-I sine table
    double* dwork = nullptr;  // 2D Dirichlet: [2H + 1][N][N] transform work
    std::vector<double*> scr;  // head-sized scratch vectors
    std::vector<double*> Vh;   // reduced GMRES basis (heads)
    int* flag = nullptr;       // device flag (any non-zero)
    int* hflag = nullptr;      // pinned host copy
  } tail;
  // diagnostics
  long long launches = 0;
  bool timing = false;
  std::vector<cudaEvent_t> evpool;          // recorded pairs, resolved lazily (no sync per phase)
  std::vector<std::pair<int, int>> evrec;   // (phase, index of begin event)
  int ev_open[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  double phase_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long phase_n[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  std::string err;
};


pd_status fail(pd_ctx* c, pd_status s, const char* fmt, ...);

#define PD_CUDA(ctx, expr)                                                                    \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(ctx, PD_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

#define PD_LAUNCH(ctx, expr) \
  do {                       \
    PD_CUDA(ctx, expr);      \
    (ctx)->launches++;       \
  } while (0)

// dist.cpp
pd_status pd_dist_setup(pd_ctx* c, const void* nccl_id, void* nccl_comm);
void pd_dist_free(pd_ctx* c);
pd_status pd_dist_apply(pd_ctx* c, const double* r, double* z, int accumulate);
pd_status pd_dist_stencil(pd_ctx* c, const double* b, const double* u, double* out, double* norm2_dev_partial_sum);
pd_status pd_dist_build_rhs(pd_ctx* c, const double* u0, const double* v0, const double* f, double* b);
// paradiag.cpp helpers used by dist.cpp and tailform.cpp
pd_status pd_apply_impl(pd_ctx* c, const double* r, double* z, int accumulate);
pd_status pd_stencil_impl(pd_ctx* c, const double* b, const double* u, double* out, double* norm2);
// reduced values are all-reduced across NCCL ranks unless global_sum is false (vectors replicated on every rank)
pd_status pd_krylov_n(pd_ctx* c, int mode, const double* const* X, const double* coef, int k, double a, double* y,
                      long long n, double* host_out, bool global_sum = true, const double* hsub = nullptr,
                      long long hlen = 0);
extern "C" void pd_report_push(pd_report* rep, double v);
void pd_tail_free(pd_ctx* c);
void pd_corner_coefs(const pd_ctx* c, pd_tail_g* gc);
pd_status pd_corner_head(pd_ctx* c, const pd_tail_g& gc, const double* tail, double* head);
pd_status pd_spatial_solve(pd_ctx* c, double2* Sh, int nfreq, int f0);
pd_status pd_gtsv_ensure(pd_ctx* c);
// Steps (a) / (c) of a local slab [Nt][S]; the spectrum rows through sp (pd_spec_local(c->Sh, S) on one GPU)
pd_status pd_time_fft_fwd(pd_ctx* c, const double* r, const pd_spec& sp, long long S);
pd_status pd_time_fft_inv(pd_ctx* c, const pd_spec& sp, double* z, long long S, int accumulate);
