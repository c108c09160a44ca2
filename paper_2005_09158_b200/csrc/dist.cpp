// Sharded ParaDiag-II apply and residual (north_star "sharded by spatial dofs for the time
// FFT, then redistributed ... so each GPU owns whole time frequencies for the spatial solves, then
// transposed back").
//
//   rank p owns the spatial slab [off_p, off_p + S_p) for all Nt time levels (1D: x-range, 2D: y-rows)
//   Step (a)  time FFT of the slab; frequency row n goes to its owner q: columns [off_p, +S_p) of Sg_q[F_q][S_glob]
//   all-to-all: block (frequencies of q) x (dofs of p) goes p -> q (fused into Step (a), see below)
//   Step (b)  spatial solves of the F_q local frequencies on full spatial rows   (no communication)
//   all-to-all back, Step (c) local inverse time FFT
//   residual: one halo column (1D) / row (2D, periodic ring) per side and time level from the neighbours
//
// The all-to-alls are fused into the time-FFT kernels: Step (a)'s epilogue stores each frequency row straight into
// its owner's Step (b) buffer Sg_q[F_q][S_glob] (at this slab's columns), and Step (c)'s prologue loads it back from
// there (pd_spec in kernels.h): no staging buffer, no copy pass.  The owners' buffers are
//   dist_mode 2: P virtual ranks of this process on one GPU (plain device pointers) - the sharded path's GPU test
//                mode (tests/test_gpu_dist.py), running the very kernels and views of mode 1;
//   dist_mode 1: NCCL ranks, one GPU each: every Sg is exported with CUDA IPC, the handles all-gathered over NCCL and
//                opened as peer mappings (NVLink); two stream-ordered NCCL barriers per apply separate the writers of
//                Step (a) from the Step (b) readers and Step (b) from the Step (c) readers.  If the peer mappings
//                cannot be opened (no P2P path, > kPdMaxRanks ranks), the plan runs as grouped ncclSend/ncclRecv
//                into a staging buffer plus one pitched copy per block (the fallback exchange).
// Plan logic is host-only (pd_make_plan) and covered by the world-size-2 gloo test (tests/test_dist_plan.py).
#include <algorithm>
#include <cstring>

#include "ctx.h"

template <class T>
static cudaError_t dalloc(T** p, size_t n) {
  return cudaMalloc((void**)p, n * sizeof(T) + 16);
}

pd_plan pd_make_plan(int op, int nx, int ny, int nt, int P) {
  pd_plan pl;
  pl.P = P;
  const bool two_d = pd_is_2d(op);
  const int ext = two_d ? ny : nx;
  const long long unit = two_d ? nx : 1;
  const int F = nt / 2 + 1;
  pl.s_off.resize(P);
  pl.s_cnt.resize(P);
  pl.f_off.resize(P);
  pl.f_cnt.resize(P);
  pl.e_off.resize(P);
  pl.e_cnt.resize(P);
  for (int p = 0; p < P; ++p) {
    const int eb = ext / P, er = ext % P;
    pl.e_off[p] = p * eb + std::min(p, er);
    pl.e_cnt[p] = eb + (p < er ? 1 : 0);
    pl.s_off[p] = pl.e_off[p] * unit;
    pl.s_cnt[p] = pl.e_cnt[p] * unit;
    const int fb = F / P, fr = F % P;
    pl.f_off[p] = p * fb + std::min(p, fr);
    pl.f_cnt[p] = fb + (p < fr ? 1 : 0);
  }
  return pl;
}

extern "C" pd_status pd_partition(int op, int nx, int ny, int nt, int size, long long* s_off, long long* s_cnt,
                                  int* f_off, int* f_cnt) {
  if (size < 1 || nt < 2 || nx < 1 || ny < 1) return PD_EINVAL;
  const pd_plan pl = pd_make_plan(op, nx, ny, nt, size);
  for (int p = 0; p < size; ++p) {
    if (s_off) s_off[p] = pl.s_off[p];
    if (s_cnt) s_cnt[p] = pl.s_cnt[p];
    if (f_off) f_off[p] = pl.f_off[p];
    if (f_cnt) f_cnt[p] = pl.f_cnt[p];
  }
  return PD_OK;
}

static int hw_of(const pd_ctx* c) { return pd_is_2d(c->g.op) ? c->g.nx : 1; }

// mode 1: export this rank's Sg, all-gather the IPC handles over NCCL, open every peer's (c->p2p on success; any
// failure leaves the fallback exchange in place)
static void open_peers(pd_ctx* c) {
  pd_shard& me = c->shards[0];
  const int P = c->size;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, me.Sg) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  char* dbuf = nullptr;
  std::vector<cudaIpcMemHandle_t> all(P);
  bool ok = cudaMalloc(&dbuf, sizeof(h) * (P + 1)) == cudaSuccess;
  ok = ok && cudaMemcpy(dbuf + sizeof(h) * P, &h, sizeof(h), cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && pd_comm_allgather(c->comm, dbuf + sizeof(h) * P, dbuf, sizeof(h)) == 0;
  ok = ok && cudaStreamSynchronize(c->st) == cudaSuccess;
  ok = ok && cudaMemcpy(all.data(), dbuf, sizeof(h) * P, cudaMemcpyDeviceToHost) == cudaSuccess;
  if (dbuf) cudaFree(dbuf);
  for (int q = 0; ok && q < P; ++q) {
    if (q == c->rank) continue;
    void* ptr = nullptr;
    ok = cudaIpcOpenMemHandle(&ptr, all[q], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
    me.peer[q] = static_cast<double2*>(ptr);
  }
  // every rank must take the same route: agree on the outcome (min over ranks)
  double flag = ok ? 1.0 : 0.0, *dflag = nullptr;
  if (cudaMalloc(&dflag, sizeof(double)) == cudaSuccess) {
    cudaMemcpy(dflag, &flag, sizeof(double), cudaMemcpyHostToDevice);
    flag = (pd_comm_allreduce_sum(c->comm, dflag, 1) == 0 && cudaStreamSynchronize(c->st) == cudaSuccess &&
            cudaMemcpy(&flag, dflag, sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess)
               ? flag
               : 0.0;
    cudaFree(dflag);
  } else {
    flag = 0.0;
  }
  c->p2p = ok && flag == (double)P;
  if (!c->p2p) {
    for (int q = 0; q < P; ++q)
      if (me.peer[q]) cudaIpcCloseMemHandle(me.peer[q]);
    for (auto& p : me.peer) p = nullptr;
    cudaGetLastError();
  }
}

pd_status pd_dist_setup(pd_ctx* c, const void* nccl_id, void* nccl_comm) {
  const int P = c->size;
  c->plan = pd_make_plan(c->g.op, c->g.nx, c->g.ny, c->nt, P);
  const pd_plan& pl = c->plan;
  const int ext = pd_is_2d(c->g.op) ? c->g.ny : c->g.nx;
  if (P > ext) return fail(c, PD_EINVAL, "more ranks (%d) than spatial slabs (%d)", P, ext);
  if (P > c->F) return fail(c, PD_EINVAL, "more ranks (%d) than frequencies (%d)", P, c->F);
  const int hw = hw_of(c);
  std::vector<int> ranks;
  if (c->dist_mode == 1) {
    c->comm = nccl_comm ? pd_comm_wrap(nccl_comm, c->rank, P, c->st) : pd_comm_create(nccl_id, c->rank, P, c->st);
    if (!c->comm) return fail(c, PD_ENCCL, "NCCL init: %s", pd_comm_last_error());
    ranks.push_back(c->rank);
  } else {
    for (int p = 0; p < P; ++p) ranks.push_back(p);
  }
  long long maxS = 0;
  for (int p = 0; p < P; ++p) maxS = std::max(maxS, pl.s_cnt[p]);
  for (int p : ranks) {
    pd_shard sh;
    sh.rank = p;
    sh.S = pl.s_cnt[p];
    sh.off = pl.s_off[p];
    sh.ext = pl.e_cnt[p];
    sh.ext_off = pl.e_off[p];
    sh.F = pl.f_cnt[p];
    sh.f0 = pl.f_off[p];
    sh.sten = c->sten;
    if (pd_is_2d(c->g.op)) {
      sh.sten.nx = c->g.nx;
      sh.sten.ny = sh.ext;
    } else {
      sh.sten.nx = sh.ext;
      sh.sten.ny = 1;
    }
    cudaError_t e = cudaSuccess;
    if (c->dist_mode == 1) {
      sh.Sh_loc = c->Sh;  // allocated by pd_setup for the local slab
      e = dalloc(&sh.stage, (size_t)std::max<long long>((long long)sh.F * c->Sg, (long long)c->F * sh.S));
      if (e == cudaSuccess) e = dalloc(&sh.sendlo, (size_t)c->nt * hw);
      if (e == cudaSuccess) e = dalloc(&sh.sendhi, (size_t)c->nt * hw);
    } else {
      e = dalloc(&sh.r_loc, (size_t)(c->nt + 1) * sh.S);
      if (e == cudaSuccess) e = dalloc(&sh.z_loc, (size_t)(c->nt + 1) * sh.S);
      if (e == cudaSuccess) e = dalloc(&sh.b_loc, (size_t)(c->nt + 1) * sh.S);
    }
    if (e == cudaSuccess) e = dalloc(&sh.Sg, (size_t)sh.F * c->Sg);
    if (e == cudaSuccess) e = dalloc(&sh.hlo, (size_t)c->nt * hw);
    if (e == cudaSuccess) e = dalloc(&sh.hhi, (size_t)c->nt * hw);
    if (e == cudaSuccess) e = dalloc(&sh.h1lo, (size_t)2 * hw);
    if (e == cudaSuccess) e = dalloc(&sh.h1hi, (size_t)2 * hw);
    c->shards.push_back(sh);
    if (e != cudaSuccess) return fail(c, PD_ENOMEM, "sharded workspace: %s", cudaGetErrorString(e));
  }
  (void)maxS;
  if (c->dist_mode == 1 && P <= kPdMaxRanks && getenv("PD_NO_P2P") == nullptr) open_peers(c);
  return PD_OK;
}

void pd_dist_free(pd_ctx* c) {
  for (pd_shard& sh : c->shards) {
    for (double2*& p : sh.peer)
      if (p) {
        cudaIpcCloseMemHandle(p);
        p = nullptr;
      }
    void* ptrs[] = {sh.Sg, sh.stage, sh.hlo, sh.hhi, sh.h1lo, sh.h1hi, sh.sendlo, sh.sendhi, sh.r_loc, sh.z_loc,
                    sh.b_loc};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
  c->shards.clear();
}

// ---- mode 2: gather / scatter a global [rows][S_glob] vector to a shard's [rows][S_p] slab ----
static cudaError_t gather(const pd_ctx* c, const pd_shard& sh, const double* g, double* loc, int rows) {
  return cudaMemcpy2DAsync(loc, sh.S * sizeof(double), g + sh.off, c->Sg * sizeof(double), sh.S * sizeof(double),
                           rows, cudaMemcpyDeviceToDevice, c->st);
}
static cudaError_t scatter(const pd_ctx* c, const pd_shard& sh, const double* loc, double* g, int rows) {
  return cudaMemcpy2DAsync(g + sh.off, c->Sg * sizeof(double), loc, sh.S * sizeof(double), sh.S * sizeof(double),
                           rows, cudaMemcpyDeviceToDevice, c->st);
}

// spectrum view of shard `sh`: frequency rows of owner q at Sg_q + (n - f_q) S_glob, this slab's columns
static pd_spec spec_of(const pd_ctx* c, const pd_shard& sh) {
  pd_spec v{};
  v.P = c->size;
  v.pitch = c->Sg;
  for (int q = 0; q < c->size; ++q) {
    double2* owner = c->dist_mode == 2 ? c->shards[q].Sg : (q == c->rank ? sh.Sg : sh.peer[q]);
    v.base[q] = owner + sh.off;
    v.f0[q] = c->plan.f_off[q];
  }
  return v;
}

#define PD_NCCL(ctx, expr) \
  do {                     \
    if ((expr) != 0) return fail(ctx, PD_ENCCL, "%s: %s", #expr, pd_comm_last_error()); \
  } while (0)

// fallback exchange (mode 1 without peer mappings): grouped ncclSend / ncclRecv into staging + pitched copies
static cudaError_t block_self(const pd_ctx* c, const pd_shard& me, bool fwd) {
  if (fwd)
    return cudaMemcpy2DAsync(me.Sg + me.off, c->Sg * sizeof(double2), me.Sh_loc + (long long)me.f0 * me.S,
                             me.S * sizeof(double2), me.S * sizeof(double2), me.F, cudaMemcpyDeviceToDevice, c->st);
  return cudaMemcpy2DAsync(me.Sh_loc + (long long)me.f0 * me.S, me.S * sizeof(double2), me.Sg + me.off,
                           c->Sg * sizeof(double2), me.S * sizeof(double2), me.F, cudaMemcpyDeviceToDevice, c->st);
}

static pd_status exchange_fwd(pd_ctx* c) {
  const pd_plan& pl = c->plan;
  pd_shard& me = c->shards[0];
  const int P = c->size, r = me.rank;
  PD_NCCL(c, pd_comm_group_start(c->comm));
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    PD_NCCL(c, pd_comm_send(c->comm, me.Sh_loc + (long long)pl.f_off[q] * me.S,
                            (size_t)pl.f_cnt[q] * me.S * sizeof(double2), q));
  }
  for (int p = 0; p < P; ++p) {
    if (p == r) continue;
    PD_NCCL(c, pd_comm_recv(c->comm, me.stage + (long long)me.F * pl.s_off[p], (size_t)me.F * pl.s_cnt[p] * sizeof(double2),
                            p));
  }
  PD_NCCL(c, pd_comm_group_end(c->comm));
  PD_CUDA(c, block_self(c, me, true));
  for (int p = 0; p < P; ++p) {
    if (p == r) continue;
    PD_CUDA(c, cudaMemcpy2DAsync(me.Sg + pl.s_off[p], c->Sg * sizeof(double2), me.stage + (long long)me.F * pl.s_off[p],
                                 pl.s_cnt[p] * sizeof(double2), pl.s_cnt[p] * sizeof(double2), me.F,
                                 cudaMemcpyDeviceToDevice, c->st));
  }
  return PD_OK;
}

static pd_status exchange_bwd(pd_ctx* c) {
  const pd_plan& pl = c->plan;
  pd_shard& me = c->shards[0];
  const int P = c->size, r = me.rank;
  for (int p = 0; p < P; ++p) {
    if (p == r) continue;
    PD_CUDA(c, cudaMemcpy2DAsync(me.stage + (long long)me.F * pl.s_off[p], pl.s_cnt[p] * sizeof(double2),
                                 me.Sg + pl.s_off[p], c->Sg * sizeof(double2), pl.s_cnt[p] * sizeof(double2), me.F,
                                 cudaMemcpyDeviceToDevice, c->st));
  }
  PD_CUDA(c, block_self(c, me, false));
  PD_NCCL(c, pd_comm_group_start(c->comm));
  for (int p = 0; p < P; ++p) {
    if (p == r) continue;
    PD_NCCL(c, pd_comm_send(c->comm, me.stage + (long long)me.F * pl.s_off[p], (size_t)me.F * pl.s_cnt[p] * sizeof(double2),
                            p));
  }
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    PD_NCCL(c, pd_comm_recv(c->comm, me.Sh_loc + (long long)pl.f_off[q] * me.S,
                            (size_t)pl.f_cnt[q] * me.S * sizeof(double2), q));
  }
  PD_NCCL(c, pd_comm_group_end(c->comm));
  return PD_OK;
}

// stream-ordered barrier over the NCCL ranks (a one-double all-reduce): the peer stores of the kernels before it are
// complete on every rank when it completes
static pd_status rank_barrier(pd_ctx* c) {
  if (pd_comm_allreduce_sum(c->comm, c->dred + 63, 1) != 0)
    return fail(c, PD_ENCCL, "barrier allreduce: %s", pd_comm_last_error());
  return PD_OK;
}

pd_status pd_dist_apply(pd_ctx* c, const double* r, double* z, int accumulate) {
  pd_status s;
  const bool fused = c->dist_mode == 2 || c->p2p;  // the all-to-alls inside the time-FFT kernels
  for (pd_shard& sh : c->shards) {
    const double* rin = r;
    if (c->dist_mode == 2) {
      PD_CUDA(c, gather(c, sh, r, sh.r_loc, c->nt));
      rin = sh.r_loc;
    }
    s = pd_time_fft_fwd(c, rin, fused ? spec_of(c, sh) : pd_spec_local(sh.Sh_loc, sh.S), sh.S);
    if (s != PD_OK) return s;
  }
  s = fused ? (c->dist_mode == 1 ? rank_barrier(c) : PD_OK) : exchange_fwd(c);
  if (s != PD_OK) return s;
  for (pd_shard& sh : c->shards) {
    s = pd_spatial_solve(c, sh.Sg, sh.F, sh.f0);
    if (s != PD_OK) return s;
  }
  s = fused ? (c->dist_mode == 1 ? rank_barrier(c) : PD_OK) : exchange_bwd(c);
  if (s != PD_OK) return s;
  for (pd_shard& sh : c->shards) {
    double* out = z;
    if (c->dist_mode == 2) {
      if (accumulate) PD_CUDA(c, gather(c, sh, z, sh.z_loc, c->nt));
      out = sh.z_loc;
    }
    s = pd_time_fft_inv(c, fused ? spec_of(c, sh) : pd_spec_local(sh.Sh_loc, sh.S), out, sh.S, accumulate);
    if (s != PD_OK) return s;
    if (c->dist_mode == 2) PD_CUDA(c, scatter(c, sh, sh.z_loc, z, c->nt));
  }
  return PD_OK;
}

// copy boundary column/row (`first` or last) of a local [rows][S_p] array into a contiguous [rows][hw]
static cudaError_t boundary(const pd_ctx* c, const pd_shard& sh, const double* loc, bool first, double* dst, int rows) {
  const int hw = hw_of(c);
  const long long col = first ? 0 : sh.S - hw;
  return cudaMemcpy2DAsync(dst, hw * sizeof(double), loc + col, sh.S * sizeof(double), hw * sizeof(double), rows,
                           cudaMemcpyDeviceToDevice, c->st);
}

// Halos of `rows` time levels of the local arrays loc[p] into hlo/hhi (rows x hw each) of every shard.
// 1D Dirichlet: the first/last rank has no lower/upper neighbour (NULL halo = zero); 2D periodic: ring.
static pd_status halos(pd_ctx* c, const std::vector<const double*>& loc, int rows, bool single_level, int level) {
  const int P = c->size;
  const bool ring = c->g.op == PD_ADE2D_PERIODIC;
  const int hw = hw_of(c);
  auto dst_lo = [&](pd_shard& sh) { return single_level ? sh.h1lo + level * hw : sh.hlo; };
  auto dst_hi = [&](pd_shard& sh) { return single_level ? sh.h1hi + level * hw : sh.hhi; };
  if (c->dist_mode == 2) {
    for (int p = 0; p < P; ++p) {
      pd_shard& sh = c->shards[p];
      const int lo = p - 1, hi = p + 1;
      if (lo >= 0 || ring) {
        const int q = (lo + P) % P;
        PD_CUDA(c, boundary(c, c->shards[q], loc[q], false, dst_lo(sh), rows));
      }
      if (hi < P || ring) {
        const int q = hi % P;
        PD_CUDA(c, boundary(c, c->shards[q], loc[q], true, dst_hi(sh), rows));
      }
    }
    return PD_OK;
  }
  pd_shard& me = c->shards[0];
  const int r = me.rank, prev = (r - 1 + P) % P, next = (r + 1) % P;
  const bool has_prev = ring || r > 0, has_next = ring || r < P - 1;
  PD_CUDA(c, boundary(c, me, loc[0], true, me.sendlo, rows));
  PD_CUDA(c, boundary(c, me, loc[0], false, me.sendhi, rows));
  const size_t bytes = (size_t)rows * hw * sizeof(double);
  // order: send last row to next, first row to prev; receive from prev into lo, from next into hi
  // (correct for P = 2 rings where prev == next, since NCCL matches messages per peer in order)
  PD_NCCL(c, pd_comm_group_start(c->comm));
  if (has_next) PD_NCCL(c, pd_comm_send(c->comm, me.sendhi, bytes, next));
  if (has_prev) PD_NCCL(c, pd_comm_send(c->comm, me.sendlo, bytes, prev));
  if (has_prev) PD_NCCL(c, pd_comm_recv(c->comm, dst_lo(me), bytes, prev));
  if (has_next) PD_NCCL(c, pd_comm_recv(c->comm, dst_hi(me), bytes, next));
  PD_NCCL(c, pd_comm_group_end(c->comm));
  return PD_OK;
}

static void set_halos(const pd_ctx* c, pd_shard& sh, pd_stencil& p, bool single) {
  const int P = c->size;
  const bool ring = c->g.op == PD_ADE2D_PERIODIC;
  p.hlo = (ring || sh.rank > 0) ? (single ? sh.h1lo : sh.hlo) : nullptr;
  p.hhi = (ring || sh.rank < P - 1) ? (single ? sh.h1hi : sh.hhi) : nullptr;
}

pd_status pd_dist_stencil(pd_ctx* c, const double* b, const double* u, double* out, double* unused) {
  (void)unused;
  std::vector<const double*> uloc;
  for (pd_shard& sh : c->shards) {
    if (c->dist_mode == 2) {
      PD_CUDA(c, gather(c, sh, u, sh.r_loc, c->nt));
      if (b) PD_CUDA(c, gather(c, sh, b, sh.b_loc, c->nt));
      uloc.push_back(sh.r_loc);
    } else {
      uloc.push_back(u);
    }
  }
  pd_status s = halos(c, uloc, c->nt, false, 0);
  if (s != PD_OK) return s;
  int off = 0;
  for (size_t i = 0; i < c->shards.size(); ++i) {
    pd_shard& sh = c->shards[i];
    pd_stencil p = sh.sten;
    set_halos(c, sh, p, false);
    const double* bb = b ? (c->dist_mode == 2 ? sh.b_loc : b) : nullptr;
    double* o = c->dist_mode == 2 ? sh.z_loc : out;
    int nb = 0;
    PD_LAUNCH(c, pd_launch_stencil(p, bb, uloc[i], o, c->partial + off, &nb, c->st));
    off += nb;
    if (c->dist_mode == 2) PD_CUDA(c, scatter(c, sh, sh.z_loc, out, c->nt));
  }
  // local sum of squares (all shards of this process) in dred[0]; mode 1 all-reduces it in the caller
  PD_LAUNCH(c, pd_launch_reduce_partials(c->partial, off, 1, c->dred, c->st));
  return PD_OK;
}

pd_status pd_dist_build_rhs(pd_ctx* c, const double* u0, const double* v0, const double* f, double* b) {
  // single-level halos of U0 (row 0) and V0 (row 1)
  std::vector<const double*> l0, l1;
  for (pd_shard& sh : c->shards) {
    if (c->dist_mode == 2) {
      PD_CUDA(c, gather(c, sh, u0, sh.r_loc, 1));
      if (v0) PD_CUDA(c, gather(c, sh, v0, sh.b_loc, 1));
      if (f) PD_CUDA(c, gather(c, sh, f, sh.z_loc, c->nt + 1));
      l0.push_back(sh.r_loc);
      l1.push_back(v0 ? sh.b_loc : sh.r_loc);
    } else {
      l0.push_back(u0);
      l1.push_back(v0 ? v0 : u0);
    }
  }
  pd_status s = halos(c, l0, 1, true, 0);
  if (s != PD_OK) return s;
  s = halos(c, l1, 1, true, 1);
  if (s != PD_OK) return s;
  for (size_t i = 0; i < c->shards.size(); ++i) {
    pd_shard& sh = c->shards[i];
    pd_stencil p = sh.sten;
    set_halos(c, sh, p, true);
    if (c->dist_mode == 2) {
      // the rhs writes [Nt][S_p] into r_loc's companion buffer; reuse b_loc after V0 is consumed is unsafe,
      // so write into r_loc + S_p .. (r_loc holds Nt+1 rows: row 0 = U0, rows 1.. free) -> use z_loc
      double* outl = sh.z_loc + (f ? 0 : 0);
      if (f) {
        // f occupies z_loc; move it behind: build into b_loc rows 1.. after copying V0 to r_loc row 1
        PD_CUDA(c, cudaMemcpyAsync(sh.r_loc + sh.S, v0 ? sh.b_loc : sh.r_loc, sh.S * sizeof(double),
                                   cudaMemcpyDeviceToDevice, c->st));
        PD_LAUNCH(c, pd_launch_rhs(p, sh.r_loc, v0 ? sh.r_loc + sh.S : nullptr, sh.z_loc, sh.b_loc, c->st));
        outl = sh.b_loc;
      } else {
        PD_LAUNCH(c, pd_launch_rhs(p, sh.r_loc, v0 ? sh.b_loc : nullptr, nullptr, sh.z_loc, c->st));
      }
      PD_CUDA(c, scatter(c, sh, outl, b, c->nt));
    } else {
      PD_LAUNCH(c, pd_launch_rhs(p, u0, v0, f, b, c->st));
    }
  }
  return PD_OK;
}
