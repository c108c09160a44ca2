// Multi-GPU plumbing of the ParaDiag-II apply (spatial slabs <-> frequency shards, halos, all-reduce).
#pragma once
#include <cuda_runtime.h>

#include "kernels.h"

struct pd_ctx;
struct pd_comm;

// read-only view of a context used by the distributed code
struct pd_ctx_view {
  int nt, F, op, nx, ny, nx_loc, ny_loc;
  long long S, Sg, off;
  cudaStream_t st;
  const double* gam;
  const double* igam;
  const double2* tw_t;
  pd_stencil sten;
  double* partial;
  double* dred;
  double2* Sh;
};
pd_ctx_view pd_ctx_get_view(pd_ctx* c);
int pd_ctx_spatial_solve(pd_ctx* c, double2* Sh, int nfreq, int f0);
void pd_ctx_count_launch(pd_ctx* c, int n);

int pd_comm_unique_id(void* out128);
pd_comm* pd_comm_create(const void* id, int rank, int size, cudaStream_t st);
void pd_comm_destroy(pd_comm* c);
const char* pd_comm_last_error();
int pd_comm_apply(pd_comm* c, pd_ctx* ctx, const double* r, double* z, int accumulate);
// out = b - A u (or A u); leaves the local sum of out^2 in view.dred[0]
int pd_comm_halo_stencil(pd_comm* c, pd_ctx* ctx, const double* b, const double* u, double* out);
int pd_comm_allreduce_sum(pd_comm* c, double* d, int n);
int pd_comm_build_rhs(pd_comm* c, pd_ctx* ctx, const double* u0, const double* v0, const double* f, double* b);
