// Multi-GPU transport (NCCL, loaded at run time).  Placeholder until the distributed apply lands:
// every entry point reports that multi-GPU runs are not available in this build.
#include "comm.h"

#include <string>

static std::string g_comm_err = "multi-GPU path not built yet";

int pd_comm_unique_id(void*) { return -1; }
pd_comm* pd_comm_create(const void*, int, int, cudaStream_t) { return nullptr; }
void pd_comm_destroy(pd_comm*) {}
const char* pd_comm_last_error() { return g_comm_err.c_str(); }
int pd_comm_apply(pd_comm*, pd_ctx*, const double*, double*, int) { return -1; }
int pd_comm_halo_stencil(pd_comm*, pd_ctx*, const double*, const double*, double*) { return -1; }
int pd_comm_allreduce_sum(pd_comm*, double*, int) { return -1; }
int pd_comm_build_rhs(pd_comm*, pd_ctx*, const double*, const double*, const double*, double*) { return -1; }
