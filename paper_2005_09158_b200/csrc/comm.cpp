// NCCL transport (grouped point-to-point send/recv for the spatial<->frequency all-to-all and the halo
// exchange; an all-reduce for norms and Gram-Schmidt dots).  NCCL is resolved with dlopen so that the
// library loads on hosts without it and single-GPU use never initialises it; inside a torch process the
// already-loaded libnccl.so.2 (torch's NCCL) is reused.
#include "comm.h"

#include <dlfcn.h>

#include <cstring>
#include <string>

namespace {

typedef int ncclResult_t;
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
constexpr int kNcclInt8 = 0, kNcclFloat64 = 8, kNcclSum = 0;

struct Api {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
};

Api g_api;
std::string g_err;

bool load() {
  if (g_api.h) return true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    g_api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (g_api.h) break;
  }
  if (!g_api.h) {
    g_err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
    return false;
  }
#define PD_SYM(field, name)                                                  \
  g_api.field = reinterpret_cast<decltype(g_api.field)>(dlsym(g_api.h, name)); \
  if (!g_api.field) {                                                        \
    g_err = std::string("missing NCCL symbol ") + name;                      \
    return false;                                                            \
  }
  PD_SYM(getUniqueId, "ncclGetUniqueId")
  PD_SYM(commInitRank, "ncclCommInitRank")
  PD_SYM(commDestroy, "ncclCommDestroy")
  PD_SYM(groupStart, "ncclGroupStart")
  PD_SYM(groupEnd, "ncclGroupEnd")
  PD_SYM(send, "ncclSend")
  PD_SYM(recv, "ncclRecv")
  PD_SYM(allReduce, "ncclAllReduce")
  PD_SYM(allGather, "ncclAllGather")
  PD_SYM(errStr, "ncclGetErrorString")
#undef PD_SYM
  return true;
}

int check(ncclResult_t r, const char* what) {
  if (r == 0) return 0;
  g_err = std::string(what) + ": " + (g_api.errStr ? g_api.errStr(r) : "nccl error");
  return -1;
}

}  // namespace

struct pd_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, size = 1;
  cudaStream_t st = nullptr;
  bool owned = true;
};

const char* pd_comm_last_error() { return g_err.c_str(); }

int pd_comm_unique_id(void* out128) {
  if (!load()) return -1;
  ncclUniqueId id;
  if (check(g_api.getUniqueId(&id), "ncclGetUniqueId")) return -1;
  std::memcpy(out128, id.internal, 128);
  return 0;
}

pd_comm* pd_comm_create(const void* id, int rank, int size, cudaStream_t st) {
  if (!load()) return nullptr;
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, 128);
  pd_comm* c = new pd_comm();
  c->rank = rank;
  c->size = size;
  c->st = st;
  if (check(g_api.commInitRank(&c->comm, size, uid, rank), "ncclCommInitRank")) {
    delete c;
    return nullptr;
  }
  return c;
}

pd_comm* pd_comm_wrap(void* nccl_comm, int rank, int size, cudaStream_t st) {
  if (!load()) return nullptr;
  pd_comm* c = new pd_comm();
  c->comm = static_cast<ncclComm_t>(nccl_comm);
  c->rank = rank;
  c->size = size;
  c->st = st;
  c->owned = false;
  return c;
}

void pd_comm_destroy(pd_comm* c) {
  if (!c) return;
  if (c->owned && c->comm && g_api.commDestroy) g_api.commDestroy(c->comm);
  delete c;
}

int pd_comm_group_start(pd_comm*) { return check(g_api.groupStart(), "ncclGroupStart"); }
int pd_comm_group_end(pd_comm*) { return check(g_api.groupEnd(), "ncclGroupEnd"); }

int pd_comm_send(pd_comm* c, const void* buf, size_t bytes, int peer) {
  if (!bytes) return 0;
  return check(g_api.send(buf, bytes, kNcclInt8, peer, c->comm, c->st), "ncclSend");
}

int pd_comm_recv(pd_comm* c, void* buf, size_t bytes, int peer) {
  if (!bytes) return 0;
  return check(g_api.recv(buf, bytes, kNcclInt8, peer, c->comm, c->st), "ncclRecv");
}

int pd_comm_allreduce_sum(pd_comm* c, double* d, int n) {
  return check(g_api.allReduce(d, d, (size_t)n, kNcclFloat64, kNcclSum, c->comm, c->st), "ncclAllReduce");
}

int pd_comm_allgather(pd_comm* c, const void* send, void* recv, size_t bytes) {
  return check(g_api.allGather(send, recv, bytes, kNcclInt8, c->comm, c->st), "ncclAllGather");
}
