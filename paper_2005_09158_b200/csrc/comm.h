// NCCL transport of the sharded ParaDiag-II path (libnccl.so.2 loaded at run time; single-GPU builds and
// CPU-only hosts never touch it).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

struct pd_comm;

int pd_comm_unique_id(void* out128);
pd_comm* pd_comm_create(const void* id, int rank, int size, cudaStream_t st);
// borrow an existing ncclComm_t (e.g. the caller's torch ProcessGroupNCCL communicator): not destroyed
pd_comm* pd_comm_wrap(void* nccl_comm, int rank, int size, cudaStream_t st);
void pd_comm_destroy(pd_comm* c);
const char* pd_comm_last_error();
int pd_comm_group_start(pd_comm* c);
int pd_comm_group_end(pd_comm* c);
int pd_comm_send(pd_comm* c, const void* buf, size_t bytes, int peer);
int pd_comm_recv(pd_comm* c, void* buf, size_t bytes, int peer);
int pd_comm_allreduce_sum(pd_comm* c, double* d, int n);
// recv[q * bytes ...] = send of rank q (device buffers, stream-ordered)
int pd_comm_allgather(pd_comm* c, const void* send, void* recv, size_t bytes);
