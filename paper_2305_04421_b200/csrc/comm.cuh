// comm.cuh — rank-to-rank exchange for time-slab sharding.
//
// Rank g of G owns the subdomains [g*Nd/G, (g+1)*Nd/G) and their node slab.
// Per GMRES iteration the sharded path exchanges
//   * halo planes (one n_sp plane with each neighbour) for the time couplings
//     of K and of the sweep's shared node,
//   * the 2*Nd coarse coefficients (all-gather of each rank's columns),
//   * one partial sum per dot product (all-gather, summed in rank order so
//     every rank gets the same, deterministic value).
// Backends: NCCL over NVLink (one process per GPU; libnccl is dlopen'ed only
// when a communicator is created) and an in-process group of host threads
// sharing one GPU — the latter exchanges with host synchronisation between
// launches (no kernel ever waits on another rank's kernel) and exists to
// test the sharded CUDA path on a single device.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace kkt {

struct Comm {
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // recv[r*n .. r*n+n) = send of rank r, for every rank (device buffers)
  virtual void allgather(const double* send, double* recv, size_t n, cudaStream_t s) = 0;
  // send `to_prev` to rank-1 and `to_next` to rank+1; receive the matching
  // planes from rank+1 into `from_next` and from rank-1 into `from_prev`.
  // Absent neighbours (first / last rank) are skipped; pointers may be null.
  virtual void halo(const double* to_prev, double* from_next, const double* to_next,
                    double* from_prev, size_t n, cudaStream_t s) = 0;
};

Comm* make_nccl_comm(const void* unique_id, int rank, int nranks);
Comm* make_local_comm(void* group, int rank);
int nccl_unique_id(void* out128);
void* local_group_create(int n);
void local_group_destroy(void* g);

}  // namespace kkt
