// hps_comm.cuh — the exchange layer of the subtree-sharded build and solve.
//
// The sharded tree needs exactly one collective: an ALL-GATHER among an aligned group of gs
// ranks (the ranks [rank / gs * gs, rank / gs * gs + gs) that share one box of a top level).
// Reductions are all-gathers followed by an ordered sum on the device, so the result does not
// depend on the transport.  Two transports:
//  - NcclComm: NCCL over NVLink/NVSwitch (one process per GPU).  libnccl is loaded at run time
//    (dlopen; the copy torch already loaded, else the system one); one split communicator per
//    group size, created collectively when the communicator is wrapped.
//  - VirtualComm: G ranks as host threads of ONE process sharing one GPU (tests and single-GPU
//    development).  Gathers are device-to-device copies ordered by CUDA events and separated by
//    host barriers; no kernel ever waits on another rank's kernel.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

struct HpsComm {
  int rank = 0, size = 1;
  virtual ~HpsComm() {}
  // recv[k * bytes, (k + 1) * bytes) = send of group rank k (group of gs aligned ranks containing
  // this rank).  Stream-ordered on st; send and recv are device buffers; send must stay valid until
  // the work enqueued on st before return has completed.
  virtual void allgather(int gs, const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
  virtual const char* kind() const = 0;
};

// The communicator a handle uses: NULL for single-GPU.
HpsComm* hps_comm_from_opts(void* comm, void* nccl_comm, int n_gpus, bool& owned);
