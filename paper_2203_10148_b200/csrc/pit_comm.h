// pit_comm.h — the slab-sharded data plane (internal).  DESIGN.md §7.
//
// One rank per GPU owns a contiguous range of slabs; the
// only traffic is
//   * the halo: the last owned block of rank r goes to rank r+1 before each
//     fine batch (apply_F / preconditioned residual);
//   * the coarse chain: G^-1 / the initial guess sweep rank by rank, W of the
//     last owned block handed to the next rank;
//   * the reductions: every rank's per-block partials all-gathered and summed
//     in global slab order on every rank (bit-identical to one GPU).
// Transports: NCCL over NVLink / NVSwitch (ncclSend / ncclRecv / ncclAllGather
// on the caller's stream, libnccl.so.2 resolved at run time so the library
// still loads where NCCL is absent), or host callbacks (any transport the
// caller has, e.g. torch.distributed gloo in the multi-process CPU-exchange
// tests).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "pit_b200.h"

struct pit_comm {
  int rank = 0, world = 1, device = 0;
  int kind = 0;             // 0 NCCL, 1 host callbacks
  void* nccl = nullptr;     // ncclComm_t
  pit_comm_ops ops{};       // kind 1
  double* h_buf = nullptr;  // pinned staging of the host transport
  size_t h_cap = 0;
};

namespace pitcomm {

// stream-ordered (NCCL) or synchronous through pinned staging (host); all
// return PIT_OK or an error code with pit_last_error set by the caller's
// set_err (the message is returned through *what)
int send(pit_comm* c, const double* dev, size_t n, int peer, cudaStream_t st, const char** what);
int recv(pit_comm* c, double* dev, size_t n, int peer, cudaStream_t st, const char** what);
// halo exchange: send `send_dev` to rank+1 (if any) and receive from rank-1
// (if any) into `recv_dev`, as one NCCL group
int shift(pit_comm* c, const double* send_dev, double* recv_dev, size_t n, cudaStream_t st,
          const char** what);
// dev_out[world*n] = concatenation of every rank's dev_in[n]
int allgather(pit_comm* c, const double* dev_in, size_t n, double* dev_out, cudaStream_t st,
              const char** what);

int unique_id(unsigned char* id, const char** what);  // NCCL_UNIQUE_ID_BYTES (128)
int create_nccl(const unsigned char* id, int rank, int world, int device, pit_comm** out,
                const char** what);
void destroy(pit_comm* c);

}  // namespace pitcomm
