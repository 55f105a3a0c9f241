// pit_comm.cpp — transports of the slab-sharded data plane (pit_comm.h).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2; an already loaded
// copy, e.g. torch's, is reused by soname), so libpit_b200.so has no link
// dependency on it and loads on hosts without NCCL.
#include "pit_comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <string>

namespace {

struct NcclApi {
  bool ok = false;
  std::string error;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = nullptr;
    if (const char* p = std::getenv("PIT_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.error = std::string("NCCL not found (libnccl.so.2): ") + dlerror();
      return a;
    }
#define PIT_NCCL_SYM(field, name)                                             \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));              \
  if (!a.field) {                                                             \
    a.error = std::string("NCCL symbol missing: ") + name;                    \
    return a;                                                                 \
  }
    PIT_NCCL_SYM(get_unique_id, "ncclGetUniqueId")
    PIT_NCCL_SYM(init_rank, "ncclCommInitRank")
    PIT_NCCL_SYM(destroy, "ncclCommDestroy")
    PIT_NCCL_SYM(send, "ncclSend")
    PIT_NCCL_SYM(recv, "ncclRecv")
    PIT_NCCL_SYM(allgather, "ncclAllGather")
    PIT_NCCL_SYM(group_start, "ncclGroupStart")
    PIT_NCCL_SYM(group_end, "ncclGroupEnd")
    PIT_NCCL_SYM(error_string, "ncclGetErrorString")
#undef PIT_NCCL_SYM
    a.ok = true;
    return a;
  }();
  return api;
}

thread_local std::string t_what;

int fail(const char** what, int code, const std::string& msg) {
  t_what = msg;
  if (what) *what = t_what.c_str();
  return code;
}

int nccl_check(ncclResult_t r, const char** what, const char* op) {
  if (r == ncclSuccess) return PIT_OK;
  return fail(what, PIT_ERR_CUDA, std::string("NCCL ") + op + ": " + nccl().error_string(r));
}

int cuda_check(cudaError_t e, const char** what, const char* op) {
  if (e == cudaSuccess) return PIT_OK;
  return fail(what, PIT_ERR_CUDA, std::string("CUDA ") + op + ": " + cudaGetErrorString(e));
}

int host_stage(pit_comm* c, size_t n, const char** what) {
  if (c->h_cap >= n) return PIT_OK;
  if (c->h_buf) cudaFreeHost(c->h_buf);
  c->h_buf = nullptr;
  c->h_cap = 0;
  if (int rc = cuda_check(cudaMallocHost(&c->h_buf, n * sizeof(double)), what, "staging")) return rc;
  c->h_cap = n;
  return PIT_OK;
}

}  // namespace

namespace pitcomm {

int send(pit_comm* c, const double* dev, size_t n, int peer, cudaStream_t st, const char** what) {
  if (c->kind == 0) {
    return nccl_check(nccl().send(dev, n, ncclDouble, peer, (ncclComm_t)c->nccl, st), what,
                      "send");
  }
  if (int rc = host_stage(c, n, what)) return rc;
  if (int rc = cuda_check(cudaMemcpyAsync(c->h_buf, dev, n * sizeof(double),
                                          cudaMemcpyDeviceToHost, st), what, "send copy"))
    return rc;
  if (int rc = cuda_check(cudaStreamSynchronize(st), what, "send sync")) return rc;
  if (c->ops.send(c->h_buf, n, peer, c->ops.user))
    return fail(what, PIT_ERR_CUDA, "host transport: send failed");
  return PIT_OK;
}

int recv(pit_comm* c, double* dev, size_t n, int peer, cudaStream_t st, const char** what) {
  if (c->kind == 0) {
    return nccl_check(nccl().recv(dev, n, ncclDouble, peer, (ncclComm_t)c->nccl, st), what,
                      "recv");
  }
  if (int rc = host_stage(c, n, what)) return rc;
  if (int rc = cuda_check(cudaStreamSynchronize(st), what, "recv sync")) return rc;
  if (c->ops.recv(c->h_buf, n, peer, c->ops.user))
    return fail(what, PIT_ERR_CUDA, "host transport: recv failed");
  if (int rc = cuda_check(cudaMemcpyAsync(dev, c->h_buf, n * sizeof(double),
                                          cudaMemcpyHostToDevice, st), what, "recv copy"))
    return rc;
  return cuda_check(cudaStreamSynchronize(st), what, "recv sync");
}

int shift(pit_comm* c, const double* send_dev, double* recv_dev, size_t n, cudaStream_t st,
          const char** what) {
  const bool to_next = c->rank + 1 < c->world, from_prev = c->rank > 0;
  if (c->kind == 0) {
    const NcclApi& a = nccl();
    if (int rc = nccl_check(a.group_start(), what, "group")) return rc;
    ncclResult_t r = ncclSuccess;
    if (to_next) r = a.send(send_dev, n, ncclDouble, c->rank + 1, (ncclComm_t)c->nccl, st);
    if (r == ncclSuccess && from_prev)
      r = a.recv(recv_dev, n, ncclDouble, c->rank - 1, (ncclComm_t)c->nccl, st);
    const ncclResult_t e = a.group_end();
    if (int rc = nccl_check(r, what, "halo")) return rc;
    return nccl_check(e, what, "group");
  }
  // host transport: even ranks send first, odd ranks receive first (no
  // cycle of blocking sends)
  if ((c->rank & 1) == 0) {
    if (to_next)
      if (int rc = send(c, send_dev, n, c->rank + 1, st, what)) return rc;
    if (from_prev)
      if (int rc = recv(c, recv_dev, n, c->rank - 1, st, what)) return rc;
  } else {
    if (from_prev)
      if (int rc = recv(c, recv_dev, n, c->rank - 1, st, what)) return rc;
    if (to_next)
      if (int rc = send(c, send_dev, n, c->rank + 1, st, what)) return rc;
  }
  return PIT_OK;
}

int allgather(pit_comm* c, const double* dev_in, size_t n, double* dev_out, cudaStream_t st,
              const char** what) {
  if (c->kind == 0)
    return nccl_check(nccl().allgather(dev_in, dev_out, n, ncclDouble, (ncclComm_t)c->nccl, st),
                      what, "allgather");
  const size_t total = n * (size_t)(c->world + 1);
  if (int rc = host_stage(c, total, what)) return rc;
  double* hin = c->h_buf;
  double* hout = c->h_buf + n;
  if (int rc = cuda_check(cudaMemcpyAsync(hin, dev_in, n * sizeof(double), cudaMemcpyDeviceToHost,
                                          st), what, "allgather copy"))
    return rc;
  if (int rc = cuda_check(cudaStreamSynchronize(st), what, "allgather sync")) return rc;
  if (c->ops.allgather(hin, n, hout, c->ops.user))
    return fail(what, PIT_ERR_CUDA, "host transport: allgather failed");
  if (int rc = cuda_check(cudaMemcpyAsync(dev_out, hout, n * c->world * sizeof(double),
                                          cudaMemcpyHostToDevice, st), what, "allgather copy"))
    return rc;
  return cuda_check(cudaStreamSynchronize(st), what, "allgather sync");
}

}  // namespace pitcomm

// ---- construction ---------------------------------------------------------

namespace pitcomm {

int unique_id(unsigned char* id, const char** what) {
  const NcclApi& a = nccl();
  if (!a.ok) return fail(what, PIT_ERR_CUDA, a.error);
  ncclUniqueId u;
  if (int rc = nccl_check(a.get_unique_id(&u), what, "get_unique_id")) return rc;
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return PIT_OK;
}

int create_nccl(const unsigned char* id, int rank, int world, int device, pit_comm** out,
                const char** what) {
  const NcclApi& a = nccl();
  if (!a.ok) return fail(what, PIT_ERR_CUDA, a.error);
  int prev = -1;
  if (int rc = cuda_check(cudaGetDevice(&prev), what, "get device")) return rc;
  if (int rc = cuda_check(cudaSetDevice(device), what, "set device")) return rc;
  ncclUniqueId u;
  std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = a.init_rank(&comm, world, u, rank);
  cudaSetDevice(prev);
  if (int rc = nccl_check(r, what, "comm init")) return rc;
  auto c = new pit_comm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->kind = 0;
  c->nccl = comm;
  *out = c;
  return PIT_OK;
}

void destroy(pit_comm* c) {
  if (!c) return;
  if (c->kind == 0 && c->nccl) nccl().destroy((ncclComm_t)c->nccl);
  if (c->h_buf) cudaFreeHost(c->h_buf);
  delete c;
}

}  // namespace pitcomm
