// pe_nccl.cc — root-parallel search over NCCL (pe.h pe_search_multi).
//
// one tree per GPU (seed + rank); every `merge_every`
// episodes the root children's (N, W) statistics are all-reduced (SUM, int64
// -- W is 2^-32 fixed point, so the merge is bit-deterministic), and at the
// end MAX reductions pick the best plan (ties -> lowest rank).  The merge is
// the only exchange on this path; messages are (ordinals + 1) x 16 bytes, so
// it is latency-bound and NVLink / NVSwitch topology does not matter.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, the library the
// process already loaded when torch created its communicators), so
// libpe_b200.so loads on hosts without NCCL and shares the caller's NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "pe.h"

namespace {

// the subset of nccl.h used here (ABI-stable since NCCL 2.0)
typedef void* Comm;
struct UniqueId {
  char internal[128];
};
enum { kInt64 = 5 };               // ncclInt64
enum { kSum = 0, kMax = 2 };       // ncclSum, ncclMax
typedef int (*GetUniqueId)(UniqueId*);
typedef int (*CommInitRank)(Comm*, int, UniqueId, int);
typedef int (*CommDestroy)(Comm);
typedef int (*CommCount)(Comm, int*);
typedef int (*CommUserRank)(Comm, int*);
typedef int (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t);
typedef const char* (*GetErrorString)(int);

struct Nccl {
  void* h = nullptr;
  GetUniqueId get_unique_id = nullptr;
  CommInitRank comm_init_rank = nullptr;
  CommDestroy comm_destroy = nullptr;
  CommCount comm_count = nullptr;
  CommUserRank comm_user_rank = nullptr;
  AllReduce all_reduce = nullptr;
  GetErrorString error_string = nullptr;
  bool ok() const { return all_reduce != nullptr; }
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      x.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // the caller's, if loaded
      if (!x.h) x.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (x.h) break;
    }
    if (!x.h) return x;
    x.get_unique_id = (GetUniqueId)dlsym(x.h, "ncclGetUniqueId");
    x.comm_init_rank = (CommInitRank)dlsym(x.h, "ncclCommInitRank");
    x.comm_destroy = (CommDestroy)dlsym(x.h, "ncclCommDestroy");
    x.comm_count = (CommCount)dlsym(x.h, "ncclCommCount");
    x.comm_user_rank = (CommUserRank)dlsym(x.h, "ncclCommUserRank");
    x.error_string = (GetErrorString)dlsym(x.h, "ncclGetErrorString");
    x.all_reduce = (AllReduce)dlsym(x.h, "ncclAllReduce");
    if (!x.get_unique_id || !x.comm_init_rank || !x.comm_destroy || !x.comm_count ||
        !x.comm_user_rank || !x.error_string)
      x.all_reduce = nullptr;
    return x;
  }();
  return n;
}

void set_err(pe_error* err, int code, const std::string& m) {
  if (!err) return;
  err->code = code;
  err->line = err->column = 0;
  std::snprintf(err->message, sizeof(err->message), "%s", m.c_str());
}

// pe_merge_fn over an NCCL communicator: the values travel through a device
// buffer on a private stream (int64 SUM or MAX across ranks).
struct NcclMerge {
  Comm comm;
  cudaStream_t stream = nullptr;
  int64_t* d_buf = nullptr;
  uint32_t cap = 0;
  int last = 0;
  static int fn(void* user, int64_t* values, uint32_t n, int32_t op) {
    NcclMerge* m = (NcclMerge*)user;
    if (n > m->cap) {
      if (m->d_buf) cudaFree(m->d_buf);
      m->d_buf = nullptr;
      if (cudaMalloc(&m->d_buf, (size_t)n * 8) != cudaSuccess) return 1;
      m->cap = n;
    }
    if (cudaMemcpyAsync(m->d_buf, values, (size_t)n * 8, cudaMemcpyHostToDevice, m->stream) !=
        cudaSuccess)
      return 1;
    int rc = nccl().all_reduce(m->d_buf, m->d_buf, n, kInt64, op == 1 ? kMax : kSum, m->comm,
                               m->stream);
    m->last = rc;
    if (rc != 0) return 1;
    if (cudaMemcpyAsync(values, m->d_buf, (size_t)n * 8, cudaMemcpyDeviceToHost, m->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(m->stream) != cudaSuccess)
      return 1;
    return 0;
  }
};

}  // namespace

extern "C" {

pe_status pe_nccl_unique_id(uint8_t* out128, pe_error* err) {
  if (!out128) return PE_ERR_INVALID_ARGUMENT;
  if (!nccl().ok()) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "libnccl.so.2 not available");
    return PE_ERR_INVALID_ARGUMENT;
  }
  UniqueId id;
  int rc = nccl().get_unique_id(&id);
  if (rc != 0) {
    set_err(err, PE_ERR_INTERNAL, std::string("ncclGetUniqueId: ") + nccl().error_string(rc));
    return PE_ERR_INTERNAL;
  }
  std::memcpy(out128, id.internal, 128);
  return PE_OK;
}

pe_status pe_nccl_comm_create(const uint8_t* id128, int32_t nranks, int32_t rank, int32_t device,
                              void** comm, pe_error* err) {
  if (!id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "bad communicator arguments");
    return PE_ERR_INVALID_ARGUMENT;
  }
  if (!nccl().ok()) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "libnccl.so.2 not available");
    return PE_ERR_INVALID_ARGUMENT;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    set_err(err, PE_ERR_CUDA, "cudaSetDevice");
    return PE_ERR_CUDA;
  }
  UniqueId id;
  std::memcpy(id.internal, id128, 128);
  Comm c = nullptr;
  int rc = nccl().comm_init_rank(&c, nranks, id, rank);
  if (rc != 0) {
    set_err(err, PE_ERR_INTERNAL, std::string("ncclCommInitRank: ") + nccl().error_string(rc));
    return PE_ERR_INTERNAL;
  }
  *comm = c;
  return PE_OK;
}

void pe_nccl_comm_destroy(void* comm) {
  if (comm && nccl().ok()) nccl().comm_destroy((Comm)comm);
}

pe_status pe_search_multi(pe_engine* e, const pe_search_config* cfg, uint32_t merge_every,
                          void* comm, pe_plan* out, pe_error* err) {
  if (!e || !comm || !out) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null argument");
    return PE_ERR_INVALID_ARGUMENT;
  }
  if (!nccl().ok()) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "libnccl.so.2 not available");
    return PE_ERR_INVALID_ARGUMENT;
  }
  int nranks = 0, rank = 0;
  if (nccl().comm_count((Comm)comm, &nranks) != 0 || nccl().comm_user_rank((Comm)comm, &rank) != 0) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "not an NCCL communicator");
    return PE_ERR_INVALID_ARGUMENT;
  }
  NcclMerge m;
  m.comm = (Comm)comm;
  if (cudaStreamCreateWithFlags(&m.stream, cudaStreamNonBlocking) != cudaSuccess) {
    set_err(err, PE_ERR_CUDA, "cudaStreamCreate");
    return PE_ERR_CUDA;
  }
  pe_status st = pe_search(e, cfg, merge_every, (uint32_t)rank, &NcclMerge::fn,
                           &m, out, err);
  if (st != PE_OK && m.last != 0)
    set_err(err, PE_ERR_INTERNAL, std::string("ncclAllReduce: ") + nccl().error_string(m.last));
  if (m.d_buf) cudaFree(m.d_buf);
  cudaStreamDestroy(m.stream);
  return st;
}

}  // extern "C"
