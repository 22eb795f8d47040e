// Multi-GPU exchange of the row-sharded SpMM (the
// reference is single-process): each rank computes a contiguous
// block of Y's rows, one ncclAllGather over NVLink assembles the whole Y in
// rank order (Y is row-major, so the gathered buffer is exactly Y).
//
// NCCL is bound at run time: dlopen("libnccl.so.2") returns the copy already
// mapped into the process (torch's, when torch.distributed initialised it) or
// loads the system one. The library therefore loads (and its CPU tests run)
// where NCCL is absent, and a process never ends up with two NCCLs.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <mutex>

#include "tcsl_internal.cuh"

namespace {

struct Nccl {
  void* handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    n.handle = h;
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_gather;
  });
  return n;
}

thread_local char g_nccl_err[160] = "";

int nccl_status(ncclResult_t r) {
  if (r == ncclSuccess) return TCSL_STATUS_OK;
  const Nccl& n = nccl();
  std::snprintf(g_nccl_err, sizeof g_nccl_err, "nccl: %s", n.error_string ? n.error_string(r) : "error");
  return TCSL_STATUS_CUDA_ERROR;
}

}  // namespace

extern "C" {

int tcsl_cuda_nccl_available(void) { return nccl().ok ? 1 : 0; }

int tcsl_cuda_nccl_unique_id(void* id128) {
  if (!id128) return TCSL_STATUS_INVALID_ARGUMENT;
  if (!nccl().ok) return TCSL_STATUS_UNSUPPORTED;
  ncclUniqueId id;
  const int st = nccl_status(nccl().get_unique_id(&id));
  if (st == TCSL_STATUS_OK) std::memcpy(id128, &id, sizeof id);
  return st;
}

int tcsl_cuda_nccl_comm_init(void** comm, int nranks, const void* id128, int rank) {
  if (!comm || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return TCSL_STATUS_INVALID_ARGUMENT;
  if (!nccl().ok) return TCSL_STATUS_UNSUPPORTED;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  const int st = nccl_status(nccl().comm_init_rank(&c, nranks, id, rank));
  *comm = st == TCSL_STATUS_OK ? static_cast<void*>(c) : nullptr;
  return st;
}

int tcsl_cuda_nccl_comm_destroy(void* comm) {
  if (!comm) return TCSL_STATUS_OK;
  if (!nccl().ok) return TCSL_STATUS_UNSUPPORTED;
  return nccl_status(nccl().comm_destroy(static_cast<ncclComm_t>(comm)));
}

int tcsl_cuda_allgather_rows(const void* dYg, void* dY, size_t rows_per_rank, int n, int out_dtype, void* comm,
                             void* stream) {
  if (!dYg || !dY || !comm || n <= 0) return TCSL_STATUS_INVALID_ARGUMENT;
  if (out_dtype != TCSL_OUT_F32 && out_dtype != TCSL_OUT_F16) return TCSL_STATUS_INVALID_ARGUMENT;
  if (!nccl().ok) return TCSL_STATUS_UNSUPPORTED;
  const size_t count = rows_per_rank * static_cast<size_t>(n);
  return nccl_status(nccl().all_gather(dYg, dY, count, out_dtype == TCSL_OUT_F16 ? ncclFloat16 : ncclFloat32,
                                       static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
