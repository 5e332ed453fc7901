// comm.cu — the opt-in NCCL entry points of the C ABI: communicator
// setup and the column all-gather of a column-sharded FlashNorm layer.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): in a process where PyTorch already
// loaded its NCCL, the same library instance is reused; without NCCL the library still loads
// and these calls return FN_ERR_NCCL.  nccl.h supplies only the types.
//
//   flashnorm_allgather_columns: ncclAllGather(z_local [M][N_local] -> workspace [P][M][N_local])
//   over NVLink / NVSwitch, then the K7 permute into z_full [M][P * N_local] on the same stream.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/flashnorm.h"
#include "kernels.h"

namespace fn {
fn_status api_fail(fn_status st, const char* fmt, ...);  // api.cu: sets flashnorm_last_error()
}

namespace {

struct NcclApi {
  bool ok = false;
  char why[256] = "";
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*commCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) {
      snprintf(api.why, sizeof(api.why), "libnccl.so.2 not loadable: %s", dlerror());
      return;
    }
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.commCount = reinterpret_cast<decltype(api.commCount)>(dlsym(h, "ncclCommCount"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.errorString = reinterpret_cast<decltype(api.errorString)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.commCount && api.allGather &&
             api.errorString;
    if (!api.ok) snprintf(api.why, sizeof(api.why), "libnccl.so.2 lacks a required symbol");
  });
  return api;
}

fn_status nccl_fail(const char* what, ncclResult_t r) {
  return fn::api_fail(FN_ERR_NCCL, "%s: %s", what, nccl().errorString ? nccl().errorString(r) : "NCCL error");
}

}  // namespace

extern "C" {

fn_status flashnorm_comm_unique_id(void* id_out) {
  if (id_out == nullptr) return fn::api_fail(FN_ERR_NULL, "id_out is NULL");
  const NcclApi& n = nccl();
  if (!n.ok) return fn::api_fail(FN_ERR_NCCL, "%s", n.why);
  ncclUniqueId id;
  const ncclResult_t r = n.getUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  static_assert(sizeof(ncclUniqueId) == FN_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
  memcpy(id_out, &id, sizeof(id));
  return FN_OK;
}

fn_status flashnorm_comm_init(const void* nccl_unique_id, int nranks, int rank, void** comm) {
  if (nccl_unique_id == nullptr || comm == nullptr)
    return fn::api_fail(FN_ERR_NULL, "nccl_unique_id=%p comm=%p: NULL", nccl_unique_id, (void*)comm);
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fn::api_fail(FN_ERR_VALUE, "rank %d of %d ranks", rank, nranks);
  const NcclApi& n = nccl();
  if (!n.ok) return fn::api_fail(FN_ERR_NCCL, "%s", n.why);
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof(id));
  ncclComm_t c = nullptr;
  const ncclResult_t r = n.commInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return nccl_fail("ncclCommInitRank", r);
  *comm = c;
  return FN_OK;
}

fn_status flashnorm_comm_destroy(void* comm) {
  if (comm == nullptr) return FN_OK;
  const NcclApi& n = nccl();
  if (!n.ok) return fn::api_fail(FN_ERR_NCCL, "%s", n.why);
  const ncclResult_t r = n.commDestroy(static_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? FN_OK : nccl_fail("ncclCommDestroy", r);
}

fn_status flashnorm_comm_count(void* comm, int* nranks) {
  if (comm == nullptr || nranks == nullptr) return fn::api_fail(FN_ERR_NULL, "comm=%p nranks=%p: NULL", comm,
                                                                (void*)nranks);
  const NcclApi& n = nccl();
  if (!n.ok) return fn::api_fail(FN_ERR_NCCL, "%s", n.why);
  const ncclResult_t r = n.commCount(static_cast<ncclComm_t>(comm), nranks);
  return r == ncclSuccess ? FN_OK : nccl_fail("ncclCommCount", r);
}

int64_t flashnorm_allgather_workspace_bytes(int64_t P, int64_t M, int64_t N_local, fn_dtype dtype) {
  if (P < 1 || M < 0 || N_local < 1) return 0;
  return P * M * N_local * (dtype == FN_F32 ? 4 : 2);
}

fn_status flashnorm_allgather_columns(const void* z_local, int64_t M, int64_t N_local, fn_dtype dtype, void* z_full,
                                      void* workspace, void* comm, void* stream) {
  if (dtype != FN_BF16 && dtype != FN_F32) return fn::api_fail(FN_ERR_DTYPE, "unknown fn_dtype %d", (int)dtype);
  if (M < 0 || N_local < 1) return fn::api_fail(FN_ERR_SHAPE, "z_local[%lld][%lld]: bad sizes", (long long)M,
                                                (long long)N_local);
  if (z_local == nullptr || z_full == nullptr || workspace == nullptr || comm == nullptr)
    return fn::api_fail(FN_ERR_NULL, "z_local=%p z_full=%p workspace=%p comm=%p: NULL", z_local, z_full, workspace,
                        comm);
  if (workspace == z_full || workspace == z_local) return fn::api_fail(FN_ERR_VALUE, "workspace must not alias z");
  const NcclApi& n = nccl();
  if (!n.ok) return fn::api_fail(FN_ERR_NCCL, "%s", n.why);
  int P = 0;
  ncclResult_t r = n.commCount(static_cast<ncclComm_t>(comm), &P);
  if (r != ncclSuccess) return nccl_fail("ncclCommCount", r);
  if (M == 0) return FN_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  r = n.allGather(z_local, workspace, (size_t)(M * N_local), dtype == FN_BF16 ? ncclBfloat16 : ncclFloat32,
                  static_cast<ncclComm_t>(comm), st);
  if (r != ncclSuccess) return nccl_fail("ncclAllGather", r);
  // [P][M][N_local] -> [M][P * N_local] (K7)
  return flashnorm_gather_columns(workspace, P, M, N_local, dtype, z_full, stream);
}

}  // extern "C"
