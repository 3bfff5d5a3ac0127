// tp_nccl.cpp -- C-ABI tensor-parallel collectives for a packed job whose base model is
// Megatron-sharded over NVLink (config C4; SURVEY.md section 8(b) "plora_tp_allreduce").
//
// A non-Python host binding libplora (the reference-facing FFI) needs the TP group's
// all-reduce without torch.  NCCL is resolved at run time with dlopen: if the process
// already loaded a libnccl.so.2 (torch does), that copy is reused, so one NCCL serves
// both torch.distributed and libplora; nothing links NCCL at build time and the library
// still loads on a CPU-only host.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/plora.h"

namespace plora {
int set_error(const std::string& msg);
}

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                 cudaStream_t) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  bool ok = false;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.reduce_scatter = reinterpret_cast<decltype(a.reduce_scatter)>(dlsym(h, "ncclReduceScatter"));
    a.reduce = reinterpret_cast<decltype(a.reduce)>(dlsym(h, "ncclReduce"));
    a.broadcast = reinterpret_cast<decltype(a.broadcast)>(dlsym(h, "ncclBroadcast"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_reduce && a.error_string &&
           a.all_gather && a.reduce_scatter && a.reduce && a.broadcast;
  });
  return a;
}

int nccl_fail(const char* what, ncclResult_t r) {
  return plora::set_error(std::string(what) + ": " + api().error_string(r));
}

int nccl_dtype(int32_t dtype, ncclDataType_t* dt) {
  switch (dtype) {
    case PLORA_TP_BF16: *dt = ncclBfloat16; return 0;
    case PLORA_TP_F32: *dt = ncclFloat32; return 0;
    default: return plora::set_error("tp: dtype must be PLORA_TP_BF16 or PLORA_TP_F32");
  }
}

}  // namespace

extern "C" {

PLORA_API int plora_tp_get_unique_id(char* id_out) {
  const NcclApi& a = api();
  if (!a.ok) return plora::set_error("tp: libnccl.so.2 not available");
  if (!id_out) return plora::set_error("tp: id buffer is NULL");
  ncclUniqueId id;
  const ncclResult_t r = a.get_unique_id(&id);
  if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  static_assert(sizeof(ncclUniqueId) == PLORA_TP_ID_BYTES, "ncclUniqueId size");
  memcpy(id_out, &id, sizeof(id));
  return 0;
}

PLORA_API int plora_tp_comm_init(void** comm, const char* id, int32_t nranks, int32_t rank) {
  const NcclApi& a = api();
  if (!a.ok) return plora::set_error("tp: libnccl.so.2 not available");
  if (!comm || !id) return plora::set_error("tp: comm / id is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks) return plora::set_error("tp: bad rank / nranks");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  const ncclResult_t r = a.comm_init_rank(&c, nranks, uid, rank);
  if (r != ncclSuccess) return nccl_fail("ncclCommInitRank", r);
  *comm = c;
  return 0;
}

PLORA_API int plora_tp_comm_destroy(void* comm) {
  const NcclApi& a = api();
  if (!a.ok) return plora::set_error("tp: libnccl.so.2 not available");
  if (!comm) return 0;
  const ncclResult_t r = a.comm_destroy(static_cast<ncclComm_t>(comm));
  return r == ncclSuccess ? 0 : nccl_fail("ncclCommDestroy", r);
}

PLORA_API int plora_tp_allreduce(void* stream, void* comm, void* buf, int64_t count, int32_t dtype, int32_t op) {
  const NcclApi& a = api();
  if (!a.ok) return plora::set_error("tp: libnccl.so.2 not available");
  if (!comm) return plora::set_error("tp: comm is NULL");
  if (count < 0) return plora::set_error("tp: negative count");
  if (count == 0) return 0;
  ncclDataType_t dt;
  switch (dtype) {
    case PLORA_TP_BF16: dt = ncclBfloat16; break;
    case PLORA_TP_F32: dt = ncclFloat32; break;
    default: return plora::set_error("tp: dtype must be PLORA_TP_BF16 or PLORA_TP_F32");
  }
  ncclRedOp_t ro;
  switch (op) {
    case PLORA_TP_SUM: ro = ncclSum; break;
    case PLORA_TP_MAX: ro = ncclMax; break;
    default: return plora::set_error("tp: op must be PLORA_TP_SUM or PLORA_TP_MAX");
  }
  const ncclResult_t r = a.all_reduce(buf, buf, static_cast<size_t>(count), dt, ro, static_cast<ncclComm_t>(comm),
                                      static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? 0 : nccl_fail("ncclAllReduce", r);
}

PLORA_API int plora_tp_allgather(void* stream, void* comm, const void* send, void* recv, int64_t count,
                                 int32_t dtype) {
  const NcclApi& a = api();
  if (!a.ok) return plora::set_error("tp: libnccl.so.2 not available");
  if (!comm) return plora::set_error("tp: comm is NULL");
  if (count <= 0) return count == 0 ? 0 : plora::set_error("tp: negative count");
  ncclDataType_t dt;
  if (nccl_dtype(dtype, &dt)) return 1;
  const ncclResult_t r = a.all_gather(send, recv, static_cast<size_t>(count), dt, static_cast<ncclComm_t>(comm),
                                      static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? 0 : nccl_fail("ncclAllGather", r);
}

PLORA_API int plora_tp_reducescatter(void* stream, void* comm, const void* send, void* recv, int64_t recv_count,
                                     int32_t dtype) {
  const NcclApi& a = api();
  if (!a.ok) return plora::set_error("tp: libnccl.so.2 not available");
  if (!comm) return plora::set_error("tp: comm is NULL");
  if (recv_count <= 0) return recv_count == 0 ? 0 : plora::set_error("tp: negative count");
  ncclDataType_t dt;
  if (nccl_dtype(dtype, &dt)) return 1;
  const ncclResult_t r = a.reduce_scatter(send, recv, static_cast<size_t>(recv_count), dt, ncclSum,
                                          static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? 0 : nccl_fail("ncclReduceScatter", r);
}

PLORA_API int plora_tp_reduce(void* stream, void* comm, void* buf, int64_t count, int32_t dtype, int32_t root) {
  const NcclApi& a = api();
  if (!a.ok) return plora::set_error("tp: libnccl.so.2 not available");
  if (!comm) return plora::set_error("tp: comm is NULL");
  if (count <= 0) return count == 0 ? 0 : plora::set_error("tp: negative count");
  ncclDataType_t dt;
  if (nccl_dtype(dtype, &dt)) return 1;
  const ncclResult_t r = a.reduce(buf, buf, static_cast<size_t>(count), dt, ncclSum, root,
                                  static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? 0 : nccl_fail("ncclReduce", r);
}

PLORA_API int plora_tp_broadcast(void* stream, void* comm, void* buf, int64_t count, int32_t dtype, int32_t root) {
  const NcclApi& a = api();
  if (!a.ok) return plora::set_error("tp: libnccl.so.2 not available");
  if (!comm) return plora::set_error("tp: comm is NULL");
  if (count <= 0) return count == 0 ? 0 : plora::set_error("tp: negative count");
  ncclDataType_t dt;
  if (nccl_dtype(dtype, &dt)) return 1;
  const ncclResult_t r = a.broadcast(buf, buf, static_cast<size_t>(count), dt, root, static_cast<ncclComm_t>(comm),
                                     static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? 0 : nccl_fail("ncclBroadcast", r);
}

}  // extern "C"
