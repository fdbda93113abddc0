// hv_runtime.cu — workspace allocation, host/device staging, call entry ordering and the in-library NCCL
// all-reduce (see hv_internal.h).
#include <dlfcn.h>
#include <nccl.h>  // types and enum values only: the symbols are resolved with dlsym (no link-time dependency)

#include <algorithm>
#include <cstring>
#include <mutex>

#include "hv_internal.h"

namespace hvrt {

int fail(hv_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

// Grow-only named device buffers owned by the context.
int ws_get(hv_ctx* c, const char* name, size_t bytes, void** out) {
  DevBuf& b = c->ws[name];
  if (b.bytes < bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    cudaError_t e = cudaMalloc(&b.p, std::max<size_t>(bytes, 256));
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(c, HV_ENOMEM,
                  std::string("cudaMalloc(") + name + ", " + std::to_string(bytes) + "): " + cudaGetErrorString(e));
    }
    b.bytes = std::max<size_t>(bytes, 256);
  }
  *out = b.p;
  return HV_OK;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Input staging: device pointers pass through; host pointers are copied into a workspace buffer.
int stage_in(hv_ctx* c, const char* name, const void* p, size_t bytes, const void** dev) {
  if (!p) return fail(c, HV_EINVAL, std::string("null pointer: ") + name);
  if (is_device_ptr(p)) {
    *dev = p;
    return HV_OK;
  }
  void* d;
  int st = ws_get(c, name, bytes, &d);
  if (st) return st;
  CU_TRY(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, c->stream));
  *dev = d;
  return HV_OK;
}

// Output staging: device pointers are written directly; host outputs go through a workspace buffer that
// finish_out copies back.
int stage_out(hv_ctx* c, const char* name, void* p, size_t bytes, OutStage* o) {
  if (!p) return fail(c, HV_EINVAL, std::string("null pointer: ") + name);
  o->user = p;
  o->bytes = bytes;
  o->host = !is_device_ptr(p);
  if (!o->host) {
    o->dev = p;
    return HV_OK;
  }
  return ws_get(c, name, bytes, &o->dev);
}

int finish_out(hv_ctx* c, const OutStage& o) {
  if (o.host) CU_TRY(cudaMemcpyAsync(o.user, o.dev, o.bytes, cudaMemcpyDeviceToHost, c->stream));
  return HV_OK;
}

int enter(hv_ctx* c) {
  CU_TRY(cudaSetDevice(c->dev));
  if (c->stream == c->own_stream) {
    if (!c->ev_legacy) CU_TRY(cudaEventCreateWithFlags(&c->ev_legacy, cudaEventDisableTiming));
    CU_TRY(cudaEventRecord(c->ev_legacy, cudaStreamLegacy));
    CU_TRY(cudaStreamWaitEvent(c->own_stream, c->ev_legacy, 0));
  }
  return HV_OK;
}

// ------------------------------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};
NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // a process that already loaded NCCL (torch) keeps its copy; otherwise the loader's libnccl.so.2
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce;
  });
  return api;
}
std::string nccl_err(ncclResult_t r) {
  const NcclApi& a = nccl();
  return a.error_string ? a.error_string(r) : ("ncclResult " + std::to_string(static_cast<int>(r)));
}
}  // namespace

int nccl_allreduce_sum(hv_ctx* c, void* buf, size_t count, int dtype) {
  if (!c->nccl_comm || count == 0) return HV_OK;
  const NcclApi& a = nccl();
  if (!a.ok) return fail(c, HV_ENCCL, "libnccl.so.2 could not be loaded");
  const ncclResult_t r = a.all_reduce(buf, buf, count, dtype == 0 ? ncclFloat32 : ncclFloat64, ncclSum,
                                      static_cast<ncclComm_t>(c->nccl_comm), c->stream);
  if (r != ncclSuccess) return fail(c, HV_ENCCL, "ncclAllReduce: " + nccl_err(r));
  return HV_OK;
}

}  // namespace hvrt

extern "C" {

int hv_nccl_unique_id(void* id_out) {
  if (!id_out) return HV_EINVAL;
  const hvrt::NcclApi& a = hvrt::nccl();
  if (!a.ok) return HV_ENCCL;
  ncclUniqueId id;
  if (a.get_unique_id(&id) != ncclSuccess) return HV_ENCCL;
  std::memcpy(id_out, &id, sizeof id);
  return HV_OK;
}

int hv_nccl_comm_create(int32_t nranks, int32_t rank, const void* id_in, int32_t device, void** comm_out) {
  if (!id_in || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return HV_EINVAL;
  *comm_out = nullptr;
  const hvrt::NcclApi& a = hvrt::nccl();
  if (!a.ok) return HV_ENCCL;
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return HV_ECUDA;
  }
  ncclUniqueId id;
  std::memcpy(&id, id_in, sizeof id);
  ncclComm_t comm = nullptr;
  if (a.comm_init_rank(&comm, nranks, id, rank) != ncclSuccess) return HV_ENCCL;
  *comm_out = comm;
  return HV_OK;
}

int hv_nccl_comm_destroy(void* comm) {
  if (!comm) return HV_EINVAL;
  const hvrt::NcclApi& a = hvrt::nccl();
  if (!a.ok) return HV_ENCCL;
  return a.comm_destroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? HV_OK : HV_ENCCL;
}

}  // extern "C"
