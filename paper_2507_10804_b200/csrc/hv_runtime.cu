// hv_runtime.cu — workspace allocation and host/device staging helpers (see hv_internal.h).
#include <algorithm>

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

}  // namespace hvrt
