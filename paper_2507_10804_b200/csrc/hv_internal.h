// hv_internal.h — runtime context and host helpers shared by hv_api.cu and psido.cu (not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cufft.h>

#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/hv.h"
#include "hv_geo.h"

namespace hvrt {
// A captured sweep (forward or backward time loop of one shot batch).
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;
  void destroy() {
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
  }
};
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};
}  // namespace hvrt

struct hv_ctx {
  hv_config cfg{};
  std::vector<int32_t> src_iz, src_ix, rec_iz, rec_ix;
  std::vector<float> wavelet;
  int nloc = 0;  // shots in this rank's shard
  int dev = 0;
  int nsm = 148;  // SMs of the device (grid sizing)
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  hvk::Geo g{};
  // persistent device arrays
  int *d_srcI = nullptr, *d_srcJ = nullptr, *d_recI = nullptr, *d_recJ = nullptr;
  int *d_trec_beg = nullptr, *d_trec_id = nullptr;
  int *d_trec2_beg = nullptr, *d_trec2_id = nullptr;  // per OX x OZ output tile of the T = 2 kernels
  int *d_tmid_beg = nullptr, *d_tmid_id = nullptr;    // per T = 2 tile: receivers inside its mid region
  float* d_src_amp = nullptr;
  // grow-only workspace
  std::map<std::string, hvrt::DevBuf> ws;
  std::map<std::tuple<int, int, int>, cufftHandle> fft_plans;  // (nz, nx, batch)
  std::map<std::string, hvrt::GraphEntry> graphs;               // captured batch time loops
  std::string err = "";
  hv_stats stats{};
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  int64_t launches = 0;
  cudaEvent_t ev_legacy = nullptr;  // orders calls on the own stream after the legacy default stream (enter)
  void* nccl_comm = nullptr;        // optional ncclComm_t: in-library all-reduce of g / H·v / phi (hv_set_comm)
};

namespace hvrt {
struct OutStage {
  void* user = nullptr;
  void* dev = nullptr;
  size_t bytes = 0;
  bool host = false;
};
int fail(hv_ctx* c, int code, const std::string& msg);
int ws_get(hv_ctx* c, const char* name, size_t bytes, void** out);
bool is_device_ptr(const void* p);
int stage_in(hv_ctx* c, const char* name, const void* p, size_t bytes, const void** dev);
int stage_out(hv_ctx* c, const char* name, void* p, size_t bytes, OutStage* o);
int finish_out(hv_ctx* c, const OutStage& o);
// Entry of every public call: selects the device and, when no stream is bound (the context's own non-blocking
// stream), makes the call wait for the work already queued on the legacy default stream (torch's default stream).
int enter(hv_ctx* c);
// In-library NCCL (dlopen'ed libnccl.so.2; no link-time dependency): sum-all-reduce on the context's stream.
// dtype: 0 float32, 1 float64. Returns HV_OK, or HV_ENCCL with the detail in the context.
int nccl_allreduce_sum(hv_ctx* c, void* buf, size_t count, int dtype);
}  // namespace hvrt

#define CU_TRY(call)                                                                           \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      return hvrt::fail(c, HV_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)
