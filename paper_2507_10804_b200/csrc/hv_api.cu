// hv_api.cu — host runtime + C ABI of libhv.so (include/hv.h).
//
// Runtime responsibilities:
//   - validate the configuration and geometry, precompute per-tile receiver lists;
//   - plan a call: storage mode (FULL / CHECKPOINT), shots in flight, fields per CTA, within the HBM budget;
//   - drive the time loops: forward sweep (fwd_step_kernel), checkpoint saves / segment replays, backward
//     sweep (bwd_step_kernel), with per-sweep CUDA-event timing;
//   - reduce the per-shot accumulators into the caller's outputs; host<->device staging when the caller
//     passes host pointers.
// Nothing here computes the method on the CPU: every step of the path runs in hv_kernels.cuh.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges per call / sweep / reduction (SURVEY.md §5 tracing)

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/hv.h"
#include "hv_internal.h"
#include "hv_kernels.cuh"
#include "hv_t2.cuh"

using namespace hvk;
using namespace hvrt;

namespace {

// 3-D tensor map over planes [nplanes][Nz][P] (logical width Nx: TMA zero-fills outside the padded grid).
int make_tmap(hv_ctx* c, const float* base, long long nplanes, int box_w, int box_h, CUtensorMap* map) {
  const Geo& g = c->g;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.Nx), static_cast<cuuint64_t>(g.Nz),
                        static_cast<cuuint64_t>(nplanes)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(g.P) * 4, static_cast<cuuint64_t>(g.plane) * 4};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = c->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, HV_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return HV_OK;
}

constexpr bool kTwoStepDefault = false;  // T = 2 forward (fwd_t2_kernel) by default
constexpr bool kT2BwdDefault = true;     // with it, the T = 2 adjoint (bwd_t2_kernel) for FULL-store calls
constexpr int kPhiBlocks = 1024;  // residual kernel grid: fixed, so phi's summation order never changes
#ifndef HV_QRES_FG
#define HV_QRES_FG 6
#endif
constexpr int kQresFG = HV_QRES_FG;  // resident-q forward: Born fields per CTA (6 q_k tiles + 3 stages: 2 CTAs/SM)
constexpr int kQresOrder = 0;        // fwd_qres_kernel grid order (FwdParams::qorder)
constexpr bool kQresClusterDefault = false;  // fwd_qres_cl_kernel for K <= 32
// Backward CTAs per (tile, field group): the batch's shots are split into this many parts, each summing its
// imaging terms into its own accumulator copy (finalize adds the copies in a fixed order). 2 halves the last
// partial wave of the backward grid at the cost of one more RED per point and field per launch; measured on
// cfg 1: 1 -> 273.9 us, 2 -> 273.8 us, 4 -> 287 us per launch, so the default keeps one part.
#ifndef HV_BWD_SPLIT
#define HV_BWD_SPLIT 1
#endif
constexpr int kBwdSplit = HV_BWD_SPLIT;

// 3-D tensor map over interior planes [nplanes][nz][PI] (the imaging-factor stores), box bw x bh.
int make_tmap_interior(hv_ctx* c, const float* base, long long nplanes, CUtensorMap* map, int bw = TX, int bh = TZ) {
  const Geo& g = c->g;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(g.PI), static_cast<cuuint64_t>(g.nz),
                        static_cast<cuuint64_t>(nplanes)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(g.PI) * 4, static_cast<cuuint64_t>(g.iplane) * 4};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = c->encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, HV_ECUDA, "cuTensorMapEncodeTiled (interior) failed: " + std::to_string(r));
  return HV_OK;
}

int grid1d(long long n) { return static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16)); }

// ------------------------------------------------------------------------------------------ the plan

enum Want { W_FORWARD = 1, W_GRAD = 2, W_HESS = 4, W_MISFIT = 8 };

// NVTX range for the lifetime of a scope (host-side markers of the call, its sweeps and its reductions).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// CUDA events of one call, destroyed on every return path.
struct Events {
  std::vector<cudaEvent_t> v;
  ~Events() {
    for (cudaEvent_t e : v) cudaEventDestroy(e);
  }
  cudaError_t make(cudaEvent_t* e) {
    const cudaError_t r = cudaEventCreate(e);
    if (r == cudaSuccess) v.push_back(*e);
    return r;
  }
};

struct Plan {
  int store = HV_STORE_FULL;
  int k = 0;           // checkpoint interval
  int nck = 0;         // checkpoints per shot
  int S = 1;           // shots in flight
  int FG = 8;
  int nslot = 1;       // field slots per shot: 0 = background / residual adjoint, 1..K Born / adjoint, K+1 replay
  int nlev = 2;        // pool planes per slot: 2 (parity, single-step kernels) or 4 (T = 2 forward, fwd_t2)
  int nacc = 0;        // accumulator slots
  double per_shot = 0; // bytes
};

int plan_call(hv_ctx* c, int want, int K, int nloc, Plan* pl) {
  const Geo& g = c->g;
  const double F4 = 4.0;
  const bool grad = want & (W_GRAD | W_MISFIT);  // background data + residual per shot
  const bool adjoint = want & (W_GRAD | W_HESS);
  pl->nslot = 1 + K + (adjoint ? 1 : 0);  // + replay slot (CHECKPOINT)
  pl->nacc = adjoint ? 1 + K : 0;
  size_t freeb = 0, totb = 0;
  if (cudaMemGetInfo(&freeb, &totb) != cudaSuccess) {
    cudaGetLastError();
    return fail(c, HV_ECUDA, "cudaMemGetInfo failed");
  }
  // the context's own workspace (grow-only, reused or re-allocated by this call) counts as available
  // (only the buffers of the H·v path: callers such as hv_lowrank_geneig hold their own across hv_hessvec calls)
  static const char* const kPathBufs[] = {"W2",   "imgc", "rec_coef", "scalars", "Q",    "pool", "dborn", "dbg",
                                          "rres", "acc",  "store",    "ring",    "sbuf", "ckpt", "seg", "phi_part",
                                          "bgD"};
  double held = 0;
  for (const char* n : kPathBufs) {
    auto it = c->ws.find(n);
    if (it != c->ws.end()) held += static_cast<double>(it->second.bytes);
  }
  double budget = c->cfg.mem_budget ? static_cast<double>(c->cfg.mem_budget)
                                    : 0.9 * (static_cast<double>(freeb) + held);
  // T = 2 forward (fwd_t2_kernel) for FULL-store and forward-only calls; HV_T2=0/1 overrides the default.
  // Default: forward-only calls (hv_forward / hv_forward_shot / hv_misfit: background only, K = 0) on grids with at
  // least one T = 2 tile per SM. There the single-step launch is latency-bound (0.26 GB per cfg 3 level in 86 us)
  // and two levels per pass win: cfg 3 misfit 85.6 -> 69.8 us per level; on small grids (cfg 1:
  // 95 tiles) the T = 2 grid is too small to fill the GPU and loses (12.8 vs 27.4 us).
  const char* t2 = std::getenv("HV_T2");
  const bool t2_fwd_only = K == 0 && !adjoint && static_cast<long long>(g.ntx2) * g.ntz2 >= c->nsm;
  const bool t2_on = t2 ? std::strcmp(t2, "0") != 0 : (kTwoStepDefault || t2_fwd_only);
  // shared (not per shot): Q, W2, imgc, rec coef, staging of V/HV/m
  const double shared = F4 * (static_cast<double>(K) * g.plane * 2 + g.plane + g.iplane + 4.0 * K * g.nz * g.nx +
                              2.0 * g.nz * g.nx + (double)kBwdSplit * pl->nacc * g.plane) + (1 << 20);
  auto per_shot = [&](int store, int k) {
    double b = F4 * (store == HV_STORE_FULL && t2_on ? 4.0 : 2.0) * pl->nslot * g.plane;  // field pool
    b += F4 * 4.0 * g.plane;  // background increments D (background + replay, 2 planes each)
    b += F4 * (double)K * g.nt * g.nrec;                                        // Born data
    if (grad) b += F4 * 2.0 * g.nt * g.nrec;                                    // data + residual
    if (adjoint) {
      if (store == HV_STORE_FULL) b += F4 * (double)g.nt * g.iplane;
      else if (store == HV_STORE_BOUNDARY) b += F4 * ((double)g.nt * ring_size(g) + 2.0 * g.iplane);
      else b += F4 * (2.0 * ((g.nt - 1 + k - 1) / k) * g.plane + (double)k * g.iplane);
    }
    return b;
  };
  int k = c->cfg.ckpt_interval > 0 ? c->cfg.ckpt_interval
                                   : std::max(1, static_cast<int>(std::lround(std::sqrt((double)g.nt))));
  int store = c->cfg.store;
  if (!adjoint) store = HV_STORE_FULL;  // forward only: nothing stored
  if (store == HV_STORE_AUTO) store = (shared + per_shot(HV_STORE_FULL, k) <= budget) ? HV_STORE_FULL
                                                                                       : HV_STORE_CHECKPOINT;
  if (store != HV_STORE_FULL && store != HV_STORE_CHECKPOINT && store != HV_STORE_BOUNDARY)
    return fail(c, HV_EINVAL, "unknown storage mode " + std::to_string(store));
  pl->store = store;
  pl->nlev = (store == HV_STORE_FULL && t2_on) ? 4 : 2;  // forward-only calls plan store = FULL (nothing kept)
  pl->k = k;
  pl->nck = (g.nt - 1 + k - 1) / k;
  pl->per_shot = per_shot(store, k);
  const double avail = budget - shared;
  int fit = avail > 0 ? static_cast<int>(avail / pl->per_shot) : 0;
  if (fit < 1)
    return fail(c, HV_ENOMEM, "plan needs " + std::to_string((shared + pl->per_shot) / 1e9) +
                                  " GB per shot in flight; budget " + std::to_string(budget / 1e9) + " GB");
  int S = c->cfg.shot_batch > 0 ? c->cfg.shot_batch : 0;
  const int ntiles = g.ntx * g.ntz;
  if (S <= 0) S = 32;  // every CTA loops over the batch's shots: more shots amortise q_k loads and imaging writes
  S = std::min(S, fit);
  S = std::max(1, std::min(S, nloc));
  if (c->cfg.shot_batch <= 0 && nloc > 0) {  // equal batches: ceil(nloc / S) of near-equal size (no 1-shot tail)
    const int nb = (nloc + S - 1) / S;
    S = (nloc + nb - 1) / nb;
  }
  pl->S = S;
  // forward Born fields per unit (groups are near-equal): fewer groups = fewer background recomputes per shot and
  // tile, more groups = finer load balance over the one-wave grid. Auto: the G minimising the busiest CTA's items,
  // ceil(S G tiles / CTAs) * (1 + ceil(K / G)) (cfg 1: G = 4 at 16 shots per rank, G = 5 at 2 shots per rank).
  if (c->cfg.field_group > 0 || K <= 0) {
    pl->FG = std::min(FWD_FG_MAX, c->cfg.field_group > 0 ? c->cfg.field_group : 16);
  } else {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fwd_step_kernel, BX * BY, fwd_smem_bytes(0)) !=
            cudaSuccess || nb < 1) {
      cudaGetLastError();
      nb = 2;
    }
    const long long ncta = static_cast<long long>(nb) * c->nsm;
    long long best = -1;
    int bestG = 1;
    for (int G = 1; G <= K; ++G) {
      const int fg = (K + G - 1) / G;
      if (fg > FWD_FG_MAX || (G > 1 && (K + G - 2) / (G - 1) == fg)) continue;  // same FG as G - 1
      const long long units = static_cast<long long>(pl->S) * G * ntiles;
      const long long cost = ((units + ncta - 1) / ncta) * (1 + fg);
      if (best < 0 || cost < best) best = cost, bestG = G;
    }
    pl->FG = (K + bestG - 1) / bestG;
  }
  // a plan that needs the memory the workspace holds releases it first (buffers are re-allocated at their new
  // sizes by this call; captured graphs refer to the old addresses and are dropped with them)
  if (!c->cfg.mem_budget && shared + pl->S * pl->per_shot > 0.9 * static_cast<double>(freeb) && held > 0) {
    for (auto& kv : c->graphs) kv.second.destroy();
    c->graphs.clear();
    for (const char* n : kPathBufs) {
      auto it = c->ws.find(n);
      if (it == c->ws.end()) continue;
      if (it->second.p) cudaFree(it->second.p);
      c->ws.erase(it);
    }
  }
  return HV_OK;
}

// ------------------------------------------------------------------------------------------ one call

// One call over the shard-local shots [lo, hi) (hi < 0: the whole shard). want: W_FORWARD (d), W_MISFIT (phi
// only), W_GRAD (phi, g), W_HESS (HV); W_GRAD | W_HESS is the fused pass.
int run(hv_ctx* c, int want, const float* m_in, const float* dobs_in, int K, const float* V_in, float* d_user,
        float* g_user, double* phi_user, float* hv_user, int lo = 0, int hi = -1) {
  if (!c) return HV_ESTATE;
  c->err.clear();
  NvtxRange nv_call((want & W_HESS) ? ((want & W_GRAD) ? "hv_gradient_hessvec" : "hv_hessvec")
                    : (want & W_GRAD) ? "hv_gradient" : (want & W_MISFIT) ? "hv_misfit" : "hv_forward");
  if (const int e_ = hvrt::enter(c)) return e_;
  const Geo& g = c->g;
  if (hi < 0) hi = c->nloc;
  const int nloc = hi - lo;  // shots of this call
  const bool grad = want & W_GRAD, hess = want & W_HESS, fwd = want & W_FORWARD, misfit = want & W_MISFIT;
  if (hess && K < 1 && !grad) return fail(c, HV_EINVAL, "K must be >= 1");
  if (K < 0) return fail(c, HV_EINVAL, "K must be >= 0");
  c->launches = 0;
  int64_t launches = 0;
  const size_t mbytes = sizeof(float) * (size_t)g.nz * g.nx;
  const size_t dbytes = sizeof(float) * (size_t)nloc * g.nt * g.nrec;

  Events evg;  // every event of this call; destroyed on all return paths
  cudaEvent_t ev0, ev1;
  CU_TRY(evg.make(&ev0));
  CU_TRY(evg.make(&ev1));
  CU_TRY(cudaEventRecord(ev0, c->stream));

  const float *m = nullptr, *dobs = nullptr, *V = nullptr;
  int st = stage_in(c, "in_m", m_in, mbytes, reinterpret_cast<const void**>(&m));
  if (st) return st;
  if ((grad || misfit) && dbytes > 0) {
    st = stage_in(c, "in_dobs", dobs_in, dbytes, reinterpret_cast<const void**>(&dobs));
    if (st) return st;
  }
  if (K > 0) {
    st = stage_in(c, "in_V", V_in, mbytes * (size_t)K, reinterpret_cast<const void**>(&V));
    if (st) return st;
  }
  OutStage o_d, o_g, o_hv;
  if (fwd && dbytes > 0 && (st = stage_out(c, "out_d", d_user, dbytes, &o_d))) return st;
  if (grad && (st = stage_out(c, "out_g", g_user, mbytes, &o_g))) return st;
  if (K > 0 && (st = stage_out(c, "out_hv", hv_user, mbytes * (size_t)K, &o_hv))) return st;

  Plan pl;
  if ((st = plan_call(c, want, K, nloc, &pl))) return st;
  const int S = pl.S;
  const bool adjoint = grad || K > 0;
  const int nslot = pl.nslot;
  const int replay_slot = nslot - 1;

  // --- a0: model-dependent coefficients
  float *W2, *imgc, *rec_coef;
  unsigned int* vmax;
  double* phi_d;
  if ((st = ws_get(c, "W2", sizeof(float) * g.plane, (void**)&W2))) return st;
  if ((st = ws_get(c, "imgc", sizeof(float) * g.iplane, (void**)&imgc))) return st;
  if ((st = ws_get(c, "rec_coef", sizeof(float) * g.nrec, (void**)&rec_coef))) return st;
  if ((st = ws_get(c, "scalars", 64, (void**)&vmax))) return st;
  unsigned int* vmin = vmax + 1;  // float bits read as int: any value <= 0 makes it <= 0
  phi_d = reinterpret_cast<double*>(reinterpret_cast<char*>(vmax) + 8);
  CU_TRY(cudaMemsetAsync(vmax, 0, 64, c->stream));
  CU_TRY(cudaMemsetAsync(vmin, 0x7f, 4, c->stream));  // 0x7f7f7f7f = 3.4e38
  const float h = c->cfg.h, dt = c->cfg.dt;
  const float dt2_h2 = dt * dt / (h * h), two_dt2_h2 = 2.0f * dt * dt / (h * h);
  model_setup_kernel<<<grid1d(g.plane), 256, 0, c->stream>>>(g, m, dt2_h2, two_dt2_h2, W2, imgc, vmax,
                                                               reinterpret_cast<int*>(vmin));
  rec_coef_kernel<<<(g.nrec + 255) / 256, 256, 0, c->stream>>>(g, m, c->d_recI, c->d_recJ, rec_coef);
  launches += 2;
  unsigned int vbits[2] = {0, 0};
  CU_TRY(cudaMemcpyAsync(vbits, vmax, 8, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(cudaStreamSynchronize(c->stream));
  float vmx, vmn;
  std::memcpy(&vmx, &vbits[0], 4);
  std::memcpy(&vmn, &vbits[1], 4);
  if (!(vmx > 0.0f) || !std::isfinite(vmx) || !(vmn > 0.0f))
    return fail(c, HV_EINVAL, "model must be positive and finite (min " + std::to_string(vmn) + ", max " +
                                  std::to_string(vmx) + ")");
  if (dt * vmx / h > 0.5546f)
    return fail(c, HV_ECFL, "CFL: dt*max(m)/h = " + std::to_string(dt * vmx / h) + " > 0.5546");

  float* Q = nullptr;
  if (K > 0) {
    if ((st = ws_get(c, "Q", sizeof(float) * g.plane * K, (void**)&Q))) return st;
    q_setup_kernel<<<grid1d(g.plane * K), 256, 0, c->stream>>>(g, m, V, K, two_dt2_h2, Q);
    launches++;
  }

  // --- workspace
  float *pool, *dborn = nullptr, *dbg = nullptr, *rres = nullptr, *acc = nullptr, *store = nullptr,
               *ckpt = nullptr, *seg = nullptr, *ring = nullptr, *sbuf = nullptr;
  const long long ringN = ring_size(g);
  const long long planes_per_shot = static_cast<long long>(pl.nlev) * nslot;
  const bool use_t2 = pl.nlev == 4;
  // T = 2 adjoint for FULL-store calls (HV_T2B=0/1 overrides; it needs the 4-plane pool of the T = 2 plan)
  bool use_t2b = use_t2 && pl.store == HV_STORE_FULL && kT2BwdDefault;
  if (const char* e = std::getenv("HV_T2B")) use_t2b = use_t2 && pl.store == HV_STORE_FULL && std::strcmp(e, "0") != 0;
  if ((st = ws_get(c, "pool", sizeof(float) * g.plane * planes_per_shot * S, (void**)&pool))) return st;
  // background increments D = u^n - u^{n-1} ([2: background, replay][S][2][plane])
  float* bgD = nullptr;
  if ((st = ws_get(c, "bgD", sizeof(float) * g.plane * 4 * S, (void**)&bgD))) return st;
  if (K > 0 && (st = ws_get(c, "dborn", sizeof(float) * (size_t)S * K * g.nt * g.nrec, (void**)&dborn))) return st;
  double* phi_part = nullptr;  // per-block partial sums of the residual kernel (fixed-order phi, no atomics)
  if (grad || misfit) {
    if ((st = ws_get(c, "dbg", sizeof(float) * (size_t)S * g.nt * g.nrec, (void**)&dbg))) return st;
    if ((st = ws_get(c, "rres", sizeof(float) * (size_t)S * g.nt * g.nrec, (void**)&rres))) return st;
    if ((st = ws_get(c, "phi_part", sizeof(double) * kPhiBlocks, (void**)&phi_part))) return st;
  }
  if (adjoint) {
    if ((st = ws_get(c, "acc", sizeof(float) * g.plane * pl.nacc * kBwdSplit, (void**)&acc))) return st;
    CU_TRY(cudaMemsetAsync(acc, 0, sizeof(float) * g.plane * pl.nacc * kBwdSplit, c->stream));
    if (pl.store == HV_STORE_FULL) {
      if ((st = ws_get(c, "store", sizeof(float) * g.iplane * g.nt * S, (void**)&store))) return st;
    } else if (pl.store == HV_STORE_BOUNDARY) {
      if ((st = ws_get(c, "ring", sizeof(float) * ringN * g.nt * S, (void**)&ring))) return st;
      if ((st = ws_get(c, "sbuf", sizeof(float) * g.iplane * 2 * S, (void**)&sbuf))) return st;
    } else {
      if ((st = ws_get(c, "ckpt", sizeof(float) * g.plane * 2 * pl.nck * S, (void**)&ckpt))) return st;
      if ((st = ws_get(c, "seg", sizeof(float) * g.iplane * pl.k * S, (void**)&seg))) return st;
    }
  }
  CUtensorMap map_halo, map_tile, map_q;
  if ((st = make_tmap(c, pool, planes_per_shot * S, HX, HZ, &map_halo))) return st;
  if ((st = make_tmap(c, pool, planes_per_shot * S, TX, TZ, &map_tile))) return st;
  if ((st = make_tmap(c, Q ? Q : pool, Q ? K : planes_per_shot * S, TX, TZ, &map_q))) return st;
  CUtensorMap map_w;
  if ((st = make_tmap(c, W2, 1, TX, TZ, &map_w))) return st;
  CUtensorMap map_d;  // background increments, TX x TZ boxes
  if ((st = make_tmap(c, bgD, 4LL * S, TX, TZ, &map_d))) return st;
  CUtensorMap map_halo_t2, map_mid_t2, map_q_t2, map_d_t2;  // T = 2 boxes: 72 x 72 halo, 64 x 64 mid region
  if (use_t2) {
    if ((st = make_tmap(c, pool, planes_per_shot * S, T2_IX, T2_IZ, &map_halo_t2))) return st;
    if ((st = make_tmap(c, pool, planes_per_shot * S, T2_MX, T2_MZ, &map_mid_t2))) return st;
    if ((st = make_tmap(c, Q ? Q : pool, Q ? K : planes_per_shot * S, T2_MX, T2_MZ, &map_q_t2))) return st;
    if ((st = make_tmap(c, bgD, 4LL * S, T2_MX, T2_MZ, &map_d_t2))) return st;
  }
  // s^j tensor map of the backward (FULL store / BOUNDARY level buffer / CHECKPOINT segment)
  CUtensorMap map_sj = map_tile, map_s_t2 = map_tile;
  if (adjoint && use_t2b && (st = make_tmap_interior(c, store, (long long)S * g.nt, &map_s_t2, OX, OZ))) return st;
  if (adjoint) {
    if (pl.store == HV_STORE_FULL) st = make_tmap_interior(c, store, (long long)S * g.nt, &map_sj);
    else if (pl.store == HV_STORE_BOUNDARY) st = make_tmap_interior(c, sbuf, 2LL * S, &map_sj);
    else st = make_tmap_interior(c, seg, (long long)S * pl.k, &map_sj);
    if (st) return st;
  }
  CU_TRY(cudaMemsetAsync(phi_d, 0, sizeof(double), c->stream));

  // --- the shot batches
  const int FG = pl.FG;
  const int Gf = K > 0 ? (K + FG - 1) / FG : 1;
  const int Fb = (grad ? 1 : 0) + K;  // adjoint fields
  const int slot0_b = grad ? 0 : 1;
  const int Gb = std::max(1, (Fb + BWD_FG - 1) / BWD_FG);
  const int fwd_smem = fwd_smem_bytes(0);
  const dim3 block(BX, BY);
  // Forward: one wave of CTAs (resident CTAs per SM x SMs) walking the shot-major unit list (hv_kernels.cuh).
  // Backward: one CTA per (tile, group), each summing its imaging terms over all the batch's shots in registers
  // (a single writer per accumulator address per launch).
  auto fwd_grid = [&](long long units) -> int {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fwd_step_kernel, BX * BY, fwd_smem_bytes(0)) !=
            cudaSuccess || nb < 1) {
      cudaGetLastError();
      nb = 1;
    }
    return static_cast<int>(std::max(1LL, std::min(static_cast<long long>(nb) * c->nsm, units)));
  };
  const long long ntiles_all = static_cast<long long>(g.ntx) * g.ntz;
  const dim3 tiles(g.ntx, g.ntz);
  double ms_f = 0, ms_b = 0;
  std::vector<cudaEvent_t> evs;
  int64_t graph_launches = 0;
  auto new_event = [&](cudaEvent_t* e) -> int {
    CU_TRY(evg.make(e));
    evs.push_back(*e);
    return HV_OK;
  };

  // One shot batch = one enqueue of the whole time loop (forward sweep, checkpoint saves / replays, backward
  // sweep). It is captured once into a CUDA graph per (call signature, buffers) and replayed afterwards.
  int64_t batch_launches = 0;
  // forward sweep kernel (decided here, not inside enqueue_batch: replayed graphs never re-run the lambda)
  bool qres_call = K > 0 && 4.0 * K * g.plane > 48e6;
  if (const char* qe = std::getenv("HV_QRES")) qres_call = K > 0 && std::strcmp(qe, "0") != 0;
  // cluster variant (fwd_qres_cl_kernel): up to 8 groups of <= 4 Born fields per tile in one cluster, the
  // background processed once per tile and shot (K <= 32); HV_QRES_CLUSTER=0/1 overrides
  bool qcl_call = qres_call && kQresClusterDefault && K <= 32;
  if (const char* qc = std::getenv("HV_QRES_CLUSTER")) qcl_call = qres_call && K <= 32 && std::strcmp(qc, "0") != 0;
  const int fwd_kernel_used = use_t2 ? 3 : (qcl_call ? 4 : (qres_call ? 1 : 0));
  // phase 0: forward sweep (+ gather); phase 1: backward sweep. Events may be null (recorded by the caller).
  auto enqueue_batch = [&](int phase, int b0, int Sb, cudaEvent_t e_f0, cudaEvent_t e_f1, cudaEvent_t e_b0,
                           cudaEvent_t e_b1) -> int {
    int64_t launches = 0;
    if (phase == 0) {
      CU_TRY(cudaMemsetAsync(pool, 0, sizeof(float) * g.plane * planes_per_shot * Sb, c->stream));
      CU_TRY(cudaMemsetAsync(bgD, 0, sizeof(float) * g.plane * 2 * Sb, c->stream));  // D^0 = 0
      if (e_f0) CU_TRY(cudaEventRecord(e_f0, c->stream));
    }

    FwdParams fp{};
    fp.g = g;
    fp.pool = pool;
    fp.nslot = nslot;
    fp.bg_slot = 0;
    fp.bg_update = 1;
    fp.born_slot0 = 1;
    fp.K = K;
    fp.S = Sb;
    fp.W2 = W2;
    fp.imgc = imgc;
    fp.shot0 = b0;
    fp.src_I = c->d_srcI;
    fp.src_J = c->d_srcJ;
    fp.src_amp = c->d_src_amp;
    fp.trec_beg = c->d_trec_beg;
    fp.trec_id = c->d_trec_id;
    fp.rec_I = c->d_recI;
    fp.rec_J = c->d_recJ;
    fp.d_born = dborn;
    if (fwd) {
      fp.d_bg = reinterpret_cast<float*>(o_d.dev);
      fp.dbg_shot0 = b0 - lo;
    } else if (grad || misfit) {
      fp.d_bg = dbg;
      fp.dbg_shot0 = 0;
    }
    const bool full = adjoint && pl.store == HV_STORE_FULL;
    const bool boundary = adjoint && pl.store == HV_STORE_BOUNDARY;
    fp.s_shot_stride = full ? g.iplane * g.nt : 0;
    fp.ring_shot_stride = ringN * g.nt;
    fp.dbuf = bgD;
    fp.dplane0 = 0;
    fp.qorder = kQresOrder;
    if (const char* qo = std::getenv("HV_QRES_ORDER")) fp.qorder = std::atoi(qo);  // tuning
    if (boundary && phase == 0) CU_TRY(cudaMemsetAsync(ring, 0, sizeof(float) * ringN * g.nt * Sb, c->stream));
    fp.G = Gf;
    // unit order: one shot per block while Q stays L2-resident; otherwise as many shots per block as keep the
    // resident window (~296 units) at two tile rows or more
    fp.sblk = 1;
    if (4.0 * K * g.plane > 48e6) fp.sblk = std::min(Sb, std::max(2, 296 / std::max(1, 2 * g.ntx)));
    if (const char* sbe = std::getenv("HV_SBLK")) fp.sblk = std::max(1, std::min(Sb, std::atoi(sbe)));  // tuning
    const dim3 gridf(fwd_grid(ntiles_all * Gf * Sb));
    // resident-q forward (q_k read once per launch) for Q too large for L2: HV_QRES=0/1 overrides (tuning)
    const bool qres = qres_call;
    const bool qcl = qcl_call;
    fp.qfg = qcl ? (K + 7) / 8 : std::min(K > 0 ? K : 1, kQresFG);
    if (!qcl)
      if (const char* qf = std::getenv("HV_QFG")) fp.qfg = std::max(1, std::min({K > 0 ? K : 1, 16, std::atoi(qf)}));
    const int Gq = K > 0 ? (K + fp.qfg - 1) / fp.qfg : 1;
    const int qres_smem = QSTAGES_BYTES + BAR_BYTES + fp.qfg * PT_BYTES + (qcl ? 2 * PT_BYTES : 0);
    cudaLaunchConfig_t qcfg{};
    cudaLaunchAttribute qattr[1];
    if (qcl) {
      qcfg.gridDim = dim3(g.ntx, g.ntz, Gq);
      qcfg.blockDim = block;
      qcfg.dynamicSmemBytes = qres_smem;
      qcfg.stream = c->stream;
      qattr[0].id = cudaLaunchAttributeClusterDimension;
      qattr[0].val.clusterDim.x = 1;
      qattr[0].val.clusterDim.y = 1;
      qattr[0].val.clusterDim.z = Gq;
      qcfg.attrs = qattr;
      qcfg.numAttrs = 1;
    }
    if (phase == 0 && use_t2) {
      T2Params t2{};
      t2.g = g;
      t2.nslot = nslot;
      t2.pool = pool;
      t2.bg_update = 1;
      t2.born_slot0 = 1;
      t2.K = K;
      t2.S = Sb;
      t2.G = K > 0 ? (K + T2_QFG - 1) / T2_QFG : 1;
      t2.ntx = g.ntx2;
      t2.ntz = g.ntz2;
      t2.W2 = W2;
      t2.imgc = imgc;
      t2.s_shot_stride = fp.s_shot_stride;
      t2.shot0 = b0;
      t2.src_I = c->d_srcI;
      t2.src_J = c->d_srcJ;
      t2.src_amp = c->d_src_amp;
      t2.trec_beg = c->d_trec2_beg;
      t2.trec_id = c->d_trec2_id;
      t2.rec_I = c->d_recI;
      t2.rec_J = c->d_recJ;
      t2.d_bg = fp.d_bg;
      t2.dbg_shot0 = fp.dbg_shot0;
      t2.d_born = dborn;
      t2.dbuf = bgD;
      t2.dplane0 = 0;
      const dim3 grid2(static_cast<unsigned>(t2.G * g.ntx2 * g.ntz2));
      const dim3 block2(BX, T2_BY);
      for (int n = 0; n <= g.nt - 2; n += 2) {
        t2.n = n;
        t2.two = n + 2 <= g.nt - 1;
        t2.dsel = (n >> 1) & 1;
        t2.s_out = full ? store + (size_t)n * g.iplane : nullptr;
        fwd_t2_kernel<<<grid2, block2, t2_fwd_smem_bytes(), c->stream>>>(map_halo_t2, map_mid_t2, map_q_t2,
                                                                            map_d_t2, t2);
        launches++;
      }
    } else if (phase == 0) {
      for (int n = 0; n <= g.nt - 2; ++n) {
        if (adjoint && pl.store == HV_STORE_CHECKPOINT && n % pl.k == 0) {
          // save (u^n, D^n) per shot; layout ckpt[S][nck][2][plane]
          for (int s = 0; s < Sb; ++s) {
            float* ck = ckpt + ((size_t)s * pl.nck + n / pl.k) * 2 * g.plane;
            CU_TRY(cudaMemcpyAsync(ck, pool + ((size_t)s * planes_per_shot + (n & 1)) * g.plane,
                                   sizeof(float) * g.plane, cudaMemcpyDeviceToDevice, c->stream));
            CU_TRY(cudaMemcpyAsync(ck + g.plane, bgD + (size_t)s * 2 * g.plane, sizeof(float) * g.plane,
                                   cudaMemcpyDeviceToDevice, c->stream));
          }
        }
        fp.n = n;
        fp.s_out = full ? store + (size_t)n * g.iplane : nullptr;
        fp.ring_out = boundary ? ring + (size_t)(n + 1) * ringN : nullptr;
        if (qcl)
          CU_TRY(cudaLaunchKernelEx(&qcfg, fwd_qres_cl_kernel, map_halo, map_tile, map_q, map_d, fp));
        else if (qres)
          fwd_qres_kernel<<<dim3(g.ntx * g.ntz * Gq), block, qres_smem, c->stream>>>(map_halo, map_tile, map_q,
                                                                                      map_d, fp);
        else
          fwd_step_kernel<<<gridf, block, fwd_smem, c->stream>>>(map_halo, map_tile, map_q, map_w, map_d, fp);
        launches++;
      }
    }
    if (phase == 0) {
      if (e_f1) CU_TRY(cudaEventRecord(e_f1, c->stream));
      {
        const dim3 gg((g.nrec + 127) / 128, 1 + K, Sb);
        gather_last_kernel<<<gg, 128, 0, c->stream>>>(g, pool, nslot, pl.nlev, (g.nt - 1) & (pl.nlev - 1),
                                                      fp.dbg_shot0, fp.d_bg, 0,
                                                      dborn, 1, K, c->d_recI, c->d_recJ);
        launches++;
      }
    CU_TRY(cudaGetLastError());
    batch_launches = launches;
    return HV_OK;
    }
    CU_TRY(cudaGetLastError());
    if (grad || misfit) {  // K4: rho = d - d_obs; phi += 1/2 |rho|^2 in a fixed order (block partials, one reducer)
      const long long nres = (long long)Sb * g.nt * g.nrec;
      residual_kernel<<<kPhiBlocks, 256, 0, c->stream>>>(nres, dbg, dobs + (size_t)(b0 - lo) * g.nt * g.nrec, rres,
                                                          phi_part);
      phi_reduce_kernel<<<1, 32, 0, c->stream>>>(phi_part, kPhiBlocks, phi_d);
      launches += 2;
    }
    if (adjoint) {
      if (boundary) {  // keep u^{nt-1}, u^{nt-2} (slot 0) in the replay slot; clear the adjoint slots
        for (int s = 0; s < Sb; ++s) {
          float* base = pool + (size_t)s * planes_per_shot * g.plane;
          CU_TRY(cudaMemcpyAsync(base + (size_t)replay_slot * 2 * g.plane, base, sizeof(float) * 2 * g.plane,
                                 cudaMemcpyDeviceToDevice, c->stream));
          CU_TRY(cudaMemsetAsync(base, 0, sizeof(float) * g.plane * 2 * replay_slot, c->stream));
        }
      } else {
        CU_TRY(cudaMemsetAsync(pool, 0, sizeof(float) * g.plane * planes_per_shot * Sb, c->stream));
      }
      BwdParams bp{};
      bp.g = g;
      bp.pool = pool;
      bp.nslot = nslot;
      bp.nlev = pl.nlev;
      bp.G = Gb;
      bp.nsplit = std::min(kBwdSplit, Sb);
      bp.acc_copy = static_cast<long long>(pl.nacc) * g.plane;
      bp.slot0 = slot0_b;
      bp.F = Fb;
      bp.S = Sb;
      bp.W2 = W2;
      bp.acc = acc;
      bp.rho_res = rres;
      bp.rho_born = dborn;
      bp.Kb = K;
      bp.rec_coef = rec_coef;
      bp.trec_beg = c->d_trec_beg;
      bp.trec_id = c->d_trec_id;
      bp.rec_I = c->d_recI;
      bp.rec_J = c->d_recJ;
      const dim3 gridb(g.ntx, g.ntz, Gb * bp.nsplit);
      if (e_b0) CU_TRY(cudaEventRecord(e_b0, c->stream));
      int cur_b = -1;
      int j_t1 = g.nt - 1;  // first level left for the single-step kernel
      if (use_t2b) {        // FULL store, T = 2 adjoint: levels j, j-1 per launch, j = nt-1, nt-3, ...
        T2BwdParams b2{};
        b2.g = g;
        b2.nslot = nslot;
        b2.pool = pool;
        b2.slot0 = slot0_b;
        b2.F = Fb;
        b2.S = Sb;
        b2.G = Gb;
        b2.ntx = g.ntx2;
        b2.ntz = g.ntz2;
        b2.W2 = W2;
        b2.sj_shot_planes = g.nt;
        b2.acc = acc;
        b2.rho_res = rres;
        b2.rho_born = dborn;
        b2.Kb = K;
        b2.rec_coef = rec_coef;
        b2.tmid_beg = c->d_tmid_beg;
        b2.tmid_id = c->d_tmid_id;
        b2.tout_beg = c->d_trec2_beg;
        b2.tout_id = c->d_trec2_id;
        b2.rec_I = c->d_recI;
        b2.rec_J = c->d_recJ;
        const dim3 gridb2(static_cast<unsigned>(Gb * g.ntx2 * g.ntz2));
        const dim3 blockb2(BX, T2_BY);
        for (int j = g.nt - 1; j >= 1; j -= 2) {
          b2.j = j;
          b2.two = j - 1 >= 1;
          b2.upd0 = j >= 2;
          b2.upd1 = j - 1 >= 2;
          b2.img0 = j <= g.nt - 2;
          b2.img1 = j - 1 >= 1 && j - 1 <= g.nt - 2;
          b2.sj_plane0 = j;
          bwd_t2_kernel<<<gridb2, blockb2, t2_bwd_smem_bytes(), c->stream>>>(map_halo_t2, map_mid_t2, map_s_t2, b2);
          launches++;
        }
        j_t1 = 0;
      }
      for (int j = j_t1; j >= 1; --j) {
        bp.j = j;
        bp.update = j >= 2;
        bp.imaging = j <= g.nt - 2;
        if (bp.imaging) {
          if (boundary) {  // a6: rebuild u^{j-1} and emit s^j
            RevParams rv{};
            rv.g = g;
            rv.nslot = nslot;
            rv.pool = pool;
            rv.slot = replay_slot;
            rv.j = j;
            rv.S = Sb;
            rv.shot0 = b0;
            rv.W2 = W2;
            rv.imgc = imgc;
            rv.s_out = sbuf + (size_t)(j & 1) * Sb * g.iplane;
            rv.s_shot_stride = g.iplane;
            rv.ring_in = ring + (size_t)(j - 1) * ringN;
            rv.ring_shot_stride = ringN * g.nt;
            rv.src_I = c->d_srcI;
            rv.src_J = c->d_srcJ;
            rv.src_amp = c->d_src_amp;
            rev_step_kernel<<<dim3(g.ntx, g.ntz, Sb), block, REV_SMEM_BYTES, c->stream>>>(map_halo, map_tile, rv);
            launches++;
            bp.s_lvl = rv.s_out;
            bp.s_shot_stride = g.iplane;
            bp.sj_plane0 = (long long)(j & 1) * Sb;
            bp.sj_shot_planes = 1;
          } else if (full) {
            bp.s_lvl = store + (size_t)j * g.iplane;
            bp.s_shot_stride = g.iplane * g.nt;
            bp.sj_plane0 = j;
            bp.sj_shot_planes = g.nt;
          } else {
            const int b = (j / pl.k) * pl.k;
            if (b != cur_b) {  // replay segment [b, e) of the background into the segment store
              const int e = std::min(b + pl.k, g.nt - 1);
              for (int s = 0; s < Sb; ++s) {  // u^b -> replay slot plane (b & 1), D^b -> the replay D plane
                const float* ck = ckpt + ((size_t)s * pl.nck + b / pl.k) * 2 * g.plane;
                CU_TRY(cudaMemcpyAsync(pool + ((size_t)s * planes_per_shot + (size_t)replay_slot * 2 + (b & 1)) *
                                                  g.plane,
                                       ck, sizeof(float) * g.plane, cudaMemcpyDeviceToDevice, c->stream));
                CU_TRY(cudaMemcpyAsync(bgD + ((size_t)(Sb + s) * 2) * g.plane, ck + g.plane,
                                       sizeof(float) * g.plane, cudaMemcpyDeviceToDevice, c->stream));
              }
              FwdParams rp = fp;
              rp.bg_slot = replay_slot;
              rp.dplane0 = Sb;
              rp.K = 0;
              rp.d_bg = nullptr;
              rp.d_born = nullptr;
              rp.s_shot_stride = g.iplane * pl.k;
              rp.G = 1;
              const dim3 gridr(fwd_grid(ntiles_all * Sb));
              for (int n = b; n < e; ++n) {
                rp.n = n;
                rp.s_out = seg + (size_t)(n - b) * g.iplane;
                fwd_step_kernel<<<gridr, block, fwd_smem_bytes(0), c->stream>>>(map_halo, map_tile, map_q, map_w,
                                                                                 map_d, rp);
                launches++;
              }
              cur_b = b;
            }
            bp.s_lvl = seg + (size_t)(j - cur_b) * g.iplane;
            bp.s_shot_stride = g.iplane * pl.k;
            bp.sj_plane0 = j - cur_b;
            bp.sj_shot_planes = pl.k;
          }
        }
        bwd_step_kernel<<<gridb, block, BWD_SMEM_BYTES, c->stream>>>(map_halo, map_tile, map_sj, bp);
        launches++;
      }
      CU_TRY(cudaGetLastError());
    } else if (e_b0) {
      CU_TRY(cudaEventRecord(e_b0, c->stream));
    }
    if (e_b1) CU_TRY(cudaEventRecord(e_b1, c->stream));
    batch_launches = launches;
    return HV_OK;
  };
  const bool use_graphs = std::getenv("HV_NO_GRAPHS") == nullptr;
  for (int b0 = lo; b0 < hi; b0 += S) {
    const int Sb = std::min(S, hi - b0);
    cudaEvent_t ev4[4];
    for (int e = 0; e < 4; ++e)
      if ((st = new_event(&ev4[e]))) return st;
    if (!use_graphs) {
      if ((st = enqueue_batch(0, b0, Sb, ev4[0], ev4[1], nullptr, nullptr))) return st;
      launches += batch_launches;
      if ((st = enqueue_batch(1, b0, Sb, nullptr, nullptr, ev4[2], ev4[3]))) return st;
      launches += batch_launches;
      continue;
    }
    for (int phase = 0; phase < 2; ++phase) {
      char keybuf[1024];
      std::snprintf(keybuf, sizeof keybuf,
                    "ph%d w%d K%d S%d Sb%d b%d st%d k%d FG%d nl%d fk%d bk%d p%p W%p i%p Q%p db%p dg%p rr%p a%p s%p "
                    "ck%p sg%p rg%p sb%p do%p od%p rc%p",
                    phase, want, K, S, Sb, b0, pl.store, pl.k, FG, pl.nlev, fwd_kernel_used, use_t2b ? 1 : 0,
                    (void*)pool, (void*)W2, (void*)imgc, (void*)Q,
                    (void*)dborn, (void*)dbg, (void*)rres, (void*)acc, (void*)store, (void*)ckpt, (void*)seg,
                    (void*)ring, (void*)sbuf, (const void*)dobs, fwd ? o_d.dev : nullptr, (void*)rec_coef);
      auto it = c->graphs.find(keybuf);
      if (it == c->graphs.end()) {
        if (c->graphs.size() >= 32) {
          for (auto& kv : c->graphs) kv.second.destroy();
          c->graphs.clear();
        }
        GraphEntry ge;
        CU_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        const int s2 = enqueue_batch(phase, b0, Sb, nullptr, nullptr, nullptr, nullptr);
        cudaGraph_t gr = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(c->stream, &gr);
        if (s2 || ec != cudaSuccess) {
          if (gr) cudaGraphDestroy(gr);
          cudaGetLastError();
          if (s2) return s2;
          return fail(c, HV_ECUDA, std::string("stream capture: ") + cudaGetErrorString(ec));
        }
        const cudaError_t ei = cudaGraphInstantiate(&ge.exec, gr, 0);
        cudaGraphDestroy(gr);
        if (ei != cudaSuccess) {
          cudaGetLastError();
          return fail(c, HV_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ei));
        }
        ge.launches = batch_launches;
        it = c->graphs.emplace(keybuf, ge).first;
      }
      // per-sweep timing events are recorded around the graph launches (events inside graphs cannot be timed)
      NvtxRange nv_sweep(phase == 0 ? "forward_sweep" : "backward_sweep");
      CU_TRY(cudaEventRecord(ev4[2 * phase], c->stream));
      CU_TRY(cudaGraphLaunch(it->second.exec, c->stream));
      CU_TRY(cudaEventRecord(ev4[2 * phase + 1], c->stream));
      launches += it->second.launches;
      ++graph_launches;
    }
  }

  // --- a8 (within the GPU): fixed-order sum over the shots in flight, into the caller's layout
  if (grad) {
    finalize_kernel<<<grid1d((long long)g.nz * g.nx), 256, 0, c->stream>>>(g, acc, kBwdSplit, pl.nacc, 0, 1,
                                                                             reinterpret_cast<float*>(o_g.dev));
    launches++;
  }
  if (K > 0) {
    finalize_kernel<<<grid1d((long long)K * g.nz * g.nx), 256, 0, c->stream>>>(
        g, acc, kBwdSplit, pl.nacc, 1, K, reinterpret_cast<float*>(o_hv.dev));
    launches++;
  }
  CU_TRY(cudaGetLastError());
  // a8 across GPUs: with a communicator attached, sum g / H·v / phi over the ranks in-library (NCCL on this stream)
  if (c->nccl_comm && (grad || misfit || K > 0)) {
    NvtxRange nv_red("nccl_allreduce");
    if (grad && (st = nccl_allreduce_sum(c, o_g.dev, (size_t)g.nz * g.nx, 0))) return st;
    if (K > 0 && (st = nccl_allreduce_sum(c, o_hv.dev, (size_t)K * g.nz * g.nx, 0))) return st;
    if ((st = nccl_allreduce_sum(c, phi_d, 1, 1))) return st;
  }
  if (fwd && dbytes > 0 && (st = finish_out(c, o_d))) return st;
  if (grad && (st = finish_out(c, o_g))) return st;
  if (K > 0 && (st = finish_out(c, o_hv))) return st;
  if (phi_user) CU_TRY(cudaMemcpyAsync(phi_user, phi_d, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(cudaEventRecord(ev1, c->stream));
  CU_TRY(cudaStreamSynchronize(c->stream));
  const std::vector<cudaEvent_t>& tev = evs;
  for (size_t i = 0; i + 3 < tev.size(); i += 4) {
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, tev[i], tev[i + 1]);
    cudaEventElapsedTime(&b, tev[i + 2], tev[i + 3]);
    ms_f += a;
    ms_b += b;
  }
  float tot = 0;
  cudaEventElapsedTime(&tot, ev0, ev1);
  c->launches = launches;
  c->stats.kernel_launches = launches;
  c->stats.graph_launches = graph_launches;
  c->stats.shot_batch = S;
  c->stats.field_group = FG;
  c->stats.store = pl.store;
  c->stats.ckpt_interval = pl.k;
  c->stats.bytes_per_shot = pl.per_shot;
  c->stats.ms_forward = ms_f;
  c->stats.ms_backward = ms_b;
  c->stats.ms_total = tot;
  c->stats.fwd_kernel = fwd_kernel_used;
  c->stats.bwd_kernel = adjoint ? (use_t2b ? 3 : 0) : -1;
  return HV_OK;
}

}  // namespace

// ============================================================================================ C ABI

extern "C" {

int hv_create(const hv_config* cfg, hv_ctx** out) {
  if (!cfg || !out) return HV_EINVAL;
  *out = nullptr;
  hv_ctx* c = new hv_ctx();
  c->cfg = *cfg;
  const hv_config& k = *cfg;
  auto bad = [&](int code, const std::string& m) {
    std::fprintf(stderr, "hv_create: %s\n", m.c_str());
    delete c;
    return code;
  };
  if (k.nz < 1 || k.nx < 1 || k.nt < 3 || k.nsrc < 1 || k.nrec < 1) return bad(HV_EINVAL, "bad sizes");
  if (!(k.h > 0) || !(k.dt > 0) || !(k.v_ref > 0)) return bad(HV_EINVAL, "h, dt, v_ref must be positive");
  if (k.sponge < R) return bad(HV_EINVAL, "sponge must be >= 4 cells");
  if (!k.src_iz || !k.src_ix || !k.rec_iz || !k.rec_ix || !k.wavelet) return bad(HV_EINVAL, "null geometry");
  const int sb = k.src_begin, se = k.src_end ? k.src_end : k.nsrc;
  if (sb < 0 || se > k.nsrc || sb > se) return bad(HV_EINVAL, "bad shot shard");  // empty shard allowed
  c->cfg.src_end = se;
  c->nloc = se - sb;
  for (int i = 0; i < k.nsrc; ++i)
    if (k.src_iz[i] < 0 || k.src_iz[i] >= k.nz || k.src_ix[i] < 0 || k.src_ix[i] >= k.nx)
      return bad(HV_EINVAL, "source index out of range");
  for (int i = 0; i < k.nrec; ++i)
    if (k.rec_iz[i] < 0 || k.rec_iz[i] >= k.nz || k.rec_ix[i] < 0 || k.rec_ix[i] >= k.nx)
      return bad(HV_EINVAL, "receiver index out of range");
  c->src_iz.assign(k.src_iz + sb, k.src_iz + se);
  c->src_ix.assign(k.src_ix + sb, k.src_ix + se);
  c->rec_iz.assign(k.rec_iz, k.rec_iz + k.nrec);
  c->rec_ix.assign(k.rec_ix, k.rec_ix + k.nrec);
  c->wavelet.assign(k.wavelet, k.wavelet + k.nt);
  c->cfg.src_iz = c->cfg.src_ix = c->cfg.rec_iz = c->cfg.rec_ix = nullptr;
  c->cfg.wavelet = nullptr;
  c->dev = k.device;
  c->nccl_comm = k.nccl_comm;

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= k.device || k.device < 0) {
    cudaGetLastError();
    return bad(HV_ECUDA, "no CUDA device (this library has no CPU fallback)");
  }
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, k.device) != cudaSuccess || prop.major < 10)
    return bad(HV_ECUDA, "device is not sm_100-class");
  c->nsm = prop.multiProcessorCount;
  if (cudaSetDevice(k.device) != cudaSuccess) return bad(HV_ECUDA, "cudaSetDevice failed");

  // geometry
  Geo& g = c->g;
  g.nz = k.nz;
  g.nx = k.nx;
  g.W = k.sponge;
  g.Nz = k.nz + 2 * k.sponge;
  g.Nx = k.nx + 2 * k.sponge;
  g.ntx = (g.Nx + TX - 1) / TX;
  g.ntz = (g.Nz + TZ - 1) / TZ;
  g.ntx2 = (g.Nx + OX - 1) / OX;
  g.ntz2 = (g.Nz + OZ - 1) / OZ;
  g.P = std::max(g.ntx * TX, (g.ntx2 * OX + 3) / 4 * 4);
  g.c0 = (g.W / 4) * 4;
  g.PI = ((g.W + g.nx - g.c0) + 3) / 4 * 4;
  g.plane = (long long)g.Nz * g.P;
  if (g.plane >= (1LL << 31)) return bad(HV_EINVAL, "padded grid too large (a plane must have < 2^31 points)");
  g.iplane = (long long)g.nz * g.PI;
  const double eta_max = 3.0 * k.v_ref * std::log(1000.0) / (2.0 * k.sponge * k.h);
  g.kc = static_cast<float>(eta_max * k.dt / (2.0 * (double)k.sponge * k.sponge));
  g.nt = k.nt;
  g.nrec = k.nrec;

  // persistent device arrays
  std::vector<int> sI(c->nloc), sJ(c->nloc), rI(k.nrec), rJ(k.nrec);
  for (int i = 0; i < c->nloc; ++i) {
    sI[i] = c->src_iz[i] + g.W;
    sJ[i] = c->src_ix[i] + g.W;
  }
  for (int i = 0; i < k.nrec; ++i) {
    rI[i] = c->rec_iz[i] + g.W;
    rJ[i] = c->rec_ix[i] + g.W;
  }
  const int ntiles = g.ntx * g.ntz;
  std::vector<int> beg(ntiles + 1, 0), ids(k.nrec);
  for (int i = 0; i < k.nrec; ++i) beg[(rI[i] / TZ) * g.ntx + rJ[i] / TX + 1]++;
  for (int t = 0; t < ntiles; ++t) beg[t + 1] += beg[t];
  {
    std::vector<int> fillp(beg.begin(), beg.end() - 1);
    for (int i = 0; i < k.nrec; ++i) ids[fillp[(rI[i] / TZ) * g.ntx + rJ[i] / TX]++] = i;
  }
  // receivers owned by each output tile of the T = 2 forward kernel
  const int ntiles2 = g.ntx2 * g.ntz2;
  std::vector<int> beg2(ntiles2 + 1, 0), ids2(k.nrec);
  for (int i = 0; i < k.nrec; ++i) beg2[(rI[i] / OZ) * g.ntx2 + rJ[i] / OX + 1]++;
  for (int t = 0; t < ntiles2; ++t) beg2[t + 1] += beg2[t];
  {
    std::vector<int> fillp(beg2.begin(), beg2.end() - 1);
    for (int i = 0; i < k.nrec; ++i) ids2[fillp[(rI[i] / OZ) * g.ntx2 + rJ[i] / OX]++] = i;
  }
  // receivers inside the mid region (output tile + R cells) of each T = 2 tile: injection into the mid level
  std::vector<int> begm(ntiles2 + 1, 0), idsm;
  for (int t = 0; t < ntiles2; ++t) {
    const int tz = t / g.ntx2, txx = t % g.ntx2;
    const int z0 = tz * OZ - R, x0 = txx * OX - R;
    for (int i = 0; i < k.nrec; ++i)
      if (rI[i] >= z0 && rI[i] < z0 + OZ + 2 * R && rJ[i] >= x0 && rJ[i] < x0 + OX + 2 * R) idsm.push_back(i);
    begm[t + 1] = static_cast<int>(idsm.size());
  }
  std::vector<float> amp(k.nt);
  for (int n = 0; n < k.nt; ++n)
    amp[n] = static_cast<float>((double)k.dt * k.dt * (double)c->wavelet[n] / ((double)k.h * k.h));
  auto up = [&](void** d, const void* h, size_t b) -> bool {
    if (cudaMalloc(d, std::max<size_t>(b, 4)) != cudaSuccess) return false;
    return cudaMemcpy(*d, h, b, cudaMemcpyHostToDevice) == cudaSuccess;
  };
  if (!up((void**)&c->d_srcI, sI.data(), sizeof(int) * sI.size()) ||
      !up((void**)&c->d_srcJ, sJ.data(), sizeof(int) * sJ.size()) ||
      !up((void**)&c->d_recI, rI.data(), sizeof(int) * rI.size()) ||
      !up((void**)&c->d_recJ, rJ.data(), sizeof(int) * rJ.size()) ||
      !up((void**)&c->d_trec_beg, beg.data(), sizeof(int) * beg.size()) ||
      !up((void**)&c->d_trec_id, ids.data(), sizeof(int) * ids.size()) ||
      !up((void**)&c->d_trec2_beg, beg2.data(), sizeof(int) * beg2.size()) ||
      !up((void**)&c->d_trec2_id, ids2.data(), sizeof(int) * ids2.size()) ||
      !up((void**)&c->d_tmid_beg, begm.data(), sizeof(int) * begm.size()) ||
      !up((void**)&c->d_tmid_id, idsm.data(), sizeof(int) * std::max<size_t>(1, idsm.size())) ||
      !up((void**)&c->d_src_amp, amp.data(), sizeof(float) * amp.size())) {
    cudaGetLastError();
    hv_destroy(c);
    std::fprintf(stderr, "hv_create: device allocation failed\n");
    return HV_ECUDA;
  }
  if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    hv_destroy(c);
    return HV_ECUDA;
  }
  c->stream = c->own_stream;
  cudaDriverEntryPointQueryResult q{};
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
      q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    hv_destroy(c);
    std::fprintf(stderr, "hv_create: cuTensorMapEncodeTiled unavailable\n");
    return HV_ECUDA;
  }
  c->encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  // opt-in shared memory per CTA (227 KB on sm_100); the tile-size knobs (HV_TZ) can ask for more than a kernel
  // variant will ever be launched with
  auto smem_cap = [](int b) { return std::min(b, 227 * 1024); };
  if (cudaFuncSetAttribute(fwd_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           smem_cap(fwd_smem_bytes(FWD_FG_MAX))) !=
          cudaSuccess ||
      cudaFuncSetAttribute(bwd_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap(BWD_SMEM_BYTES)) !=
          cudaSuccess ||
      cudaFuncSetAttribute(fwd_qres_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           smem_cap(QSTAGES_BYTES + BAR_BYTES + 16 * PT_BYTES)) != cudaSuccess ||
      cudaFuncSetAttribute(fwd_t2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap(t2_fwd_smem_bytes())) !=
          cudaSuccess ||
      cudaFuncSetAttribute(fwd_qres_cl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           smem_cap(QSTAGES_BYTES + BAR_BYTES + 6 * PT_BYTES)) != cudaSuccess ||
      cudaFuncSetAttribute(bwd_t2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap(t2_bwd_smem_bytes())) !=
          cudaSuccess ||
      cudaFuncSetAttribute(rev_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cap(REV_SMEM_BYTES)) !=
          cudaSuccess) {
    cudaGetLastError();
    hv_destroy(c);
    return HV_ECUDA;
  }
  *out = c;
  return HV_OK;
}

int hv_destroy(hv_ctx* c) {
  if (!c) return HV_ESTATE;
  cudaSetDevice(c->dev);
  for (auto& kv : c->ws)
    if (kv.second.p) cudaFree(kv.second.p);
  for (auto& kv : c->fft_plans) cufftDestroy(kv.second);
  for (auto& kv : c->graphs) kv.second.destroy();
  cudaFree(c->d_srcI);
  cudaFree(c->d_srcJ);
  cudaFree(c->d_recI);
  cudaFree(c->d_recJ);
  cudaFree(c->d_trec_beg);
  cudaFree(c->d_trec_id);
  cudaFree(c->d_trec2_beg);
  cudaFree(c->d_trec2_id);
  cudaFree(c->d_tmid_beg);
  cudaFree(c->d_tmid_id);
  cudaFree(c->d_src_amp);
  if (c->ev_legacy) cudaEventDestroy(c->ev_legacy);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
  return HV_OK;
}

int hv_set_stream(hv_ctx* c, void* s) {
  if (!c) return HV_ESTATE;
  c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
  return HV_OK;
}

int hv_set_comm(hv_ctx* c, void* comm) {
  if (!c) return HV_ESTATE;
  c->nccl_comm = comm;
  c->cfg.nccl_comm = comm;
  return HV_OK;
}

int hv_forward(hv_ctx* c, const float* m, float* d) {
  if (!c) return HV_ESTATE;
  return run(c, W_FORWARD, m, nullptr, 0, nullptr, d, nullptr, nullptr, nullptr);
}

int hv_forward_shot(hv_ctx* c, const float* m, int32_t isrc, float* d) {
  if (!c) return HV_ESTATE;
  const int lo = isrc - c->cfg.src_begin;
  if (lo < 0 || lo >= c->nloc)
    return fail(c, HV_EINVAL, "shot " + std::to_string(isrc) + " is not in this context's shard [" +
                                  std::to_string(c->cfg.src_begin) + ", " + std::to_string(c->cfg.src_end) + ")");
  return run(c, W_FORWARD, m, nullptr, 0, nullptr, d, nullptr, nullptr, nullptr, lo, lo + 1);
}

int hv_misfit(hv_ctx* c, const float* m, const float* d_obs, double* phi) {
  if (!c) return HV_ESTATE;
  if (!phi) return fail(c, HV_EINVAL, "null pointer: phi");
  return run(c, W_MISFIT, m, d_obs, 0, nullptr, nullptr, nullptr, phi, nullptr);
}

int hv_gradient(hv_ctx* c, const float* m, const float* d_obs, float* g, double* phi) {
  if (!c) return HV_ESTATE;
  return run(c, W_GRAD, m, d_obs, 0, nullptr, nullptr, g, phi, nullptr);
}

int hv_hessvec(hv_ctx* c, const float* m, int32_t K, const float* V, float* HV) {
  if (!c) return HV_ESTATE;
  if (K < 1) return fail(c, HV_EINVAL, "K must be >= 1");
  return run(c, W_HESS, m, nullptr, K, V, nullptr, nullptr, nullptr, HV);
}

int hv_gradient_hessvec(hv_ctx* c, const float* m, const float* d_obs, int32_t K, const float* V, float* g,
                        double* phi, float* HV) {
  if (!c) return HV_ESTATE;
  if (K < 0) return fail(c, HV_EINVAL, "K must be >= 0");
  return run(c, W_GRAD | (K > 0 ? W_HESS : 0), m, d_obs, K, V, nullptr, g, phi, HV);
}

int hv_get_stats(const hv_ctx* c, hv_stats* out) {
  if (!c) return HV_ESTATE;
  if (!out) return HV_EINVAL;
  *out = c->stats;
  return HV_OK;
}

const char* hv_last_error(const hv_ctx* c) { return c ? c->err.c_str() : "null hv_ctx"; }

}  // extern "C"
