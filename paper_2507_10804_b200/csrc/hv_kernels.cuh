// hv_kernels.cuh — sm_100a device code of the Gauss-Newton H·v hot path.
//
// Every kernel here is a step of SURVEY.md §8(a):
//   fwd_step_kernel  a1 + a2 + a3 (+ a4 FULL write): background leapfrog step, K Born steps sharing L u^n,
//                    point-source injection, receiver sampling, sponge damping, imaging-factor store
//   bwd_step_kernel  a5 + a7 (+ a3 injection): K adjoint steps with fused zero-lag imaging accumulation
//   setup / gather / residual (K4) / finalize (a8 within a GPU) helpers
// The scheme they implement is the one restated in include/hv.h and DESIGN.md §3 (PAPER.md:44-49, 108-112,
// 157-164 for what is computed; the discretisation is our reading, the paper gives none).
//
// B200 design: 2-D tiles of TZ x TX outputs; the (TZ+8) x (TX+8) halo tile of the stencil field is staged
// into shared memory by TMA (cp.async.bulk.tensor.3d; out-of-bounds boxes are zero-filled, which *is* the
// zero-outside-the-padded-grid boundary of the Laplacian), NSTAGE-deep mbarrier ring over the fields a CTA
// handles; pointwise streams (u^{n-1}, q_k, accumulators) are float4, coalesced, no halo.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "hv_geo.h"

namespace hvk {

// ------------------------------------------------------------------------------------------------ PTX

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// try_wait with a suspend-time hint: the warp is parked (not spinning on issue slots) until the phase completes
// or the hint (ns) expires.
#ifndef HV_WAIT_HINT_NS
#define HV_WAIT_HINT_NS 1000000
#endif
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(HV_WAIT_HINT_NS)
      : "memory");
  return ok != 0;
}
// Waits for the phase; a pipeline bug that would hang the GPU traps instead after ~2^34 cycles (~9 s), so the
// call fails with a CUDA error rather than wedging the device. The clock is read once per 64 failed polls so
// the guard costs no issue slots in the common case.
#ifndef HV_WAIT_GUARD
#define HV_WAIT_GUARD 1
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if !HV_WAIT_GUARD
  while (!mbar_try_wait_hint(bar, parity)) {
  }
  return;
#endif
  if (mbar_try_wait_hint(bar, parity)) return;
  const long long t0 = clock64();
  for (uint32_t k = 1;; ++k) {
    if (mbar_try_wait_hint(bar, parity)) return;
    if ((k & 63u) == 0 && clock64() - t0 > (1LL << 34)) __trap();
  }
}
__device__ __forceinline__ void tma_load_3d(float* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                            int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
// Same, with an L2 eviction-priority hint (a policy from createpolicy): q_k tiles are re-read by every shot and
// are loaded evict_last so they stay L2-resident; single-use pointwise tiles go evict_first.
__device__ __forceinline__ void tma_load_3d_hint(float* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                                 int z, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Thread-block clusters: distributed shared memory reads and the cluster-wide barrier.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 ld_dsmem4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float f4(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// Paired fp32 arithmetic (sm_100 FADD2 / FMUL2 / FFMA2: two lanes per instruction, each lane rounded exactly
// like the scalar FADD / FMUL / FFMA, so results are bit-identical to the scalar formulation).
#ifndef HV_PAIRED
#define HV_PAIRED 1
#endif
#if HV_PAIRED
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
// a - b as one FFMA2 (-1 * b + a is exact before the single rounding, so it equals FADD(a, -b))
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __ffma2_rn(b, make_float2(-1.0f, -1.0f), a); }
#else  // scalar lanes (same roundings)
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  return make_float2(__fmaf_rn(a.x, b.x, c.x), __fmaf_rn(a.y, b.y, c.y));
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return make_float2(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y)); }
#endif
__device__ __forceinline__ float2 splat2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 lo2(const float4& v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(const float4& v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float2 half2of(const float4& v, int h) { return h == 0 ? lo2(v) : hi2(v); }

// Unscaled 8th-order Laplacian of this thread's RZ x 4 points from a halo tile in shared memory, as column pairs
// (h = 0: columns 0-1, h = 1: columns 2-3). Thread (tx, ty) owns tile rows ty*RZ .. ty*RZ+RZ-1 and columns
// 4tx .. 4tx+3. t points at element (0, 0) of a buffer of row width W whose element (ty*RZ + r + R, 4tx + i + R) is
// the stencil centre of the thread's point (r, i) (W = HX: a staged halo tile).
//
// Difference form for the two large weights: since 2 a0 + 4 (a1 + a2 + a3 + a4) = 0,
//   L u = sum_{k=1,2} a_k [ (u[x+k] - u) + (u[x-k] - u) + (u[z+k] - u) + (u[z-k] - u) ]
//       + sum_{k=3,4} a_k [ u[x+k] + u[x-k] + u[z+k] + u[z-k] ] - 4 (a3 + a4) u.
// For the smooth fields of this problem (5 Hz at h = 8 m: 37-137 cells per wavelength) |L u| is 1e-2 - 1e-3 of |u|;
// the plain sum 2 a0 u + sum a_k (...) loses that factor of fp32 precision to cancellation, while differences of
// neighbouring values are exact (Sterbenz) and the rounding is then relative to the small differences.
// fp32 numpy on cfg 2 (nt 4000, sharp model, increment-form background): receiver-data error vs the fp64 oracle
// 1.6e-4 (plain) -> 6e-7 (all four terms as differences) -> 1.0e-6 (this form: k = 1, 2 only, ~4.5 fewer FP
// instructions per point than the full difference form).
// DIFF = false: the plain form 2 a0 u + sum_k a_k (pair sums), ~5 fewer FP instructions per point, kept for
// experiments only. Measured on cfg 2 shot 31 at nt 4000 (H·v row 0 / gradient vs the fp64 oracle): DIFF for every
// field 2.4e-5 / 5.2e-6 (the default); plain for Born and adjoint fields 1.1e-5 / 2.3e-4 (the gradient's adjoint,
// driven by the residual at every step, needs DIFF); plain for the Born fields only 6.0e-5 / 5.2e-6 — and only
// 1 % faster at cfg 3, so every field uses DIFF.
template <int W, bool DIFF = true>
__device__ __forceinline__ void lap_points_w(const float* __restrict__ t, int tx, int ty, float2 (&L)[RZ][2],
                                             float2 (&C)[RZ][2]) {
  const int col = R + tx * 4;
  float4 zw[RZ + 2 * R];
#pragma unroll
  for (int k = 0; k < RZ + 2 * R; ++k) zw[k] = ld4(t + (ty * RZ + k) * W + col);
  // z differences shared by the thread's RZ rows (the d = 1, 2 terms below): f1[k] = z[k + 1] - z[k] for
  // k = R - 1 .. R + RZ - 1, f2[k] = z[k + 2] - z[k] for k = R - 2 .. R + RZ - 1 (index k - (R - 2) in the arrays).
  // (z[c+d] - z[c]) + (z[c-d] - z[c]) = f_d[c] - f_d[c-d] exactly (negating a rounded difference is exact), so the
  // bits are those of the per-row form.
  float2 f1[RZ + 2][2], f2[RZ + 2][2];
  if constexpr (DIFF) {
#pragma unroll
    for (int k = 0; k < RZ + 2; ++k)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = k + R - 2;
        if (k >= 1) f1[k][h] = sub2(half2of(zw[a + 1], h), half2of(zw[a], h));
        f2[k][h] = sub2(half2of(zw[a + 2], h), half2of(zw[a], h));
      }
  }
#pragma unroll
  for (int r = 0; r < RZ; ++r) {
    const float* row = t + (ty * RZ + r + R) * W + tx * 4;
    const float4 a = ld4(row);
    const float4 b = zw[r + R];
    const float4 c = ld4(row + 8);
    const float xs[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
    if constexpr (!DIFF) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = 2 * h;
        auto P = [&](int k) { return make_float2(xs[k + i], xs[k + i + 1]); };
        auto Z = [&](int k) { return half2of(zw[r + k], h); };
        auto X = [&](int d) {
          if (d % 2 == 0) return add2(P(4 - d), P(4 + d));
          return make_float2(__fadd_rn(xs[4 - d + i], xs[4 + d + i]), __fadd_rn(xs[5 - d + i], xs[5 + d + i]));
        };
        const float2 ctr = P(4);
        float2 s = mul2(splat2(HV_A1), add2(X(1), add2(Z(3), Z(5))));
        s = fma2(splat2(HV_A2), add2(X(2), add2(Z(2), Z(6))), s);
        s = fma2(splat2(HV_A3), add2(X(3), add2(Z(1), Z(7))), s);
        s = fma2(splat2(HV_A4), add2(X(4), add2(Z(0), Z(8))), s);
        L[r][h] = fma2(splat2(2.0f * HV_A0), ctr, s);
        C[r][h] = ctr;
      }
      continue;
    }
    // first differences e_k = x[k+4] - x[k+3] (k = 0..4) shared by neighbouring points: the d = 1 term of point p
    // is (x[p+1] - x[p]) + (x[p-1] - x[p]) = e_p - e_{p-1} (negation is exact: the same bits, 3 fewer FADDs a row)
    float e[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) e[k] = __fsub_rn(xs[k + 4], xs[k + 3]);
    // d = 2 differences of register-aligned pairs, shared by the two column pairs: gx[m] = x[2m + 4 .. 2m + 5] -
    // x[2m + 2 .. 2m + 3]
    float2 gx[3];
#pragma unroll
    for (int m = 0; m < 3; ++m)
      gx[m] = sub2(make_float2(xs[2 * m + 4], xs[2 * m + 5]), make_float2(xs[2 * m + 2], xs[2 * m + 3]));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = 2 * h;
      auto P = [&](int k) { return make_float2(xs[k + i], xs[k + i + 1]); };
      auto Z = [&](int k) { return half2of(zw[r + k], h); };
      const float2 ctr = P(4);
      // (x+d - c) + (x-d - c) as differences of shared first differences (d = 1: scalar e, the pairs straddle the
      // float4s; d = 2: the aligned pairs gx); d = 3 straddles too and is not shared
      auto DX = [&](int d) {
        if (d == 2) return sub2(gx[h + 1], gx[h]);
        if (d == 1) return make_float2(__fsub_rn(e[i + 1], e[i]), __fsub_rn(e[i + 2], e[i + 1]));
        return make_float2(__fadd_rn(__fsub_rn(xs[4 + d + i], xs[4 + i]), __fsub_rn(xs[4 - d + i], xs[4 + i])),
                           __fadd_rn(__fsub_rn(xs[5 + d + i], xs[5 + i]), __fsub_rn(xs[5 - d + i], xs[5 + i])));
      };
      auto DZ = [&](int d) {
        if (d == 1) return sub2(f1[r + 2][h], f1[r + 1][h]);
        return sub2(f2[r + 2][h], f2[r][h]);
      };
      // plain pair sums for the small outer weights (|a3|, |a4| <= 0.025): their rounding is 60x below the
      // first two terms', which is where the cancellation happened
      auto X = [&](int d) {
        if (d % 2 == 0) return add2(P(4 - d), P(4 + d));
        return make_float2(__fadd_rn(xs[4 - d + i], xs[4 + d + i]), __fadd_rn(xs[5 - d + i], xs[5 + d + i]));
      };
      float2 s = mul2(splat2(HV_A1), add2(DX(1), DZ(1)));
      s = fma2(splat2(HV_A2), add2(DX(2), DZ(2)), s);
      s = fma2(splat2(HV_A3), add2(X(3), add2(Z(1), Z(7))), s);
      s = fma2(splat2(HV_A4), add2(X(4), add2(Z(0), Z(8))), s);
      L[r][h] = fma2(splat2(-4.0f * (HV_A3 + HV_A4)), ctr, s);
      C[r][h] = ctr;
    }
  }
}
__device__ __forceinline__ void lap_points(const float* __restrict__ t, int tx, int ty, float2 (&L)[RZ][2],
                                           float2 (&C)[RZ][2]) {  // Born fields (forward)
  lap_points_w<HX, true>(t, tx, ty, L, C);
}
__device__ __forceinline__ void lap_points_adj(const float* __restrict__ t, int tx, int ty, float2 (&L)[RZ][2],
                                               float2 (&C)[RZ][2]) {  // adjoint fields: the gradient's needs DIFF
  lap_points_w<HX, true>(t, tx, ty, L, C);
}
__device__ __forceinline__ void lap_points_bg(const float* __restrict__ t, int tx, int ty, float2 (&L)[RZ][2],
                                              float2 (&C)[RZ][2]) {  // background field
  lap_points_w<HX, true>(t, tx, ty, L, C);
}

// Sponge coefficient c = kc (d_z^2 + d_x^2), d_z = max(0, W - I, I - (W + nz - 1)) (C10).
__device__ __forceinline__ float sponge_c(const Geo& g, int I, int J) {
  const int dz = max(0, max(g.W - I, I - (g.W + g.nz - 1)));
  const int dx = max(0, max(g.W - J, J - (g.W + g.nx - 1)));
  return g.kc * static_cast<float>(dz * dz + dx * dx);
}

__device__ __forceinline__ bool tile_is_interior(const Geo& g, int x0, int z0) {
  return z0 >= g.W && z0 + TZ <= g.W + g.nz && x0 >= g.W && x0 + TX <= g.W + g.nx;
}

// BOUNDARY store: index of padded cell (I, J) in the RING-cell band around the interior, or -1.
// Layout: top band [R][nx + 2R], bottom band [R][nx + 2R], left band [nz][R], right band [nz][R].
__device__ __forceinline__ int ring_index(const Geo& g, int I, int J) {
  const int zi = I - (g.W - R), xi = J - (g.W - R);
  const int wz = g.nz + 2 * R, wx = g.nx + 2 * R;
  if (zi < 0 || zi >= wz || xi < 0 || xi >= wx) return -1;
  if (zi < R) return zi * wx + xi;
  if (zi >= R + g.nz) return R * wx + (zi - R - g.nz) * wx + xi;
  if (xi < R) return 2 * R * wx + (zi - R) * R + xi;
  if (xi >= R + g.nx) return 2 * R * wx + g.nz * R + (zi - R) * R + (xi - R - g.nx);
  return -1;  // interior
}
__host__ __device__ __forceinline__ int ring_size(const Geo& g) { return 2 * R * (g.nx + 2 * R) + 2 * R * g.nz; }

// ------------------------------------------------------------------------------------------------ forward


struct FwdParams {
  Geo g;
  int nslot;              // pool plane index = ((s_local * nslot) + slot) * 2 + parity
  float* pool;
  int n;                  // this launch computes level n+1 from levels n, n-1
  int bg_slot;            // slot of the background u
  int bg_update;          // write u^{n+1}? (1; 0 = sampling-only use)
  int born_slot0;         // Born field k lives in slot born_slot0 + k
  int K;                  // Born fields
  int S;                  // shots of the batch
  int G;                  // Born-field groups (near-equal sizes, group_begin); work unit = (group, shot, tile)
  int sblk;               // shots per block of the unit order (fwd_unit_decode), 1 <= sblk <= S
  int qfg;                // fwd_qres_kernel: Born fields per CTA (q_k tiles resident in shared memory)
  const float* W2;        // [Nz][P]   dt^2 v^2 / h^2 (0 outside the padded grid)
  const float* imgc;      // [nz][PI]  2 dt^2 / (v h^2); with s_out: store s^n = imgc * Lu^n
  float* s_out;           // level-n slot of the imaging-factor store for s_local = 0, or null
  long long s_shot_stride;
  int shot0;              // shard-local index of batch shot 0
  const int* src_I;       // [local shots] padded source row / column
  const int* src_J;
  const float* src_amp;   // [nt] dt^2 s[n] / h^2
  const int* trec_beg;    // [ntiles + 1] receivers owned by each tile
  const int* trec_id;
  const int* rec_I;
  const int* rec_J;
  float* d_bg;            // background data [..][nt][nrec], row dbg_shot0 + s_local, or null
  int dbg_shot0;
  float* d_born;          // [S][K][nt][nrec] Born data (batch-local) or null
  float* ring_out;        // BOUNDARY store: ring of u^{n+1} for batch shot 0, or null
  long long ring_shot_stride;
  // Background in increment form (compensated leapfrog): the second state plane of the background
  // holds D^n = u^n - u^{n-1} (not u^{n-1}); D is updated in place. D of batch shot s is plane (dplane0 + s) * 2
  // of the D tensor map / buffer dbuf ([.][2][Nz][P]; the second plane of a pair is used by the T = 2 kernel).
  float* dbuf;
  int dplane0;
  int qorder;             // fwd_qres_kernel linear grid order: 0 = tiles (x, then z) fastest, group slowest;
                          // 1 = group fastest (the groups of a tile share its background halo in L2);
                          // q >= 2: blocks of q groups, group fastest within a block
};

// Per-point damping of this thread's points (SP: the tile touches the sponge): (1 - c) and 1 / (1 + c), as
// column pairs h = 0 (columns 0-1), h = 1 (columns 2-3).
template <bool SP>
struct Damp {
  float2 cm[RZ][2], ci_[RZ][2];
  __device__ __forceinline__ void init(const Geo& g, int I0, int J0) {
#pragma unroll
    for (int r = 0; r < RZ; ++r)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float c0 = sponge_c(g, I0 + r, J0 + 2 * h), c1 = sponge_c(g, I0 + r, J0 + 2 * h + 1);
        cm[r][h] = make_float2(1.0f - c0, 1.0f - c1);
        ci_[r][h] = make_float2(1.0f / (1.0f + c0), 1.0f / (1.0f + c1));
      }
  }
  __device__ __forceinline__ float ci(int r, int i) const { return (i & 1) ? ci_[r][i >> 1].y : ci_[r][i >> 1].x; }
  // [2 C - (1 - c) prev + rhs] / (1 + c)
  __device__ __forceinline__ float2 upd(int r, int h, float2 C, float2 prev, float2 rhs) const {
    const float2 t = fma2(splat2(2.0f), C, rhs);
    return mul2(fma2(make_float2(-cm[r][h].x, -cm[r][h].y), prev, t), ci_[r][h]);
  }
  __device__ __forceinline__ float upd1(int r, int i, float C, float prev, float rhs) const {
    const float cmi = (i & 1) ? cm[r][i >> 1].y : cm[r][i >> 1].x;
    return (fmaf(2.0f, C, rhs) - cmi * prev) * ci(r, i);
  }
  // increment form: D^{n+1} = [(1 - c) D^n + rhs] / (1 + c)   (u^{n+1} = u^n + D^{n+1})
  __device__ __forceinline__ float2 updd(int r, int h, float2 D, float2 rhs) const {
    return mul2(fma2(cm[r][h], D, rhs), ci_[r][h]);
  }
};
template <>
struct Damp<false> {
  __device__ __forceinline__ void init(const Geo&, int, int) {}
  __device__ __forceinline__ float2 upd(int, int, float2 C, float2 prev, float2 rhs) const {
    return sub2(fma2(splat2(2.0f), C, rhs), prev);
  }
  __device__ __forceinline__ float upd1(int, int, float C, float prev, float rhs) const {
    return fmaf(2.0f, C, rhs) - prev;
  }
  __device__ __forceinline__ float2 updd(int, int, float2 D, float2 rhs) const { return add2(D, rhs); }
};
template <bool SP>
using BwdDamp = Damp<SP>;
#ifndef HV_BWD_PAIRED
#define HV_BWD_PAIRED 1  // backward arithmetic on column pairs (FFMA2), like the forward
#endif

template <bool SP>
__device__ __forceinline__ float dmp_ci(const Damp<SP>& d, int r, int i) {
  if constexpr (SP) return d.ci(r, i);
  else return 1.0f;
}

// Consumer/producer bookkeeping of an N-deep TMA ring (no divisions in the item loop).
template <int N>
struct RingN {
  int stage = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void advance() {
    if (++stage == N) {
      stage = 0;
      phase ^= 1u;
    }
  }
};
using Ring = RingN<NSTAGE>;     // backward / reverse kernels
using RingF = RingN<NSTAGE_F>;  // forward kernel

// Forward schedule (v4). Work unit = (shot s, field group grp, tile): the background item of shot s on the tile
// (its Laplacian L u^n feeds the group's Born sources) followed by the group's nf Born items. Units are numbered
// shot-major (s, grp, tile) and CTA c of n takes units c, c + n, c + 2n, ...: every launch is one balanced wave
// (no partial last wave), and at any moment the resident CTAs work on the same shot, so halo overlaps between
// neighbouring tiles and the background tile shared by the groups are L2 hits. Each item's q_k tile travels in
// its pipeline stage (q stays L2-resident across shots), so the TMA ring runs across unit boundaries.
#ifndef HV_L2_HINTS
#define HV_L2_HINTS 1
#endif
#ifndef HV_FWD_EMPTY
#define HV_FWD_EMPTY 1  // forward: per-stage empty mbarriers instead of a block barrier per item
#endif
// Forward unit u -> (group, shot, tile). Units are ordered (group, shot block, tile, shot within the block) with
// blocks of p.sblk shots: the resident window of ~296 units then covers 296 / sblk tiles x sblk shots. sblk = 1
// keeps the window on neighbouring tiles of one shot (vertical halo overlaps and the background tile are L2 hits;
// a group's q_k tiles stay L2-resident while Q fits), larger sblk shares each q_k tile among the window's
// shots (Q larger than L2) as long as the window still spans a tile row (sblk <= 296 / ntx).
__device__ __forceinline__ void fwd_unit_decode(const FwdParams& p, int u, int ntl, int& grp, int& s, int& tile) {
  grp = u / (p.S * ntl);
  const int rem = u - grp * p.S * ntl;
  const int blk = rem / (p.sblk * ntl);
  const int rem2 = rem - blk * p.sblk * ntl;
  const int nb = min(p.sblk, p.S - blk * p.sblk);  // shots in this block (the last one may be short)
  tile = rem2 / nb;
  s = blk * p.sblk + (rem2 - tile * nb);
}

// Born fields of forward group grp: [group_begin(grp), group_begin(grp + 1)), G near-equal groups.
__device__ __forceinline__ int group_begin(int K, int G, int grp) { return (K * grp) / G; }

struct FwdProducer {  // thread 0's walk over this CTA's items (decoded once per unit: no divisions per item)
  const CUtensorMap *mh, *mt, *mq, *mw, *md;
  float* stages;
  uint64_t* bars;
  int u, t;                 // current unit, next item within it (0 = background, 1..nf = Born fields)
  int U, nstep, ntl;
  int x0, z0, pl_bg, pl_born, fb, nf, dpl;  // decoded unit
  bool upd;
  uint64_t pol_first, pol_last;
  RingF ring;
  RingF ering;       // stage whose consumers the next refill waits for
  int consumed = 0;  // items this CTA's warp 0 has finished
  // Barrier-free refill (HV_FWD_EMPTY): after warp 0 finishes item c - 1, refill the stage of item c - 2 once
  // all consumer warps have released it (empty barrier), i.e. one item of slack for the slowest warp.
  __device__ __forceinline__ void after_consume(const FwdParams& p, uint64_t* empty) {
    if (++consumed < 2) return;
    mbar_wait(&empty[ering.stage], ering.phase);
    ering.advance();
    issue(p);
  }
  __device__ __forceinline__ void decode(const FwdParams& p) {
    if (u >= U) return;
    int grp, s, tile;
    fwd_unit_decode(p, u, ntl, grp, s, tile);
    const int by = tile / p.g.ntx;
    x0 = (tile - by * p.g.ntx) * TX, z0 = by * TZ;
    fb = group_begin(p.K, p.G, grp);
    nf = group_begin(p.K, p.G, grp + 1) - fb;
    upd = grp == 0 && p.bg_update;
    pl_bg = (s * p.nslot + p.bg_slot) * 2;
    dpl = (p.dplane0 + s) * 2;
    pl_born = (s * p.nslot + p.born_slot0 + fb) * 2;
  }
  __device__ __forceinline__ void issue(const FwdParams& p) {
    if (u >= U) return;
    const int par_n = p.n & 1, par_new = par_n ^ 1;
    float* st = stages + ring.stage * FSTAGE_FLOATS;
    uint64_t* bar = &bars[ring.stage];
    if (t == 0) {  // background: halo u^n, (leader) tile u^{n-1}, and the unit's w = dt^2 v^2 / h^2 tile
      mbar_expect_tx(bar, TILE_BYTES + (upd ? PT_BYTES : 0) + PT_BYTES);
      tma_load_3d(st, mh, bar, x0 - R, z0 - R, pl_bg + par_n);
      tma_load_3d(st + TILE_FLOATS + PT_FLOATS, mw, bar, x0, z0, 0);
#if HV_L2_HINTS
      if (upd) tma_load_3d_hint(st + TILE_FLOATS, md, bar, x0, z0, dpl, pol_first);  // D^n (increment form)
#else
      if (upd) tma_load_3d(st + TILE_FLOATS, md, bar, x0, z0, dpl);
#endif
    } else {
      const int pl = pl_born + 2 * (t - 1);
      mbar_expect_tx(bar, TILE_BYTES + 2 * PT_BYTES);
      tma_load_3d(st, mh, bar, x0 - R, z0 - R, pl + par_n);
#if HV_L2_HINTS
      tma_load_3d_hint(st + TILE_FLOATS, mt, bar, x0, z0, pl + par_new, pol_first);
      tma_load_3d_hint(st + TILE_FLOATS + PT_FLOATS, mq, bar, x0, z0, fb + t - 1, pol_last);
#else
      tma_load_3d(st + TILE_FLOATS, mt, bar, x0, z0, pl + par_new);
      tma_load_3d(st + TILE_FLOATS + PT_FLOATS, mq, bar, x0, z0, fb + t - 1);
#endif
    }
    ring.advance();
    if (++t > nf) {
      t = 0;
      u += nstep;
      decode(p);
    }
  }
};

template <bool SP>
__device__ __forceinline__ void fwd_unit(const FwdParams& p, const float* stages, uint64_t* bars, int s, int grp,
                                         int bx, int by, RingF& cons, FwdProducer& prod) {
  const Geo& g = p.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
  const int x0 = bx * TX, z0 = by * TZ;
  const int fb = group_begin(p.K, p.G, grp);
  const int nf = group_begin(p.K, p.G, grp + 1) - fb;
  const int par_n = p.n & 1, par_new = par_n ^ 1;
  const bool leader = (grp == 0) && p.bg_update;

  const int I0 = z0 + ty * RZ;
  const int J0 = x0 + tx * 4;
  const int so = ty * RZ * TX + tx * 4;                       // smem offset of this thread's first point
  const int go = I0 * g.P + J0;  // within-plane offset of this thread's first point (plane < 2^31 floats)
  float2 w[RZ][2];  // from the background item's stage (TMA), below
  bool row_ok[RZ];
#pragma unroll
  for (int r = 0; r < RZ; ++r) row_ok[r] = !SP || I0 + r < g.Nz;
  Damp<SP> dmp;
  dmp.init(g, I0, J0);
  const int tile_id = by * g.ntx + bx;
  const int rb = p.trec_beg[tile_id], re = p.trec_beg[tile_id + 1];
  const long long data_stride = static_cast<long long>(g.nt) * g.nrec;

  auto release = [&]() {
#if HV_FWD_EMPTY
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&bars[NSTAGE_F + cons.stage]);  // this warp is done with the stage
    cons.advance();
    if (tid == 0) prod.after_consume(p, bars + NSTAGE_F);
#else
    __syncthreads();  // every thread is done with this stage
    cons.advance();
    if (tid == 0) {
      fence_proxy_async();
      prod.issue(p);
    }
#endif
  };
  auto sample = [&](const float* st, float* out) {  // d[n][r] = field^n[rec_r] from the staged tile
    for (int q = rb + tid; q < re; q += NTHREADS) {
      const int rid = p.trec_id[q];
      const int lz = p.rec_I[rid] - z0 + R, lx = p.rec_J[rid] - x0 + R;
      out[static_cast<long long>(p.n) * g.nrec + rid] = st[lz * HX + lx];
    }
  };
  auto store_row = [&](float* dst, int r, float (&v)[4]) {
    if (SP) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (J0 + i >= g.Nx) v[i] = 0.0f;
    }
    if (row_ok[r]) st4(dst + (go + r * g.P), make_float4(v[0], v[1], v[2], v[3]));
  };

  // ---------------- background u of shot s: L u^n (kept for the Born sources), leader updates u
  float2 Lb[RZ][2];
  {
    const float* st = stages + cons.stage * FSTAGE_FLOATS;
    mbar_wait(&bars[cons.stage], cons.phase);
#pragma unroll
    for (int r = 0; r < RZ; ++r) {
      const float4 wv = ld4(st + TILE_FLOATS + PT_FLOATS + so + r * TX);
      w[r][0] = lo2(wv), w[r][1] = hi2(wv);
    }
    float2 C[RZ][2];
    lap_points_bg(st, tx, ty, Lb, C);
    if (leader) {
      float* dst = p.pool + (static_cast<long long>(s * p.nslot + p.bg_slot) * 2 + par_new) * g.plane;
      float* dD = p.dbuf + static_cast<long long>((p.dplane0 + s) * 2) * g.plane;
      const int sI = p.src_I[p.shot0 + s], sJ = p.src_J[p.shot0 + s];
      const float amp = p.src_amp[p.n];
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        const float4 dv = ld4(st + TILE_FLOATS + so + r * TX);  // D^n = u^n - u^{n-1}
        float v[4], dn[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2 d1 = dmp.updd(r, h, half2of(dv, h), mul2(w[r][h], Lb[r][h]));
          dn[2 * h] = d1.x, dn[2 * h + 1] = d1.y;
        }
        if (I0 + r == sI && sJ >= J0 && sJ < J0 + 4) {  // point source dt^2 s[n] / h^2 (/(1 + c))
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (J0 + i == sJ) dn[i] += amp * dmp_ci(dmp, r, i);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // u^{n+1} = u^n + D^{n+1}
          const float2 u = add2(C[r][h], make_float2(dn[2 * h], dn[2 * h + 1]));
          v[2 * h] = u.x, v[2 * h + 1] = u.y;
        }
        if (SP && p.ring_out != nullptr) {  // BOUNDARY store: the ring of u^{n+1}
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int q = ring_index(g, I0 + r, J0 + i);
            if (q >= 0) p.ring_out[s * p.ring_shot_stride + q] = v[i];
          }
        }
        store_row(dst, r, v);
        store_row(dD, r, dn);
      }
      // imaging-factor store s^n = 2 dt^2 / (v h^2) * L~u^n on the interior (FULL store / replay segments)
      const int jc = J0 - g.c0;
      if (p.s_out != nullptr && jc >= 0 && jc < g.PI) {
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
          const int iz = I0 + r - g.W;
          if (iz < 0 || iz >= g.nz) continue;
          const float4 ic = ldg4(p.imgc + static_cast<long long>(iz) * g.PI + jc);
          const float2 o01 = mul2(lo2(ic), Lb[r][0]), o23 = mul2(hi2(ic), Lb[r][1]);
          float o[4] = {o01.x, o01.y, o23.x, o23.y};
          if (SP) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int ix = J0 + i - g.W;
              if (ix < 0 || ix >= g.nx) o[i] = 0.0f;
            }
          }
          st4(p.s_out + s * p.s_shot_stride + static_cast<long long>(iz) * g.PI + jc,
              make_float4(o[0], o[1], o[2], o[3]));
        }
      }
      if (re > rb && p.d_bg) sample(st, p.d_bg + (p.dbg_shot0 + s) * data_stride);
    }
    release();
  }
  // ---------------- Born fields du_k of shot s: source q_k L u^n
  float* born_base = p.pool + (static_cast<long long>(s * p.nslot + p.born_slot0 + fb) * 2 + par_new) * g.plane;
  for (int t = 0; t < nf; ++t) {
    const float* st = stages + cons.stage * FSTAGE_FLOATS;
    mbar_wait(&bars[cons.stage], cons.phase);
    float2 L[RZ][2], C[RZ][2];
    lap_points(st, tx, ty, L, C);
    float* dst = born_base + static_cast<long long>(t) * 2 * g.plane;
    const float* qk = st + TILE_FLOATS + PT_FLOATS + so;
#pragma unroll
    for (int r = 0; r < RZ; ++r) {
      const float4 pv = ld4(st + TILE_FLOATS + so + r * TX);
      const float4 qv = ld4(qk + r * TX);
      float v[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float2 u = dmp.upd(r, h, C[r][h], half2of(pv, h),
                                 fma2(half2of(qv, h), Lb[r][h], mul2(w[r][h], L[r][h])));
        v[2 * h] = u.x, v[2 * h + 1] = u.y;
      }
      store_row(dst, r, v);
    }
    if (re > rb && p.d_born) sample(st, p.d_born + (static_cast<long long>(s) * p.K + fb + t) * data_stride);
    release();
  }
}

#ifndef HV_FWD_MINB
#define HV_FWD_MINB MINB
#endif
#ifndef HV_BWD_SJ_LAST
#define HV_BWD_SJ_LAST 1  // measured: backward 584 -> 566 us per cfg 3 launch, DRAM reads -150 MB
#endif
#ifndef HV_BWD_PREV_FIRST
#define HV_BWD_PREV_FIRST 0
#endif
#ifndef HV_QRES_HINTS
#define HV_QRES_HINTS 0
#endif
#ifndef HV_BWD_MINB
#define HV_BWD_MINB MINB
#endif
__global__ void __launch_bounds__(NTHREADS, HV_FWD_MINB)
    fwd_step_kernel(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mt,
                    const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mw,
                    const __grid_constant__ CUtensorMap md, const FwdParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stages = reinterpret_cast<float*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + FSTAGES_BYTES);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    tma_prefetch_desc(&mh);
    tma_prefetch_desc(&mt);
    tma_prefetch_desc(&mq);
    for (int i = 0; i < NSTAGE_F; ++i) mbar_init(&bars[i], 1);
    for (int i = 0; i < NSTAGE_F; ++i) mbar_init(&bars[NSTAGE_F + i], NTHREADS / 32);  // empty: one per warp
    fence_mbar_init();
  }
  __syncthreads();
  const int ntl = p.g.ntx * p.g.ntz;
  const int U = p.S * p.G * ntl;
  const int nstep = gridDim.x;
  FwdProducer prod;
  prod.mh = &mh, prod.mt = &mt, prod.mq = &mq, prod.mw = &mw, prod.md = &md, prod.stages = stages, prod.bars = bars;
  prod.u = blockIdx.x, prod.t = 0, prod.U = U, prod.nstep = nstep, prod.ntl = ntl;
  prod.pol_first = policy_evict_first(), prod.pol_last = policy_evict_last();
  prod.decode(p);
  if (threadIdx.x == 0 && threadIdx.y == 0)
    for (int i = 0; i < NSTAGE_F; ++i) prod.issue(p);
  RingF cons;
  for (int u = blockIdx.x; u < U; u += nstep) {
    int grp, s, tile;
    fwd_unit_decode(p, u, ntl, grp, s, tile);
    const int bx = tile % p.g.ntx, by = tile / p.g.ntx;
    if (tile_is_interior(p.g, bx * TX, by * TZ))
      fwd_unit<false>(p, stages, bars, s, grp, bx, by, cons, prod);
    else
      fwd_unit<true>(p, stages, bars, s, grp, bx, by, cons, prod);
  }
}

// ------------------------------------------------------------------------------------------------ forward, resident q
// Forward for large Q (Q = K x plane does not fit L2: cfg 3, the cfg 4 grid): one CTA per (tile, group of qfg Born
// fields) loops over all the batch's shots; the group's q_k tiles are loaded into shared memory once and reused by
// every shot (q_k is read from DRAM once per launch), the resident CTAs step through the shots in lockstep (halo
// overlaps are L2 hits). Same paired-fp32 (FFMA2) arithmetic as fwd_step_kernel (bit-identical fields).
// CL: thread-block-cluster variant (fwd_qres_cl_kernel): the G field groups of a tile form one cluster; only the
// leader (group 0) processes the background item and publishes L u^n through distributed shared memory (lbuf,
// double-buffered by shot), so the background halo is loaded and its Laplacian computed once per tile and shot
// instead of once per group. One cluster barrier per shot.
template <bool SP, bool CL>
__device__ __forceinline__ void fwd_qres_body(const CUtensorMap* mh, const CUtensorMap* mt, const CUtensorMap* mq,
                                         const CUtensorMap* md, const FwdParams& p, float* stages, float* qs,
                                         uint64_t* bars, int bx, int by, int grp, float* lbuf = nullptr) {
  const Geo& g = p.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
  const int x0 = bx * TX, z0 = by * TZ;
  const int fb = grp * p.qfg;
  const int nf = max(0, min(p.K, fb + p.qfg) - fb);   // Born fields of this CTA
  const int par_n = p.n & 1, par_new = par_n ^ 1;
  const bool leader = (grp == 0) && p.bg_update;
  const bool has_bg = !CL || grp == 0;                   // this CTA processes the background item
  const int nitems = p.S * ((has_bg ? 1 : 0) + nf);      // per shot: [background], then its Born fields
  uint64_t* qbar = bars + NSTAGE_Q;

  // producer (thread 0): next item (ps, pt) -> stage; pt = 0 is the background item
  int ps = 0, pt = has_bg ? 0 : 1, issued = 0;
  RingN<NSTAGE_Q> prod;
  auto issue_next = [&]() {
    float* st = stages + prod.stage * STAGE_FLOATS;
    const bool upd = pt > 0 || leader;
    const int slot = pt == 0 ? p.bg_slot : p.born_slot0 + fb + pt - 1;
    const int pl = (ps * p.nslot + slot) * 2;
    mbar_expect_tx(&bars[prod.stage], TILE_BYTES + (upd ? PT_BYTES : 0));
#if HV_QRES_HINTS
    // the background halo of a shot is read by every field group's CTA of the tile (different waves): evict_last;
    // the level n-1 / D tiles are single-use: evict_first
    if (pt == 0)
      tma_load_3d_hint(st, mh, &bars[prod.stage], x0 - R, z0 - R, pl + par_n, policy_evict_last());
    else
      tma_load_3d(st, mh, &bars[prod.stage], x0 - R, z0 - R, pl + par_n);
    if (upd && pt == 0)  // background: D^n (increment form)
      tma_load_3d_hint(st + TILE_FLOATS, md, &bars[prod.stage], x0, z0, (p.dplane0 + ps) * 2, policy_evict_first());
    else if (upd)
      tma_load_3d_hint(st + TILE_FLOATS, mt, &bars[prod.stage], x0, z0, pl + par_new, policy_evict_first());
#else
    tma_load_3d(st, mh, &bars[prod.stage], x0 - R, z0 - R, pl + par_n);
    if (upd && pt == 0)  // background: D^n (increment form)
      tma_load_3d(st + TILE_FLOATS, md, &bars[prod.stage], x0, z0, (p.dplane0 + ps) * 2);
    else if (upd)
      tma_load_3d(st + TILE_FLOATS, mt, &bars[prod.stage], x0, z0, pl + par_new);
#endif
    prod.advance();
    if (++pt > nf) {
      pt = has_bg ? 0 : 1;
      ++ps;
    }
    ++issued;
  };
  if (tid == 0) {
    if (nf > 0) {  // q_k tiles of the group, once for all shots
      mbar_expect_tx(qbar, nf * PT_BYTES);
      for (int t = 0; t < nf; ++t) tma_load_3d(qs + t * PT_FLOATS, mq, qbar, x0, z0, fb + t);
    }
    while (issued < min(NSTAGE_Q, nitems)) issue_next();
  }

  const int I0 = z0 + ty * RZ;
  const int J0 = x0 + tx * 4;
  const int so = ty * RZ * TX + tx * 4;                       // smem offset of this thread's first point
  const int go = I0 * g.P + J0;  // within-plane offset of this thread's first point (plane < 2^31 floats)
  float2 w[RZ][2];
#pragma unroll
  for (int r = 0; r < RZ; ++r) {
    const float4 wv = ldg4(p.W2 + static_cast<long long>(min(I0 + r, g.Nz - 1)) * g.P + J0);
    w[r][0] = lo2(wv), w[r][1] = hi2(wv);
  }
  bool row_ok[RZ];
#pragma unroll
  for (int r = 0; r < RZ; ++r) row_ok[r] = !SP || I0 + r < g.Nz;
  Damp<SP> dmp;
  dmp.init(g, I0, J0);
  const int tile_id = by * g.ntx + bx;
  const int rb = p.trec_beg[tile_id], re = p.trec_beg[tile_id + 1];
  const float amp = p.src_amp[p.n];
  const long long data_stride = static_cast<long long>(g.nt) * g.nrec;
  if (nf > 0) mbar_wait(qbar, 0);

  RingN<NSTAGE_Q> cons;
  // a block barrier per item, then thread 0 refills the stage just consumed (NSTAGE_Q items of lead). Per-warp
  // release (empty mbarriers, refill of item c - 1 after item c) measured slower here: 698 vs 594 us per launch
  // on cfg 3 (the refill lost one item of lead and thread 0 waited on the slowest warp).
  auto release = [&]() {
    __syncthreads();  // every thread is done with this stage
    cons.advance();
    if (tid == 0 && issued < nitems) {
      fence_proxy_async();
      issue_next();
    }
  };
  auto sample = [&](const float* st, float* out) {  // d[n][r] = field^n[rec_r] from the staged tile
    for (int q = rb + tid; q < re; q += NTHREADS) {
      const int rid = p.trec_id[q];
      const int lz = p.rec_I[rid] - z0 + R, lx = p.rec_J[rid] - x0 + R;
      out[static_cast<long long>(p.n) * g.nrec + rid] = st[lz * HX + lx];
    }
  };
  auto store_row = [&](float* dst, int r, float (&v)[4]) {
    if (SP) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (J0 + i >= g.Nx) v[i] = 0.0f;
    }
    if (row_ok[r]) st4(dst + (go + r * g.P), make_float4(v[0], v[1], v[2], v[3]));
  };

  float2 Lb[RZ][2];
  for (int s = 0; s < p.S; ++s) {
    // ---------------- background u of shot s: L u^n (kept for the Born sources), leader updates u
    if (has_bg) {
      const float* st = stages + cons.stage * STAGE_FLOATS;
      mbar_wait(&bars[cons.stage], cons.phase);
      float2 C[RZ][2];
      lap_points_bg(st, tx, ty, Lb, C);
      if constexpr (CL) {  // publish L u^n for the cluster's other field groups
#pragma unroll
        for (int r = 0; r < RZ; ++r)
          st4(lbuf + (s & 1) * PT_FLOATS + so + r * TX, make_float4(Lb[r][0].x, Lb[r][0].y, Lb[r][1].x, Lb[r][1].y));
      }
      if (leader) {
        float* dst = p.pool + (static_cast<long long>(s * p.nslot + p.bg_slot) * 2 + par_new) * g.plane;
        float* dD = p.dbuf + static_cast<long long>((p.dplane0 + s) * 2) * g.plane;
        const int sI = p.src_I[p.shot0 + s], sJ = p.src_J[p.shot0 + s];
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
          const float4 dv = ld4(st + TILE_FLOATS + so + r * TX);  // D^n = u^n - u^{n-1}
          float v[4], dn[4];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float2 d1 = dmp.updd(r, h, half2of(dv, h), mul2(w[r][h], Lb[r][h]));
            dn[2 * h] = d1.x, dn[2 * h + 1] = d1.y;
          }
          if (I0 + r == sI && sJ >= J0 && sJ < J0 + 4) {  // point source dt^2 s[n] / h^2 (/(1 + c))
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (J0 + i == sJ) dn[i] += amp * dmp_ci(dmp, r, i);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {  // u^{n+1} = u^n + D^{n+1}
            const float2 u = add2(C[r][h], make_float2(dn[2 * h], dn[2 * h + 1]));
            v[2 * h] = u.x, v[2 * h + 1] = u.y;
          }
          store_row(dD, r, dn);
          if (SP && p.ring_out != nullptr) {  // BOUNDARY store: the ring of u^{n+1}
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int q = ring_index(g, I0 + r, J0 + i);
              if (q >= 0) p.ring_out[s * p.ring_shot_stride + q] = v[i];
            }
          }
          store_row(dst, r, v);
        }
        // imaging-factor store s^n = 2 dt^2 / (v h^2) * L~u^n on the interior (FULL store / replay segments)
        const int jc = J0 - g.c0;
        if (p.s_out != nullptr && jc >= 0 && jc < g.PI) {
#pragma unroll
          for (int r = 0; r < RZ; ++r) {
            const int iz = I0 + r - g.W;
            if (iz < 0 || iz >= g.nz) continue;
            const float4 ic = ldg4(p.imgc + static_cast<long long>(iz) * g.PI + jc);
            const float2 o01 = mul2(lo2(ic), Lb[r][0]), o23 = mul2(hi2(ic), Lb[r][1]);
            float o[4] = {o01.x, o01.y, o23.x, o23.y};
            if (SP) {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int ix = J0 + i - g.W;
                if (ix < 0 || ix >= g.nx) o[i] = 0.0f;
              }
            }
            st4(p.s_out + s * p.s_shot_stride + static_cast<long long>(iz) * g.PI + jc,
                make_float4(o[0], o[1], o[2], o[3]));
          }
        }
        if (re > rb && p.d_bg) sample(st, p.d_bg + (p.dbg_shot0 + s) * data_stride);
      }
      release();
    }
    if constexpr (CL) {
      cluster_sync_all();  // lbuf[s & 1] of the leader is complete (and every CTA is done with shot s - 1's)
      if (!has_bg) {
        const uint32_t src = mapa_shared(smem_u32(lbuf + (s & 1) * PT_FLOATS + so), 0);
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
          const float4 v = ld_dsmem4(src + r * TX * 4);
          Lb[r][0] = lo2(v), Lb[r][1] = hi2(v);
        }
      }
    }
    // ---------------- Born fields du_k of shot s: source q_k L u^n
    float* born_base = p.pool + (static_cast<long long>(s * p.nslot + p.born_slot0 + fb) * 2 + par_new) * g.plane;
    for (int t = 0; t < nf; ++t) {
      const float* st = stages + cons.stage * STAGE_FLOATS;
      mbar_wait(&bars[cons.stage], cons.phase);
      float2 L[RZ][2], C[RZ][2];
      lap_points(st, tx, ty, L, C);
      float* dst = born_base + static_cast<long long>(t) * 2 * g.plane;
      const float* qk = qs + t * PT_FLOATS + so;
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        const float4 pv = ld4(st + TILE_FLOATS + so + r * TX);
        const float4 qv = ld4(qk + r * TX);
        float v[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2 u = dmp.upd(r, h, C[r][h], half2of(pv, h),
                                   fma2(half2of(qv, h), Lb[r][h], mul2(w[r][h], L[r][h])));
          v[2 * h] = u.x, v[2 * h + 1] = u.y;
        }
        store_row(dst, r, v);
      }
      if (re > rb && p.d_born) sample(st, p.d_born + (static_cast<long long>(s) * p.K + fb + t) * data_stride);
      release();
    }
  }
}

#ifndef HV_FWD_MINB
#define HV_FWD_MINB 2
#endif
#ifndef HV_BWD_MINB
#define HV_BWD_MINB 2
#endif
__global__ void __launch_bounds__(NTHREADS, HV_FWD_MINB)
    fwd_qres_kernel(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mt,
                    const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap md,
                    const FwdParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stages = reinterpret_cast<float*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + QSTAGES_BYTES);
  float* qs = reinterpret_cast<float*>(smem_raw + QSTAGES_BYTES + BAR_BYTES);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    tma_prefetch_desc(&mh);
    tma_prefetch_desc(&mt);
    tma_prefetch_desc(&mq);
    for (int i = 0; i < NSTAGE_Q + 1; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // linear grid of ntx * ntz * G CTAs
  const int ntl = p.g.ntx * p.g.ntz;
  const int G = (gridDim.x + ntl - 1) / ntl;
  int grp, tile;
  if (p.qorder == 1) {
    grp = blockIdx.x % G, tile = blockIdx.x / G;
  } else if (p.qorder >= 2) {  // blocks of qorder groups, group fastest within a block: (block, tile, group)
    const int blk = blockIdx.x / (p.qorder * ntl), base = blk * p.qorder;
    const int gs = min(p.qorder, G - base), rem = blockIdx.x - blk * p.qorder * ntl;
    tile = rem / gs, grp = base + (rem - tile * gs);
  } else {
    grp = blockIdx.x / ntl, tile = blockIdx.x - grp * ntl;
  }
  const int by = tile / p.g.ntx, bx = tile - by * p.g.ntx;
  if (tile_is_interior(p.g, bx * TX, by * TZ))
    fwd_qres_body<false, false>(&mh, &mt, &mq, &md, p, stages, qs, bars, bx, by, grp);
  else
    fwd_qres_body<true, false>(&mh, &mt, &mq, &md, p, stages, qs, bars, bx, by, grp);
}

// Cluster variant: grid (ntx, ntz, G) launched with cluster dimensions (1, 1, G), G <= 8; p.qfg Born fields per
// group. Shared memory: stages | barriers | q tiles (qfg) | lbuf (2 planes of the tile's L u^n).
__global__ void __launch_bounds__(NTHREADS, HV_FWD_MINB)
    fwd_qres_cl_kernel(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mt,
                       const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap md,
                       const FwdParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stages = reinterpret_cast<float*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + QSTAGES_BYTES);
  float* qs = reinterpret_cast<float*>(smem_raw + QSTAGES_BYTES + BAR_BYTES);
  float* lbuf = qs + p.qfg * PT_FLOATS;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    tma_prefetch_desc(&mh);
    tma_prefetch_desc(&mt);
    tma_prefetch_desc(&mq);
    for (int i = 0; i < NSTAGE_Q + 1; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int bx = blockIdx.x, by = blockIdx.y, grp = blockIdx.z;  // cluster (1, 1, G): rank = group
  if (tile_is_interior(p.g, bx * TX, by * TZ))
    fwd_qres_body<false, true>(&mh, &mt, &mq, &md, p, stages, qs, bars, bx, by, grp, lbuf);
  else
    fwd_qres_body<true, true>(&mh, &mt, &mq, &md, p, stages, qs, bars, bx, by, grp, lbuf);
  cluster_sync_all();  // the leader's lbuf must outlive every remote read
}

// ------------------------------------------------------------------------------------------------ backward

struct BwdParams {
  Geo g;
  int nslot;
  int nlev;               // planes per slot (2: parity; 4: level & 3, after/between two-step launches)
  float* pool;
  int j;                  // computes lambda^j from lambda^{j+1} (halo) and lambda^{j+2} (pointwise)
  int update;             // compute lambda^j (j >= 2; lambda^1 is never used)
  int imaging;            // accumulate s^j lambda^{j+1} (j <= nt-2)
  int slot0, F;           // adjoint fields in slots slot0 .. slot0 + F - 1; BWD_FG per group
  int S;                  // shots of the batch
  int G;                  // field groups (grid.z = nsplit x G)
  int nsplit;             // shot parts: part h loops over shots [h S / nsplit, (h+1) S / nsplit)
  long long acc_copy;     // floats between the per-part accumulator copies (single writer per copy and launch)
  const float* W2;
  const float* s_lvl;     // s^j for batch shot 0 (two-step kernel / reference of the plane indices below)
  long long s_shot_stride;
  long long sj_plane0;    // plane of s^j for batch shot 0 in the s-tensor map (interior planes [nz][PI])
  int sj_shot_planes;     // planes between consecutive shots' s^j
  float* acc;             // [nacc][Nz][P], index by slot (summed over shots and batches)
  const float* rho_res;   // slot 0 injection data [S][nt][nrec] (gradient), or null
  const float* rho_born;  // slot k >= 1 injection data [S][K][nt][nrec]
  int Kb;                 // K of rho_born
  const float* rec_coef;  // [nrec] v^2 / (1 + c) at each receiver
  const int* trec_beg;
  const int* trec_id;
  const int* rec_I;
  const int* rec_J;
};

template <bool SP>
__device__ __forceinline__ void bwd_body(const CUtensorMap* mh, const CUtensorMap* mt, const CUtensorMap* msj, const BwdParams& p,
                                         float* stages, uint64_t* bars) {
  const Geo& g = p.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
  const int x0 = blockIdx.x * TX, z0 = blockIdx.y * TZ;
  // grid.z = (shot part h) x (field group): part h owns the batch's shots [sb, se) and its own accumulator copy
  const int h = blockIdx.z / p.G, grp = blockIdx.z - h * p.G;
  const int sb = (h * p.S) / p.nsplit, se = ((h + 1) * p.S) / p.nsplit;
  const int fb = grp * BWD_FG;
  const int nf = min(p.F, fb + BWD_FG) - fb;
  if (nf <= 0 || se <= sb) return;
  const int nitems = (se - sb) * nf;
  // planes of lambda^{j+1} (halo), lambda^{j+2} (pointwise) and lambda^j (written): with 2 planes per field
  // lambda^j overwrites lambda^{j+2} in place; with 4 (after T = 2 forward sweeps) they are distinct planes
  const int par_in = (p.j + 1) & (p.nlev - 1), par_out = p.j & (p.nlev - 1), par_prev = (p.j + 2) & (p.nlev - 1);
  int ps = sb, pt = 0, issued = 0;
  Ring prod;
  auto issue_next = [&]() {
    float* st = stages + prod.stage * BSTAGE_FLOATS;
    const int pl = (ps * p.nslot + p.slot0 + fb + pt) * p.nlev;
    const bool with_sj = p.imaging && pt == 0;  // s^j of the shot travels with its first field's stage
    mbar_expect_tx(&bars[prod.stage], TILE_BYTES + (p.update ? PT_BYTES : 0) + (with_sj ? PT_BYTES : 0));
    tma_load_3d(st, mh, &bars[prod.stage], x0 - R, z0 - R, pl + par_in);
#if HV_BWD_PREV_FIRST
    if (p.update)  // lambda^{j+2}: single use
      tma_load_3d_hint(st + TILE_FLOATS, mt, &bars[prod.stage], x0, z0, pl + par_prev, policy_evict_first());
#else
    if (p.update) tma_load_3d(st + TILE_FLOATS, mt, &bars[prod.stage], x0, z0, pl + par_prev);
#endif
    if (with_sj) {  // interior store: padded (x0, z0) is interior (x0 - c0, z0 - W); outside -> TMA zero fill
      const int sj_plane = static_cast<int>(p.sj_plane0 + static_cast<long long>(ps) * p.sj_shot_planes);
#if HV_BWD_SJ_LAST
      // s^j of a shot is read by every field group's CTA of the tile, in different waves: keep it in L2
      tma_load_3d_hint(st + TILE_FLOATS + PT_FLOATS, msj, &bars[prod.stage], x0 - g.c0, z0 - g.W, sj_plane,
                       policy_evict_last());
#else
      tma_load_3d(st + TILE_FLOATS + PT_FLOATS, msj, &bars[prod.stage], x0 - g.c0, z0 - g.W, sj_plane);
#endif
    }
    prod.advance();
    if (++pt == nf) {
      pt = 0;
      ++ps;
    }
    ++issued;
  };
  if (tid == 0) {
    while (issued < min(NSTAGE, nitems)) issue_next();
  }
  const int I0 = z0 + ty * RZ;
  const int J0 = x0 + tx * 4;
  const int so = ty * RZ * TX + tx * 4;
  const int go = I0 * g.P + J0;  // within-plane offset (plane < 2^31 floats)
  const int jc = J0 - g.c0;
#if HV_BWD_PAIRED
  float2 w2[RZ][2];
#endif
  float w[RZ][4];
  bool img_rows[RZ], row_ok[RZ];
  bool any_img = false;
#pragma unroll
  for (int r = 0; r < RZ; ++r) {
    const int I = I0 + r;
    const float4 wv = ldg4(p.W2 + static_cast<long long>(min(I, g.Nz - 1)) * g.P + J0);
    w[r][0] = wv.x, w[r][1] = wv.y, w[r][2] = wv.z, w[r][3] = wv.w;
#if HV_BWD_PAIRED
    w2[r][0] = lo2(wv), w2[r][1] = hi2(wv);
#endif
    const int iz = I - g.W;
    img_rows[r] = p.imaging && iz >= 0 && iz < g.nz && J0 + 3 >= g.W && J0 < g.W + g.nx && jc >= 0 &&
                  jc < g.PI;
    any_img |= img_rows[r];
    row_ok[r] = !SP || I < g.Nz;
  }
  BwdDamp<SP> dmp;
  dmp.init(g, I0, J0);
  const int tile_id = blockIdx.y * g.ntx + blockIdx.x;
  const int rb = p.trec_beg[tile_id], re = p.trec_beg[tile_id + 1];
  const long long data_stride = static_cast<long long>(g.nt) * g.nrec;
#if HV_BWD_PAIRED
  float2 acc[BWD_FG][RZ][2];
#pragma unroll
  for (int t = 0; t < BWD_FG; ++t)
#pragma unroll
    for (int r = 0; r < RZ; ++r) acc[t][r][0] = acc[t][r][1] = make_float2(0.0f, 0.0f);
#else
  float acc[BWD_FG][RZ][4];
#pragma unroll
  for (int t = 0; t < BWD_FG; ++t)
#pragma unroll
    for (int r = 0; r < RZ; ++r)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[t][r][i] = 0.0f;
#endif

  Ring cons;
  for (int s = sb; s < se; ++s) {
    float sj[RZ][4];  // s^j of shot s at this thread's points, read from the first field's stage
    float* out_base = p.pool + (static_cast<long long>(s * p.nslot + p.slot0 + fb) * p.nlev + par_out) * g.plane;
#pragma unroll
    for (int t = 0; t < BWD_FG; ++t) {
      if (t >= nf) break;
      const float* st = stages + cons.stage * BSTAGE_FLOATS;
      float* dst = out_base + static_cast<long long>(t) * p.nlev * g.plane;
      mbar_wait(&bars[cons.stage], cons.phase);
      if (t == 0) {
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
          const float4 v = p.imaging ? ld4(st + TILE_FLOATS + PT_FLOATS + so + r * TX) : make_float4(0.f, 0.f, 0.f, 0.f);
          sj[r][0] = v.x, sj[r][1] = v.y, sj[r][2] = v.z, sj[r][3] = v.w;
        }
      }
#if HV_BWD_PAIRED
      float2 L2[RZ][2], C2[RZ][2];
      lap_points_adj(st, tx, ty, L2, C2);
      if (p.update) {
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
          const float4 pv = ld4(st + TILE_FLOATS + so + r * TX);
          float v[4];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const float2 uu = dmp.upd(r, hh, C2[r][hh], half2of(pv, hh), mul2(w2[r][hh], L2[r][hh]));
            v[2 * hh] = uu.x, v[2 * hh + 1] = uu.y;
          }
          if (SP) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (J0 + i >= g.Nx) v[i] = 0.0f;
          }
          if (row_ok[r]) st4(dst + (go + r * g.P), make_float4(v[0], v[1], v[2], v[3]));
        }
      }
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        acc[t][r][0] = fma2(make_float2(sj[r][0], sj[r][1]), C2[r][0], acc[t][r][0]);
        acc[t][r][1] = fma2(make_float2(sj[r][2], sj[r][3]), C2[r][1], acc[t][r][1]);
      }
#else
      float L[RZ][4], C[RZ][4];
      {
        float2 L2[RZ][2], C2[RZ][2];
        lap_points_adj(st, tx, ty, L2, C2);
#pragma unroll
        for (int r = 0; r < RZ; ++r)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            L[r][2 * h] = L2[r][h].x, L[r][2 * h + 1] = L2[r][h].y;
            C[r][2 * h] = C2[r][h].x, C[r][2 * h + 1] = C2[r][h].y;
          }
      }
      if (p.update) {
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
          const float4 pv = ld4(st + TILE_FLOATS + so + r * TX);
          float v[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) v[i] = dmp.upd1(r, i, C[r][i], f4(pv, i), w[r][i] * L[r][i]);
          if (SP) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (J0 + i >= g.Nx) v[i] = 0.0f;
          }
          if (row_ok[r]) st4(dst + (go + r * g.P), make_float4(v[0], v[1], v[2], v[3]));
        }
      }
      // zero-lag imaging, summed over the batch's shots in registers: acc += s^j * lambda^{j+1}
#pragma unroll
      for (int r = 0; r < RZ; ++r)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[t][r][i] = fmaf(sj[r][i], C[r][i], acc[t][r][i]);
#endif
      __syncthreads();  // stage consumed and lambda^j of this tile stored
      cons.advance();
      if (tid == 0 && issued < nitems) {
        fence_proxy_async();
        issue_next();
      }
      // receiver injection into lambda^j: += v^2 / (1 + c) * rho[j][r]   (R^T scatter-add)
      if (p.update && re > rb) {
        const int slot = p.slot0 + fb + t;
        const float* rho = (slot == 0) ? p.rho_res + s * data_stride
                                       : p.rho_born + (static_cast<long long>(s) * p.Kb + (slot - 1)) * data_stride;
        for (int q = rb + tid; q < re; q += NTHREADS) {
          const int rid = p.trec_id[q];
          const float val = p.rec_coef[rid] * rho[static_cast<long long>(p.j) * g.nrec + rid];
          atomicAdd(dst + static_cast<long long>(p.rec_I[rid]) * g.P + p.rec_J[rid], val);
        }
      }
    }
  }
  if (any_img) {  // one writer per (field, point) per step: RED.128, deterministic order over steps
#pragma unroll
    for (int t = 0; t < BWD_FG; ++t) {
      if (t >= nf) break;
      float* a = p.acc + h * p.acc_copy + static_cast<long long>(p.slot0 + fb + t) * g.plane + go;
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        if (!img_rows[r]) continue;
#if HV_BWD_PAIRED
        atomicAdd(reinterpret_cast<float4*>(a + static_cast<long long>(r) * g.P),
                  make_float4(acc[t][r][0].x, acc[t][r][0].y, acc[t][r][1].x, acc[t][r][1].y));
#else
        atomicAdd(reinterpret_cast<float4*>(a + static_cast<long long>(r) * g.P),
                  make_float4(acc[t][r][0], acc[t][r][1], acc[t][r][2], acc[t][r][3]));
#endif
      }
    }
  }
}

__global__ void __launch_bounds__(NTHREADS, HV_BWD_MINB)
    bwd_step_kernel(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mt,
                    const __grid_constant__ CUtensorMap msj, const BwdParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stages = reinterpret_cast<float*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + BSTAGES_BYTES);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    tma_prefetch_desc(&mh);
    tma_prefetch_desc(&mt);
    tma_prefetch_desc(&msj);
    for (int i = 0; i < NSTAGE; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tile_is_interior(p.g, blockIdx.x * TX, blockIdx.y * TZ))
    bwd_body<false>(&mh, &mt, &msj, p, stages, bars);
  else
    bwd_body<true>(&mh, &mt, &msj, p, stages, bars);
}

// ------------------------------------------------------------------------------------------------ reverse (a6)

// BOUNDARY mode: rebuild the background backwards, u^{j-1} = 2 u^j - u^{j+1} + w L u^j + dt^2 f^j on the interior
// (c = 0 there) and the stored ring elsewhere in the Laplacian's reach, and emit s^j = 2 dt^2 / (v h^2) L~u^j.
struct RevParams {
  Geo g;
  int nslot;
  float* pool;
  int slot;               // background replay slot
  int j;                  // level whose Laplacian is taken; writes level j-1 in place over level j+1
  int S;
  int shot0;
  const float* W2;
  const float* imgc;
  float* s_out;           // s^j for batch shot 0 ([nz][PI] per shot)
  long long s_shot_stride;
  const float* ring_in;   // ring of level j-1 for batch shot 0
  long long ring_shot_stride;
  const int* src_I;
  const int* src_J;
  const float* src_amp;
};

template <bool SP>
__device__ __forceinline__ void rev_body(const CUtensorMap* mh, const CUtensorMap* mt, const RevParams& p,
                                         float* stages, uint64_t* bars) {
  const Geo& g = p.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
  const int x0 = blockIdx.x * TX, z0 = blockIdx.y * TZ;
  const int par_j = p.j & 1, par_o = par_j ^ 1;
  // grid.z splits the batch's shots: this CTA rebuilds shots [s0, s1)
  const int s0 = (blockIdx.z * p.S) / gridDim.z, s1 = ((blockIdx.z + 1) * p.S) / gridDim.z;
  int issued = s0;
  Ring prod;
  auto issue_next = [&]() {
    float* st = stages + prod.stage * STAGE_FLOATS;
    const int pl = (issued * p.nslot + p.slot) * 2;
    mbar_expect_tx(&bars[prod.stage], TILE_BYTES + PT_BYTES);
    tma_load_3d(st, mh, &bars[prod.stage], x0 - R, z0 - R, pl + par_j);
    tma_load_3d(st + TILE_FLOATS, mt, &bars[prod.stage], x0, z0, pl + par_o);
    prod.advance();
    ++issued;
  };
  if (tid == 0) {
    while (issued < min(s0 + NSTAGE, s1)) issue_next();
  }
  const int I0 = z0 + ty * RZ;
  const int J0 = x0 + tx * 4;
  const int so = ty * RZ * TX + tx * 4;
  const int go = I0 * g.P + J0;  // within-plane offset (plane < 2^31 floats)
  float w[RZ][4];
  int rq[RZ][4];       // ring index (>= 0), interior (-1), or neither (-2)
#pragma unroll
  for (int r = 0; r < RZ; ++r) {
    const float4 wv = ldg4(p.W2 + static_cast<long long>(min(I0 + r, g.Nz - 1)) * g.P + J0);
    w[r][0] = wv.x, w[r][1] = wv.y, w[r][2] = wv.z, w[r][3] = wv.w;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int I = I0 + r, J = J0 + i;
      const bool in = I >= g.W && I < g.W + g.nz && J >= g.W && J < g.W + g.nx;
      rq[r][i] = SP ? (in ? -1 : (ring_index(g, I, J) >= 0 ? ring_index(g, I, J) : -2)) : -1;
    }
  }
  const float amp = p.src_amp[p.j];
  const int jc = J0 - g.c0;
  Ring cons;
  for (int s = s0; s < s1; ++s) {
    const float* st = stages + cons.stage * STAGE_FLOATS;
    mbar_wait(&bars[cons.stage], cons.phase);
    float2 L2[RZ][2], C2[RZ][2];
    lap_points_bg(st, tx, ty, L2, C2);
    float L[RZ][4], C[RZ][4];
#pragma unroll
    for (int r = 0; r < RZ; ++r)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        L[r][2 * h] = L2[r][h].x, L[r][2 * h + 1] = L2[r][h].y;
        C[r][2 * h] = C2[r][h].x, C[r][2 * h + 1] = C2[r][h].y;
      }
    float* dst = p.pool + (static_cast<long long>(s * p.nslot + p.slot) * 2 + par_o) * g.plane;
    const int sI = p.src_I[p.shot0 + s], sJ = p.src_J[p.shot0 + s];
#pragma unroll
    for (int r = 0; r < RZ; ++r) {
      const float4 nx1 = ld4(st + TILE_FLOATS + so + r * TX);  // u^{j+1}
      float v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v[i] = fmaf(2.0f, C[r][i], fmaf(w[r][i], L[r][i], -f4(nx1, i)));
        if (I0 + r == sI && J0 + i == sJ) v[i] += amp;
        if (SP && rq[r][i] >= 0) v[i] = p.ring_in[s * p.ring_shot_stride + rq[r][i]];
      }
      if (!SP) {
        st4(dst + (go + r * g.P), make_float4(v[0], v[1], v[2], v[3]));
      } else if (I0 + r < g.Nz) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (rq[r][i] != -2) dst[(go + r * g.P) + i] = v[i];
      }
      // s^j on the interior
      const int iz = I0 + r - g.W;
      if (iz >= 0 && iz < g.nz && jc >= 0 && jc < g.PI) {
        const float4 ic = ldg4(p.imgc + static_cast<long long>(iz) * g.PI + jc);
        float o[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = (!SP || rq[r][i] == -1) ? f4(ic, i) * L[r][i] : 0.0f;
        st4(p.s_out + s * p.s_shot_stride + static_cast<long long>(iz) * g.PI + jc,
            make_float4(o[0], o[1], o[2], o[3]));
      }
    }
    __syncthreads();
    cons.advance();
    if (tid == 0 && issued < s1) {
      fence_proxy_async();
      issue_next();
    }
  }
}

__global__ void __launch_bounds__(NTHREADS, MINB)
    rev_step_kernel(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mt,
                    const RevParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stages = reinterpret_cast<float*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + STAGES_BYTES);
  const int x0 = blockIdx.x * TX, z0 = blockIdx.y * TZ;
  const Geo& g = p.g;
  // tiles entirely outside interior + ring have nothing to rebuild
  if (z0 + TZ <= g.W - R || z0 >= g.W + g.nz + R || x0 + TX <= g.W - R || x0 >= g.W + g.nx + R) return;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    tma_prefetch_desc(&mh);
    tma_prefetch_desc(&mt);
    for (int i = 0; i < NSTAGE; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tile_is_interior(g, x0, z0))
    rev_body<false>(&mh, &mt, p, stages, bars);
  else
    rev_body<true>(&mh, &mt, p, stages, bars);
}

// ------------------------------------------------------------------------------------------------ helpers

// a0: padded coefficient planes from the interior model m (edge-replicated into the sponge, C13).
// vmax_bits: atomicMax of the float bits (finite positive values order like their bits; NaN / negative values
// exceed +inf); vmin_bits: atomicMin of the bits read as int (any value <= 0 gives an int <= 0).
__global__ void model_setup_kernel(Geo g, const float* __restrict__ m, float dt2_h2, float two_dt2_h2,
                                   float* __restrict__ W2, float* __restrict__ imgc, unsigned int* vmax_bits,
                                   int* vmin_bits) {
  const long long n = static_cast<long long>(g.Nz) * g.P;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int I = static_cast<int>(q / g.P), J = static_cast<int>(q % g.P);
    float wv = 0.0f;
    if (J < g.Nx) {
      const int iz = min(max(I - g.W, 0), g.nz - 1), ix = min(max(J - g.W, 0), g.nx - 1);
      const float v = m[static_cast<long long>(iz) * g.nx + ix];
      wv = dt2_h2 * v * v;
      if (I == iz + g.W && J == ix + g.W) {
        atomicMax(vmax_bits, __float_as_uint(v));
        atomicMin(vmin_bits, __float_as_int(v));
      }
    }
    W2[q] = wv;
  }
  const long long ni = static_cast<long long>(g.nz) * g.PI;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < ni;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int iz = static_cast<int>(q / g.PI), ix = static_cast<int>(q % g.PI) + g.c0 - g.W;
    float c = 0.0f;
    if (ix >= 0 && ix < g.nx) c = two_dt2_h2 / m[static_cast<long long>(iz) * g.nx + ix];
    imgc[q] = c;
  }
}

__global__ void rec_coef_kernel(Geo g, const float* __restrict__ m, const int* rec_I,
                                const int* rec_J, float* coef) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= g.nrec) return;
  const int I = rec_I[r], J = rec_J[r];
  const float v = m[static_cast<long long>(I - g.W) * g.nx + (J - g.W)];
  const float c = sponge_c(g, I, J);
  coef[r] = v * v / (1.0f + c);
}

// K5: q_k = 2 dt^2 v dv_k / h^2 on the interior, 0 in the sponge and the row padding.
__global__ void q_setup_kernel(Geo g, const float* __restrict__ m, const float* __restrict__ V, int K,
                               float two_dt2_h2, float* __restrict__ Q) {
  const long long n = static_cast<long long>(K) * g.Nz * g.P;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long k = q / g.plane;
    const long long rem = q % g.plane;
    const int I = static_cast<int>(rem / g.P), J = static_cast<int>(rem % g.P);
    const int iz = I - g.W, ix = J - g.W;
    float val = 0.0f;
    if (iz >= 0 && iz < g.nz && ix >= 0 && ix < g.nx) {
      const long long o = static_cast<long long>(iz) * g.nx + ix;
      val = two_dt2_h2 * m[o] * V[k * g.nz * static_cast<long long>(g.nx) + o];
    }
    Q[q] = val;
  }
}

// d[n = nt-1] for every field of the batch: the level the last forward step produced.
// Pool planes per slot: nlev (2: parity planes of the single-step kernels; 4: level & 3 of fwd2); par = the
// plane of level nt-1 within a slot.
__global__ void gather_last_kernel(Geo g, const float* __restrict__ pool, int nslot, int nlev, int par, int dbg_shot0,
                                    float* d_bg, int bg_slot, float* d_born, int born_slot0, int K,
                                    const int* rec_I, const int* rec_J) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int f = blockIdx.y;  // 0 = background, 1..K Born
  const int s = blockIdx.z;
  if (r >= g.nrec) return;
  const long long off = static_cast<long long>(rec_I[r]) * g.P + rec_J[r];
  if (f == 0) {
    if (!d_bg) return;
    const long long pl = (static_cast<long long>(s) * nslot + bg_slot) * nlev + par;
    d_bg[(static_cast<long long>(dbg_shot0 + s) * g.nt + (g.nt - 1)) * g.nrec + r] = pool[pl * g.plane + off];
  } else {
    if (!d_born) return;
    const long long pl = (static_cast<long long>(s) * nslot + born_slot0 + f - 1) * nlev + par;
    d_born[((static_cast<long long>(s) * K + (f - 1)) * g.nt + (g.nt - 1)) * g.nrec + r] =
        pool[pl * g.plane + off];
  }
}

// K4: residual rho = d - d_obs and the block partials of phi = 1/2 sum rho^2 in float64 (part[blockIdx.x]); with
// a fixed grid every partial sums the same elements in the same order, and phi_reduce_kernel adds them in index
// order: phi is bit-deterministic.
__global__ void residual_kernel(long long n, const float* __restrict__ d, const float* __restrict__ dobs,
                                float* __restrict__ res, double* part) {
  double acc = 0.0;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float r = d[q] - dobs[q];
    res[q] = r;
    acc += 0.5 * static_cast<double>(r) * static_cast<double>(r);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

// phi += sum_b part[b] (one warp, fixed order: lane l sums b = l, l + 32, ..., then a fixed butterfly).
__global__ void phi_reduce_kernel(const double* __restrict__ part, int nb, double* phi) {
  double v = 0.0;
  for (int b = threadIdx.x; b < nb; b += 32) v += part[b];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (threadIdx.x == 0) *phi += v;
}

// a8 within a GPU: out[f][iz][ix] = sum_s acc[s][slot f][iz + W][ix + W] in a fixed order (deterministic).
__global__ void finalize_kernel(Geo g, const float* __restrict__ acc, int S, int nacc, int slot0, int F,
                                float* __restrict__ out) {
  const long long n = static_cast<long long>(F) * g.nz * g.nx;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long f = q / (static_cast<long long>(g.nz) * g.nx);
    const long long rem = q % (static_cast<long long>(g.nz) * g.nx);
    const int iz = static_cast<int>(rem / g.nx), ix = static_cast<int>(rem % g.nx);
    float s = 0.0f;
    for (int k = 0; k < S; ++k)
      s += acc[(static_cast<long long>(k) * nacc + slot0 + f) * g.plane + static_cast<long long>(iz + g.W) * g.P +
               ix + g.W];
    out[q] = s;
  }
}

}  // namespace hvk
