// hv_bwd2.cuh — two-step (temporally blocked) adjoint sweep: a5 + a7 (+ a3 injection) for levels j AND j-1 in
// one launch ("bwd2"). Same scheme and per-point arithmetic as bwd_step_kernel (hv_kernels.cuh).
//
// Launch "top level" j >= 2 (the host runs j = nt-1, nt-3, ...; a final j = 1 launch, imaging only, uses the
// single-step kernel):
//   step 1 (TX x TZ ext region): lambda^j = upd(lambda^{j+1}, lambda^{j+2}) -> shared `mid`, then the receiver
//           injection v^2/(1+c) rho[j] for every receiver inside the ext region (shared atomics: duplicates add);
//   step 2 (OX x OZ core): lambda^{j-1} = upd(lambda^j = mid, lambda^{j+1}) when j - 1 >= 2;
//   imaging  HV += s^j lambda^{j+1} (j <= nt-2) + s^{j-1} lambda^j, summed over the batch's shots in registers;
//   stores   lambda^j, lambda^{j-1} on the core; then the injection rho[j-1] into lambda^{j-1} (global atomics).
// Levels live in four planes per field (level & 3), as in hv_fwd2.cuh.
#pragma once
#include "hv_fwd2.cuh"

namespace hvk {

struct Bwd2Params {
  Geo g;
  int nslot;
  float* pool;            // plane ((s * nslot) + slot) * 4 + (level & 3)
  int j;                  // top level (>= 2): computes lambda^j and, if j >= 3, lambda^{j-1}
  int img_top;            // accumulate s^j lambda^{j+1} (j <= nt-2)
  int slot0, F;           // adjoint fields in slots slot0 .. slot0 + F - 1; BWD_FG per group (grid.z)
  int S;
  const float* W2;
  const float* s_lvl;     // s^j for batch shot 0 (s^{j-1} = s_lvl - iplane)
  long long s_shot_stride;
  float* acc;             // [nacc][Nz][P]
  const float* rho_res;   // slot 0 injection data [S][nt][nrec] (gradient), or null
  const float* rho_born;  // slot k >= 1: [S][K][nt][nrec]
  int Kb;
  const float* rec_coef;  // [nrec] v^2 / (1 + c)
  const int* trec_beg;    // receivers owned by each core tile (level j-1 injection)
  const int* trec_id;
  const int* trecx_beg;   // receivers inside each ext region (level j injection into mid)
  const int* trecx_id;
  const int* rec_I;
  const int* rec_J;
};

template <bool SP>
__device__ __forceinline__ void bwd2_body(const CUtensorMap* mh, const CUtensorMap* mt, const Bwd2Params& p,
                                          float* stages, float* mid, uint64_t* bars) {
  const Geo& g = p.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
  const int bx = blockIdx.x, by = blockIdx.y;
  const int ox0 = bx * OX, oz0 = by * OZ;
  const int ex0 = ox0 - R, ez0 = oz0 - R;
  const int fb = blockIdx.z * BWD_FG;
  const int nf = min(p.F, fb + BWD_FG) - fb;
  if (nf <= 0) return;
  const int nitems = p.S * nf;
  const int j = p.j;
  const bool upd2 = j >= 3;  // lambda^{j-1} is needed (lambda^1 never is)
  const int lin = (j + 1) & 3, lprev = (j + 2) & 3, l1 = j & 3, l2 = (j - 1) & 3;
  int ps = 0, pt = 0, issued = 0;
  Ring prod;
  auto issue_next = [&]() {
    float* st = stages + prod.stage * STAGE_FLOATS;
    const int pl = (ps * p.nslot + p.slot0 + fb + pt) * 4;
    mbar_expect_tx(&bars[prod.stage], TILE_BYTES + PT_BYTES);
    tma_load_3d(st, mh, &bars[prod.stage], ex0 - R, ez0 - R, pl + lin);
    tma_load_3d(st + TILE_FLOATS, mt, &bars[prod.stage], ex0, ez0, pl + lprev);
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
  const int I0 = ez0 + ty * RZ;
  const int J0 = ex0 + tx * 4;
  const int so = ty * RZ * TX + tx * 4;
  const bool inner = tx >= 1 && tx <= BX - 2 && ty >= R / RZ && ty < BY - R / RZ;
  const long long go = static_cast<long long>(I0) * g.P + J0;
  const int jc = J0 - g.c0;
  bool row_in[RZ], col_in[4], img_rows[RZ];
  bool any_img = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) col_in[i] = !SP || (J0 + i >= 0 && J0 + i < g.Nx);
  float2 w[RZ][2];
#pragma unroll
  for (int r = 0; r < RZ; ++r) {
    const int I = I0 + r;
    row_in[r] = !SP || (I >= 0 && I < g.Nz);
    float4 wv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!SP || (row_in[r] && J0 >= 0 && J0 < g.P)) wv = ldg4(p.W2 + static_cast<long long>(I) * g.P + J0);
    w[r][0] = lo2(wv), w[r][1] = hi2(wv);
    const int iz = I - g.W;
    img_rows[r] = inner && iz >= 0 && iz < g.nz && J0 + 3 >= g.W && J0 < g.W + g.nx && jc >= 0 && jc < g.PI;
    any_img |= img_rows[r];
  }
  // imaging factors s^j, s^{j-1} of shot s at this thread's (core) points, zero outside the interior
  auto load_s = [&](int s, float2 (&a)[RZ][2], float2 (&b)[RZ][2]) {
#pragma unroll
    for (int r = 0; r < RZ; ++r) {
      float4 va = make_float4(0.f, 0.f, 0.f, 0.f), vb = va;
      if (img_rows[r]) {
        const float* q = p.s_lvl + s * p.s_shot_stride + static_cast<long long>(I0 + r - g.W) * g.PI + jc;
        va = ldg4(q);
        vb = ldg4(q - g.iplane);
      }
      float x[4] = {va.x, va.y, va.z, va.w}, y[4] = {vb.x, vb.y, vb.z, vb.w};
      if (SP) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int ix = J0 + i - g.W;
          if (ix < 0 || ix >= g.nx) x[i] = 0.0f, y[i] = 0.0f;
        }
      }
      a[r][0] = make_float2(x[0], x[1]), a[r][1] = make_float2(x[2], x[3]);
      b[r][0] = make_float2(y[0], y[1]), b[r][1] = make_float2(y[2], y[3]);
    }
  };
  BwdDamp<SP> dmp;
  dmp.init(g, I0, J0);
  const int tile_id = by * g.ntx2 + bx;
  const int rb = p.trec_beg[tile_id], re = p.trec_beg[tile_id + 1];
  const int xb = p.trecx_beg[tile_id], xe = p.trecx_beg[tile_id + 1];
  const long long data_stride = static_cast<long long>(g.nt) * g.nrec;
  float2 acc[BWD_FG][RZ][2];
#pragma unroll
  for (int t = 0; t < BWD_FG; ++t)
#pragma unroll
    for (int r = 0; r < RZ; ++r)
#pragma unroll
      for (int h = 0; h < 2; ++h) acc[t][r][h] = make_float2(0.0f, 0.0f);

  Ring cons;
  for (int s = 0; s < p.S; ++s) {
    float2 s0[RZ][2], s1[RZ][2];  // s^j, s^{j-1}
    load_s(s, s0, s1);
    if (!p.img_top) {
#pragma unroll
      for (int r = 0; r < RZ; ++r) s0[r][0] = s0[r][1] = make_float2(0.0f, 0.0f);
    }
    float* out_base = p.pool + static_cast<long long>(s * p.nslot + p.slot0 + fb) * 4 * g.plane;
#pragma unroll
    for (int t = 0; t < BWD_FG; ++t) {
      if (t >= nf) break;
      const float* st = stages + cons.stage * STAGE_FLOATS;
      float* fbase = out_base + static_cast<long long>(t) * 4 * g.plane;
      const int slot = p.slot0 + fb + t;
      const float* rho = (slot == 0) ? p.rho_res + s * data_stride
                                     : p.rho_born + (static_cast<long long>(s) * p.Kb + (slot - 1)) * data_stride;
      mbar_wait(&bars[cons.stage], cons.phase);
      float2 L0[RZ][2], C0[RZ][2];
      lap_points(st, tx, ty, L0, C0);
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        const float4 pv = ld4(st + TILE_FLOATS + so + r * TX);
        float v[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2 u = dmp.upd(r, h, C0[r][h], half2of(pv, h), mul2(w[r][h], L0[r][h]));
          v[2 * h] = u.x, v[2 * h + 1] = u.y;
        }
        if (SP) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (!row_in[r] || !col_in[i]) v[i] = 0.0f;
        }
        st4(mid + so + r * TX, make_float4(v[0], v[1], v[2], v[3]));
      }
      if (xe > xb) {  // receiver injection into lambda^j on the ext region (shared atomics)
        __syncthreads();
        for (int q = xb + tid; q < xe; q += NTHREADS) {
          const int rid = p.trecx_id[q];
          const float val = p.rec_coef[rid] * rho[static_cast<long long>(j) * g.nrec + rid];
          atomicAdd(mid + (p.rec_I[rid] - ez0) * TX + (p.rec_J[rid] - ex0), val);
        }
      }
      __syncthreads();  // mid = lambda^j (injected) on the ext region
      if (inner) {
        float2 L1[RZ][2], C1[RZ][2];
        lap_points_w<TX>(mid - R * TX - R, tx, ty, L1, C1);
        float* d1 = fbase + static_cast<long long>(l1) * g.plane;
        float* d2 = fbase + static_cast<long long>(l2) * g.plane;
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
          const bool row_ok = !SP || I0 + r < g.Nz;
          float v1[4] = {C1[r][0].x, C1[r][0].y, C1[r][1].x, C1[r][1].y};
          if (SP) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (J0 + i >= g.Nx) v1[i] = 0.0f;
          }
          if (row_ok) st4(d1 + go + static_cast<long long>(r) * g.P, make_float4(v1[0], v1[1], v1[2], v1[3]));
          if (upd2) {
            float v[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const float2 u = dmp.upd(r, h, C1[r][h], C0[r][h], mul2(w[r][h], L1[r][h]));
              v[2 * h] = u.x, v[2 * h + 1] = u.y;
            }
            if (SP) {
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (J0 + i >= g.Nx) v[i] = 0.0f;
            }
            if (row_ok) st4(d2 + go + static_cast<long long>(r) * g.P, make_float4(v[0], v[1], v[2], v[3]));
          }
          // zero-lag imaging: acc += s^j lambda^{j+1} + s^{j-1} lambda^j
#pragma unroll
          for (int h = 0; h < 2; ++h)
            acc[t][r][h] = fma2(s1[r][h], C1[r][h], fma2(s0[r][h], C0[r][h], acc[t][r][h]));
        }
      }
      __syncthreads();  // stage and mid consumed, lambda^j / lambda^{j-1} of this tile stored
      cons.advance();
      if (tid == 0 && issued < nitems) {
        fence_proxy_async();
        issue_next();
      }
      if (upd2 && re > rb) {  // receiver injection into lambda^{j-1} (core receivers)
        float* d2 = fbase + static_cast<long long>(l2) * g.plane;
        for (int q = rb + tid; q < re; q += NTHREADS) {
          const int rid = p.trec_id[q];
          const float val = p.rec_coef[rid] * rho[static_cast<long long>(j - 1) * g.nrec + rid];
          atomicAdd(d2 + static_cast<long long>(p.rec_I[rid]) * g.P + p.rec_J[rid], val);
        }
      }
    }
  }
  if (any_img) {  // one writer per (field, point) per launch: RED.128, deterministic order over launches
#pragma unroll
    for (int t = 0; t < BWD_FG; ++t) {
      if (t >= nf) break;
      float* a = p.acc + static_cast<long long>(p.slot0 + fb + t) * g.plane + go;
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        if (!img_rows[r]) continue;
        atomicAdd(reinterpret_cast<float4*>(a + static_cast<long long>(r) * g.P),
                  make_float4(acc[t][r][0].x, acc[t][r][0].y, acc[t][r][1].x, acc[t][r][1].y));
      }
    }
  }
}

__global__ void __launch_bounds__(NTHREADS, MINB)
    bwd2_kernel(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mt,
                const Bwd2Params p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stages = reinterpret_cast<float*>(smem_raw);
  float* mid = reinterpret_cast<float*>(smem_raw + STAGES_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + STAGES_BYTES + PT_FLOATS * 4);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    tma_prefetch_desc(&mh);
    tma_prefetch_desc(&mt);
    for (int i = 0; i < NSTAGE; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (ext_is_interior(p.g, blockIdx.x * OX - R, blockIdx.y * OZ - R))
    bwd2_body<false>(&mh, &mt, p, stages, mid, bars);
  else
    bwd2_body<true>(&mh, &mt, p, stages, mid, bars);
}

}  // namespace hvk
