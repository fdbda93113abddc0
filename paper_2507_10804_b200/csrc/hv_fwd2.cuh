// hv_fwd2.cuh — two-step (temporally blocked) forward sweep: a1 + a2 + a3 + a4 FULL for levels n+1 AND n+2 in
// one launch ("fwd2"). Same scheme and arithmetic as fwd_step_kernel (hv_kernels.cuh): every
// level is computed by exactly the same per-point operations, so the two kernels give bit-identical fields.
//
// Why: a single-step pass reads u^n, u^{n-1} and writes u^{n+1} (12 B of DRAM per field update). Two steps per
// pass read u^n, u^{n-1} and write u^{n+1}, u^{n+2}: 16 B per two updates. The price is recomputation:
//   - level n+1 is computed on the TX x TZ "ext" region (the output tile + R cells on each side), from the
//     (TX + 2R) x (TZ + 2R) halo tile of u^n and the TX x TZ tile of u^{n-1} (the same TMA boxes as the
//     single-step kernel, shifted by R), into a shared-memory buffer `mid`;
//   - level n+2 is computed on the OX x OZ = (TX - 2R) x (TZ - 2R) output tile from `mid` (halo R) and u^n.
// Each thread keeps the same RZ x 4 points in both steps (the ext mapping); threads whose points are output
// points (1 <= tx <= BX-2, 2 <= ty <= BY-3 for R = 4, RZ = 2) do the second step.
// Points of the ext region outside the padded grid are forced to zero in `mid` (the Laplacian's zero boundary).
//
// Levels live in four planes per field (level & 3): a launch reads planes n, n-1 and writes n+1, n+2, so no CTA
// overwrites a level another CTA still reads (the single-step kernel's two parity planes would race here).
#pragma once
#include "hv_kernels.cuh"

namespace hvk {

struct Fwd2Params {
  Geo g;
  int nslot;              // pool plane index = ((s_local * nslot) + slot) * 4 + (level & 3)
  float* pool;
  int n;                  // this launch computes level n+1 (and n+2 if two) from levels n, n-1
  int two;                // 1: two steps; 0: only level n+1 (the last, odd step)
  int born_slot0;         // background in slot 0, Born field k in slot born_slot0 + k
  int K, S, G;            // Born fields, shots of the batch, Born-field groups (group_begin)
  const float* W2;        // [Nz][P]   dt^2 v^2 / h^2
  const float* imgc;      // [nz][PI]  2 dt^2 / (v h^2); with s_out: s^n, s^{n+1} = imgc * L u
  float* s_out;           // level-n slot of the FULL store for s_local = 0 (level n+1 = s_out + iplane), or null
  long long s_shot_stride;
  int shot0;
  const int* src_I;
  const int* src_J;
  const float* src_amp;   // [nt] dt^2 s[n] / h^2
  const int* trec_beg;    // [ntiles2 + 1] receivers owned by each output tile
  const int* trec_id;
  const int* rec_I;
  const int* rec_J;
  float* d_bg;            // background data [..][nt][nrec], row dbg_shot0 + s_local, or null
  int dbg_shot0;
  float* d_born;          // [S][K][nt][nrec] or null
};

struct Fwd2Producer {  // thread 0's walk over this CTA's items (decoded once per unit)
  const CUtensorMap *mh, *mt, *mq;
  float* stages;
  uint64_t* bars;
  int u, t;
  int U, nstep, ntl;
  int ex0, ez0, pl_bg, pl_born, fb, nf;
  bool upd;
  uint64_t pol_first, pol_last;
  RingN<NSTAGE_F2> ring;
  __device__ __forceinline__ void decode(const Fwd2Params& p) {
    if (u >= U) return;
    const int s = u / (p.G * ntl);
    const int rem = u - s * p.G * ntl;
    const int grp = rem / ntl, tile = rem - grp * ntl;
    const int by = tile / p.g.ntx2;
    ex0 = (tile - by * p.g.ntx2) * OX - R, ez0 = by * OZ - R;
    fb = group_begin(p.K, p.G, grp);
    nf = group_begin(p.K, p.G, grp + 1) - fb;
    upd = grp == 0;
    pl_bg = (s * p.nslot) * 4;
    pl_born = (s * p.nslot + p.born_slot0 + fb) * 4;
  }
  __device__ __forceinline__ void issue(const Fwd2Params& p) {
    if (u >= U) return;
    const int ln = p.n & 3, lp = (p.n + 3) & 3;  // planes of levels n and n-1
    float* st = stages + ring.stage * FSTAGE_FLOATS;
    uint64_t* bar = &bars[ring.stage];
    if (t == 0) {
      mbar_expect_tx(bar, TILE_BYTES + PT_BYTES);
      tma_load_3d(st, mh, bar, ex0 - R, ez0 - R, pl_bg + ln);
      tma_load_3d_hint(st + TILE_FLOATS, mt, bar, ex0, ez0, pl_bg + lp, pol_first);
    } else {
      const int pl = pl_born + 4 * (t - 1);
      mbar_expect_tx(bar, TILE_BYTES + 2 * PT_BYTES);
      tma_load_3d(st, mh, bar, ex0 - R, ez0 - R, pl + ln);
      tma_load_3d_hint(st + TILE_FLOATS, mt, bar, ex0, ez0, pl + lp, pol_first);
      tma_load_3d_hint(st + TILE_FLOATS + PT_FLOATS, mq, bar, ex0, ez0, fb + t - 1, pol_last);
    }
    ring.advance();
    if (++t > nf) {
      t = 0;
      u += nstep;
      decode(p);
    }
  }
};

__device__ __forceinline__ bool ext_is_interior(const Geo& g, int ex0, int ez0) {
  return ez0 >= g.W && ez0 + TZ <= g.W + g.nz && ex0 >= g.W && ex0 + TX <= g.W + g.nx;
}

template <bool SP>
__device__ __forceinline__ void fwd2_unit(const Fwd2Params& p, const float* stages, float* mid, uint64_t* bars,
                                          int s, int grp, int bx, int by, RingN<NSTAGE_F2>& cons,
                                          Fwd2Producer& prod) {
  const Geo& g = p.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
  const int ox0 = bx * OX, oz0 = by * OZ;
  const int ex0 = ox0 - R, ez0 = oz0 - R;
  const int fb = group_begin(p.K, p.G, grp);
  const int nf = group_begin(p.K, p.G, grp + 1) - fb;
  const bool leader = grp == 0;
  const bool two = p.two != 0;
  const int l1 = (p.n + 1) & 3, l2 = (p.n + 2) & 3;

  const int I0 = ez0 + ty * RZ;
  const int J0 = ex0 + tx * 4;
  const int so = ty * RZ * TX + tx * 4;  // offset of the thread's first point in a TX x TZ buffer
  // output (second-step) points: whole float4s of the OX x OZ core
  const bool inner = tx >= 1 && tx <= BX - 2 && ty >= R / RZ && ty < BY - R / RZ;
  bool row_in[RZ];   // row inside the padded grid
  bool col_in[4];
#pragma unroll
  for (int r = 0; r < RZ; ++r) row_in[r] = !SP || (I0 + r >= 0 && I0 + r < g.Nz);
#pragma unroll
  for (int i = 0; i < 4; ++i) col_in[i] = !SP || (J0 + i >= 0 && J0 + i < g.Nx);
  float2 w[RZ][2];
#pragma unroll
  for (int r = 0; r < RZ; ++r) {
    float4 wv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!SP || (row_in[r] && J0 >= 0 && J0 < g.P)) wv = ldg4(p.W2 + static_cast<long long>(I0 + r) * g.P + J0);
    w[r][0] = lo2(wv), w[r][1] = hi2(wv);
  }
  Damp<SP> dmp;
  dmp.init(g, I0, J0);
  const int tile_id = by * g.ntx2 + bx;
  const int rb = p.trec_beg[tile_id], re = p.trec_beg[tile_id + 1];
  const long long data_stride = static_cast<long long>(g.nt) * g.nrec;
  const long long go = static_cast<long long>(I0) * g.P + J0;  // plane offset (valid for inner threads)

  auto release = [&]() {
    __syncthreads();  // stage and mid consumed
    cons.advance();
    if (tid == 0) {
      fence_proxy_async();
      prod.issue(p);
    }
  };
  // d[n] from the staged halo tile of level n, d[n+1] from mid
  auto sample = [&](const float* st, float* out) {
    for (int q = rb + tid; q < re; q += NTHREADS) {
      const int rid = p.trec_id[q];
      const int lz = p.rec_I[rid] - ez0, lx = p.rec_J[rid] - ex0;
      out[static_cast<long long>(p.n) * g.nrec + rid] = st[(lz + R) * HX + lx + R];
      if (two) out[static_cast<long long>(p.n + 1) * g.nrec + rid] = mid[lz * TX + lx];
    }
  };
  // step 1 result -> mid (zero outside the padded grid)
  auto put_mid = [&](int r, float (&v)[4]) {
    if (SP) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (!row_in[r] || !col_in[i]) v[i] = 0.0f;
    }
    st4(mid + so + r * TX, make_float4(v[0], v[1], v[2], v[3]));
  };
  auto store_row = [&](float* dst, int r, float (&v)[4]) {
    if (SP) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (J0 + i >= g.Nx) v[i] = 0.0f;
      if (I0 + r >= g.Nz) return;
    }
    st4(dst + go + static_cast<long long>(r) * g.P, make_float4(v[0], v[1], v[2], v[3]));
  };
  auto plane = [&](int slot, int lvl) {
    return p.pool + (static_cast<long long>(s * p.nslot + slot) * 4 + lvl) * g.plane;
  };

  // ---------------- background: L u^n (ext), u^{n+1} (ext) -> mid, L u^{n+1} (core), u^{n+2} (core)
  float2 Lb0[RZ][2], Lb1[RZ][2];
  {
    const float* st = stages + cons.stage * FSTAGE_FLOATS;
    mbar_wait(&bars[cons.stage], cons.phase);
    float2 C0[RZ][2];
    lap_points(st, tx, ty, Lb0, C0);
    const int sI = p.src_I[p.shot0 + s], sJ = p.src_J[p.shot0 + s];
    const float amp0 = p.src_amp[p.n], amp1 = two ? p.src_amp[p.n + 1] : 0.0f;
#pragma unroll
    for (int r = 0; r < RZ; ++r) {
      const float4 pv = ld4(st + TILE_FLOATS + so + r * TX);
      float v[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float2 u = dmp.upd(r, h, C0[r][h], half2of(pv, h), mul2(w[r][h], Lb0[r][h]));
        v[2 * h] = u.x, v[2 * h + 1] = u.y;
      }
      if (I0 + r == sI && sJ >= J0 && sJ < J0 + 4) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (J0 + i == sJ) v[i] += amp0 * dmp_ci(dmp, r, i);
      }
      put_mid(r, v);
    }
    __syncthreads();  // mid = u^{n+1} on the ext region
    if (inner) {
      float2 C1[RZ][2];
      lap_points_w<TX>(mid - R * TX - R, tx, ty, Lb1, C1);
      if (leader) {
        float* d1 = plane(0, l1);
        float* d2 = plane(0, l2);
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
          float v1[4] = {C1[r][0].x, C1[r][0].y, C1[r][1].x, C1[r][1].y};
          store_row(d1, r, v1);
          if (two) {
            float v[4];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const float2 u = dmp.upd(r, h, C1[r][h], C0[r][h], mul2(w[r][h], Lb1[r][h]));
              v[2 * h] = u.x, v[2 * h + 1] = u.y;
            }
            if (I0 + r == sI && sJ >= J0 && sJ < J0 + 4) {
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (J0 + i == sJ) v[i] += amp1 * dmp_ci(dmp, r, i);
            }
            store_row(d2, r, v);
          }
        }
        // FULL store: s^n (and s^{n+1}) = imgc * L u on the interior part of the core
        const int jc = J0 - g.c0;
        if (p.s_out != nullptr && jc >= 0 && jc < g.PI) {
#pragma unroll
          for (int r = 0; r < RZ; ++r) {
            const int iz = I0 + r - g.W;
            if (iz < 0 || iz >= g.nz) continue;
            const float4 ic = ldg4(p.imgc + static_cast<long long>(iz) * g.PI + jc);
            float* so0 = p.s_out + s * p.s_shot_stride + static_cast<long long>(iz) * g.PI + jc;
#pragma unroll
            for (int lv = 0; lv < 2; ++lv) {
              if (lv == 1 && !two) break;
              const float2 (&Lx)[RZ][2] = lv == 0 ? Lb0 : Lb1;
              const float2 o01 = mul2(lo2(ic), Lx[r][0]), o23 = mul2(hi2(ic), Lx[r][1]);
              float o[4] = {o01.x, o01.y, o23.x, o23.y};
              if (SP) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const int ix = J0 + i - g.W;
                  if (ix < 0 || ix >= g.nx) o[i] = 0.0f;
                }
              }
              st4(so0 + lv * g.iplane, make_float4(o[0], o[1], o[2], o[3]));
            }
          }
        }
      }
    }
    if (leader && re > rb && p.d_bg) sample(st, p.d_bg + (p.dbg_shot0 + s) * data_stride);
    release();
  }
  // ---------------- Born fields of the group: sources q_k L u^n, q_k L u^{n+1}
  for (int t = 0; t < nf; ++t) {
    const float* st = stages + cons.stage * FSTAGE_FLOATS;
    mbar_wait(&bars[cons.stage], cons.phase);
    float2 L0[RZ][2], C0[RZ][2];
    lap_points(st, tx, ty, L0, C0);
    const float* qk = st + TILE_FLOATS + PT_FLOATS + so;
#pragma unroll
    for (int r = 0; r < RZ; ++r) {
      const float4 pv = ld4(st + TILE_FLOATS + so + r * TX);
      const float4 qv = ld4(qk + r * TX);
      float v[4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float2 u = dmp.upd(r, h, C0[r][h], half2of(pv, h),
                                 fma2(half2of(qv, h), Lb0[r][h], mul2(w[r][h], L0[r][h])));
        v[2 * h] = u.x, v[2 * h + 1] = u.y;
      }
      put_mid(r, v);
    }
    __syncthreads();  // mid = du^{n+1} on the ext region
    if (inner) {
      float2 L1[RZ][2], C1[RZ][2];
      lap_points_w<TX>(mid - R * TX - R, tx, ty, L1, C1);
      float* d1 = plane(p.born_slot0 + fb + t, l1);
      float* d2 = plane(p.born_slot0 + fb + t, l2);
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        float v1[4] = {C1[r][0].x, C1[r][0].y, C1[r][1].x, C1[r][1].y};
        store_row(d1, r, v1);
        if (two) {
          const float4 qv = ld4(qk + r * TX);
          float v[4];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float2 u = dmp.upd(r, h, C1[r][h], C0[r][h],
                                     fma2(half2of(qv, h), Lb1[r][h], mul2(w[r][h], L1[r][h])));
            v[2 * h] = u.x, v[2 * h + 1] = u.y;
          }
          store_row(d2, r, v);
        }
      }
    }
    if (re > rb && p.d_born) sample(st, p.d_born + (static_cast<long long>(s) * p.K + fb + t) * data_stride);
    release();
  }
}

__global__ void __launch_bounds__(NTHREADS, MINB)
    fwd2_kernel(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mt,
                const __grid_constant__ CUtensorMap mq, const Fwd2Params p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stages = reinterpret_cast<float*>(smem_raw);
  float* mid = reinterpret_cast<float*>(smem_raw + NSTAGE_F2 * FSTAGE_FLOATS * 4);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + NSTAGE_F2 * FSTAGE_FLOATS * 4 + PT_FLOATS * 4);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    tma_prefetch_desc(&mh);
    tma_prefetch_desc(&mt);
    tma_prefetch_desc(&mq);
    for (int i = 0; i < NSTAGE_F2; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int ntl = p.g.ntx2 * p.g.ntz2;
  const int U = p.S * p.G * ntl;
  const int nstep = gridDim.x;
  Fwd2Producer prod;
  prod.mh = &mh, prod.mt = &mt, prod.mq = &mq, prod.stages = stages, prod.bars = bars;
  prod.u = blockIdx.x, prod.t = 0, prod.U = U, prod.nstep = nstep, prod.ntl = ntl;
  prod.pol_first = policy_evict_first(), prod.pol_last = policy_evict_last();
  prod.decode(p);
  if (threadIdx.x == 0 && threadIdx.y == 0)
    for (int i = 0; i < NSTAGE_F2; ++i) prod.issue(p);
  RingN<NSTAGE_F2> cons;
  for (int u = blockIdx.x; u < U; u += nstep) {
    const int s = u / (p.G * ntl);
    const int rem = u - s * p.G * ntl;
    const int grp = rem / ntl, tile = rem - grp * ntl;
    const int by = tile / p.g.ntx2, bx = tile - by * p.g.ntx2;
    if (ext_is_interior(p.g, bx * OX - R, by * OZ - R))
      fwd2_unit<false>(p, stages, mid, bars, s, grp, bx, by, cons, prod);
    else
      fwd2_unit<true>(p, stages, mid, bars, s, grp, bx, by, cons, prod);
  }
}

}  // namespace hvk
