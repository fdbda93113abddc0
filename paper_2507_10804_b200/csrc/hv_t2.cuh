// hv_t2.cuh — temporally blocked (T = 2) forward sweep: a1 + a2 + a3 + a4 (FULL store) for levels n+1 AND n+2
// in one launch (DESIGN.md §5 "fwd_t2"; BASELINE.json north_star: "temporal blocking where registers allow").
//
// Why: a single-step pass reads u^n, u^{n-1} and writes u^{n+1}: 12 B of DRAM per field update. Two levels per
// pass read u^n, u^{n-1} and write u^{n+1}, u^{n+2}: 16 B per two updates (8 B per update).
//
// Scheme (same per-point arithmetic as fwd_step_kernel / fwd_qres_kernel, so every field level is bit-identical
// to the single-step path):
//   - CTA = (56 x 56 output tile, group of up to T2_QFG Born fields); it loops over ALL shots of the batch with
//     the group's q_k tiles resident in shared memory (q read from DRAM once per launch, as in fwd_qres_kernel);
//   - 512 threads, each owning 2 rows x 4 columns of the 64 x 64 "mid" region (output tile + R on each side);
//   - phase 1: level n+1 on the mid region from the 72 x 72 TMA halo box of level n and the 64 x 64 box of level
//     n-1, into a shared-memory buffer (zero outside the padded grid: the Laplacian's boundary);
//   - one block barrier;
//   - phase 2: the 392 threads whose points lie in the output tile compute level n+2 at their OWN points from
//     the mid buffer (Laplacian) and their own level-n values (registers from phase 1);
//   - the mid buffer is double-buffered across items, so the barrier of item i+1 also guarantees that every
//     warp has finished reading item i: one barrier per item, and the TMA refill of the stage of item i-1 is
//     issued right after the barrier of item i (no empty barriers needed).
// Level planes: 4 per field (plane = level & 3): levels n, n-1 are read, n+1, n+2 written, nothing is written
// over a level another CTA still reads.
#pragma once
#include "hv_kernels.cuh"

#ifndef HV_T2_GROUP_FASTEST
#define HV_T2_GROUP_FASTEST 0
#endif

namespace hvk {

constexpr int T2_OX = OX, T2_OZ = OZ;                      // output tile (level n+2): 56 x 56
constexpr int T2_MX = T2_OX + 2 * R, T2_MZ = T2_OZ + 2 * R;  // mid region (level n+1): 64 x 64
constexpr int T2_IX = T2_MX + 2 * R, T2_IZ = T2_MZ + 2 * R;  // input halo box (level n): 72 x 72
constexpr int T2_BY = T2_MZ / RZ;                          // thread rows (RZ rows each)
constexpr int T2_NT = BX * T2_BY;                          // 512 threads
constexpr int T2_MINB = T2_NT * RZ / 2 <= 256 ? 2 : 1;     // resident CTAs per SM the registers are sized for
constexpr int T2_IN_FLOATS = T2_IX * T2_IZ;
constexpr int T2_MID_FLOATS = T2_MX * T2_MZ;
constexpr int T2_STAGE_FLOATS = T2_IN_FLOATS + T2_MID_FLOATS;  // halo of level n + level n-1 on the mid region
#ifndef HV_T2_NSTAGE
#define HV_T2_NSTAGE 3
#endif
constexpr int T2_NSTAGE = HV_T2_NSTAGE;
#ifndef HV_T2_QFG
#define HV_T2_QFG 4
#endif
constexpr int T2_QFG = HV_T2_QFG;  // Born fields per CTA (q_k tiles resident in shared memory)
constexpr int T2_BAR_BYTES = 128;
constexpr int t2_fwd_smem_bytes() {
  return (T2_NSTAGE * T2_STAGE_FLOATS + 2 * T2_MID_FLOATS + T2_QFG * T2_MID_FLOATS) * 4 + T2_BAR_BYTES;
}

struct T2Params {
  Geo g;
  int nslot;              // pool plane index = ((s_local * nslot) + slot) * 4 + (level & 3)
  float* pool;
  int n;                  // this launch computes level n+1 (and n+2 if two) from levels n, n-1
  int two;                // 1: two levels; 0: only level n+1 (the last, odd step)
  int bg_update;          // group 0 writes the background levels (0: sampling-only use)
  int born_slot0;         // background in slot 0, Born field k in slot born_slot0 + k
  int K, S, G;            // Born fields, shots of the batch, Born-field groups of <= T2_QFG
  int ntx, ntz;           // output-tile grid
  const float* W2;        // [Nz][P]   dt^2 v^2 / h^2 (0 outside the padded grid)
  const float* imgc;      // [nz][PI]  2 dt^2 / (v h^2); with s_out: s^n, s^{n+1} = imgc * L u
  float* s_out;           // level-n plane of the FULL store for s_local = 0 (level n+1 = s_out + iplane), or null
  long long s_shot_stride;
  int shot0;
  const int* src_I;
  const int* src_J;
  const float* src_amp;   // [nt] dt^2 s[n] / h^2
  const int* trec_beg;    // [ntx * ntz + 1] receivers owned by each output tile
  const int* trec_id;
  const int* rec_I;
  const int* rec_J;
  float* d_bg;            // background data [..][nt][nrec], row dbg_shot0 + s_local, or null
  int dbg_shot0;
  float* d_born;          // [S][K][nt][nrec] or null
  float* ring_out;        // BOUNDARY store: ring of level n+1 for batch shot 0 (level n+2 = + ringN), or null
  long long ring_shot_stride;
  int ringN;
  // background increment D = u^n - u^{n-1} (compensated leapfrog, as FwdParams): shot s reads plane
  // (dplane0 + s) * 2 + dsel (D^n) and writes plane (dplane0 + s) * 2 + (dsel ^ 1) (D^{n+2}, or D^{n+1})
  float* dbuf;
  int dplane0, dsel;
};

template <bool SP>
__device__ __forceinline__ void fwd_t2_body(const CUtensorMap* mh, const CUtensorMap* mt, const CUtensorMap* mq,
                                            const CUtensorMap* md, const T2Params& p, float* stages, float* midb,
                                            float* qs, uint64_t* bars, int bx, int bz, int grp) {
  const Geo& g = p.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
  const int ox0 = bx * T2_OX, oz0 = bz * T2_OZ;   // output tile origin (padded coordinates)
  const int ex0 = ox0 - R, ez0 = oz0 - R;         // mid region origin
  const int fb = group_begin(p.K, p.G, grp);
  const int nf = group_begin(p.K, p.G, grp + 1) - fb;
  const bool leader = grp == 0 && p.bg_update;
  const bool two = p.two != 0;
  const int ln = p.n & 3, lp = (p.n + 3) & 3, l1 = (p.n + 1) & 3, l2 = (p.n + 2) & 3;
  const int nitems = p.S * (1 + nf);
  uint64_t* qbar = bars + T2_NSTAGE;

  // producer (thread 0): item i = (shot i / (1 + nf), field i % (1 + nf)) -> stage i % T2_NSTAGE
  int ps = 0, pt = 0, issued = 0;
  RingN<T2_NSTAGE> prod;
  auto issue_next = [&]() {
    float* st = stages + prod.stage * T2_STAGE_FLOATS;
    const int slot = pt == 0 ? 0 : p.born_slot0 + fb + pt - 1;
    const int pl = (ps * p.nslot + slot) * 4;
    mbar_expect_tx(&bars[prod.stage], (T2_IN_FLOATS + T2_MID_FLOATS) * 4);
    tma_load_3d(st, mh, &bars[prod.stage], ex0 - R, ez0 - R, pl + ln);
    if (pt == 0)  // background: D^n on the mid region (increment form)
      tma_load_3d(st + T2_IN_FLOATS, md, &bars[prod.stage], ex0, ez0, (p.dplane0 + ps) * 2 + p.dsel);
    else
      tma_load_3d(st + T2_IN_FLOATS, mt, &bars[prod.stage], ex0, ez0, pl + lp);
    prod.advance();
    if (++pt > nf) {
      pt = 0;
      ++ps;
    }
    ++issued;
  };
  if (tid == 0) {
    if (nf > 0) {  // q_k tiles of the group (mid region), once for all shots
      mbar_expect_tx(qbar, nf * T2_MID_FLOATS * 4);
      for (int t = 0; t < nf; ++t) tma_load_3d(qs + t * T2_MID_FLOATS, mq, qbar, ex0, ez0, fb + t);
    }
    // NSTAGE items in flight: phase 2 reads no stage data, so item i's stage is refilled at item i's barrier
    while (issued < min(T2_NSTAGE, nitems)) issue_next();
  }

  const int I0 = ez0 + ty * RZ;
  const int J0 = ex0 + tx * 4;
  const int so = ty * RZ * T2_MX + tx * 4;           // offset of the thread's first point in a mid-region buffer
  const bool inner = tx >= 1 && tx <= BX - 2 && ty >= R / RZ && ty < T2_BY - R / RZ;  // output-tile points
  bool row_in[RZ], col_in[4];
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
  const int tile_id = bz * p.ntx + bx;
  const int rb = p.trec_beg[tile_id], re = p.trec_beg[tile_id + 1];
  const long long data_stride = static_cast<long long>(g.nt) * g.nrec;
  const long long go = static_cast<long long>(I0) * g.P + J0;  // plane offset (inner threads)
  const int jc = J0 - g.c0;
  const bool store_s = leader && p.s_out != nullptr && inner && jc >= 0 && jc < g.PI;
  const float amp0 = p.src_amp[p.n], amp1 = two ? p.src_amp[p.n + 1] : 0.0f;
  if (nf > 0) mbar_wait(qbar, 0);

  auto store_row = [&](float* dst, int r, float (&v)[4]) {
    if (SP) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (J0 + i >= g.Nx) v[i] = 0.0f;
      if (I0 + r >= g.Nz) return;
    }
    st4(dst + go + static_cast<long long>(r) * g.P, make_float4(v[0], v[1], v[2], v[3]));
  };
  auto put_mid = [&](float* mid, int r, float (&v)[4]) {  // zero outside the padded grid
    if (SP) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (!row_in[r] || !col_in[i]) v[i] = 0.0f;
    }
    st4(mid + so + r * T2_MX, make_float4(v[0], v[1], v[2], v[3]));
  };
  // d[n] from the staged halo of level n (before the barrier: the stage is refilled at it), d[n+1] from mid
  auto sample_n = [&](const float* st, float* out) {
    for (int q = rb + tid; q < re; q += T2_NT) {
      const int rid = p.trec_id[q];
      const int lz = p.rec_I[rid] - ez0, lx = p.rec_J[rid] - ex0;
      out[static_cast<long long>(p.n) * g.nrec + rid] = st[(lz + R) * T2_IX + lx + R];
    }
  };
  auto sample_n1 = [&](const float* mid, float* out) {
    if (!two) return;
    for (int q = rb + tid; q < re; q += T2_NT) {
      const int rid = p.trec_id[q];
      const int lz = p.rec_I[rid] - ez0, lx = p.rec_J[rid] - ex0;
      out[static_cast<long long>(p.n + 1) * g.nrec + rid] = mid[lz * T2_MX + lx];
    }
  };
  auto ring_store = [&](float* ring, int r, const float (&v)[4]) {  // BOUNDARY store (own output points)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = ring_index(g, I0 + r, J0 + i);
      if (q >= 0) ring[q] = v[i];
    }
  };

  RingN<T2_NSTAGE> cons;
  int it = 0;  // item counter: mid buffer = it & 1
  auto barrier_and_refill = [&]() {
    __syncthreads();  // mid complete; every warp is done with item it's stage and with item it - 1
    if (tid == 0 && issued < nitems) {
      fence_proxy_async();
      issue_next();  // into the stage of item it (phase 2 reads registers and mid only)
    }
  };
  float2 Lb0[RZ][2], Lb1[RZ][2];  // background L u^n, L u^{n+1} at this thread's points (shot s)
  for (int s = 0; s < p.S; ++s) {
    // ---------------- background of shot s: L u^n, u^{n+1} (mid) -> L u^{n+1}, u^{n+2} (output tile)
    {
      const float* st = stages + cons.stage * T2_STAGE_FLOATS;
      float* mid = midb + (it & 1) * T2_MID_FLOATS;
      mbar_wait(&bars[cons.stage], cons.phase);
      float2 C0[RZ][2];
      lap_points_w<T2_IX, true>(st, tx, ty, Lb0, C0);
      const int sI = p.src_I[p.shot0 + s], sJ = p.src_J[p.shot0 + s];
      float v1s[RZ][4], d1s[RZ][4];  // u^{n+1}, D^{n+1} at this thread's points
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        const float4 dv = ld4(st + T2_IN_FLOATS + so + r * T2_MX);  // D^n
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2 d1 = dmp.updd(r, h, half2of(dv, h), mul2(w[r][h], Lb0[r][h]));
          d1s[r][2 * h] = d1.x, d1s[r][2 * h + 1] = d1.y;
        }
        if (I0 + r == sI && sJ >= J0 && sJ < J0 + 4) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (J0 + i == sJ) d1s[r][i] += amp0 * dmp_ci(dmp, r, i);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2 u = add2(C0[r][h], make_float2(d1s[r][2 * h], d1s[r][2 * h + 1]));
          v1s[r][2 * h] = u.x, v1s[r][2 * h + 1] = u.y;
        }
        put_mid(mid, r, v1s[r]);
      }
      if (leader && re > rb && p.d_bg) sample_n(st, p.d_bg + (p.dbg_shot0 + s) * data_stride);
      barrier_and_refill();
      if (inner) {
        float2 C1[RZ][2];
        lap_points_w<T2_MX, true>(mid - R * T2_MX - R, tx, ty, Lb1, C1);
        if (leader) {
          float* d1 = p.pool + (static_cast<long long>(s * p.nslot) * 4 + l1) * g.plane;
          float* d2 = p.pool + (static_cast<long long>(s * p.nslot) * 4 + l2) * g.plane;
          float* dD = p.dbuf + static_cast<long long>((p.dplane0 + s) * 2 + (p.dsel ^ 1)) * g.plane;
#pragma unroll
          for (int r = 0; r < RZ; ++r) {
            store_row(d1, r, v1s[r]);
            if (SP && p.ring_out) ring_store(p.ring_out + s * p.ring_shot_stride, r, v1s[r]);
            if (two) {
              float v[4], dn[4];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const float2 d2v = dmp.updd(r, h, make_float2(d1s[r][2 * h], d1s[r][2 * h + 1]),
                                            mul2(w[r][h], Lb1[r][h]));
                dn[2 * h] = d2v.x, dn[2 * h + 1] = d2v.y;
              }
              if (I0 + r == sI && sJ >= J0 && sJ < J0 + 4) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                  if (J0 + i == sJ) dn[i] += amp1 * dmp_ci(dmp, r, i);
              }
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const float2 u = add2(C1[r][h], make_float2(dn[2 * h], dn[2 * h + 1]));
                v[2 * h] = u.x, v[2 * h + 1] = u.y;
              }
              if (SP && p.ring_out) ring_store(p.ring_out + s * p.ring_shot_stride + p.ringN, r, v);
              store_row(d2, r, v);
              store_row(dD, r, dn);
            } else {
              store_row(dD, r, d1s[r]);
            }
          }
          if (store_s) {  // FULL store: s^n (and s^{n+1}) = imgc * L u on the interior
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
      if (leader && re > rb && p.d_bg) sample_n1(mid, p.d_bg + (p.dbg_shot0 + s) * data_stride);
      cons.advance();
      ++it;
    }
    // ---------------- Born fields of the group: sources q_k L u^n (mid), q_k L u^{n+1} (output tile)
    for (int t = 0; t < nf; ++t) {
      const float* st = stages + cons.stage * T2_STAGE_FLOATS;
      float* mid = midb + (it & 1) * T2_MID_FLOATS;
      const float* qk = qs + t * T2_MID_FLOATS + so;
      mbar_wait(&bars[cons.stage], cons.phase);
      float2 L0[RZ][2], C0[RZ][2];
      lap_points_w<T2_IX, true>(st, tx, ty, L0, C0);
      float v1s[RZ][4];
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        const float4 pv = ld4(st + T2_IN_FLOATS + so + r * T2_MX);
        const float4 qv = ld4(qk + r * T2_MX);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2 u = dmp.upd(r, h, C0[r][h], half2of(pv, h),
                                   fma2(half2of(qv, h), Lb0[r][h], mul2(w[r][h], L0[r][h])));
          v1s[r][2 * h] = u.x, v1s[r][2 * h + 1] = u.y;
        }
        put_mid(mid, r, v1s[r]);
      }
      if (re > rb && p.d_born) sample_n(st, p.d_born + (static_cast<long long>(s) * p.K + fb + t) * data_stride);
      barrier_and_refill();
      if (inner) {
        float2 L1[RZ][2], C1[RZ][2];
        lap_points_w<T2_MX, true>(mid - R * T2_MX - R, tx, ty, L1, C1);
        const long long pl = static_cast<long long>(s * p.nslot + p.born_slot0 + fb + t) * 4;
        float* d1 = p.pool + (pl + l1) * g.plane;
        float* d2 = p.pool + (pl + l2) * g.plane;
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
          store_row(d1, r, v1s[r]);
          if (two) {
            const float4 qv = ld4(qk + r * T2_MX);
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
      if (re > rb && p.d_born) sample_n1(mid, p.d_born + (static_cast<long long>(s) * p.K + fb + t) * data_stride);
      cons.advance();
      ++it;
    }
  }
}

__device__ __forceinline__ bool t2_mid_is_interior(const Geo& g, int ex0, int ez0) {
  return ez0 >= g.W && ez0 + T2_MZ <= g.W + g.nz && ex0 >= g.W && ex0 + T2_MX <= g.W + g.nx;
}

// grid.x = G x ntz x ntx. Default order: tiles fastest, group slowest (HV_T2_GROUP_FASTEST=1: group fastest, so
// the groups of a tile share the background halo in L2 but neighbouring tiles' halos miss: 19 % L2 hit rate).
__global__ void __launch_bounds__(T2_NT, T2_MINB)
    fwd_t2_kernel(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mt,
                  const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap md, const T2Params p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stages = reinterpret_cast<float*>(smem_raw);
  float* midb = stages + T2_NSTAGE * T2_STAGE_FLOATS;
  float* qs = midb + 2 * T2_MID_FLOATS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(qs + T2_QFG * T2_MID_FLOATS);
#if HV_T2_GROUP_FASTEST
  const int grp = blockIdx.x % p.G;
  const int tile = blockIdx.x / p.G;
  const int bz = tile % p.ntz, bx = tile / p.ntz;
#else  // tiles fastest (x, then z), group slowest: a wave holds most tiles of one group, all stepping through the
       // same (shot, field) items, so the halo reads of neighbouring tiles are L2 hits
  const int ntl = p.ntx * p.ntz;
  const int grp = blockIdx.x / ntl;
  const int tile = blockIdx.x - grp * ntl;
  const int bz = tile / p.ntx, bx = tile - bz * p.ntx;
#endif
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    tma_prefetch_desc(&mh);
    tma_prefetch_desc(&mt);
    tma_prefetch_desc(&mq);
    for (int i = 0; i < T2_NSTAGE + 1; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (t2_mid_is_interior(p.g, bx * T2_OX - R, bz * T2_OZ - R))
    fwd_t2_body<false>(&mh, &mt, &mq, &md, p, stages, midb, qs, bars, bx, bz, grp);
  else
    fwd_t2_body<true>(&mh, &mt, &mq, &md, p, stages, midb, qs, bars, bx, bz, grp);
}

// ------------------------------------------------------------------------------------------------ backward

// T = 2 adjoint sweep (a5 + a7 + a3 injection) for levels j AND j-1 in one launch, same per-point arithmetic as
// bwd_step_kernel (bit-identical lambda levels; the imaging sums add two levels per launch before the
// per-launch RED, so H·v / g agree with the single-step path to fp32 summation order):
//   - CTA = (56 x 56 output tile, BWD_FG adjoint fields); it loops over all shots of the batch and keeps the
//     imaging sums of its output points in registers (one RED.128 per point and field per launch);
//   - phase 1 (512 threads, mid region): lambda^j = step(lambda^{j+1} halo, lambda^{j+2}) -> mid buffer;
//     receiver injection v^2/(1+c) rho[j] into the mid buffer (receivers anywhere in the mid region; tiles
//     with receivers take one extra barrier); imaging s^j lambda^{j+1} at the output points;
//   - phase 2 (the 392 output-tile threads): lambda^{j-1} = step(lambda^j (mid), lambda^{j+1} (own registers));
//     imaging s^{j-1} lambda^j; lambda^j (post-injection, from mid) and lambda^{j-1} stored; rho[j-1] is added to
//     lambda^{j-1} in global memory after the next barrier (one atomic per owned receiver).
// s^j, s^{j-1} (FULL store, 56 x 56 boxes of the interior store) travel with the stage of a shot's first field.
constexpr int T2_S_FLOATS = T2_OX * T2_OZ;
constexpr int T2_BSTAGE_FLOATS = T2_IN_FLOATS + T2_MID_FLOATS + 2 * T2_S_FLOATS;
constexpr int t2_bwd_smem_bytes() { return (T2_NSTAGE * T2_BSTAGE_FLOATS + 2 * T2_MID_FLOATS) * 4 + T2_BAR_BYTES; }

struct T2BwdParams {
  Geo g;
  int nslot;
  float* pool;            // plane = ((s_local * nslot) + slot) * 4 + (level & 3)
  int j;                  // computes lambda^j and, if two, lambda^{j-1}
  int two;
  int upd0, upd1;         // lambda^j / lambda^{j-1} are computed (level >= 2)
  int img0, img1;         // imaging s^j lambda^{j+1} / s^{j-1} lambda^j
  int slot0, F, S, G;     // adjoint fields in slots slot0 .. slot0 + F - 1, BWD_FG per group
  int ntx, ntz;
  const float* W2;
  long long sj_plane0;    // plane of s^j of batch shot 0 in the interior-store tensor map (s^{j-1}: plane - 1)
  int sj_shot_planes;
  float* acc;             // [nacc][Nz][P] (single copy)
  const float* rho_res;   // slot 0 injection data [S][nt][nrec] (gradient), or null
  const float* rho_born;  // slot k >= 1 injection data [S][K][nt][nrec]
  int Kb;
  const float* rec_coef;  // [nrec] v^2 / (1 + c)
  const int* tmid_beg;    // [ntx * ntz + 1] receivers inside each tile's MID region
  const int* tmid_id;
  const int* tout_beg;    // [ntx * ntz + 1] receivers owned by each output tile
  const int* tout_id;
  const int* rec_I;
  const int* rec_J;
};

template <bool SP>
__device__ __forceinline__ void bwd_t2_body(const CUtensorMap* mh, const CUtensorMap* mt, const CUtensorMap* ms,
                                            const T2BwdParams& p, float* stages, float* midb, uint64_t* bars,
                                            int bx, int bz, int grp) {
  const Geo& g = p.g;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BX + tx;
  const int ox0 = bx * T2_OX, oz0 = bz * T2_OZ;
  const int ex0 = ox0 - R, ez0 = oz0 - R;
  const int fb = grp * BWD_FG;
  const int nf = min(p.F, fb + BWD_FG) - fb;
  if (nf <= 0) return;
  const bool two = p.two != 0;
  const int lin = (p.j + 1) & 3, lpr = (p.j + 2) & 3, l0 = p.j & 3, l1 = (p.j + 3) & 3;
  const int nitems = p.S * nf;

  int ps = 0, pt = 0, issued = 0;
  RingN<T2_NSTAGE> prod;
  auto issue_next = [&]() {
    float* st = stages + prod.stage * T2_BSTAGE_FLOATS;
    const int pl = (ps * p.nslot + p.slot0 + fb + pt) * 4;
    const bool with_s = pt == 0 && (p.img0 || p.img1);
    mbar_expect_tx(&bars[prod.stage], (T2_IN_FLOATS + T2_MID_FLOATS + (with_s ? 2 * T2_S_FLOATS : 0)) * 4);
    tma_load_3d(st, mh, &bars[prod.stage], ex0 - R, ez0 - R, pl + lin);
    tma_load_3d(st + T2_IN_FLOATS, mt, &bars[prod.stage], ex0, ez0, pl + lpr);
    if (with_s) {  // interior store: padded (ox0, oz0) is interior (ox0 - c0, oz0 - W); outside -> zero fill
      const int plane = static_cast<int>(p.sj_plane0 + static_cast<long long>(ps) * p.sj_shot_planes);
      tma_load_3d(st + T2_IN_FLOATS + T2_MID_FLOATS, ms, &bars[prod.stage], ox0 - g.c0, oz0 - g.W, plane);
      tma_load_3d(st + T2_IN_FLOATS + T2_MID_FLOATS + T2_S_FLOATS, ms, &bars[prod.stage], ox0 - g.c0, oz0 - g.W,
                  plane - 1);
    }
    prod.advance();
    if (++pt == nf) {
      pt = 0;
      ++ps;
    }
    ++issued;
  };
  if (tid == 0)  // NSTAGE items in flight: phase 2 reads no stage data (s^j is copied to registers first)
    while (issued < min(T2_NSTAGE, nitems)) issue_next();

  const int I0 = ez0 + ty * RZ;
  const int J0 = ex0 + tx * 4;
  const int so = ty * RZ * T2_MX + tx * 4;
  const bool inner = tx >= 1 && tx <= BX - 2 && ty >= R / RZ && ty < T2_BY - R / RZ;
  const int soo = (ty * RZ - R) * T2_OX + tx * 4 - R;  // offset in the output-tile boxes (inner threads)
  bool row_in[RZ], col_in[4];
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
  // imaging rows: interior rows and columns of this thread's output points
  bool img_row[RZ];
  bool any_img = false;
#pragma unroll
  for (int r = 0; r < RZ; ++r) {
    const int iz = I0 + r - g.W;
    img_row[r] = inner && iz >= 0 && iz < g.nz && J0 + 3 >= g.W && J0 < g.W + g.nx;
    any_img |= img_row[r];
  }
  Damp<SP> dmp;
  dmp.init(g, I0, J0);
  const int tile_id = bz * p.ntx + bx;
  const int mb = p.tmid_beg[tile_id], me = p.tmid_beg[tile_id + 1];
  const int ob = p.tout_beg[tile_id], oe = p.tout_beg[tile_id + 1];
  const long long data_stride = static_cast<long long>(g.nt) * g.nrec;
  const long long go = static_cast<long long>(I0) * g.P + J0;

  auto put_mid = [&](float* mid, int r, float (&v)[4]) {
    if (SP) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (!row_in[r] || !col_in[i]) v[i] = 0.0f;
    }
    st4(mid + so + r * T2_MX, make_float4(v[0], v[1], v[2], v[3]));
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
  auto rho_of = [&](int s, int f) -> const float* {
    const int slot = p.slot0 + fb + f;
    return slot == 0 ? p.rho_res + s * data_stride
                     : p.rho_born + (static_cast<long long>(s) * p.Kb + (slot - 1)) * data_stride;
  };

  float2 acc[BWD_FG][RZ][2];
#pragma unroll
  for (int t = 0; t < BWD_FG; ++t)
#pragma unroll
    for (int r = 0; r < RZ; ++r) acc[t][r][0] = acc[t][r][1] = make_float2(0.0f, 0.0f);

  RingN<T2_NSTAGE> cons;
  int it = 0;
  int pend_s = -1, pend_f = 0;  // item whose lambda^{j-1} still needs its receiver injection (after a barrier)
  auto inject_pending = [&]() {  // rho[j-1] into lambda^{j-1} at the receivers this tile owns (global atomics)
    if (pend_s < 0 || oe <= ob || !p.upd1) return;
    const float* rho = rho_of(pend_s, pend_f);
    float* dst = p.pool + (static_cast<long long>(pend_s * p.nslot + p.slot0 + fb + pend_f) * 4 + l1) * g.plane;
    for (int q = ob + tid; q < oe; q += T2_NT) {
      const int rid = p.tout_id[q];
      atomicAdd(dst + static_cast<long long>(p.rec_I[rid]) * g.P + p.rec_J[rid],
                p.rec_coef[rid] * rho[static_cast<long long>(p.j - 1) * g.nrec + rid]);
    }
  };
  for (int s = 0; s < p.S; ++s) {
    float2 sj0[RZ][2], sj1[RZ][2];  // s^j, s^{j-1} of shot s at this thread's output points
#pragma unroll
    for (int f = 0; f < BWD_FG; ++f) {  // unrolled: the imaging sums acc[f] stay in registers
      if (f >= nf) break;
      const float* st = stages + cons.stage * T2_BSTAGE_FLOATS;
      float* mid = midb + (it & 1) * T2_MID_FLOATS;
      mbar_wait(&bars[cons.stage], cons.phase);
      if (f == 0) {
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
          float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
          if (inner && (p.img0 || p.img1)) {
            a = ld4(st + T2_IN_FLOATS + T2_MID_FLOATS + soo + r * T2_OX);
            b = ld4(st + T2_IN_FLOATS + T2_MID_FLOATS + T2_S_FLOATS + soo + r * T2_OX);
          }
          sj0[r][0] = lo2(a), sj0[r][1] = hi2(a);
          sj1[r][0] = lo2(b), sj1[r][1] = hi2(b);
        }
      }
      float2 L0[RZ][2], C0[RZ][2];
      lap_points_w<T2_IX, true>(st, tx, ty, L0, C0);
      float v1s[RZ][4];
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        const float4 pv = ld4(st + T2_IN_FLOATS + so + r * T2_MX);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float2 u = p.upd0 ? dmp.upd(r, h, C0[r][h], half2of(pv, h), mul2(w[r][h], L0[r][h]))
                                  : make_float2(0.0f, 0.0f);
          v1s[r][2 * h] = u.x, v1s[r][2 * h + 1] = u.y;
        }
        put_mid(mid, r, v1s[r]);
      }
      // imaging of level j: s^j lambda^{j+1} (C0 = lambda^{j+1} at this thread's points)
      if (p.img0 && any_img) {
#pragma unroll
        for (int r = 0; r < RZ; ++r) {
          acc[f][r][0] = fma2(sj0[r][0], C0[r][0], acc[f][r][0]);
          acc[f][r][1] = fma2(sj0[r][1], C0[r][1], acc[f][r][1]);
        }
      }
      if (me > mb && p.upd0 && two) {  // receivers in the mid region: rho[j] into the mid buffer before phase 2
        __syncthreads();
        const float* rho = rho_of(s, f);
        for (int q = mb + tid; q < me; q += T2_NT) {
          const int rid = p.tmid_id[q];
          atomicAdd(mid + (p.rec_I[rid] - ez0) * T2_MX + (p.rec_J[rid] - ex0),
                    p.rec_coef[rid] * rho[static_cast<long long>(p.j) * g.nrec + rid]);
        }
      }
      __syncthreads();  // mid complete; every warp is done with item it - 1
      if (tid == 0 && issued < nitems) {
        fence_proxy_async();
        issue_next();
      }
      inject_pending();  // lambda^{j-1} of item it - 1 is stored (all warps passed this barrier)
      pend_s = -1;
      if (inner) {
        float* d0 = p.pool + (static_cast<long long>(s * p.nslot + p.slot0 + fb + f) * 4 + l0) * g.plane;
        if (two) {
          float2 L1[RZ][2], C1[RZ][2];
          lap_points_w<T2_MX, true>(mid - R * T2_MX - R, tx, ty, L1, C1);
          float* d1 = p.pool + (static_cast<long long>(s * p.nslot + p.slot0 + fb + f) * 4 + l1) * g.plane;
#pragma unroll
          for (int r = 0; r < RZ; ++r) {
            float v0[4] = {C1[r][0].x, C1[r][0].y, C1[r][1].x, C1[r][1].y};  // lambda^j after injection
            if (p.upd0) store_row(d0, r, v0);
            if (p.upd1) {
              float v[4];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const float2 u = dmp.upd(r, h, C1[r][h], C0[r][h], mul2(w[r][h], L1[r][h]));
                v[2 * h] = u.x, v[2 * h + 1] = u.y;
              }
              store_row(d1, r, v);
            }
            if (p.img1 && img_row[r]) {  // imaging of level j-1: s^{j-1} lambda^j
              acc[f][r][0] = fma2(sj1[r][0], C1[r][0], acc[f][r][0]);
              acc[f][r][1] = fma2(sj1[r][1], C1[r][1], acc[f][r][1]);
            }
          }
        } else if (p.upd0) {  // single level (the last launch): lambda^j, injection added in global below
#pragma unroll
          for (int r = 0; r < RZ; ++r) store_row(d0, r, v1s[r]);
        }
      }
      if (two && p.upd1) pend_s = s, pend_f = f;
      if (!two && p.upd0 && oe > ob) {  // single level: rho[j] into lambda^j after the stores are visible
        __syncthreads();
        const float* rho = rho_of(s, f);
        float* d0 = p.pool + (static_cast<long long>(s * p.nslot + p.slot0 + fb + f) * 4 + l0) * g.plane;
        for (int q = ob + tid; q < oe; q += T2_NT) {
          const int rid = p.tout_id[q];
          atomicAdd(d0 + static_cast<long long>(p.rec_I[rid]) * g.P + p.rec_J[rid],
                    p.rec_coef[rid] * rho[static_cast<long long>(p.j) * g.nrec + rid]);
        }
      }
      cons.advance();
      ++it;
    }
  }
  if (pend_s >= 0 && oe > ob) {
    __syncthreads();
    inject_pending();
  }
  if (any_img && (p.img0 || p.img1)) {  // one writer per (field, point) per launch: RED.128
#pragma unroll
    for (int t = 0; t < BWD_FG; ++t) {
      if (t >= nf) break;
      float* a = p.acc + static_cast<long long>(p.slot0 + fb + t) * g.plane + go;
#pragma unroll
      for (int r = 0; r < RZ; ++r) {
        if (!img_row[r]) continue;
        atomicAdd(reinterpret_cast<float4*>(a + static_cast<long long>(r) * g.P),
                  make_float4(acc[t][r][0].x, acc[t][r][0].y, acc[t][r][1].x, acc[t][r][1].y));
      }
    }
  }
}

__global__ void __launch_bounds__(T2_NT, T2_MINB)
    bwd_t2_kernel(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mt,
                  const __grid_constant__ CUtensorMap ms, const T2BwdParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stages = reinterpret_cast<float*>(smem_raw);
  float* midb = stages + T2_NSTAGE * T2_BSTAGE_FLOATS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(midb + 2 * T2_MID_FLOATS);
#if HV_T2_GROUP_FASTEST
  const int grp = blockIdx.x % p.G;
  const int tile = blockIdx.x / p.G;
  const int bz = tile % p.ntz, bx = tile / p.ntz;
#else  // tiles fastest (x, then z), group slowest: a wave holds most tiles of one group, all stepping through the
       // same (shot, field) items, so the halo reads of neighbouring tiles are L2 hits
  const int ntl = p.ntx * p.ntz;
  const int grp = blockIdx.x / ntl;
  const int tile = blockIdx.x - grp * ntl;
  const int bz = tile / p.ntx, bx = tile - bz * p.ntx;
#endif
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    tma_prefetch_desc(&mh);
    tma_prefetch_desc(&mt);
    tma_prefetch_desc(&ms);
    for (int i = 0; i < T2_NSTAGE; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (t2_mid_is_interior(p.g, bx * T2_OX - R, bz * T2_OZ - R))
    bwd_t2_body<false>(&mh, &mt, &ms, p, stages, midb, bars, bx, bz, grp);
  else
    bwd_t2_body<true>(&mh, &mt, &ms, p, stages, midb, bars, bx, bz, grp);
}

}  // namespace hvk
