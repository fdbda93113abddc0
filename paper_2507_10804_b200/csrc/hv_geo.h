// hv_geo.h — tile constants and the padded-grid geometry shared by kernels and the host runtime.
#pragma once

namespace hvk {

constexpr int R = 4;                 // stencil radius (8th order)
constexpr int TX = 64;               // tile width  (x, contiguous)
#ifndef HV_TZ
#define HV_TZ 32
#endif
constexpr int TZ = HV_TZ;            // tile height (z)
constexpr int BX = 16;               // threads along x, 4 consecutive points (one float4) each
#ifndef HV_RZ
#define HV_RZ 4
#endif
constexpr int RZ = HV_RZ;            // consecutive rows per thread
constexpr int BY = TZ / RZ;          // threads along z
constexpr int NTHREADS = BX * BY;
// resident CTAs per SM the registers are sized for (2 x 256 threads at 2 rows; 2 x 128 threads at 4 rows).
// 4 rows (default): the per-item overhead (barrier waits, addressing, loop control) is shared by 16 points instead
// of 8: -18 % instructions per cfg 3 forward launch, +2.2 % H·v/s in the power-capped bench
constexpr int MINB = NTHREADS * RZ / 2 >= 512 ? 1 : 512 / (NTHREADS * RZ / 2);
constexpr int HX = TX + 2 * R;       // halo tile width  (72 floats = 288 B, a multiple of 16 B for TMA)
constexpr int HZ = TZ + 2 * R;       // halo tile height
constexpr int TILE_FLOATS = HX * HZ;          // halo tile (stencil input)
constexpr int TILE_BYTES = TILE_FLOATS * 4;
constexpr int PT_FLOATS = TX * TZ;            // pointwise tile (no halo)
constexpr int PT_BYTES = PT_FLOATS * 4;
#ifndef HV_NSTAGE
#define HV_NSTAGE 3
#endif
#ifndef HV_BWD_FG
#define HV_BWD_FG 2
#endif
constexpr int NSTAGE = HV_NSTAGE;             // TMA pipeline depth (items in flight per CTA)
// one pipeline stage: halo of level n (stencil input) + pointwise tile of level n-1 (updated in place)
constexpr int STAGE_FLOATS = TILE_FLOATS + PT_FLOATS;
constexpr int STAGES_BYTES = NSTAGE * STAGE_FLOATS * 4;
// resident-q forward: its own stage count (fewer stages leave room for more resident q_k tiles, i.e. fewer
// background recomputes per shot)
#ifndef HV_NSTAGE_Q
#define HV_NSTAGE_Q 3
#endif
constexpr int NSTAGE_Q = HV_NSTAGE_Q;
constexpr int QSTAGES_BYTES = NSTAGE_Q * STAGE_FLOATS * 4;
constexpr int BAR_BYTES = 128;              // keeps the q tiles behind the barriers 128-byte aligned (TMA)
// forward CTA: NSTAGE_F stages of halo u^n + tile u^{n-1} + tile q_k
#ifndef HV_NSTAGE_F
#define HV_NSTAGE_F 4
#endif
constexpr int NSTAGE_F = HV_NSTAGE_F;
constexpr int FSTAGE_FLOATS = TILE_FLOATS + 2 * PT_FLOATS;
constexpr int FSTAGES_BYTES = NSTAGE_F * FSTAGE_FLOATS * 4;
constexpr int FWD_FG_MAX = 64;
constexpr int fwd_smem_bytes(int) { return FSTAGES_BYTES + BAR_BYTES; }
// backward CTA: stages; its BWD_FG adjoint fields keep their imaging sums over the batch's shots in registers
constexpr int BWD_FG = HV_BWD_FG;
// backward stage: halo lambda^{j+1} + tile lambda^{j+2} + tile s^j (first field of a shot)
constexpr int BSTAGE_FLOATS = TILE_FLOATS + 2 * PT_FLOATS;
constexpr int BSTAGES_BYTES = NSTAGE * BSTAGE_FLOATS * 4;
constexpr int BWD_SMEM_BYTES = BSTAGES_BYTES + BAR_BYTES;
constexpr int REV_SMEM_BYTES = STAGES_BYTES + BAR_BYTES;  // BOUNDARY reverse kernel: halo + tile stages

// standard 8th-order central second-derivative weights (unscaled; h^-2 is folded into the coefficients)
#define HV_A0 (-205.0f / 72.0f)
#define HV_A1 (8.0f / 5.0f)
#define HV_A2 (-1.0f / 5.0f)
#define HV_A3 (8.0f / 315.0f)
#define HV_A4 (-1.0f / 560.0f)

// T = 2 forward kernel (hv_t2.cuh): OX x OZ output tiles, level n+1 on the (OX + 2R) x (OZ + 2R) mid region
constexpr int OX = 56;
#ifndef HV_T2_OZ
#define HV_T2_OZ 24
#endif
// 24: 32-row mid region = 8 thread rows of 4 -> 128-thread CTAs, 2 per SM (the forward-only default path, the
// fastest measured: 69.8 vs 79.2 us per cfg 3 misfit level with 56); 56: 256-thread CTAs, 1 per SM
constexpr int OZ = HV_T2_OZ;


struct Geo {
  int nz, nx, W;        // interior grid, sponge width
  int Nz, Nx;           // padded grid
  int P;                // row pitch of padded planes (floats) >= ntx * TX and >= ntx2 * OX
  int PI, c0;           // interior-store row pitch and first padded column stored (c0 % 4 == 0)
  int ntx, ntz;         // tile grid (TX x TZ tiles: single-step kernels)
  int ntx2, ntz2;       // tile grid of the T = 2 forward kernel (OX x OZ output tiles)
  long long plane;      // Nz * P
  long long iplane;     // nz * PI
  float kc;             // eta_max * dt / (2 W^2): c = kc (d_z^2 + d_x^2)
  int nt, nrec;
};

}  // namespace hvk
