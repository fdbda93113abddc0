/*
 * hv.h — C ABI of the B200-native Gauss-Newton Hessian-vector-product library (libhv.so).
 *
 * What it computes (arxiv 2507.10804, PAPER.md; discrete readings in DESIGN.md §3):
 *   forward   f(m) -> d       "values of u(x,t) at receiver locations"            PAPER.md:49 (§2)
 *                              for (1/m^2) u_tt - lap u = s(t) delta(x - x_s)      PAPER.md:44-47 (Eq. equ:pde)
 *   gradient  F* (f(m) - d)    misfit term of grad Phi, F = Born, F* = migration  PAPER.md:108-112 (Eq. equ:grad)
 *   hessvec   H_d v = F* F v   misfit (Gauss-Newton) Hessian "accessed via matrix-vector products"
 *                              "two wave equations per source"                      PAPER.md:9, 157-164 (§3)
 *   psido     sum_k D_{a_k} F^-1 D_{b_k} F v  low-rank-symbol PsiDO apply          PAPER.md:240-247 (Eq. equ:lr-psido)
 *                              (apply_psf / apply_pdo on assembled approximations)
 *
 * Discretisation (none is given by the paper; SURVEY.md §8(c) O1-O11 / DESIGN.md §3):
 *   2-D constant-density acoustic u_tt = v^2 lap u + f, leapfrog in time, 8th-order 17-point Laplacian
 *   (zero outside the padded grid), W-cell sponge with centred damping, point source s[n]/h^2, point receivers,
 *   discretise-then-optimise exact adjoint, Gauss-Newton H_d = J^T J, Euclidean inner products, sigma = 1.
 *
 * Layout: every model-space array is [nz][nx] float32, z-major row-major (row iz, column ix), contiguous.
 *         data arrays are [shot][nt][nrec] float32; probe batches are [K][nz][nx]; symbols are [r][nz][nx].
 * Pointers: any array argument may be a HOST pointer or a DEVICE pointer of the context's device (the library
 *         asks the CUDA runtime which). Host inputs are copied in and host outputs copied back inside the call.
 *         Ownership stays with the caller; the library owns only its context workspace. Outputs are overwritten,
 *         never accumulated into.
 * Calls are blocking (they return when the result is complete) and are serialised per context; use one context
 * per GPU. No call falls back to the CPU: without a usable sm_100a device hv_create fails with HV_ECUDA.
 * Multi-GPU: each rank passes its shot shard [src_begin, src_end) (may be empty); gradient / hessvec / misfit
 * return RANK-LOCAL partial sums over that shard (the per-source terms of PAPER.md:164) unless a NCCL communicator
 * is attached (hv_config.nccl_comm / hv_set_comm): then the library all-reduces g, H.v and phi in-library on its
 * stream before returning, and every rank receives the sum over all shots.
 * Streams: with no stream bound (hv_set_stream NULL) a call first waits for the work already queued on the legacy
 * default stream (e.g. torch's default stream), so device inputs produced there are complete; with a bound stream
 * the call is ordered on that stream.
 */
#ifndef HV_H
#define HV_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define HV_API __attribute__((visibility("default")))
#else
#define HV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define HV_OK      0
#define HV_EINVAL  1  /* bad argument: null pointer, index out of range, K < 1, r < 1, mode unknown      */
#define HV_EGRID   2  /* array / grid shape does not match the configuration                             */
#define HV_ECFL    3  /* dt * max(m) / h exceeds the stability limit 0.5546 (leapfrog + 8th order, 2-D)  */
#define HV_ENOMEM  4  /* the plan exceeds the device-memory budget                                        */
#define HV_ECUDA   5  /* CUDA / cuFFT error, or no sm_100 device                                          */
#define HV_ESTATE  6  /* null / destroyed context                                                         */
#define HV_ENCCL   7  /* NCCL unavailable (libnccl.so.2 not loadable) or an NCCL call failed              */

/* forward-history storage for the reverse pass (not in the paper) */
#define HV_STORE_AUTO       0  /* FULL when it fits the budget, else CHECKPOINT                      */
#define HV_STORE_FULL       1  /* keep the imaging factor (2 dt^2 / v) L u^n of every level in HBM    */
#define HV_STORE_CHECKPOINT 2  /* keep (u^n, u^{n-1}) every ckpt_interval levels, replay segments      */
#define HV_STORE_BOUNDARY   3  /* keep the 4-cell ring around the interior of every level; rebuild the
                                  background backwards (time-reversed leapfrog on the interior)          */

typedef struct hv_ctx hv_ctx;

typedef struct {
  int32_t nz, nx;        /* interior grid (rows = depth), >= 1                                           */
  float   h;             /* grid spacing [m]                                                             */
  float   dt;            /* time step [s]                                                                */
  int32_t nt;            /* time levels t_n = n dt, n = 0..nt-1, >= 3                                     */
  int32_t sponge;        /* W: absorbing cells added on each side (>= 4)                                 */
  float   v_ref;         /* fixed sponge reference speed [m/s]; eta_max = 3 v_ref ln(1e3) / (2 W h)       */
  int32_t nsrc;          /* total shots; src_iz/src_ix: HOST arrays [nsrc], interior indices (copied)     */
  const int32_t *src_iz, *src_ix;
  int32_t nrec;          /* receivers (same for every shot); rec_iz/rec_ix: HOST arrays [nrec] (copied)   */
  const int32_t *rec_iz, *rec_ix;
  const float *wavelet;  /* HOST [nt]: source function s[n] (copied)                                     */
  int32_t src_begin, src_end; /* this rank's shot shard [begin, end); end = 0 means nsrc                  */
  int32_t store;         /* HV_STORE_* (AUTO: FULL if it fits, else CHECKPOINT)                         */
  int32_t ckpt_interval; /* CHECKPOINT spacing in levels; 0 = round(sqrt(nt))                            */
  int32_t shot_batch;    /* shots propagated concurrently; 0 = auto: the most that fit the budget (<= 32),
                            then ceil(nshard / S) near-equal batches                                      */
  int32_t field_group;   /* max Born fields per forward work unit (tuning); 0 = auto (busiest-CTA model)   */
  int32_t device;        /* CUDA device ordinal                                                          */
  size_t  mem_budget;    /* bytes of device memory the plan may use; 0 = 90 % of (free memory + the
                            context's own H.v workspace, which a larger plan releases and re-allocates)   */
  void   *nccl_comm;     /* optional ncclComm_t (NULL: rank-local partial sums). Borrowed, not owned: it must
                            outlive the context's calls. One rank per GPU; every rank must make the same
                            sequence of gradient / hessvec / misfit calls (the all-reduces are collective).   */
} hv_config;

/* Create / destroy. Validates geometry (indices inside the interior grid) -> HV_EINVAL. An empty shard
 * (src_begin == src_end, e.g. more ranks than shots) is allowed: its partial sums are zero. */
HV_API int hv_create(const hv_config* cfg, hv_ctx** out);
HV_API int hv_destroy(hv_ctx* ctx);

/* Run subsequent work on this cudaStream_t (NULL = the context's own stream). */
HV_API int hv_set_stream(hv_ctx* ctx, void* cuda_stream);

/* Attach (or detach with NULL) a NCCL communicator for in-library reductions (see hv_config.nccl_comm). */
HV_API int hv_set_comm(hv_ctx* ctx, void* nccl_comm);

/* d = f(m) for the shard's shots: m [nz][nx] (m/s); d [src_end - src_begin][nt][nrec]; d[:,0,:] = 0. */
HV_API int hv_forward(hv_ctx* ctx, const float* m, float* d);

/* d = f(m) for ONE shot ("given a source location x_s ... solve the wave equation"): isrc is the
 * GLOBAL shot index, src_begin <= isrc < src_end (else HV_EINVAL); d [nt][nrec]. */
HV_API int hv_forward_shot(hv_ctx* ctx, const float* m, int32_t isrc, float* d);

/* Data misfit only, Phi_d(m) = 1/2 sum_s sum_{n,r} (f_s(m) - d_obs,s)^2 (the likelihood term of Phi, PAPER.md:104-106;
 * what each gpCN proposal evaluates): forward sweeps + residual, no history store, no adjoint.
 * d_obs [local shots][nt][nrec]; *phi float64, summed in a fixed order (bit-deterministic). */
HV_API int hv_misfit(hv_ctx* ctx, const float* m, const float* d_obs, double* phi);

/* Misfit gradient and value over the shard: d_obs [local shots][nt][nrec]; g [nz][nx];
 * *phi = 1/2 sum (d - d_obs)^2 accumulated in float64 in a fixed order (phi may be NULL). g and phi are
 * bit-deterministic for a given shard and shot batching. */
HV_API int hv_gradient(hv_ctx* ctx, const float* m, const float* d_obs, float* g, double* phi);

/* Gauss-Newton H_d [v_1..v_K] over the shard: V, HV [K][nz][nx]. K >= 1. All K probes of a shot share one
 * background wavefield (batched probing). Bit-deterministic for a given shard and shot
 * batching (every accumulator address has one writer per launch; launches are ordered), and row k does not
 * depend on the other probes of the batch. */
HV_API int hv_hessvec(hv_ctx* ctx, const float* m, int32_t K, const float* V, float* HV);

/* Fused: gradient and K Hessian-vector products in one pass over the shard (1 + K fields forward,
 * 1 + K adjoint fields backward). K >= 0. */
HV_API int hv_gradient_hessvec(hv_ctx* ctx, const float* m, const float* d_obs, int32_t K, const float* V,
                        float* g, double* phi, float* HV);

/* Low-rank-symbol PsiDO apply on an nz x nx grid (Eq. equ:lr-psido):
 *   mode 0: out = Re sum_k a_k . IDFT(b_k . DFT(v))
 *   mode 1: out = Re sum_k IDFT(conj(b_k) . DFT(a_k . v))   (adjoint, Euclidean inner product)
 *   mode 2: (mode 0 + mode 1) / 2                             (symmetrised)
 * a [r][nz][nx] float32 (real spatial factors), b [r][nz][nx] interleaved complex64 (frequency factors at the
 * unshifted DFT frequencies), v, out [nz][nx]. DFT unnormalised, IDFT scaled 1/(nz nx), so b == 1 is the
 * identity. apply_psf == (a = PSF weights w_k, b = symbol rows); apply_pdo == (a = symbol columns, b = weights).
 * mode + 4: the spatial factors a are interleaved complex64 [r][nz][nx] (PSF+ factors); out = Re sum_k a_k . IDFT(..),
 * adjoint Re sum_k IDFT(conj(b_k) . DFT(conj(a_k) . v)). */
HV_API int hv_psido_apply(hv_ctx* ctx, int32_t nz, int32_t nx, int32_t r, const float* a, const float* b,
                   const float* v, float* out, int32_t mode);

/* ---- Probe -> symbol assembly, feeding hv_psido_apply. Discrete conventions: DESIGN.md §3
 * R-probe (unnormalised DFT, unit-spike probes, periodic interior grid). Complex outputs are interleaved complex64.
 *
 * PSF symbol rows: responses [nb][nz][nx] = H_d v_b for probes v_b that are sums of
 * unit spikes; point k at (pt_iz[k], pt_ix[k]) was probed in batch pt_batch[k]. rows [np][nz][nx] =
 * conj(DFT(p_k)) with p_k = the (2 radius + 1)^2 window of the response around the point, rolled to the origin
 * (the paper's s(x_k, xi) = (2 pi)^2 conj(p^_k(xi))). Index arrays may be host or device pointers. */
HV_API int hv_psf_rows(hv_ctx* ctx, int32_t nz, int32_t nx, int32_t nb, const float* responses, int32_t np,
                       const int32_t* pt_iz, const int32_t* pt_ix, const int32_t* pt_batch, int32_t radius,
                       float* rows);

/* PSF spatial weights ("interpolation weights"): bilinear hats on the lattice
 * lat_z[nlz] x lat_x[nlx] (sorted), constant outside it; w [nlz * nlx][nz][nx], k = i * nlx + j. Partition of
 * unity; w_k(x_j) = delta_kj. apply_psf == hv_psido_apply(a = w, b = rows). */
HV_API int hv_psf_weights(hv_ctx* ctx, int32_t nz, int32_t nx, int32_t nlz, const int32_t* lat_z, int32_t nlx,
                          const int32_t* lat_x, float* w);

/* PDO symbol columns (Eq. equ:symbol): response [nz][nx] = H_d v_p, v_p = sum_k phi_{xi_k};
 * xi_k given as DFT indices (kz[k], kx[k]); cols [r][nz][nx] = IDFT(M_k . DFT(response)) / phi_{xi_k}, M_k = disc
 * of mask_radius frequency cells around xi_k with a 2-cell raised-cosine roll-off. */
HV_API int hv_pdo_columns(hv_ctx* ctx, int32_t nz, int32_t nx, const float* response, int32_t r, const int32_t* kz,
                          const int32_t* kx, float mask_radius, float* cols);

/* PDO frequency weights (Eq. equ:pdo-w): w [r][nz][nx] (complex64, imaginary 0) =
 * (|xi| / rho0) t(theta(xi) - theta_k), t(phi) = sin(r phi / 2) cot(phi / 2) / r (r even), xi at the unshifted
 * DFT frequencies of spacing h, theta = atan2(xi_z, xi_x). apply_pdo == hv_psido_apply(a = Re cols, b = w). */
HV_API int hv_pdo_weights(hv_ctx* ctx, int32_t nz, int32_t nx, float h, float rho0, int32_t r, const float* thetas,
                          float* w);

/* ---- High-pass wrapper ("apply a high-pass filter to H_d before the
 * approximation"): out = Q v for K fields v, out [K][nz][nx], Q = IDFT diag(q) DFT with q(|xi|) = 0 below
 * cutoff - width/2, 1 above cutoff + width/2, raised cosine between (angular frequencies, grid spacing h). The
 * wrapped operator Q H_d Q is hv_highpass -> hv_hessvec -> hv_highpass. */
HV_API int hv_highpass(hv_ctx* ctx, int32_t nz, int32_t nx, float h, float cutoff, float width, int32_t K,
                       const float* v, float* out);

/* ---- Randomized low-rank generalized eigensolver (Eq. equ:eig):
 * leading r pairs of H_d v = lambda R v over the shard's shots, V^T R V = I, with R = (delta I - gamma Delta)^2 the
 * biharmonic prior precision applied as the periodic spectral multiplier (delta + gamma |xi|^2)^2.
 * Double-pass randomized algorithm with power_iters power iterations; each pass is ONE batched hv_hessvec on
 * K = r + oversampling probes. Omega [K][nz][nx] are the caller's random probes (e.g. N(0,1) draws).
 * evals [r] float64 descending (host or device), evecs [r][nz][nx] float32 (may be NULL). Multi-GPU note: the
 * eigensolve needs the FULL H_d, so call it on a context whose shard covers every shot. */
HV_API int hv_lowrank_geneig(hv_ctx* ctx, const float* m, int32_t r, int32_t K, const float* Omega,
                             int32_t power_iters, double delta, double gamma, double* evals, float* evecs);

/* ---- PSF+ (Eq. equ:psfplus): from symbol rows [nr][nz][nx] (complex64,
 * hv_psf_rows), their PSF weights w [nr][nz][nx] (hv_psf_weights) and symbol columns [nc][nz][nx] (complex64,
 * hv_pdo_columns) at DFT indices (col_kz, col_kx): B = leading `rank` right singular vectors of the rows,
 * A_0 = W U_r Sigma_r, A = (S_c B_c^H + alpha A_0)(B_c B_c^H + alpha I)^-1 with alpha = ||B_c||^2 / ||B||^2.
 * Outputs A [rank][nz][nx] (column k = a_k, complex64), B [rank][nz][nx] (complex64), *alpha (may be NULL).
 * Apply with hv_psido_apply(a = A, b = B, mode + 4). */
HV_API int hv_psf_plus(hv_ctx* ctx, int32_t nz, int32_t nx, int32_t nr, const float* rows, const float* w, int32_t nc,
                       const float* cols, const int32_t* col_kz, const int32_t* col_kx, int32_t rank, float* A,
                       float* B, double* alpha);

/* ---- NCCL helpers (the library dlopens libnccl.so.2; nothing links against it). Rank 0 calls hv_nccl_unique_id
 * and shares the 128 bytes with the other ranks (e.g. a torch.distributed broadcast); every rank then calls
 * hv_nccl_comm_create with its rank and CUDA device. The caller owns the communicator (hv_nccl_comm_destroy). */
HV_API int hv_nccl_unique_id(void* id_out /* 128 bytes */);
HV_API int hv_nccl_comm_create(int32_t nranks, int32_t rank, const void* id /* 128 bytes */, int32_t device,
                               void** comm_out);
HV_API int hv_nccl_comm_destroy(void* comm);

/* Counters of the last call (for benches). */
typedef struct {
  int64_t kernel_launches;   /* launches of this library's kernels in the last call           */
  int64_t graph_launches;    /* CUDA-graph replays in the last call                           */
  int32_t shot_batch;        /* shots in flight used                                          */
  int32_t field_group;       /* max Born fields per forward work unit used                    */
  int32_t store;             /* storage mode used                                             */
  int32_t ckpt_interval;
  double  bytes_per_shot;    /* device bytes per shot in flight                               */
  double  ms_forward;        /* device time of the forward sweeps (CUDA events), last call    */
  double  ms_backward;       /* device time of the backward sweeps, last call                 */
  double  ms_total;          /* device time of the whole call                                 */
  int32_t fwd_kernel;        /* forward sweep kernel used: 0 one-wave (fwd_step_kernel), 1 resident-q
                                (fwd_qres_kernel, Q > 48 MB), 3 two levels per launch (fwd_t2_kernel),
                                4 resident-q with thread-block clusters (fwd_qres_cl_kernel)        */
  int32_t bwd_kernel;        /* adjoint sweep kernel used: 0 bwd_step_kernel, 3 bwd_t2_kernel, -1 none   */
} hv_stats;
HV_API int hv_get_stats(const hv_ctx* ctx, hv_stats* out);

/* Human-readable detail of the last error on this context (never NULL). */
HV_API const char* hv_last_error(const hv_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* HV_H */
