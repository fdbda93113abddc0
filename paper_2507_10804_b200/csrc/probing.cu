// probing.cu — probe -> symbol assembly on the GPU, feeding hv_psido_apply.
//
// PSF: symbol row s(x_k, xi) = conj(DFT(p_k)), p_k = window of the response
//   H v_b around x_k rolled to the origin; spatial weights = bilinear hats on the sample lattice.
// PDO: column s(., xi_k) = IDFT(M_k . DFT(H v_p)) / phi_{xi_k}; frequency weights
//   w_k(xi) = (|xi| / rho0) t(theta - theta_k), t the even-r trigonometric interpolation kernel.
// Discrete conventions: DESIGN.md §3 R-probe. Transforms: cuFFT C2C; everything else is this file's kernels.
#include <cufft.h>

#include "hv_internal.h"

using namespace hvrt;

namespace {


int grid_for(long long n) { return static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16)); }

// p_k[z][x] = R_b[(iz_k + dz) mod nz][(ix_k + dx) mod nx] for |dz|, |dx| <= radius (dz = signed offset of z)
__global__ void psf_window_kernel(int nz, int nx, int np, const float* __restrict__ R, const int* __restrict__ piz,
                                  const int* __restrict__ pix, const int* __restrict__ pb, int radius,
                                  cufftComplex* __restrict__ out) {
  const long long n = (long long)nz * nx;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * np; q += (long long)gridDim.x * blockDim.x) {
    const int k = static_cast<int>(q / n);
    const int rem = static_cast<int>(q % n);
    const int z = rem / nx, x = rem % nx;
    const int dz = z <= nz / 2 ? z : z - nz;
    const int dx = x <= nx / 2 ? x : x - nx;
    float v = 0.0f;
    if (dz >= -radius && dz <= radius && dx >= -radius && dx <= radius) {
      const int sz = ((piz[k] + dz) % nz + nz) % nz, sx = ((pix[k] + dx) % nx + nx) % nx;
      v = R[(long long)pb[k] * n + (long long)sz * nx + sx];
    }
    out[q] = make_cuFloatComplex(v, 0.0f);
  }
}

__global__ void conj_kernel(long long n, cufftComplex* __restrict__ a) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    a[q].y = -a[q].y;
}

// 1-D hat basis on sorted lattice coordinates, constant outside: H[j][x]
__global__ void hat_kernel(int n, int nl, const int* __restrict__ lat, float* __restrict__ H) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n * nl; q += gridDim.x * blockDim.x) {
    const int j = q / n, x = q % n;
    float v;
    if (nl == 1) {
      v = 1.0f;
    } else if (x <= lat[0]) {
      v = j == 0 ? 1.0f : 0.0f;
    } else if (x >= lat[nl - 1]) {
      v = j == nl - 1 ? 1.0f : 0.0f;
    } else {
      int s = 0;
      while (s + 1 < nl - 1 && x >= lat[s + 1]) ++s;  // segment [lat[s], lat[s+1])
      const float t = static_cast<float>(x - lat[s]) / static_cast<float>(lat[s + 1] - lat[s]);
      v = (j == s) ? 1.0f - t : (j == s + 1 ? t : 0.0f);
    }
    H[q] = v;
  }
}

__global__ void outer_kernel(int nz, int nx, int nlz, int nlx, const float* __restrict__ hz,
                             const float* __restrict__ hx, float* __restrict__ w) {
  const long long n = (long long)nz * nx;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * nlz * nlx;
       q += (long long)gridDim.x * blockDim.x) {
    const int k = static_cast<int>(q / n);
    const int rem = static_cast<int>(q % n);
    const int z = rem / nx, x = rem % nx;
    w[q] = hz[(k / nlx) * nz + z] * hx[(k % nlx) * nx + x];
  }
}

__global__ void real_to_complex(long long n, const float* __restrict__ v, cufftComplex* __restrict__ X) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    X[q] = make_cuFloatComplex(v[q], 0.0f);
}

// T[k][f] = M_k(f) X[f], M_k = disc of `radius` cells around (kz_k, kx_k) (periodic index distance) with a
// raised-cosine roll-off of `rolloff` cells
__global__ void pdo_mask_kernel(int nz, int nx, int r, const int* __restrict__ kz, const int* __restrict__ kx,
                                float radius, float rolloff, const cufftComplex* __restrict__ X,
                                cufftComplex* __restrict__ T) {
  const long long n = (long long)nz * nx;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * r; q += (long long)gridDim.x * blockDim.x) {
    const int k = static_cast<int>(q / n);
    const int rem = static_cast<int>(q % n);
    const int z = rem / nx, x = rem % nx;
    const int dz = ((z - kz[k] + nz / 2) % nz + nz) % nz - nz / 2;
    const int dx = ((x - kx[k] + nx / 2) % nx + nx) % nx - nx / 2;
    const float d = sqrtf(static_cast<float>(dz * dz + dx * dx));
    float m = 0.0f;
    if (d <= radius) m = 1.0f;
    else if (d < radius + rolloff) m = 0.5f * (1.0f + cospif((d - radius) / rolloff));
    const cufftComplex v = X[rem];
    T[q] = make_cuFloatComplex(m * v.x, m * v.y);
  }
}

// col_k[z][x] = T_k[z][x] / (N phi_k), phi_k = exp(2 pi i (kz z / nz + kx x / nx))
__global__ void pdo_demod_kernel(int nz, int nx, int r, const int* __restrict__ kz, const int* __restrict__ kx,
                                 cufftComplex* __restrict__ T) {
  const long long n = (long long)nz * nx;
  const float inv_n = 1.0f / static_cast<float>(n);
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * r; q += (long long)gridDim.x * blockDim.x) {
    const int k = static_cast<int>(q / n);
    const int rem = static_cast<int>(q % n);
    const int z = rem / nx, x = rem % nx;
    // phase in turns, reduced exactly in integers before the float conversion
    const long long pz = ((long long)kz[k] * z) % nz, px = ((long long)kx[k] * x) % nx;
    const float turns = static_cast<float>(pz) / nz + static_cast<float>(px) / nx;
    float s, c;
    sincospif(2.0f * turns, &s, &c);
    const cufftComplex v = T[q];
    // v * conj(phi) / N
    T[q] = make_cuFloatComplex((v.x * c + v.y * s) * inv_n, (v.y * c - v.x * s) * inv_n);
  }
}

// w_k(f) = (|xi| / rho0) t(theta(xi) - theta_k), t(phi) = sin(r phi / 2) cot(phi / 2) / r (t -> cos(r phi / 2) at
// sin(phi / 2) = 0); xi from the unshifted DFT index, theta = atan2(xi_z, xi_x). Written as complex (imag 0).
__global__ void pdo_weight_kernel(int nz, int nx, float h, float rho0, int r, const float* __restrict__ thetas,
                                  cufftComplex* __restrict__ W) {
  const long long n = (long long)nz * nx;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * r; q += (long long)gridDim.x * blockDim.x) {
    const int k = static_cast<int>(q / n);
    const int rem = static_cast<int>(q % n);
    const int z = rem / nx, x = rem % nx;
    // unshifted DFT order, symmetric range [-n/2, n/2): index >= ceil(n/2) is negative
    const int fz = z >= (nz + 1) / 2 ? z - nz : z, fx = x >= (nx + 1) / 2 ? x - nx : x;
    const double xz = 2.0 * 3.14159265358979323846 * fz / (nz * (double)h);
    const double xx = 2.0 * 3.14159265358979323846 * fx / (nx * (double)h);
    const double rho = sqrt(xz * xz + xx * xx);
    const double phi = atan2(xz, xx) - (double)thetas[k];
    const double s = sin(phi / 2.0);
    double t;
    if (fabs(s) < 1e-12) t = cos(r * phi / 2.0);
    else t = sin(r * phi / 2.0) * cos(phi / 2.0) / (r * s);
    W[q] = make_cuFloatComplex(static_cast<float>(rho / rho0 * t), 0.0f);
  }
}

int plan_for(hv_ctx* c, int nz, int nx, int batch, cufftHandle* out) {
  auto key = std::make_tuple(nz, nx, batch);
  auto it = c->fft_plans.find(key);
  if (it == c->fft_plans.end()) {
    cufftHandle p;
    int dims[2] = {nz, nx};
    if (cufftPlanMany(&p, 2, dims, nullptr, 1, nz * nx, nullptr, 1, nz * nx, CUFFT_C2C, batch) != CUFFT_SUCCESS)
      return fail(c, HV_ECUDA, "cufftPlanMany failed");
    it = c->fft_plans.emplace(key, p).first;
  }
  if (cufftSetStream(it->second, c->stream) != CUFFT_SUCCESS) return fail(c, HV_ECUDA, "cufftSetStream failed");
  *out = it->second;
  return HV_OK;
}

int finish(hv_ctx* c, const OutStage& o, int64_t launches) {
  CU_TRY(cudaGetLastError());
  int st = finish_out(c, o);
  if (st) return st;
  CU_TRY(cudaStreamSynchronize(c->stream));
  c->stats = hv_stats{};
  c->stats.kernel_launches = launches;
  return HV_OK;
}

}  // namespace

extern "C" {

int hv_psf_rows(hv_ctx* c, int32_t nz, int32_t nx, int32_t nb, const float* responses, int32_t np,
                const int32_t* pt_iz, const int32_t* pt_ix, const int32_t* pt_batch, int32_t radius, float* rows) {
  if (!c) return HV_ESTATE;
  c->err.clear();
  if (nz < 1 || nx < 1 || nb < 1 || np < 1) return fail(c, HV_EGRID, "bad sizes");
  if (radius < 0 || 2 * radius + 1 > nz || 2 * radius + 1 > nx) return fail(c, HV_EINVAL, "bad radius");
  if (!pt_batch || !pt_iz || !pt_ix) return fail(c, HV_EINVAL, "null point arrays");
  if (!is_device_ptr(pt_batch))
    for (int k = 0; k < np; ++k)
      if (pt_batch[k] < 0 || pt_batch[k] >= nb) return fail(c, HV_EINVAL, "point batch index out of range");
  if (const int e_ = hvrt::enter(c)) return e_;
  const long long n = (long long)nz * nx;
  const float* R;
  const int *iz, *ix, *pb;
  int st;
  if ((st = stage_in(c, "psf_R", responses, sizeof(float) * n * nb, (const void**)&R))) return st;
  if ((st = stage_in(c, "psf_iz", pt_iz, sizeof(int) * np, (const void**)&iz))) return st;
  if ((st = stage_in(c, "psf_ix", pt_ix, sizeof(int) * np, (const void**)&ix))) return st;
  if ((st = stage_in(c, "psf_b", pt_batch, sizeof(int) * np, (const void**)&pb))) return st;
  OutStage o;
  if ((st = stage_out(c, "psf_rows", rows, sizeof(cufftComplex) * n * np, &o))) return st;
  cufftComplex* out = reinterpret_cast<cufftComplex*>(o.dev);
  psf_window_kernel<<<grid_for(n * np), 256, 0, c->stream>>>(nz, nx, np, R, iz, ix, pb, radius, out);
  cufftHandle p;
  if ((st = plan_for(c, nz, nx, np, &p))) return st;
  if (cufftExecC2C(p, out, out, CUFFT_FORWARD) != CUFFT_SUCCESS) return fail(c, HV_ECUDA, "cufftExecC2C");
  conj_kernel<<<grid_for(n * np), 256, 0, c->stream>>>(n * np, out);
  return finish(c, o, 2);
}

int hv_psf_weights(hv_ctx* c, int32_t nz, int32_t nx, int32_t nlz, const int32_t* lat_z, int32_t nlx,
                   const int32_t* lat_x, float* w) {
  if (!c) return HV_ESTATE;
  c->err.clear();
  if (nz < 1 || nx < 1 || nlz < 1 || nlx < 1) return fail(c, HV_EGRID, "bad sizes");
  if (const int e_ = hvrt::enter(c)) return e_;
  const int *lz, *lx;
  int st;
  if ((st = stage_in(c, "lat_z", lat_z, sizeof(int) * nlz, (const void**)&lz))) return st;
  if ((st = stage_in(c, "lat_x", lat_x, sizeof(int) * nlx, (const void**)&lx))) return st;
  float *hz, *hx;
  if ((st = ws_get(c, "hat_z", sizeof(float) * nz * nlz, (void**)&hz))) return st;
  if ((st = ws_get(c, "hat_x", sizeof(float) * nx * nlx, (void**)&hx))) return st;
  OutStage o;
  const long long n = (long long)nz * nx;
  if ((st = stage_out(c, "psf_w", w, sizeof(float) * n * nlz * nlx, &o))) return st;
  hat_kernel<<<grid_for((long long)nz * nlz), 256, 0, c->stream>>>(nz, nlz, lz, hz);
  hat_kernel<<<grid_for((long long)nx * nlx), 256, 0, c->stream>>>(nx, nlx, lx, hx);
  outer_kernel<<<grid_for(n * nlz * nlx), 256, 0, c->stream>>>(nz, nx, nlz, nlx, hz, hx,
                                                                 reinterpret_cast<float*>(o.dev));
  return finish(c, o, 3);
}

int hv_pdo_columns(hv_ctx* c, int32_t nz, int32_t nx, const float* response, int32_t r, const int32_t* kz_in,
                   const int32_t* kx_in, float mask_radius, float* cols) {
  if (!c) return HV_ESTATE;
  c->err.clear();
  if (nz < 1 || nx < 1 || r < 1) return fail(c, HV_EGRID, "bad sizes");
  if (!(mask_radius >= 0.0f)) return fail(c, HV_EINVAL, "bad mask radius");
  if (const int e_ = hvrt::enter(c)) return e_;
  const long long n = (long long)nz * nx;
  const float* R;
  const int *kz, *kx;
  int st;
  if ((st = stage_in(c, "pdo_R", response, sizeof(float) * n, (const void**)&R))) return st;
  if ((st = stage_in(c, "pdo_kz", kz_in, sizeof(int) * r, (const void**)&kz))) return st;
  if ((st = stage_in(c, "pdo_kx", kx_in, sizeof(int) * r, (const void**)&kx))) return st;
  cufftComplex* X;
  if ((st = ws_get(c, "pdo_X", sizeof(cufftComplex) * n, (void**)&X))) return st;
  OutStage o;
  if ((st = stage_out(c, "pdo_cols", cols, sizeof(cufftComplex) * n * r, &o))) return st;
  cufftComplex* T = reinterpret_cast<cufftComplex*>(o.dev);
  cufftHandle p1, pr;
  if ((st = plan_for(c, nz, nx, 1, &p1)) || (st = plan_for(c, nz, nx, r, &pr))) return st;
  real_to_complex<<<grid_for(n), 256, 0, c->stream>>>(n, R, X);
  if (cufftExecC2C(p1, X, X, CUFFT_FORWARD) != CUFFT_SUCCESS) return fail(c, HV_ECUDA, "cufftExecC2C");
  pdo_mask_kernel<<<grid_for(n * r), 256, 0, c->stream>>>(nz, nx, r, kz, kx, mask_radius, 2.0f, X, T);
  if (cufftExecC2C(pr, T, T, CUFFT_INVERSE) != CUFFT_SUCCESS) return fail(c, HV_ECUDA, "cufftExecC2C");
  pdo_demod_kernel<<<grid_for(n * r), 256, 0, c->stream>>>(nz, nx, r, kz, kx, T);
  return finish(c, o, 3);
}

int hv_pdo_weights(hv_ctx* c, int32_t nz, int32_t nx, float h, float rho0, int32_t r, const float* thetas_in,
                   float* w) {
  if (!c) return HV_ESTATE;
  c->err.clear();
  if (nz < 1 || nx < 1 || r < 2 || (r % 2)) return fail(c, HV_EINVAL, "r must be even and >= 2");
  if (!(h > 0.0f) || !(rho0 > 0.0f)) return fail(c, HV_EINVAL, "h and rho0 must be positive");
  if (const int e_ = hvrt::enter(c)) return e_;
  const long long n = (long long)nz * nx;
  const float* th;
  int st;
  if ((st = stage_in(c, "pdo_th", thetas_in, sizeof(float) * r, (const void**)&th))) return st;
  OutStage o;
  if ((st = stage_out(c, "pdo_w", w, sizeof(cufftComplex) * n * r, &o))) return st;
  pdo_weight_kernel<<<grid_for(n * r), 256, 0, c->stream>>>(nz, nx, h, rho0, r, th,
                                                             reinterpret_cast<cufftComplex*>(o.dev));
  return finish(c, o, 1);
}

}  // extern "C"
