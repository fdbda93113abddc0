// psido.cu — low-rank-symbol PsiDO apply, hv_psido_apply (include/hv.h, Eq. equ:lr-psido).
//
//   mode 0: out = Re sum_k a_k . IDFT(b_k . DFT(v))          "one Fourier transform, r inverse Fourier transforms,
//                                                              and 2r pointwise multiplications"
//   mode 1: out = Re IDFT(sum_k conj(b_k) . DFT(a_k . v))    adjoint: r forward transforms, one inverse
//   mode 2: (mode 0 + mode 1) / 2
// The 2-D DFTs are cuFFT C2C (library FFT, like cuBLAS for a GEMM); the pointwise multiplies and the
// r-way reductions are this file's kernels, fused so each complex plane is touched once per pass.
#include <cufft.h>

#include "hv_internal.h"

using namespace hvrt;

namespace {

__global__ void psido_real_to_complex(long long n, const float* __restrict__ v, cufftComplex* __restrict__ X) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    X[q] = make_cuFloatComplex(v[q], 0.0f);
}

// T[k][p] = b_k[p] * X[p]
__global__ void psido_symbol_mul(long long n, int r, const cufftComplex* __restrict__ b,
                                 const cufftComplex* __restrict__ X, cufftComplex* __restrict__ T) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * r;
       q += (long long)gridDim.x * blockDim.x)
    T[q] = cuCmulf(b[q], X[q % n]);
}

// out[p] (+)= scale * sum_k Re(a_k[p] T[k][p])   (a real, or complex when ca)
__global__ void psido_combine(long long n, int r, const float* __restrict__ a, int ca,
                              const cufftComplex* __restrict__ T, float scale, int accumulate, float* __restrict__ out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    float s = 0.0f;
    for (int k = 0; k < r; ++k) {
      const cufftComplex t = T[k * n + q];
      if (ca) {
        const float2 ak = reinterpret_cast<const float2*>(a)[k * n + q];
        s = fmaf(ak.x, t.x, fmaf(-ak.y, t.y, s));
      } else {
        s = fmaf(a[k * n + q], cuCrealf(t), s);
      }
    }
    out[q] = accumulate ? out[q] + scale * s : scale * s;
  }
}

// Y[k][p] = conj(a_k[p]) v[p]   (a real, or complex when ca)
__global__ void psido_weight(long long n, int r, const float* __restrict__ a, int ca, const float* __restrict__ v,
                             cufftComplex* __restrict__ Y) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * r;
       q += (long long)gridDim.x * blockDim.x) {
    const float vv = v[q % n];
    if (ca) {
      const float2 ak = reinterpret_cast<const float2*>(a)[q];
      Y[q] = make_cuFloatComplex(ak.x * vv, -ak.y * vv);
    } else {
      Y[q] = make_cuFloatComplex(a[q] * vv, 0.0f);
    }
  }
}

// Z[p] = sum_k conj(b_k[p]) Y[k][p]
__global__ void psido_conj_reduce(long long n, int r, const cufftComplex* __restrict__ b,
                                  const cufftComplex* __restrict__ Y, cufftComplex* __restrict__ Z) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    cufftComplex s = make_cuFloatComplex(0.f, 0.f);
    for (int k = 0; k < r; ++k) s = cuCaddf(s, cuCmulf(cuConjf(b[k * n + q]), Y[k * n + q]));
    Z[q] = s;
  }
}

// out[p] (+)= scale * Re Z[p]
__global__ void psido_real_out(long long n, const cufftComplex* __restrict__ Z, float scale, int accumulate,
                               float* __restrict__ out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    out[q] = accumulate ? out[q] + scale * cuCrealf(Z[q]) : scale * cuCrealf(Z[q]);
}

// High-pass multiplier q(|xi|) (raised cosine between cutoff -+ width/2), applied in place to K spectra; scale 1/N
__global__ void highpass_mul(int nz, int nx, int K, float h, float cutoff, float width, cufftComplex* __restrict__ T) {
  const long long n = (long long)nz * nx;
  const float lo = cutoff - 0.5f * width, hi = cutoff + 0.5f * width;
  const float inv_n = 1.0f / static_cast<float>(n);
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * K; q += (long long)gridDim.x * blockDim.x) {
    const int rem = static_cast<int>(q % n);
    const int z = rem / nx, x = rem % nx;
    const int fz = z >= (nz + 1) / 2 ? z - nz : z, fx = x >= (nx + 1) / 2 ? x - nx : x;
    const float xz = 6.283185307179586f * fz / (nz * h), xx = 6.283185307179586f * fx / (nx * h);
    const float rho = sqrtf(xz * xz + xx * xx);
    float m;
    if (rho >= hi) m = 1.0f;
    else if (rho <= lo) m = 0.0f;
    else m = 0.5f * (1.0f - cospif((rho - lo) / width));
    m *= inv_n;
    T[q] = make_cuFloatComplex(m * T[q].x, m * T[q].y);
  }
}

__global__ void real_part_out(long long n, const cufftComplex* __restrict__ T, float* __restrict__ out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    out[q] = cuCrealf(T[q]);
}

__global__ void reals_to_complex(long long n, const float* __restrict__ v, cufftComplex* __restrict__ X) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    X[q] = make_cuFloatComplex(v[q], 0.0f);
}

int grid_for(long long n) { return static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16)); }

int get_plan(hv_ctx* c, int nz, int nx, int batch, cufftHandle* out) {
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

}  // namespace

extern "C" int hv_psido_apply(hv_ctx* c, int32_t nz, int32_t nx, int32_t r, const float* a_in, const float* b_in,
                              const float* v_in, float* out_user, int32_t mode) {
  if (!c) return HV_ESTATE;
  c->err.clear();
  if (nz < 1 || nx < 1) return fail(c, HV_EGRID, "bad grid");
  if (r < 1) return fail(c, HV_EINVAL, "r must be >= 1");
  const int ca = (mode & 4) ? 1 : 0;  // complex spatial factors (PSF+)
  mode &= 3;
  if (mode > 2) return fail(c, HV_EINVAL, "mode must be 0, 1 or 2 (+4 for complex a)");
  if (const int e_ = hvrt::enter(c)) return e_;
  const long long n = (long long)nz * nx;
  const float *a, *b, *v;
  int st;
  if ((st = stage_in(c, "psido_a", a_in, sizeof(float) * n * r * (ca ? 2 : 1), (const void**)&a))) return st;
  if ((st = stage_in(c, "psido_b", b_in, sizeof(cufftComplex) * n * r, (const void**)&b))) return st;
  if ((st = stage_in(c, "psido_v", v_in, sizeof(float) * n, (const void**)&v))) return st;
  OutStage o;
  if ((st = stage_out(c, "psido_out", out_user, sizeof(float) * n, &o))) return st;
  float* out = reinterpret_cast<float*>(o.dev);
  cufftComplex *X, *T;
  if ((st = ws_get(c, "psido_X", sizeof(cufftComplex) * n, (void**)&X))) return st;
  if ((st = ws_get(c, "psido_T", sizeof(cufftComplex) * n * r, (void**)&T))) return st;
  const cufftComplex* bc = reinterpret_cast<const cufftComplex*>(b);
  cufftHandle p1, pr;
  if ((st = get_plan(c, nz, nx, 1, &p1)) || (st = get_plan(c, nz, nx, r, &pr))) return st;
  const float inv_n = 1.0f / static_cast<float>(n);
  const float half = (mode == 2) ? 0.5f : 1.0f;
  int64_t launches = 0;
  if (mode == 0 || mode == 2) {
    psido_real_to_complex<<<grid_for(n), 256, 0, c->stream>>>(n, v, X);
    if (cufftExecC2C(p1, X, X, CUFFT_FORWARD) != CUFFT_SUCCESS) return fail(c, HV_ECUDA, "cufftExecC2C");
    psido_symbol_mul<<<grid_for(n * r), 256, 0, c->stream>>>(n, r, bc, X, T);
    if (cufftExecC2C(pr, T, T, CUFFT_INVERSE) != CUFFT_SUCCESS) return fail(c, HV_ECUDA, "cufftExecC2C");
    psido_combine<<<grid_for(n), 256, 0, c->stream>>>(n, r, a, ca, T, half * inv_n, 0, out);
    launches += 3;
  }
  if (mode == 1 || mode == 2) {
    psido_weight<<<grid_for(n * r), 256, 0, c->stream>>>(n, r, a, ca, v, T);
    if (cufftExecC2C(pr, T, T, CUFFT_FORWARD) != CUFFT_SUCCESS) return fail(c, HV_ECUDA, "cufftExecC2C");
    psido_conj_reduce<<<grid_for(n), 256, 0, c->stream>>>(n, r, bc, T, X);
    if (cufftExecC2C(p1, X, X, CUFFT_INVERSE) != CUFFT_SUCCESS) return fail(c, HV_ECUDA, "cufftExecC2C");
    psido_real_out<<<grid_for(n), 256, 0, c->stream>>>(n, X, half * inv_n, mode == 2, out);
    launches += 3;
  }
  CU_TRY(cudaGetLastError());
  if ((st = finish_out(c, o))) return st;
  CU_TRY(cudaStreamSynchronize(c->stream));
  c->stats = hv_stats{};
  c->stats.kernel_launches = launches;
  return HV_OK;
}

// High-pass filter Q = IDFT diag(q) DFT on K fields. v, out [K][nz][nx].
extern "C" int hv_highpass(hv_ctx* c, int32_t nz, int32_t nx, float h, float cutoff, float width, int32_t K,
                           const float* v_in, float* out_user) {
  if (!c) return HV_ESTATE;
  c->err.clear();
  if (nz < 1 || nx < 1 || K < 1) return fail(c, HV_EGRID, "bad sizes");
  if (!(h > 0.0f) || !(width > 0.0f) || !(cutoff >= 0.0f)) return fail(c, HV_EINVAL, "bad filter parameters");
  if (const int e_ = hvrt::enter(c)) return e_;
  const long long n = (long long)nz * nx;
  const float* v;
  int st;
  if ((st = stage_in(c, "hp_v", v_in, sizeof(float) * n * K, (const void**)&v))) return st;
  OutStage o;
  if ((st = stage_out(c, "hp_out", out_user, sizeof(float) * n * K, &o))) return st;
  cufftComplex* T;
  if ((st = ws_get(c, "hp_T", sizeof(cufftComplex) * n * K, (void**)&T))) return st;
  cufftHandle p;
  if ((st = get_plan(c, nz, nx, K, &p))) return st;
  reals_to_complex<<<grid_for(n * K), 256, 0, c->stream>>>(n * K, v, T);
  if (cufftExecC2C(p, T, T, CUFFT_FORWARD) != CUFFT_SUCCESS) return fail(c, HV_ECUDA, "cufftExecC2C");
  highpass_mul<<<grid_for(n * K), 256, 0, c->stream>>>(nz, nx, K, h, cutoff, width, T);
  if (cufftExecC2C(p, T, T, CUFFT_INVERSE) != CUFFT_SUCCESS) return fail(c, HV_ECUDA, "cufftExecC2C");
  real_part_out<<<grid_for(n * K), 256, 0, c->stream>>>(n * K, T, reinterpret_cast<float*>(o.dev));
  CU_TRY(cudaGetLastError());
  if ((st = finish_out(c, o))) return st;
  CU_TRY(cudaStreamSynchronize(c->stream));
  c->stats = hv_stats{};
  c->stats.kernel_launches = 3;
  return HV_OK;
}
