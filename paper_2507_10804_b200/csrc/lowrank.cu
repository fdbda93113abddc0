// lowrank.cu — randomized low-rank generalized eigensolver H_d v = lambda R v (PAPER.md:168-195,
// Eq. equ:eig). Double pass with power iterations (N2):
//   Y = R^-1 H_d Omega; [Q = R-orth(Y); Y = R^-1 H_d Q] x power_iters; Q = R-orth(Y); T = Q^T H_d Q = U L U^T;
//   V = Q U (leading r).
// H_d products: this library's batched hv_hessvec (one call per pass, K = r + oversampling probes).
// R^{+-1}: periodic spectral multiplier (delta + gamma |xi|^2)^{+-2} (cuFFT Z2Z + this file's kernel).
// Small dense algebra in fp64: cuBLAS DGEMM / DTRSM, cuSOLVER DPOTRF / DSYEVD (plain library calls).
#include <cublas_v2.h>
#include <cufft.h>
#include <cusolverDn.h>

#include <cmath>
#include <vector>

#include "hv_internal.h"

using namespace hvrt;

namespace {

int grid_for(long long n) { return static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16)); }

__global__ void d_to_z(long long n, const double* __restrict__ a, cufftDoubleComplex* __restrict__ z) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    z[q] = make_cuDoubleComplex(a[q], 0.0);
}
__global__ void z_real_to_d(long long n, const cufftDoubleComplex* __restrict__ z, double* __restrict__ a) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    a[q] = z[q].x;
}
__global__ void d_to_f32(long long n, const double* __restrict__ a, float* __restrict__ b) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    b[q] = static_cast<float>(a[q]);
}
__global__ void f32_to_d(long long n, const float* __restrict__ a, double* __restrict__ b) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    b[q] = static_cast<double>(a[q]);
}
// spectra *= (delta + gamma |xi|^2)^(2 power) / N
__global__ void prior_mul(int nz, int nx, int K, double h, double delta, double gamma, double power,
                          cufftDoubleComplex* __restrict__ Z) {
  const long long n = (long long)nz * nx;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n * K; q += (long long)gridDim.x * blockDim.x) {
    const int rem = static_cast<int>(q % n);
    const int z = rem / nx, x = rem % nx;
    const int fz = z >= (nz + 1) / 2 ? z - nz : z, fx = x >= (nx + 1) / 2 ? x - nx : x;
    const double xz = 2.0 * 3.14159265358979323846 * fz / (nz * h);
    const double xx = 2.0 * 3.14159265358979323846 * fx / (nx * h);
    const double s = pow(delta + gamma * (xz * xz + xx * xx), 2.0 * power) / static_cast<double>(n);
    Z[q] = make_cuDoubleComplex(Z[q].x * s, Z[q].y * s);
  }
}

struct Dense {
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t sol = nullptr;
  ~Dense() {
    if (blas) cublasDestroy(blas);
    if (sol) cusolverDnDestroy(sol);
  }
};

}  // namespace

extern "C" int hv_lowrank_geneig(hv_ctx* c, const float* m, int32_t r, int32_t K, const float* omega_in,
                                 int32_t power_iters, double delta, double gamma, double* evals_user,
                                 float* evecs_user) {
  if (!c) return HV_ESTATE;
  c->err.clear();
  if (r < 1 || K < r || power_iters < 0) return fail(c, HV_EINVAL, "need 1 <= r <= K, power_iters >= 0");
  if (!(delta > 0.0) || !(gamma >= 0.0)) return fail(c, HV_EINVAL, "delta must be > 0, gamma >= 0");
  if (!evals_user) return fail(c, HV_EINVAL, "null evals");
  if (const int e_ = hvrt::enter(c)) return e_;
  const int nz = c->g.nz, nx = c->g.nx;
  const long long N = (long long)nz * nx;
  const double h = c->cfg.h;
  const float *md, *Om;
  int st;
  if ((st = stage_in(c, "le_m", m, sizeof(float) * N, (const void**)&md))) return st;
  // Omega is read through hv_hessvec and must stay valid while "le_m" staging is reused -> copy to own buffer
  if ((st = stage_in(c, "le_om", omega_in, sizeof(float) * N * K, (const void**)&Om))) return st;
  OutStage ov;
  if (evecs_user && (st = stage_out(c, "le_vec", evecs_user, sizeof(float) * N * r, &ov))) return st;
  float *Yf, *HQf;
  double *Yd, *RYd, *G, *T, *Wv, *Vd;
  cufftDoubleComplex* Z;
  if ((st = ws_get(c, "le_Yf", sizeof(float) * N * K, (void**)&Yf))) return st;
  if ((st = ws_get(c, "le_HQf", sizeof(float) * N * K, (void**)&HQf))) return st;
  if ((st = ws_get(c, "le_Yd", sizeof(double) * N * K, (void**)&Yd))) return st;
  if ((st = ws_get(c, "le_RYd", sizeof(double) * N * K, (void**)&RYd))) return st;
  if ((st = ws_get(c, "le_Z", sizeof(cufftDoubleComplex) * N * K, (void**)&Z))) return st;
  if ((st = ws_get(c, "le_G", sizeof(double) * K * K, (void**)&G))) return st;
  if ((st = ws_get(c, "le_T", sizeof(double) * K * K, (void**)&T))) return st;
  if ((st = ws_get(c, "le_W", sizeof(double) * K, (void**)&Wv))) return st;
  if ((st = ws_get(c, "le_Vd", sizeof(double) * N * r, (void**)&Vd))) return st;
  int* info;
  if ((st = ws_get(c, "le_info", sizeof(int) * 4, (void**)&info))) return st;

  Dense dn;
  if (cublasCreate(&dn.blas) != CUBLAS_STATUS_SUCCESS) return fail(c, HV_ECUDA, "cublasCreate");
  if (cusolverDnCreate(&dn.sol) != CUSOLVER_STATUS_SUCCESS) return fail(c, HV_ECUDA, "cusolverDnCreate");
  cublasSetStream(dn.blas, c->stream);
  cusolverDnSetStream(dn.sol, c->stream);
  cufftHandle pz;
  int dims[2] = {nz, nx};
  if (cufftPlanMany(&pz, 2, dims, nullptr, 1, (int)N, nullptr, 1, (int)N, CUFFT_Z2Z, K) != CUFFT_SUCCESS)
    return fail(c, HV_ECUDA, "cufftPlanMany Z2Z");
  struct PlanGuard {
    cufftHandle p;
    ~PlanGuard() { cufftDestroy(p); }
  } pg{pz};
  cufftSetStream(pz, c->stream);

  int64_t launches = 0, hv_calls = 0;
  // out (fp64) = R^power applied to the K fp64 fields in `in`
  auto prior = [&](const double* in, double* out, double power) -> int {
    d_to_z<<<grid_for(N * K), 256, 0, c->stream>>>(N * K, in, Z);
    if (cufftExecZ2Z(pz, Z, Z, CUFFT_FORWARD) != CUFFT_SUCCESS) return fail(c, HV_ECUDA, "cufftExecZ2Z");
    prior_mul<<<grid_for(N * K), 256, 0, c->stream>>>(nz, nx, K, h, delta, gamma, power, Z);
    if (cufftExecZ2Z(pz, Z, Z, CUFFT_INVERSE) != CUFFT_SUCCESS) return fail(c, HV_ECUDA, "cufftExecZ2Z");
    z_real_to_d<<<grid_for(N * K), 256, 0, c->stream>>>(N * K, Z, out);
    launches += 3;
    return HV_OK;
  };
  // Yd = R^-1 H_d (fp32 fields `in`)
  auto rinv_h = [&](const float* in) -> int {
    int s2 = hv_hessvec(c, md, K, in, HQf);
    if (s2) return s2;
    ++hv_calls;
    launches += c->stats.kernel_launches;
    f32_to_d<<<grid_for(N * K), 256, 0, c->stream>>>(N * K, HQf, Yd);
    return prior(Yd, Yd, -1.0);
  };
  // Yd <- R-orthonormal basis (Cholesky QR in the R inner product, twice); column-major N x K
  auto r_orth = [&]() -> int {
    for (int pass = 0; pass < 2; ++pass) {
      int s2 = prior(Yd, RYd, 1.0);
      if (s2) return s2;
      const double one = 1.0, zero = 0.0;
      if (cublasDgemm(dn.blas, CUBLAS_OP_T, CUBLAS_OP_N, K, K, (int)N, &one, Yd, (int)N, RYd, (int)N, &zero, G, K) !=
          CUBLAS_STATUS_SUCCESS)
        return fail(c, HV_ECUDA, "cublasDgemm (Gram)");
      int lw = 0;
      cusolverDnDpotrf_bufferSize(dn.sol, CUBLAS_FILL_MODE_LOWER, K, G, K, &lw);
      double* work;
      if ((s2 = ws_get(c, "le_work", sizeof(double) * std::max(lw, 1), (void**)&work))) return s2;
      if (cusolverDnDpotrf(dn.sol, CUBLAS_FILL_MODE_LOWER, K, G, K, work, lw, info) != CUSOLVER_STATUS_SUCCESS)
        return fail(c, HV_ECUDA, "cusolverDnDpotrf");
      int hinfo = 0;
      CU_TRY(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CU_TRY(cudaStreamSynchronize(c->stream));
      if (hinfo != 0) return fail(c, HV_ECUDA, "R-Gram matrix not positive definite (probes dependent)");
      // Y <- Y L^-T
      if (cublasDtrsm(dn.blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, (int)N, K,
                      &one, G, K, Yd, (int)N) != CUBLAS_STATUS_SUCCESS)
        return fail(c, HV_ECUDA, "cublasDtrsm");
    }
    return HV_OK;
  };

  if ((st = rinv_h(Om))) return st;
  for (int q = 0; q < power_iters; ++q) {
    if ((st = r_orth())) return st;
    d_to_f32<<<grid_for(N * K), 256, 0, c->stream>>>(N * K, Yd, Yf);
    if ((st = rinv_h(Yf))) return st;
  }
  if ((st = r_orth())) return st;
  d_to_f32<<<grid_for(N * K), 256, 0, c->stream>>>(N * K, Yd, Yf);
  if ((st = hv_hessvec(c, md, K, Yf, HQf))) return st;
  ++hv_calls;
  launches += c->stats.kernel_launches;
  f32_to_d<<<grid_for(N * K), 256, 0, c->stream>>>(N * K, HQf, RYd);
  const double one = 1.0, zero = 0.0;
  if (cublasDgemm(dn.blas, CUBLAS_OP_T, CUBLAS_OP_N, K, K, (int)N, &one, Yd, (int)N, RYd, (int)N, &zero, T, K) !=
      CUBLAS_STATUS_SUCCESS)
    return fail(c, HV_ECUDA, "cublasDgemm (T)");
  // symmetrise T and take its eigen-decomposition (ascending)
  {
    std::vector<double> hT((size_t)K * K);
    CU_TRY(cudaMemcpyAsync(hT.data(), T, sizeof(double) * K * K, cudaMemcpyDeviceToHost, c->stream));
    CU_TRY(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < K; ++i)
      for (int j = 0; j < i; ++j) hT[(size_t)i * K + j] = hT[(size_t)j * K + i] = 0.5 * (hT[(size_t)i * K + j] + hT[(size_t)j * K + i]);
    CU_TRY(cudaMemcpyAsync(T, hT.data(), sizeof(double) * K * K, cudaMemcpyHostToDevice, c->stream));
  }
  int lw = 0;
  cusolverDnDsyevd_bufferSize(dn.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, K, T, K, Wv, &lw);
  double* work;
  if ((st = ws_get(c, "le_work2", sizeof(double) * std::max(lw, 1), (void**)&work))) return st;
  if (cusolverDnDsyevd(dn.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, K, T, K, Wv, work, lw, info) !=
      CUSOLVER_STATUS_SUCCESS)
    return fail(c, HV_ECUDA, "cusolverDnDsyevd");
  // leading r (descending): columns K-1 .. K-r of T
  std::vector<double> w(K);
  CU_TRY(cudaMemcpyAsync(w.data(), Wv, sizeof(double) * K, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(cudaStreamSynchronize(c->stream));
  std::vector<double> ev(r);
  for (int i = 0; i < r; ++i) ev[i] = w[K - 1 - i];
  if (is_device_ptr(evals_user)) {
    CU_TRY(cudaMemcpyAsync(evals_user, ev.data(), sizeof(double) * r, cudaMemcpyHostToDevice, c->stream));
  } else {
    for (int i = 0; i < r; ++i) evals_user[i] = ev[i];
  }
  if (evecs_user) {
    for (int i = 0; i < r; ++i) {  // V[:, i] = Q U[:, K-1-i]
      if (cublasDgemv(dn.blas, CUBLAS_OP_N, (int)N, K, &one, Yd, (int)N, T + (size_t)(K - 1 - i) * K, 1, &zero,
                      Vd + (size_t)i * N, 1) != CUBLAS_STATUS_SUCCESS)
        return fail(c, HV_ECUDA, "cublasDgemv");
    }
    d_to_f32<<<grid_for(N * r), 256, 0, c->stream>>>(N * r, Vd, reinterpret_cast<float*>(ov.dev));
    if ((st = finish_out(c, ov))) return st;
  }
  CU_TRY(cudaGetLastError());
  CU_TRY(cudaStreamSynchronize(c->stream));
  c->stats = hv_stats{};
  c->stats.kernel_launches = launches;
  (void)hv_calls;
  return HV_OK;
}
