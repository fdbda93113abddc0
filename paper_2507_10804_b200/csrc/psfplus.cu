// psfplus.cu — PSF+ (Eq. equ:psfplus), restated in DESIGN.md §1 (N3):
//  (ii)  SVD of the symbol rows S~[I_r,:] (nr x N) through the nr x nr Gram matrix: B = Sigma_r^-1 U_r^H S~[I_r,:],
//        A_0 = W U_r Sigma_r (so S_psf = W S~[I_r,:] = A_0 B up to the discarded singular values)
//  (iii) A = (S~[:,I_c] B_c^H + alpha A_0)(B_c B_c^H + alpha I)^-1, alpha = ||B_c||_F^2 / ||B||_F^2, B_c = B[:, I_c].
// Dense algebra in complex128: cuBLAS ZGEMM, cuSOLVER ZHEEVD (library calls); the rank x rank inverse on the host.
// Layout: a field list [k][N] row-major is the column-major N x k matrix cuBLAS sees.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <cmath>
#include <complex>
#include <vector>

#include "hv_internal.h"

using namespace hvrt;
using zc = cuDoubleComplex;

namespace {

int grid_for(long long n) { return static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 16)); }

__global__ void c64_to_z(long long n, const float2* __restrict__ a, zc* __restrict__ z) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    z[q] = make_cuDoubleComplex(a[q].x, a[q].y);
}
__global__ void f32_to_zr(long long n, const float* __restrict__ a, zc* __restrict__ z) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    z[q] = make_cuDoubleComplex(a[q], 0.0);
}
__global__ void z_to_c64(long long n, const zc* __restrict__ z, float2* __restrict__ a) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
    a[q] = make_float2(static_cast<float>(z[q].x), static_cast<float>(z[q].y));
}
// Bc[j + rank * c] = Bm[ic[c] + N * j]
__global__ void gather_cols(long long N, int rank, int nc, const int* __restrict__ ic, const zc* __restrict__ Bm,
                            zc* __restrict__ Bc) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= rank * nc) return;
  const int j = q % rank, c = q / rank;
  Bc[q] = Bm[ic[c] + N * j];
}

struct Dense {
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t sol = nullptr;
  ~Dense() {
    if (blas) cublasDestroy(blas);
    if (sol) cusolverDnDestroy(sol);
  }
};

// host Gauss-Jordan inverse of a small complex matrix (column-major n x n)
bool invert(std::vector<std::complex<double>>& M, int n) {
  std::vector<std::complex<double>> I(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) I[i + (size_t)n * i] = 1.0;
  auto at = [n](std::vector<std::complex<double>>& X, int r, int c) -> std::complex<double>& { return X[r + (size_t)n * c]; };
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::abs(at(M, r, col)) > std::abs(at(M, piv, col))) piv = r;
    if (std::abs(at(M, piv, col)) == 0.0) return false;
    if (piv != col)
      for (int c = 0; c < n; ++c) {
        std::swap(at(M, piv, c), at(M, col, c));
        std::swap(at(I, piv, c), at(I, col, c));
      }
    const std::complex<double> d = 1.0 / at(M, col, col);
    for (int c = 0; c < n; ++c) {
      at(M, col, c) *= d;
      at(I, col, c) *= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      const std::complex<double> f = at(M, r, col);
      if (f == 0.0) continue;
      for (int c = 0; c < n; ++c) {
        at(M, r, c) -= f * at(M, col, c);
        at(I, r, c) -= f * at(I, col, c);
      }
    }
  }
  M = I;
  return true;
}

}  // namespace

extern "C" int hv_psf_plus(hv_ctx* c, int32_t nz, int32_t nx, int32_t nr, const float* rows_in, const float* w_in,
                           int32_t nc, const float* cols_in, const int32_t* col_kz, const int32_t* col_kx,
                           int32_t rank, float* A_user, float* B_user, double* alpha_user) {
  if (!c) return HV_ESTATE;
  c->err.clear();
  if (nz < 1 || nx < 1 || nr < 1 || nc < 1) return fail(c, HV_EGRID, "bad sizes");
  if (rank < 1 || rank > nr) return fail(c, HV_EINVAL, "need 1 <= rank <= nr");
  if (!col_kz || !col_kx) return fail(c, HV_EINVAL, "null column indices");
  if (const int e_ = hvrt::enter(c)) return e_;
  const long long N = (long long)nz * nx;
  std::vector<int> ic(nc);
  {
    std::vector<int> kz(nc), kx(nc);
    if (is_device_ptr(col_kz)) {
      CU_TRY(cudaMemcpy(kz.data(), col_kz, sizeof(int) * nc, cudaMemcpyDeviceToHost));
      CU_TRY(cudaMemcpy(kx.data(), col_kx, sizeof(int) * nc, cudaMemcpyDeviceToHost));
    } else {
      for (int i = 0; i < nc; ++i) kz[i] = col_kz[i], kx[i] = col_kx[i];
    }
    for (int i = 0; i < nc; ++i) {
      if (kz[i] < 0 || kz[i] >= nz || kx[i] < 0 || kx[i] >= nx) return fail(c, HV_EINVAL, "column index out of range");
      ic[i] = kz[i] * nx + kx[i];
    }
  }
  const float *rows, *w, *cols;
  int st;
  if ((st = stage_in(c, "pp_rows", rows_in, sizeof(float2) * N * nr, (const void**)&rows))) return st;
  if ((st = stage_in(c, "pp_w", w_in, sizeof(float) * N * nr, (const void**)&w))) return st;
  if ((st = stage_in(c, "pp_cols", cols_in, sizeof(float2) * N * nc, (const void**)&cols))) return st;
  OutStage oA, oB;
  if ((st = stage_out(c, "pp_A", A_user, sizeof(float2) * N * rank, &oA))) return st;
  if ((st = stage_out(c, "pp_B", B_user, sizeof(float2) * N * rank, &oB))) return st;
  zc *Rm, *Wm, *Sc, *Bm, *A0, *RHS, *G, *E, *Bc, *Msm, *tmp;
  double* ev;
  int* dic;
  int* info;
  if ((st = ws_get(c, "pp_Rm", sizeof(zc) * N * nr, (void**)&Rm)) || (st = ws_get(c, "pp_Wm", sizeof(zc) * N * nr, (void**)&Wm)) ||
      (st = ws_get(c, "pp_Sc", sizeof(zc) * N * nc, (void**)&Sc)) || (st = ws_get(c, "pp_Bm", sizeof(zc) * N * rank, (void**)&Bm)) ||
      (st = ws_get(c, "pp_A0", sizeof(zc) * N * rank, (void**)&A0)) ||
      (st = ws_get(c, "pp_RHS", sizeof(zc) * N * rank, (void**)&RHS)) ||
      (st = ws_get(c, "pp_G", sizeof(zc) * nr * nr, (void**)&G)) || (st = ws_get(c, "pp_E", sizeof(zc) * nr * rank, (void**)&E)) ||
      (st = ws_get(c, "pp_Bc", sizeof(zc) * rank * nc, (void**)&Bc)) ||
      (st = ws_get(c, "pp_M", sizeof(zc) * rank * rank, (void**)&Msm)) ||
      (st = ws_get(c, "pp_tmp", sizeof(zc) * nr * rank, (void**)&tmp)) ||
      (st = ws_get(c, "pp_ev", sizeof(double) * nr, (void**)&ev)) || (st = ws_get(c, "pp_ic", sizeof(int) * nc, (void**)&dic)) ||
      (st = ws_get(c, "pp_info", sizeof(int) * 4, (void**)&info)))
    return st;
  CU_TRY(cudaMemcpyAsync(dic, ic.data(), sizeof(int) * nc, cudaMemcpyHostToDevice, c->stream));
  c64_to_z<<<grid_for(N * nr), 256, 0, c->stream>>>(N * nr, reinterpret_cast<const float2*>(rows), Rm);
  f32_to_zr<<<grid_for(N * nr), 256, 0, c->stream>>>(N * nr, w, Wm);
  c64_to_z<<<grid_for(N * nc), 256, 0, c->stream>>>(N * nc, reinterpret_cast<const float2*>(cols), Sc);
  Dense dn;
  if (cublasCreate(&dn.blas) != CUBLAS_STATUS_SUCCESS) return fail(c, HV_ECUDA, "cublasCreate");
  if (cusolverDnCreate(&dn.sol) != CUSOLVER_STATUS_SUCCESS) return fail(c, HV_ECUDA, "cusolverDnCreate");
  cublasSetStream(dn.blas, c->stream);
  cusolverDnSetStream(dn.sol, c->stream);
  const zc one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
  // (ii) Rm^H Rm = conj(S S^H) = E diag(sigma^2) E^H, E = conj(U)
  if (cublasZgemm(dn.blas, CUBLAS_OP_C, CUBLAS_OP_N, nr, nr, (int)N, &one, Rm, (int)N, Rm, (int)N, &zero, G, nr) !=
      CUBLAS_STATUS_SUCCESS)
    return fail(c, HV_ECUDA, "cublasZgemm (Gram)");
  int lw = 0;
  cusolverDnZheevd_bufferSize(dn.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, nr, G, nr, ev, &lw);
  zc* work;
  if ((st = ws_get(c, "pp_work", sizeof(zc) * std::max(lw, 1), (void**)&work))) return st;
  if (cusolverDnZheevd(dn.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, nr, G, nr, ev, work, lw, info) !=
      CUSOLVER_STATUS_SUCCESS)
    return fail(c, HV_ECUDA, "cusolverDnZheevd");
  std::vector<double> hev(nr);
  std::vector<std::complex<double>> hG((size_t)nr * nr);
  CU_TRY(cudaMemcpyAsync(hev.data(), ev, sizeof(double) * nr, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(cudaMemcpyAsync(hG.data(), G, sizeof(zc) * nr * nr, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(cudaStreamSynchronize(c->stream));
  // leading `rank` (descending): E_r [nr][rank] / sigma, and conj(E_r) sigma for A0
  std::vector<std::complex<double>> hE((size_t)nr * rank), hU((size_t)nr * rank);
  for (int j = 0; j < rank; ++j) {
    const int col = nr - 1 - j;
    const double sig = std::sqrt(std::max(hev[col], 0.0));
    if (!(sig > 0.0)) return fail(c, HV_EINVAL, "rank exceeds the numerical rank of the symbol rows");
    for (int k = 0; k < nr; ++k) {
      const std::complex<double> e = hG[k + (size_t)nr * col];
      hE[k + (size_t)nr * j] = e / sig;
      hU[k + (size_t)nr * j] = std::conj(e) * sig;
    }
  }
  CU_TRY(cudaMemcpyAsync(E, hE.data(), sizeof(zc) * nr * rank, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(cudaMemcpyAsync(tmp, hU.data(), sizeof(zc) * nr * rank, cudaMemcpyHostToDevice, c->stream));
  // Bm (N x rank) = Rm E_r Sigma^-1 ; A0 (N x rank) = Wm conj(E_r) Sigma
  if (cublasZgemm(dn.blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)N, rank, nr, &one, Rm, (int)N, E, nr, &zero, Bm, (int)N) !=
          CUBLAS_STATUS_SUCCESS ||
      cublasZgemm(dn.blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)N, rank, nr, &one, Wm, (int)N, tmp, nr, &zero, A0, (int)N) !=
          CUBLAS_STATUS_SUCCESS)
    return fail(c, HV_ECUDA, "cublasZgemm (B, A0)");
  // (iii) Bc = B[:, I_c] (rank x nc); alpha = ||Bc||^2 / ||B||^2
  gather_cols<<<(rank * nc + 127) / 128, 128, 0, c->stream>>>(N, rank, nc, dic, Bm, Bc);
  double nBc = 0, nB = 0;
  if (cublasDznrm2(dn.blas, rank * nc, Bc, 1, &nBc) != CUBLAS_STATUS_SUCCESS ||
      cublasDznrm2(dn.blas, (int)(N * rank), Bm, 1, &nB) != CUBLAS_STATUS_SUCCESS)
    return fail(c, HV_ECUDA, "cublasDznrm2");
  CU_TRY(cudaStreamSynchronize(c->stream));
  const double alpha = (nBc * nBc) / (nB * nB);
  // M = Bc Bc^H + alpha I (host inverse), RHS = Sc Bc^H + alpha A0, A = RHS M^-1
  if (cublasZgemm(dn.blas, CUBLAS_OP_N, CUBLAS_OP_C, rank, rank, nc, &one, Bc, rank, Bc, rank, &zero, Msm, rank) !=
      CUBLAS_STATUS_SUCCESS)
    return fail(c, HV_ECUDA, "cublasZgemm (M)");
  std::vector<std::complex<double>> hM((size_t)rank * rank);
  CU_TRY(cudaMemcpyAsync(hM.data(), Msm, sizeof(zc) * rank * rank, cudaMemcpyDeviceToHost, c->stream));
  CU_TRY(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < rank; ++i) hM[i + (size_t)rank * i] += alpha;
  if (!invert(hM, rank)) return fail(c, HV_EINVAL, "singular PSF+ normal matrix");
  CU_TRY(cudaMemcpyAsync(Msm, hM.data(), sizeof(zc) * rank * rank, cudaMemcpyHostToDevice, c->stream));
  CU_TRY(cudaMemcpyAsync(RHS, A0, sizeof(zc) * N * rank, cudaMemcpyDeviceToDevice, c->stream));
  const zc za = make_cuDoubleComplex(alpha, 0);
  if (cublasZgemm(dn.blas, CUBLAS_OP_N, CUBLAS_OP_C, (int)N, rank, nc, &one, Sc, (int)N, Bc, rank, &za, RHS, (int)N) !=
          CUBLAS_STATUS_SUCCESS ||
      cublasZgemm(dn.blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)N, rank, rank, &one, RHS, (int)N, Msm, rank, &zero, A0, (int)N) !=
          CUBLAS_STATUS_SUCCESS)
    return fail(c, HV_ECUDA, "cublasZgemm (A)");
  z_to_c64<<<grid_for(N * rank), 256, 0, c->stream>>>(N * rank, A0, reinterpret_cast<float2*>(oA.dev));
  z_to_c64<<<grid_for(N * rank), 256, 0, c->stream>>>(N * rank, Bm, reinterpret_cast<float2*>(oB.dev));
  CU_TRY(cudaGetLastError());
  if ((st = finish_out(c, oA)) || (st = finish_out(c, oB))) return st;
  CU_TRY(cudaStreamSynchronize(c->stream));
  if (alpha_user) *alpha_user = alpha;
  c->stats = hv_stats{};
  c->stats.kernel_launches = 7;
  return HV_OK;
}
