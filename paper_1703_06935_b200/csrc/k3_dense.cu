// K3-K6: dense tall-skinny stages of simultaneous iteration and Rayleigh-Ritz.
//
//  K3  orthonormalisation (reference spectral.py:165-169, Householder QR +
//      re-QR when max|Q^T Q - I| > 1e-8) is done as CholeskyQR: Gram G = B^T B
//      in fp64, G = R^T R, Q = B R^-1.  Only span(Q) reaches the output and
//      CholeskyQR's Q equals Householder's up to column signs, so the
//      decomposition is unchanged.  Householder (cuSOLVER geqrf/orgqr) remains
//      as the fallback for rank-deficient blocks.
//  K4  C = Q^T B (spectral.py:186), fp64.
//  K5  (C + C^T)/2, eigh (cuSOLVER syevd, fp64), keep the r algebraically
//      largest in stable argsort(-lambda) order (spectral.py:187-189,141-144).
//  K6  U = Q V (spectral.py:190), column sign fix (spectral.py:133-138) and
//      row norms eta (spectral.py:127-130).
//
// Layout: row-major n x k blocks are column-major k x n for cuBLAS, so
// A^T A = A_c A_c^T etc.  Float32 blocks are accumulated into fp64 Gram /
// projection matrices through row chunks upcast into scratch.
#include <algorithm>
#include <vector>

#include <cstring>

#include "fsr_common.cuh"

namespace {

template <typename T>
__global__ void upcast_rows_kernel(int64_t rows, int64_t k, const T* __restrict__ A, int64_t lda,
                                   double* __restrict__ out) {
  const int64_t total = rows * k;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = f / k, j = f - i * k;
    out[f] = (double)A[i * lda + j];
  }
}

__global__ void symmetrize_kernel(int64_t k, double* __restrict__ C) {
  // C <- (C + C^T) / 2, each unordered pair handled once
  const int64_t total = k * k;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = f / k, j = f - i * k;
    if (j < i) continue;
    const double v = (C[i * k + j] + C[j * k + i]) / 2.0;
    C[i * k + j] = v;
    C[j * k + i] = v;
  }
}

__global__ void max_offdiag_kernel(int64_t k, const double* __restrict__ G, unsigned long long* out) {
  double m = 0.0;
  const int64_t total = k * k;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = f / k, j = f - i * k;
    const double d = fabs(G[f] - (i == j ? 1.0 : 0.0));
    m = d > m || d != d ? d : m;
  }
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__global__ void gather_cols_kernel(int64_t k, int64_t r, const double* __restrict__ Vc,
                                   const int64_t* __restrict__ perm, double* __restrict__ V) {
  // Vc: column-major k x k eigenvectors; V: row-major k x r with V[a, j] = Vc[a, perm[j]]
  const int64_t total = k * r;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = f / r, j = f - a * r;
    V[f] = Vc[perm[j] * k + a];
  }
}

// min over columns j of |R^-1_jj| / max_i |R^-1_ij| (column-major upper-triangular R^-1),
// as float bits (nonnegative floats order like unsigned ints)
__global__ void diag_ratio_kernel(int64_t k, const double* __restrict__ Rinv, unsigned* __restrict__ worst) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < k; j += nwarps) {
    double m = 0.0;
    for (int64_t i = lane; i <= j; i += 32) m = fmax(m, fabs(Rinv[j * k + i]));
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (!lane) {
      const float r = m > 0.0 ? (float)(fabs(Rinv[j * k + j]) / m) : 0.0f;
      atomicMin(worst, __float_as_uint(r));
    }
  }
}

__global__ void identity_kernel(int64_t k, double* __restrict__ M) {
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < k * k; f += (int64_t)gridDim.x * blockDim.x)
    M[f] = (f / k == f % k) ? 1.0 : 0.0;
}

__global__ void d2s_kernel(int64_t n, const double* __restrict__ in, float* __restrict__ out) {
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < n; f += (int64_t)gridDim.x * blockDim.x)
    out[f] = (float)in[f];
}

// Column |max| with the first (lowest) row on ties.  Phase 1: block (32 cols x 8
// row lanes) scans a row chunk; phase 2 folds the chunks.
struct Best {
  double a;
  int64_t row;
  double v;
};
__device__ __forceinline__ bool better(const Best& x, const Best& y) {
  return x.a > y.a || (x.a == y.a && x.row < y.row);
}

template <typename T>
__global__ void col_absmax_partial(int64_t n_rows, int64_t r, const T* __restrict__ U, int64_t ldu,
                                   int64_t row_offset, int64_t chunk, double* pa, int64_t* prow, double* pv) {
  __shared__ Best sh[8][32];
  const int64_t j = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * chunk, r1 = min(n_rows, r0 + chunk);
  Best b{-1.0, INT64_MAX, 0.0};
  if (j < r)
    for (int64_t i = r0 + threadIdx.y; i < r1; i += 8) {
      const double v = (double)U[i * ldu + j];
      const double a = fabs(v);
      if (a > b.a) b = Best{a, row_offset + i, v};
    }
  sh[threadIdx.y][threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.y == 0 && j < r) {
    for (int t = 1; t < 8; ++t)
      if (better(sh[t][threadIdx.x], b)) b = sh[t][threadIdx.x];
    const int64_t o = (int64_t)blockIdx.y * r + j;
    pa[o] = b.a;
    prow[o] = b.row;
    pv[o] = b.v;
  }
}

__global__ void col_absmax_final(int64_t r, int64_t nchunks, const double* pa, const int64_t* prow,
                                 const double* pv, double* best_abs, int64_t* best_row, double* best_val) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < r; j += (int64_t)gridDim.x * blockDim.x) {
    Best b{-1.0, INT64_MAX, 0.0};
    for (int64_t c = 0; c < nchunks; ++c) {
      Best x{pa[c * r + j], prow[c * r + j], pv[c * r + j]};
      if (better(x, b)) b = x;
    }
    best_abs[j] = b.a;
    best_row[j] = b.row;
    best_val[j] = b.v;
  }
}

template <typename T, bool APPLY>
__global__ void __launch_bounds__(256) signs_rownorm_kernel(int64_t n_rows, int64_t r, T* __restrict__ U,
                                                            int64_t ldu, const double* __restrict__ best_val,
                                                            double* __restrict__ eta) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_rows; i += nwarps) {
    T* row = U + i * ldu;
    double ss = 0.0;
    for (int64_t j = lane; j < r; j += 32) {
      T v = row[j];
      if (APPLY) {
        if (best_val[j] < 0.0) {
          v = -v;
          row[j] = v;
        }
      }
      const double d = (double)v;
      ss = fma(d, d, ss);
    }
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (!lane && eta) eta[i] = sqrt(ss);
  }
}

// Rows per chunk when a float32 block is upcast into fp64 scratch.
inline int64_t chunk_rows(int64_t n_rows, int64_t k, int operands) {
  const int64_t budget = (int64_t)1 << 29;  // 512 MB of fp64 per operand
  (void)operands;
  const int64_t m = budget / std::max<int64_t>(1, k * 8);
  return std::max<int64_t>(1, std::min(m, n_rows));
}

template <typename T>
int upcast(fsr_ctx* ctx, int64_t rows, int64_t k, const T* A, int64_t lda, double* out) {
  const int64_t total = rows * k;
  upcast_rows_kernel<T><<<fsr::grid_for(total, 256, ctx, 16), 256, 0, ctx->stream>>>(rows, k, A, lda, out);
  return fsr::launched(ctx, "upcast_rows_kernel");
}

int dgemm_nt_accum(fsr_ctx* ctx, int64_t k, int64_t rows, const double* A, int64_t lda, const double* B,
                   int64_t ldb, double* C, double beta) {
  const double one = 1.0;
  FSR_BLAS(ctx, cublasDgemm_64(ctx->blas, CUBLAS_OP_N, CUBLAS_OP_T, k, k, rows, &one, A, lda, B, ldb, &beta, C, k));
  return FSR_OK;
}

// C (k x k) (+)= A^T B over n_rows rows (A, B row-major); B may alias A.
int cross_impl(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, const void* A, int64_t lda, const void* B,
               int64_t ldb, double* C, int accumulate, bool sym_hint = false) {
  FSR_REQUIRE(ctx, n_rows >= 0 && k >= 1 && lda >= k && ldb >= k, "gram/cross: bad shape");
  fsr::StageTimer timer(ctx, FSR_STAGE_GRAM);
  if (n_rows == 0) {
    if (!accumulate) FSR_CUDA(ctx, cudaMemsetAsync(C, 0, k * k * 8, ctx->stream));
    return FSR_OK;
  }
  if (dtype == FSR_F64)
    return dgemm_nt_accum(ctx, k, n_rows, (const double*)A, lda, (const double*)B, ldb, C, accumulate ? 1.0 : 0.0);
  const bool same = A == B && lda == ldb;
  if (ctx->dense_path == 0)
    return fsr::tc_gram(ctx, n_rows, k, (const float*)A, lda, k, (const float*)B, ldb, C, accumulate, 4,
                        same || sym_hint);
  const int64_t m = chunk_rows(n_rows, k, same ? 1 : 2);
  void* buf = nullptr;
  FSR_TRY(fsr::scratch(ctx, (size_t)m * k * 8 * (same ? 1 : 2), &buf));
  double* a64 = (double*)buf;
  double* b64 = same ? a64 : a64 + m * k;
  for (int64_t s = 0; s < n_rows; s += m) {
    const int64_t rows = std::min(m, n_rows - s);
    FSR_TRY(upcast<float>(ctx, rows, k, (const float*)A + s * lda, lda, a64));
    if (!same) FSR_TRY(upcast<float>(ctx, rows, k, (const float*)B + s * ldb, ldb, b64));
    const double beta = (s == 0 && !accumulate) ? 0.0 : 1.0;
    FSR_TRY(dgemm_nt_accum(ctx, k, rows, a64, k, b64, k, C, beta));
  }
  return FSR_OK;
}

}  // namespace

extern "C" {

int fsr_gram(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, const void* A, int64_t lda, double* G,
             int accumulate) {
  return cross_impl(ctx, dtype, n_rows, k, A, lda, A, lda, G, accumulate);
}

int fsr_cross(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, const void* Q, int64_t ldq, const void* B,
              int64_t ldb, double* C, int accumulate) {
  return cross_impl(ctx, dtype, n_rows, k, Q, ldq, B, ldb, C, accumulate);
}

int fsr_cross_sym(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, const void* Q, int64_t ldq, const void* B,
                  int64_t ldb, double* C, int accumulate) {
  // F32 tensor-core path: upper triangle only, mirrored; other paths: full product
  return cross_impl(ctx, dtype, n_rows, k, Q, ldq, B, ldb, C, accumulate, dtype == FSR_F32);
}

int fsr_gram_levels(fsr_ctx* ctx, int64_t n_rows, int64_t k, const float* A, int64_t lda, double* G, int accumulate,
                    int levels) {
  FSR_REQUIRE(ctx, n_rows >= 0 && k >= 1 && lda >= k && (levels == 1 || levels == 4), "gram_levels: bad args");
  fsr::StageTimer timer(ctx, FSR_STAGE_GRAM);
  if (n_rows == 0) {
    if (!accumulate) FSR_CUDA(ctx, cudaMemsetAsync(G, 0, k * k * 8, ctx->stream));
    return FSR_OK;
  }
  if (ctx->dense_path != 0) return cross_impl(ctx, FSR_F32, n_rows, k, A, lda, A, lda, G, accumulate);
  return fsr::tc_gram(ctx, n_rows, k, A, lda, k, A, lda, G, accumulate, levels, 1);
}

int fsr_cholesky(fsr_ctx* ctx, int64_t k, double* G) {
  FSR_REQUIRE(ctx, k >= 1, "cholesky: bad shape");
  fsr::StageTimer timer(ctx, FSR_STAGE_CHOLESKY);
  int lwork = 0;
  FSR_SOLVER(ctx, cusolverDnDpotrf_bufferSize(ctx->solver, CUBLAS_FILL_MODE_UPPER, (int)k, G, (int)k, &lwork));
  void* work = nullptr;
  FSR_TRY(fsr::scratch(ctx, (size_t)lwork * 8 + 64, &work));
  FSR_SOLVER(ctx, cusolverDnDpotrf(ctx->solver, CUBLAS_FILL_MODE_UPPER, (int)k, G, (int)k, (double*)work, lwork,
                                   ctx->dev_info));
  int info = 0;
  FSR_CUDA(ctx, cudaMemcpyAsync(&info, ctx->dev_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (info > 0) return fsr::set_error(ctx, FSR_ENOTSPD, "cholesky: leading minor %d not positive definite", info);
  if (info < 0) return fsr::set_error(ctx, FSR_ELIBRARY, "cholesky: bad argument %d", -info);
  return FSR_OK;
}

int fsr_apply_rinv(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, const double* R, void* A, int64_t lda) {
  return fsr_apply_rinv_levels(ctx, dtype, n_rows, k, R, A, lda, 4);
}

int fsr_apply_rinv_levels(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, const double* R, void* A, int64_t lda,
                          int m_slices) {
  FSR_REQUIRE(ctx, n_rows >= 0 && k >= 1 && lda >= k, "apply_rinv: bad shape");
  FSR_REQUIRE(ctx, m_slices == 1 || m_slices == 4, "apply_rinv: m_slices must be 1 or 4");
  if (!n_rows) return FSR_OK;
  fsr::StageTimer timer(ctx, FSR_STAGE_APPLY);
  // (A R^-1)^T = R^-T A^T: solve R^T X = A_c with A_c the column-major k x n view
  if (dtype == FSR_F64) {
    const double one = 1.0;
    FSR_BLAS(ctx, cublasDtrsm_64(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T,
                                 CUBLAS_DIAG_NON_UNIT, k, n_rows, &one, R, k, (double*)A, lda));
    return FSR_OK;
  }
  if (ctx->dense_path == 0) {
    // explicit R^-1 (fp64 TRSM on the identity; measured faster than trtri at k = 5500),
    // then Q = B R^-1 on tensor cores
    void* aux = nullptr;
    FSR_TRY(fsr::scratch_aux(ctx, (size_t)k * k * 8, &aux));
    double* Rinv = (double*)aux;
    identity_kernel<<<fsr::grid_for(k * k, 256, ctx), 256, 0, ctx->stream>>>(k, Rinv);
    FSR_TRY(fsr::launched(ctx, "identity_kernel"));
    const double done = 1.0;
    FSR_BLAS(ctx, cublasDtrsm_64(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                                 CUBLAS_DIAG_NON_UNIT, k, k, &done, R, k, Rinv, k));
    if (m_slices == 1) {
      // the 7-bit R^-1 must stay a good preconditioner: every diagonal entry
      // (triangular: its determinant) within 2^-4 of its column's maximum
      unsigned* worst = (unsigned*)ctx->dev_info;  // 4 device bytes, free between solver calls
      const unsigned one_bits = 0x3f800000u;
      FSR_CUDA(ctx, cudaMemcpyAsync(worst, &one_bits, sizeof(unsigned), cudaMemcpyHostToDevice, ctx->stream));
      diag_ratio_kernel<<<fsr::grid_for(k * 32, 256, ctx, 8), 256, 0, ctx->stream>>>(k, Rinv, worst);
      FSR_TRY(fsr::launched(ctx, "diag_ratio_kernel"));
      unsigned h = 0;
      FSR_CUDA(ctx, cudaMemcpyAsync(&h, worst, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
      FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
      float ratio;
      memcpy(&ratio, &h, 4);
      if (!(ratio >= 0.0625f)) m_slices = 4;
    }
    return fsr::tc_apply(ctx, n_rows, k, (const float*)A, lda, k, Rinv, k, 1, (float*)A, lda, m_slices);
  }
  void* buf = nullptr;
  FSR_TRY(fsr::scratch(ctx, (size_t)k * k * 4, &buf));
  d2s_kernel<<<fsr::grid_for(k * k, 256, ctx), 256, 0, ctx->stream>>>(k * k, R, (float*)buf);
  FSR_TRY(fsr::launched(ctx, "d2s_kernel"));
  const float one = 1.0f;
  FSR_BLAS(ctx, cublasStrsm_64(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T,
                               CUBLAS_DIAG_NON_UNIT, k, n_rows, &one, (const float*)buf, k, (float*)A, lda));
  return FSR_OK;
}

int fsr_householder_qr(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, void* A, int64_t lda) {
  FSR_REQUIRE(ctx, n_rows >= k && k >= 1 && lda >= k, "householder_qr: need n_rows >= k");
  FSR_REQUIRE(ctx, n_rows < (1ll << 31) && n_rows * k < (1ll << 40), "householder_qr: too large");
  const int m = (int)n_rows, kk = (int)k;
  fsr::StageTimer timer(ctx, FSR_STAGE_HOUSEHOLDER);
  const size_t es = fsr::dtype_size(dtype);
  int lw1 = 0, lw2 = 0;
  void* buf = nullptr;
  FSR_TRY(fsr::scratch(ctx, ((size_t)m * kk + kk) * es + 256, &buf));
  {
    void* T0 = buf;
    void* tau0 = (char*)buf + (size_t)m * kk * es;
    if (dtype == FSR_F64) {
      FSR_SOLVER(ctx, cusolverDnDgeqrf_bufferSize(ctx->solver, m, kk, (double*)T0, m, &lw1));
      FSR_SOLVER(ctx, cusolverDnDorgqr_bufferSize(ctx->solver, m, kk, kk, (double*)T0, m, (double*)tau0, &lw2));
    } else {
      FSR_SOLVER(ctx, cusolverDnSgeqrf_bufferSize(ctx->solver, m, kk, (float*)T0, m, &lw1));
      FSR_SOLVER(ctx, cusolverDnSorgqr_bufferSize(ctx->solver, m, kk, kk, (float*)T0, m, (float*)tau0, &lw2));
    }
  }
  const size_t lw = (size_t)std::max(lw1, lw2);
  const size_t bytes = ((size_t)m * kk + kk + lw) * es + 256;
  FSR_TRY(fsr::scratch(ctx, bytes, &buf));
  char* base = (char*)buf;
  void* T = base;                                  // column-major m x k
  void* tau = base + (size_t)m * kk * es;          // k
  void* work = (char*)tau + (size_t)kk * es;       // lw
  if (dtype == FSR_F64) {
    const double one = 1.0, zero = 0.0;
    // T (m x k col-major) = (A_c)^T where A_c is k x m col-major with ld lda
    FSR_BLAS(ctx, cublasDgeam(ctx->blas, CUBLAS_OP_T, CUBLAS_OP_N, m, kk, &one, (const double*)A, (int)lda, &zero,
                              (const double*)T, m, (double*)T, m));
    FSR_SOLVER(ctx, cusolverDnDgeqrf(ctx->solver, m, kk, (double*)T, m, (double*)tau, (double*)work, (int)lw,
                                     ctx->dev_info));
    FSR_SOLVER(ctx, cusolverDnDorgqr(ctx->solver, m, kk, kk, (double*)T, m, (const double*)tau, (double*)work,
                                     (int)lw, ctx->dev_info));
    FSR_BLAS(ctx, cublasDgeam(ctx->blas, CUBLAS_OP_T, CUBLAS_OP_N, kk, m, &one, (const double*)T, m, &zero,
                              (const double*)A, (int)lda, (double*)A, (int)lda));
  } else {
    const float one = 1.0f, zero = 0.0f;
    FSR_BLAS(ctx, cublasSgeam(ctx->blas, CUBLAS_OP_T, CUBLAS_OP_N, m, kk, &one, (const float*)A, (int)lda, &zero,
                              (const float*)T, m, (float*)T, m));
    FSR_SOLVER(ctx, cusolverDnSgeqrf(ctx->solver, m, kk, (float*)T, m, (float*)tau, (float*)work, (int)lw,
                                     ctx->dev_info));
    FSR_SOLVER(ctx, cusolverDnSorgqr(ctx->solver, m, kk, kk, (float*)T, m, (const float*)tau, (float*)work,
                                     (int)lw, ctx->dev_info));
    FSR_BLAS(ctx, cublasSgeam(ctx->blas, CUBLAS_OP_T, CUBLAS_OP_N, kk, m, &one, (const float*)T, m, &zero,
                              (const float*)A, (int)lda, (float*)A, (int)lda));
  }
  return FSR_OK;
}

int fsr_max_offdiag_error(fsr_ctx* ctx, int64_t k, const double* G, double* err_host) {
  FSR_REQUIRE(ctx, k >= 1 && err_host, "max_offdiag_error: bad args");
  void* buf = nullptr;
  FSR_TRY(fsr::scratch(ctx, 64, &buf));
  FSR_CUDA(ctx, cudaMemsetAsync(buf, 0, 8, ctx->stream));
  max_offdiag_kernel<<<fsr::grid_for(k * k, 256, ctx, 4), 256, 0, ctx->stream>>>(k, G, (unsigned long long*)buf);
  FSR_TRY(fsr::launched(ctx, "max_offdiag_kernel"));
  FSR_CUDA(ctx, cudaMemcpyAsync(err_host, buf, 8, cudaMemcpyDeviceToHost, ctx->stream));
  FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FSR_OK;
}

// Shared by fsr_eigh_desc (C v = lambda v) and fsr_eigh_gen_desc (C v = lambda G v).
static int eigh_impl(fsr_ctx* ctx, int64_t k, double* C, double* G, int64_t r, double* lam_host, double* V) {
  FSR_REQUIRE(ctx, k >= 1 && r >= 1 && r <= k && lam_host, "eigh_desc: bad shape");
  FSR_REQUIRE(ctx, k < (1 << 20), "eigh_desc: k too large");
  fsr::StageTimer timer(ctx, FSR_STAGE_EIGH);
  symmetrize_kernel<<<fsr::grid_for(k * k, 256, ctx, 8), 256, 0, ctx->stream>>>(k, C);
  FSR_TRY(fsr::launched(ctx, "symmetrize_kernel"));
  if (G) {
    symmetrize_kernel<<<fsr::grid_for(k * k, 256, ctx, 8), 256, 0, ctx->stream>>>(k, G);
    FSR_TRY(fsr::launched(ctx, "symmetrize_kernel"));
  }
  int lwork = 0;
  void* buf = nullptr;
  if (G)
    FSR_SOLVER(ctx, cusolverDnDsygvd_bufferSize(ctx->solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                                CUBLAS_FILL_MODE_UPPER, (int)k, C, (int)k, G, (int)k, C, &lwork));
  else
    FSR_SOLVER(ctx, cusolverDnDsyevd_bufferSize(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, (int)k,
                                                C, (int)k, C, &lwork));
  const size_t bytes = ((size_t)lwork + k) * 8 + (size_t)r * 8 + 256;
  FSR_TRY(fsr::scratch(ctx, bytes, &buf));
  double* W = (double*)buf;
  int64_t* perm_dev = (int64_t*)(W + k);
  double* work = (double*)(perm_dev + r);
  if (G)
    FSR_SOLVER(ctx, cusolverDnDsygvd(ctx->solver, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR,
                                     CUBLAS_FILL_MODE_UPPER, (int)k, C, (int)k, G, (int)k, W, work, lwork,
                                     ctx->dev_info));
  else
    FSR_SOLVER(ctx, cusolverDnDsyevd(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, (int)k, C,
                                     (int)k, W, work, lwork, ctx->dev_info));
  std::vector<double> lam(k);
  int info = 0;
  FSR_CUDA(ctx, cudaMemcpyAsync(lam.data(), W, k * 8, cudaMemcpyDeviceToHost, ctx->stream));
  FSR_CUDA(ctx, cudaMemcpyAsync(&info, ctx->dev_info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (info != 0)
    return fsr::set_error(ctx, FSR_ENUMERICAL, "%s failed (info=%d)%s", G ? "sygvd" : "syevd", info,
                          G && info > k ? ": G not positive definite" : "");
  for (int64_t i = 0; i < k; ++i)
    if (!(lam[i] == lam[i])) return fsr::set_error(ctx, FSR_ENUMERICAL, "syevd produced NaN eigenvalues");
  // argsort(-lambda, kind="stable")[:r]
  std::vector<int64_t> order(k);
  for (int64_t i = 0; i < k; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return -lam[a] < -lam[b]; });
  order.resize(r);
  for (int64_t j = 0; j < r; ++j) lam_host[j] = lam[order[j]];
  FSR_CUDA(ctx, cudaMemcpyAsync(perm_dev, order.data(), r * 8, cudaMemcpyHostToDevice, ctx->stream));
  gather_cols_kernel<<<fsr::grid_for(k * r, 256, ctx, 8), 256, 0, ctx->stream>>>(k, r, C, perm_dev, V);
  FSR_TRY(fsr::launched(ctx, "gather_cols_kernel"));
  // perm_dev lives in scratch: make sure the gather consumed it before reuse
  FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FSR_OK;
}

int fsr_eigh_desc(fsr_ctx* ctx, int64_t k, double* C, int64_t r, double* lam_host, double* V) {
  return eigh_impl(ctx, k, C, nullptr, r, lam_host, V);
}

int fsr_eigh_gen_desc(fsr_ctx* ctx, int64_t k, double* C, double* G, int64_t r, double* lam_host, double* V) {
  FSR_REQUIRE(ctx, G != nullptr, "eigh_gen_desc: missing G");
  return eigh_impl(ctx, k, C, G, r, lam_host, V);
}

int fsr_lift(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t k, int64_t r, const void* Q, int64_t ldq,
             const double* V, void* U, int64_t ldu) {
  FSR_REQUIRE(ctx, n_rows >= 0 && k >= 1 && r >= 1 && r <= k && ldq >= k && ldu >= r, "lift: bad shape");
  if (!n_rows) return FSR_OK;
  fsr::StageTimer timer(ctx, FSR_STAGE_LIFT);
  // U_c (r x n) = V_c' (r x k; row-major V viewed column-major) * Q_c (k x n)
  if (dtype == FSR_F64) {
    const double one = 1.0, zero = 0.0;
    FSR_BLAS(ctx, cublasDgemm_64(ctx->blas, CUBLAS_OP_N, CUBLAS_OP_N, r, n_rows, k, &one, V, r, (const double*)Q,
                                 ldq, &zero, (double*)U, ldu));
    return FSR_OK;
  }
  if (ctx->dense_path == 0)
    return fsr::tc_apply(ctx, n_rows, k, (const float*)Q, ldq, r, V, r, 0, (float*)U, ldu);
  void* buf = nullptr;
  FSR_TRY(fsr::scratch(ctx, (size_t)k * r * 4, &buf));
  d2s_kernel<<<fsr::grid_for(k * r, 256, ctx), 256, 0, ctx->stream>>>(k * r, V, (float*)buf);
  FSR_TRY(fsr::launched(ctx, "d2s_kernel"));
  const float one = 1.0f, zero = 0.0f;
  FSR_BLAS(ctx, cublasSgemm_64(ctx->blas, CUBLAS_OP_N, CUBLAS_OP_N, r, n_rows, k, &one, (const float*)buf, r,
                               (const float*)Q, ldq, &zero, (float*)U, ldu));
  return FSR_OK;
}

int fsr_col_absmax(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t r, const void* U, int64_t ldu,
                   int64_t row_offset, double* best_abs, int64_t* best_row, double* best_val) {
  FSR_REQUIRE(ctx, n_rows >= 0 && r >= 1 && ldu >= r, "col_absmax: bad shape");
  fsr::StageTimer timer(ctx, FSR_STAGE_SIGNS);
  const int64_t col_blocks = fsr::ceil_div(r, 32);
  int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(fsr::ceil_div((int64_t)ctx->num_sms * 8, col_blocks),
                                                           fsr::ceil_div(std::max<int64_t>(n_rows, 1), 64)));
  nchunks = std::min<int64_t>(nchunks, 65535);
  const int64_t chunk = fsr::ceil_div(std::max<int64_t>(n_rows, 1), nchunks);
  nchunks = fsr::ceil_div(std::max<int64_t>(n_rows, 1), chunk);
  void* buf = nullptr;
  FSR_TRY(fsr::scratch(ctx, (size_t)nchunks * r * 24 + 64, &buf));
  double* pa = (double*)buf;
  int64_t* prow = (int64_t*)(pa + nchunks * r);
  double* pv = (double*)(prow + nchunks * r);
  dim3 grid((unsigned)col_blocks, (unsigned)nchunks), block(32, 8);
  if (dtype == FSR_F64)
    col_absmax_partial<double><<<grid, block, 0, ctx->stream>>>(n_rows, r, (const double*)U, ldu, row_offset, chunk,
                                                                 pa, prow, pv);
  else
    col_absmax_partial<float><<<grid, block, 0, ctx->stream>>>(n_rows, r, (const float*)U, ldu, row_offset, chunk,
                                                                pa, prow, pv);
  FSR_TRY(fsr::launched(ctx, "col_absmax_partial"));
  col_absmax_final<<<fsr::grid_for(r, 256, ctx), 256, 0, ctx->stream>>>(r, nchunks, pa, prow, pv, best_abs,
                                                                         best_row, best_val);
  return fsr::launched(ctx, "col_absmax_final");
}

int fsr_apply_signs_rownorm(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t r, void* U, int64_t ldu,
                            const double* best_val, double* eta) {
  FSR_REQUIRE(ctx, n_rows >= 0 && r >= 1 && ldu >= r, "apply_signs: bad shape");
  if (!n_rows) return FSR_OK;
  fsr::StageTimer timer(ctx, FSR_STAGE_SIGNS);
  const int grid = fsr::grid_for(n_rows * 32, 256, ctx, 8);
  if (dtype == FSR_F64)
    signs_rownorm_kernel<double, true><<<grid, 256, 0, ctx->stream>>>(n_rows, r, (double*)U, ldu, best_val, eta);
  else
    signs_rownorm_kernel<float, true><<<grid, 256, 0, ctx->stream>>>(n_rows, r, (float*)U, ldu, best_val, eta);
  return fsr::launched(ctx, "signs_rownorm_kernel");
}

int fsr_row_norms(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t r, const void* U, int64_t ldu, double* eta) {
  FSR_REQUIRE(ctx, n_rows >= 0 && r >= 1 && ldu >= r, "row_norms: bad shape");
  if (!n_rows) return FSR_OK;
  fsr::StageTimer timer(ctx, FSR_STAGE_SIGNS);
  const int grid = fsr::grid_for(n_rows * 32, 256, ctx, 8);
  if (dtype == FSR_F64)
    signs_rownorm_kernel<double, false><<<grid, 256, 0, ctx->stream>>>(n_rows, r, (double*)U, ldu, nullptr, eta);
  else
    signs_rownorm_kernel<float, false><<<grid, 256, 0, ctx->stream>>>(n_rows, r, (float*)U, ldu, nullptr, eta);
  return fsr::launched(ctx, "rownorm_kernel");
}

}  // extern "C"
