// K10: the reference's epilogues around the online path.
//
//   fsr_fsrw_correct   ranking.py:256-274  x + (1 - eta) * (V . sum_regions q)
//   fsr_pool_rows      ranking.py:329-334  U_bar = P U      (pooled_basis)
//   fsr_pool_scores    ranking.py:322-326  x_pooled = P x   (pool), b queries
//   fsr_dense_scores   ranking.py:337-353  X = Z A^T        (filter_pooled: A = U_bar)
//
// P is the (N x n) region->image pooling matrix in CSR (each region column
// owned by exactly one image row).  Orders of accumulation follow scipy where
// the reference goes through scipy (CSR @ dense, CSR @ CSR, CSR @ vector):
// per output element, sequential over the CSR row, fp64 multiply and add
// rounded separately -- so fp64 results are bitwise scipy's.  The two dense
// products (V q and U_bar z) go through cuBLAS like the reference's BLAS
// (summation order differs; ~1 ulp).
#include "spmm.cuh"

namespace {

// X[j, i] = X[j, i] + (1 - eta_i) * E[j, i]   (numpy: x + (1.0 - eta) * euclid)
template <typename T>
__global__ void fsrw_axpy_kernel(int64_t b, int64_t n, const T* __restrict__ E, const double* __restrict__ eta,
                                 T* __restrict__ X, int64_t ldx) {
  const int64_t total = b * n;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total; f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = f / n, i = f - j * n;
    const double s = __dsub_rn(1.0, eta[i]);
    if (sizeof(T) == 8) {
      X[j * ldx + i] = (T)__dadd_rn((double)X[j * ldx + i], __dmul_rn(s, (double)E[f]));
    } else {
      // numpy in float32 mode would promote to float64 through eta; round once at the end
      X[j * ldx + i] = (T)((double)X[j * ldx + i] + s * (double)E[f]);
    }
  }
}

// U_bar[I, :] = sum_{e in P row I} P_e * U~[p_col_e, :]   (sparse U~, scipy csr_matmat order)
// one CTA per image row; the dense output row lives in shared memory.
template <typename T>
__global__ void __launch_bounds__(256) pool_sparse_rows_kernel(int64_t N, int64_t r, const int64_t* __restrict__ p_ptr,
                                                               const int32_t* __restrict__ p_idx,
                                                               const T* __restrict__ p_val,
                                                               const int64_t* __restrict__ u_ptr,
                                                               const int32_t* __restrict__ u_idx,
                                                               const T* __restrict__ u_val, T* __restrict__ Ub,
                                                               int64_t ldb) {
  extern __shared__ __align__(16) unsigned char dyn[];
  T* acc = (T*)dyn;
  for (int64_t I = blockIdx.x; I < N; I += gridDim.x) {
    for (int64_t c = threadIdx.x; c < r; c += blockDim.x) acc[c] = T(0);
    __syncthreads();
    for (int64_t e = p_ptr[I]; e < p_ptr[I + 1]; ++e) {
      const int64_t i = p_idx[e];
      const T a = p_val[e];
      for (int64_t s = u_ptr[i] + threadIdx.x; s < u_ptr[i + 1]; s += blockDim.x) {
        const int32_t c = u_idx[s];  // distinct within a canonical row: no write conflicts
        acc[c] = fsr::mul_add_rn(acc[c], a, u_val[s]);
      }
      __syncthreads();
    }
    for (int64_t c = threadIdx.x; c < r; c += blockDim.x) Ub[I * ldb + c] = acc[c];
    __syncthreads();
  }
}

// Xp[j, I] = sum_{e in P row I} P_e * X[j, p_col_e]   (scipy csr_matvec order)
template <typename T>
__global__ void pool_scores_kernel(int64_t b, int64_t N, const int64_t* __restrict__ p_ptr,
                                   const int32_t* __restrict__ p_idx, const T* __restrict__ p_val,
                                   const T* __restrict__ X, int64_t ldx, T* __restrict__ Xp, int64_t ldp) {
  const int64_t j = blockIdx.y;
  for (int64_t I = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; I < N; I += (int64_t)gridDim.x * blockDim.x) {
    T s = T(0);
    for (int64_t e = p_ptr[I]; e < p_ptr[I + 1]; ++e) s = fsr::mul_add_rn(s, p_val[e], X[j * ldx + p_idx[e]]);
    Xp[j * ldp + I] = s;
  }
}

// Out (b x N, row-major) = Z (b x k, ld ldz) * A^T, A (N x k row-major, ld lda)
template <typename T>
int gemm_rows(fsr_ctx* ctx, int64_t N, int64_t k, const T* A, int64_t lda, int64_t b, const T* Z, int64_t ldz,
              T* Out, int64_t ldo) {
  // column-major view: Out_c (N x b) = A_c^T (N x k) * Z_c (k x b)
  if (sizeof(T) == 8) {
    const double one = 1.0, zero = 0.0;
    FSR_BLAS(ctx, cublasDgemm_64(ctx->blas, CUBLAS_OP_T, CUBLAS_OP_N, N, b, k, &one, (const double*)A, lda,
                                 (const double*)Z, ldz, &zero, (double*)Out, ldo));
  } else {
    const float one = 1.0f, zero = 0.0f;
    FSR_BLAS(ctx, cublasSgemm_64(ctx->blas, CUBLAS_OP_T, CUBLAS_OP_N, N, b, k, &one, (const float*)A, lda,
                                 (const float*)Z, ldz, &zero, (float*)Out, ldo));
  }
  return FSR_OK;
}

}  // namespace

extern "C" {

int fsr_fsrw_correct(fsr_ctx* ctx, int dtype, int64_t b, int64_t n, int64_t d, const void* V, int64_t ldv,
                     const void* Qsum, int64_t ldq, const double* eta, void* X, int64_t ldx) {
  FSR_REQUIRE(ctx, b >= 0 && n >= 1 && d >= 1 && ldv >= d && ldq >= d && ldx >= n && V && Qsum && eta && X,
              "fsrw_correct: bad args");
  if (!b) return FSR_OK;
  const size_t es = fsr::dtype_size(dtype);
  // E = Qsum V^T in row chunks of queries so the scratch stays bounded
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(b, ((int64_t)1 << 30) / (n * (int64_t)es)));
  void* buf = nullptr;
  FSR_TRY(fsr::scratch(ctx, (size_t)chunk * n * es, &buf));
  for (int64_t j0 = 0; j0 < b; j0 += chunk) {
    const int64_t m = std::min(chunk, b - j0);
    if (dtype == FSR_F64) {
      FSR_TRY(gemm_rows<double>(ctx, n, d, (const double*)V, ldv, m, (const double*)Qsum + j0 * ldq, ldq,
                                (double*)buf, n));
      fsrw_axpy_kernel<double><<<fsr::grid_for(m * n, 256, ctx, 8), 256, 0, ctx->stream>>>(
          m, n, (const double*)buf, eta, (double*)X + j0 * ldx, ldx);
    } else {
      FSR_TRY(gemm_rows<float>(ctx, n, d, (const float*)V, ldv, m, (const float*)Qsum + j0 * ldq, ldq, (float*)buf,
                               n));
      fsrw_axpy_kernel<float><<<fsr::grid_for(m * n, 256, ctx, 8), 256, 0, ctx->stream>>>(
          m, n, (const float*)buf, eta, (float*)X + j0 * ldx, ldx);
    }
    FSR_TRY(fsr::launched(ctx, "fsrw_axpy_kernel"));
  }
  return FSR_OK;
}

int fsr_pool_rows(fsr_ctx* ctx, int dtype, int64_t N, const int64_t* p_indptr, const int32_t* p_indices,
                  const void* p_values, int64_t n, int64_t r, int u_sparse, const int64_t* u_indptr,
                  const int32_t* u_indices, const void* u_values, const void* u_dense, int64_t ldu, void* Ubar,
                  int64_t ldb) {
  FSR_REQUIRE(ctx, N >= 0 && n >= 1 && r >= 1 && ldb >= r && p_indptr && Ubar, "pool_rows: bad args");
  FSR_REQUIRE(ctx, u_sparse ? (u_indptr && u_indices && u_values) : (u_dense && ldu >= r), "pool_rows: missing U");
  if (!N) return FSR_OK;
  if (!u_sparse) {  // CSR x dense: the K2 kernel (CSR order per element)
    if (dtype == FSR_F64)
      return fsr::launch_spmm<double>(ctx, N, p_indptr, p_indices, (const double*)p_values, r,
                                      (const double*)u_dense, ldu, (double*)Ubar, ldb);
    return fsr::launch_spmm<float>(ctx, N, p_indptr, p_indices, (const float*)p_values, r, (const float*)u_dense,
                                   ldu, (float*)Ubar, ldb);
  }
  const size_t es = fsr::dtype_size(dtype);
  const size_t smem = (size_t)r * es;
  FSR_REQUIRE(ctx, smem <= 200 * 1024, "pool_rows: r = %lld too large for the sparse path", (long long)r);
  const int grid = (int)std::min<int64_t>(N, (int64_t)ctx->num_sms * 4);
  if (dtype == FSR_F64) {
    FSR_CUDA(ctx, cudaFuncSetAttribute(pool_sparse_rows_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    pool_sparse_rows_kernel<double><<<grid, 256, smem, ctx->stream>>>(
        N, r, p_indptr, p_indices, (const double*)p_values, u_indptr, u_indices, (const double*)u_values,
        (double*)Ubar, ldb);
  } else {
    FSR_CUDA(ctx, cudaFuncSetAttribute(pool_sparse_rows_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    pool_sparse_rows_kernel<float><<<grid, 256, smem, ctx->stream>>>(
        N, r, p_indptr, p_indices, (const float*)p_values, u_indptr, u_indices, (const float*)u_values, (float*)Ubar,
        ldb);
  }
  return fsr::launched(ctx, "pool_sparse_rows_kernel");
}

int fsr_pool_scores(fsr_ctx* ctx, int dtype, int64_t b, int64_t N, const int64_t* p_indptr,
                    const int32_t* p_indices, const void* p_values, const void* X, int64_t ldx, void* Xp,
                    int64_t ldp) {
  FSR_REQUIRE(ctx, b >= 0 && N >= 0 && ldp >= N && p_indptr && X && Xp, "pool_scores: bad args");
  if (!b || !N) return FSR_OK;
  FSR_REQUIRE(ctx, b <= 65535, "pool_scores: at most 65535 queries per call");
  dim3 grid((unsigned)std::min<int64_t>(fsr::ceil_div(N, 256), 1024), (unsigned)b);
  if (dtype == FSR_F64)
    pool_scores_kernel<double><<<grid, 256, 0, ctx->stream>>>(b, N, p_indptr, p_indices, (const double*)p_values,
                                                              (const double*)X, ldx, (double*)Xp, ldp);
  else
    pool_scores_kernel<float><<<grid, 256, 0, ctx->stream>>>(b, N, p_indptr, p_indices, (const float*)p_values,
                                                             (const float*)X, ldx, (float*)Xp, ldp);
  return fsr::launched(ctx, "pool_scores_kernel");
}

int fsr_dense_scores(fsr_ctx* ctx, int dtype, int64_t N, int64_t k, const void* A, int64_t lda, int64_t b,
                     const void* Z, int64_t ldz, void* Out, int64_t ldo) {
  FSR_REQUIRE(ctx, N >= 0 && k >= 1 && b >= 0 && lda >= k && ldz >= k && ldo >= N, "dense_scores: bad args");
  if (!N || !b) return FSR_OK;
  if (dtype == FSR_F64)
    return gemm_rows<double>(ctx, N, k, (const double*)A, lda, b, (const double*)Z, ldz, (double*)Out, ldo);
  return gemm_rows<float>(ctx, N, k, (const float*)A, lda, b, (const float*)Z, ldz, (float*)Out, ldo);
}

}  // extern "C"
