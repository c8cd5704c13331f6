// K8/K9: online batched filtering X = U h(Lambda) U^T Y with fused
// copy-uncovered and an exact top-k, for b observation columns at once.
//
// Reference (per query, one at a time): ranking.py:229-255 `filter`:
//   z = U[y.indices]^T y.values           (_project, ranking.py:219-226)
//   x = U @ (weights * z)                 (ranking.py:246)
//   x[i] = y_i where eta_i == 0, i in supp(y)   (ranking.py:248-254)
// and ranking.py:390-395 `rank` (descending, ties by ascending index).
//
// Device: one CTA per query gathers its k rows of U (sparse CSR or dense) into
// z (rows processed in order, so the fp sums follow the reference order),
// scales by w = h(lambda) and writes both a query-major copy Zt (b x r) and a
// rank-major copy Zs (r x b).  The sparse product runs the K2 row-panel SpMM
// on (U~, Zs); the dense one a cuBLAS GEMM.  Copy-uncovered patches X in
// place, and the top-k is an exact radix select per query (one histogram pass
// + candidate compaction in shared memory + bitonic sort), with a general
// multi-pass fallback when the candidate set overflows shared memory.
#include <cub/cub.cuh>

#include "spmm.cuh"

namespace {

constexpr int kTopkThreads = 512;
constexpr int kTopkCap = 4096;  // candidates held in shared memory
constexpr int kHistBits = 12;

template <typename T, bool SPARSE>
__global__ void __launch_bounds__(256) project_kernel(int64_t r, int64_t b, const int64_t* __restrict__ u_indptr,
                                                      const int32_t* __restrict__ u_indices,
                                                      const T* __restrict__ u_values, const T* __restrict__ u_dense,
                                                      int64_t ldu, const T* __restrict__ w,
                                                      const int64_t* __restrict__ y_ptr,
                                                      const int64_t* __restrict__ y_idx, const T* __restrict__ y_val,
                                                      T* __restrict__ Zt, T* __restrict__ Zs) {
  const int64_t j = blockIdx.x;
  T* z = Zt + j * r;
  for (int64_t c = threadIdx.x; c < r; c += blockDim.x) z[c] = T(0);
  __syncthreads();
  const int64_t e1 = y_ptr[j + 1];
  for (int64_t e = y_ptr[j]; e < e1; ++e) {
    const int64_t i = y_idx[e];
    const T v = y_val[e];
    if (SPARSE) {
      const int64_t s1 = u_indptr[i + 1];
      for (int64_t s = u_indptr[i] + threadIdx.x; s < s1; s += blockDim.x) {
        const int32_t c = u_indices[s];
        z[c] = fsr::mul_add_rn(z[c], u_values[s], v);
      }
    } else {
      const T* row = u_dense + i * ldu;
      for (int64_t c = threadIdx.x; c < r; c += blockDim.x) z[c] = fsr::mul_add_rn(z[c], row[c], v);
    }
    __syncthreads();
  }
  for (int64_t c = threadIdx.x; c < r; c += blockDim.x) {
    const T s = w[c] * z[c];
    z[c] = s;
    if (Zs) Zs[c * b + j] = s;
  }
}

template <typename T>
__global__ void transpose_kernel(int64_t rows, int64_t cols, const T* __restrict__ in, T* __restrict__ out) {
  // in: rows x cols row-major -> out: cols x rows row-major
  __shared__ T tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t rr = r0 + k, cc = c0 + threadIdx.x;
    if (rr < rows && cc < cols) tile[k][threadIdx.x] = in[rr * cols + cc];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {
    const int64_t cc = c0 + k, rr = r0 + threadIdx.x;
    if (rr < rows && cc < cols) out[cc * rows + rr] = tile[threadIdx.x][k];
  }
}

template <typename T>
__global__ void copy_uncovered_kernel(int64_t n, const int64_t* __restrict__ y_ptr, const int64_t* __restrict__ y_idx,
                                      const T* __restrict__ y_val, const double* __restrict__ eta, T* __restrict__ X,
                                      int64_t ldx) {
  const int64_t j = blockIdx.x;
  for (int64_t e = y_ptr[j] + threadIdx.x; e < y_ptr[j + 1]; e += blockDim.x) {
    const int64_t i = y_idx[e];
    if (eta[i] == 0.0) X[j * ldx + i] = y_val[e];
  }
}

// ---- exact top-k ---------------------------------------------------------
__device__ __forceinline__ uint64_t order_key(float x) {
  if (x == 0.0f) x = 0.0f;  // -0 ties with +0 (numpy compares values)
  const uint32_t u = __float_as_uint(x);
  return (uint64_t)((u & 0x80000000u) ? ~u : (u | 0x80000000u));
}
__device__ __forceinline__ uint64_t order_key(double x) {
  if (x == 0.0) x = 0.0;
  const uint64_t u = (uint64_t)__double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
template <typename T>
struct KeyBits {
  static constexpr int value = sizeof(T) * 8;
};

struct TopkShared {
  unsigned int hist[1 << kHistBits];
  unsigned int count;
  unsigned int found_bin;
  unsigned long long above;
  unsigned long long warp_sums[kTopkThreads / 32];
};

// Find, among bins [0, nb) read from high to low, the bin where the running
// count first reaches `need`.  Writes found_bin and the count strictly above.
__device__ void find_bin(TopkShared& sh, int nb, unsigned long long need) {
  typedef cub::BlockScan<unsigned long long, kTopkThreads> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;
  const int per = nb / kTopkThreads > 0 ? nb / kTopkThreads : 1;
  // thread t owns bins nb-1-t*per ... nb-(t+1)*per (descending)
  unsigned long long mine = 0;
  const int hi = nb - 1 - threadIdx.x * per;
  for (int q = 0; q < per; ++q) {
    const int bin = hi - q;
    if (bin >= 0) mine += sh.hist[bin];
  }
  unsigned long long before = 0;
  Scan(scan_tmp).ExclusiveSum(mine, before);
  unsigned long long run = before;
  for (int q = 0; q < per; ++q) {
    const int bin = hi - q;
    if (bin < 0) break;
    const unsigned long long h = sh.hist[bin];
    if (run < need && run + h >= need) {
      sh.found_bin = (unsigned)bin;
      sh.above = run;
    }
    run += h;
  }
  __syncthreads();
}

__device__ __forceinline__ bool before_in_rank(uint64_t ka, int64_t ia, uint64_t kb, int64_t ib) {
  return ka > kb || (ka == kb && ia < ib);
}

__device__ void bitonic_sort(uint64_t* key, int64_t* idx, int count) {
  int P = 1;
  while (P < count) P <<= 1;
  for (int t = count + threadIdx.x; t < P; t += blockDim.x) {
    key[t] = 0;
    idx[t] = INT64_MAX;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < P / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;  // "up" = rank order
        const bool swap = up ? before_in_rank(key[hi], idx[hi], key[lo], idx[lo])
                             : before_in_rank(key[lo], idx[lo], key[hi], idx[hi]);
        if (swap) {
          const uint64_t tk = key[lo];
          key[lo] = key[hi];
          key[hi] = tk;
          const int64_t ti = idx[lo];
          idx[lo] = idx[hi];
          idx[hi] = ti;
        }
      }
      __syncthreads();
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kTopkThreads) topk_kernel(int64_t n, const T* __restrict__ X, int64_t ldx,
                                                            int64_t K, int64_t* __restrict__ top_idx,
                                                            T* __restrict__ top_val) {
  extern __shared__ __align__(16) unsigned char dyn[];
  uint64_t* ckey = (uint64_t*)dyn;
  int64_t* cidx = (int64_t*)(ckey + kTopkCap);
  __shared__ TopkShared sh;
  const T* x = X + (int64_t)blockIdx.x * ldx;
  constexpr int KB = KeyBits<T>::value;
  constexpr int nb = 1 << kHistBits;

  // pass 1: histogram of the top 12 key bits
  for (int t = threadIdx.x; t < nb; t += blockDim.x) sh.hist[t] = 0;
  if (!threadIdx.x) sh.count = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    atomicAdd(&sh.hist[order_key(x[i]) >> (KB - kHistBits)], 1u);
  __syncthreads();
  find_bin(sh, nb, (unsigned long long)K);
  uint64_t prefix = sh.found_bin;
  int pbits = kHistBits;
  unsigned long long above = sh.above;
  const unsigned long long in_bin = sh.hist[prefix];
  __syncthreads();

  if (above + in_bin <= (unsigned long long)kTopkCap) {
    // pass 2: every entry at or above the threshold bin is a candidate
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t k = order_key(x[i]);
      if ((k >> (KB - kHistBits)) >= prefix) {
        const unsigned slot = atomicAdd(&sh.count, 1u);
        ckey[slot] = k;
        cidx[slot] = i;
      }
    }
    __syncthreads();
    bitonic_sort(ckey, cidx, (int)sh.count);
  } else {
    // general path: pin the exact threshold key T, then take ties in index order
    unsigned long long need = (unsigned long long)K - above;
    while (pbits < KB) {
      const int d = KB - pbits < kHistBits ? KB - pbits : kHistBits;
      const int shift = KB - pbits - d;
      for (int t = threadIdx.x; t < nb; t += blockDim.x) sh.hist[t] = 0;
      __syncthreads();
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t k = order_key(x[i]);
        if ((k >> (KB - pbits)) == prefix) atomicAdd(&sh.hist[(k >> shift) & ((1u << d) - 1u)], 1u);
      }
      __syncthreads();
      find_bin(sh, 1 << d, need);
      need -= sh.above;
      prefix = (prefix << d) | sh.found_bin;
      pbits += d;
      __syncthreads();
    }
    const uint64_t Tk = prefix;
    const unsigned long long gt_total = (unsigned long long)K - need;
    // entries strictly above T (< K of them): any order
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint64_t k = order_key(x[i]);
      if (k > Tk) {
        const unsigned slot = atomicAdd(&sh.count, 1u);
        ckey[slot] = k;
        cidx[slot] = i;
      }
    }
    __syncthreads();
    // the first `need` ties in index order
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long taken = 0;
    for (int64_t base = 0; base < n && taken < need; base += blockDim.x) {
      const int64_t i = base + threadIdx.x;
      const bool tie = i < n && order_key(x[i]) == Tk;
      const unsigned m = __ballot_sync(0xffffffffu, tie);
      if (!lane) sh.warp_sums[wid] = __popc(m);
      __syncthreads();
      unsigned long long off = 0;
      for (int w = 0; w < wid; ++w) off += sh.warp_sums[w];
      unsigned long long tot = 0;
      for (int w = 0; w < kTopkThreads / 32; ++w) tot += sh.warp_sums[w];
      const unsigned long long rank_in = taken + off + __popc(m & ((1u << lane) - 1u));
      if (tie && rank_in < need) {
        ckey[gt_total + rank_in] = Tk;
        cidx[gt_total + rank_in] = i;
      }
      taken += tot;
      __syncthreads();
    }
    bitonic_sort(ckey, cidx, (int)K);
  }
  for (int64_t m = threadIdx.x; m < K; m += blockDim.x) {
    const int64_t i = cidx[m];
    top_idx[(int64_t)blockIdx.x * K + m] = i;
    top_val[(int64_t)blockIdx.x * K + m] = x[i];
  }
}

template <typename T>
int launch_topk(fsr_ctx* ctx, int64_t b, int64_t n, const T* X, int64_t ldx, int64_t K, int64_t* top_idx,
                T* top_val) {
  const size_t smem = (size_t)kTopkCap * 16;
  static bool configured[2] = {false, false};
  if (!configured[sizeof(T) == 8]) {
    FSR_CUDA(ctx, cudaFuncSetAttribute(topk_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[sizeof(T) == 8] = true;
  }
  topk_kernel<T><<<(unsigned)b, kTopkThreads, smem, ctx->stream>>>(n, X, ldx, K, top_idx, top_val);
  return fsr::launched(ctx, "topk_kernel");
}

inline size_t align256(size_t x) { return (x + 255) / 256 * 256; }

template <typename T>
int filter_impl(fsr_ctx* ctx, int64_t n, int64_t r, int u_sparse, const int64_t* u_indptr, const int32_t* u_indices,
                const T* u_values, const T* u_dense, int64_t ldu, const T* w, const double* eta, int64_t b,
                const int64_t* y_ptr, const int64_t* y_idx, const T* y_val, int copy_uncovered, void* workspace,
                T* X, int64_t topk, int64_t* top_idx, T* top_val) {
  char* ws = (char*)workspace;
  const size_t es = sizeof(T);
  T* Zt = (T*)ws;
  ws += align256((size_t)b * r * es);
  T* Zs = nullptr;
  if (u_sparse) {
    Zs = (T*)ws;
    ws += align256((size_t)r * b * es);
  }
  T* Xout = X;
  if (!Xout) Xout = (T*)ws;

  {
  fsr::StageTimer timer(ctx, FSR_STAGE_PROJECT);
  if (u_sparse)
    project_kernel<T, true><<<(unsigned)b, 256, 0, ctx->stream>>>(r, b, u_indptr, u_indices, u_values, nullptr, 0, w,
                                                                  y_ptr, y_idx, y_val, Zt, Zs);
  else
    project_kernel<T, false><<<(unsigned)b, 256, 0, ctx->stream>>>(r, b, nullptr, nullptr, nullptr, u_dense, ldu, w,
                                                                   y_ptr, y_idx, y_val, Zt, nullptr);
  FSR_TRY(fsr::launched(ctx, "project_kernel"));
  }

  if (u_sparse) {
    if (b == 1) {
      fsr::StageTimer timer(ctx, FSR_STAGE_FILTER_SPMM);
      FSR_TRY(fsr::launch_spmm<T>(ctx, n, u_indptr, u_indices, u_values, 1, Zs, 1, Xout, 1));
    } else {
      // K9 writes X (b x n) directly: smem-staged transposed tiles, no separate pass
      fsr::StageTimer timer(ctx, FSR_STAGE_FILTER_SPMM);
      FSR_TRY(fsr::launch_spmm_T<T>(ctx, n, u_indptr, u_indices, u_values, b, Zs, b, Xout, n));
    }
  } else {
    fsr::StageTimer timer(ctx, FSR_STAGE_FILTER_SPMM);
    // X_c (n x b, col-major) = U_c^T (n x r) * Zt_c (r x b)
    if (sizeof(T) == 8) {
      const double one = 1.0, zero = 0.0;
      FSR_BLAS(ctx, cublasDgemm_64(ctx->blas, CUBLAS_OP_T, CUBLAS_OP_N, n, b, r, &one, (const double*)u_dense, ldu,
                                   (const double*)Zt, r, &zero, (double*)Xout, n));
    } else {
      const float one = 1.0f, zero = 0.0f;
      FSR_BLAS(ctx, cublasSgemm_64(ctx->blas, CUBLAS_OP_T, CUBLAS_OP_N, n, b, r, &one, (const float*)u_dense, ldu,
                                   (const float*)Zt, r, &zero, (float*)Xout, n));
    }
  }
  if (copy_uncovered && eta) {
    fsr::StageTimer timer(ctx, FSR_STAGE_COPY_UNCOVERED);
    copy_uncovered_kernel<T><<<(unsigned)b, 128, 0, ctx->stream>>>(n, y_ptr, y_idx, y_val, eta, Xout, n);
    FSR_TRY(fsr::launched(ctx, "copy_uncovered_kernel"));
  }
  if (topk > 0) {
    fsr::StageTimer timer(ctx, FSR_STAGE_TOPK);
    FSR_TRY(launch_topk<T>(ctx, b, n, Xout, n, topk, top_idx, top_val));
  }
  return FSR_OK;
}

}  // namespace

extern "C" {

int64_t fsr_filter_workspace_bytes(int dtype, int64_t n, int64_t r, int64_t b, int need_x) {
  const size_t es = fsr::dtype_size(dtype);
  size_t total = align256((size_t)b * r * es) + align256((size_t)r * b * es);
  if (need_x) total += align256((size_t)n * b * es);
  return (int64_t)total + 256;
}

int fsr_filter_batch(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, int u_sparse, const int64_t* u_indptr,
                     const int32_t* u_indices, const void* u_values, const void* u_dense, int64_t ldu, const void* w,
                     const double* eta, int64_t b, const int64_t* y_ptr, const int64_t* y_idx, const void* y_val,
                     int copy_uncovered, void* workspace, void* X, int64_t topk, int64_t* top_idx, void* top_val) {
  FSR_REQUIRE(ctx, n >= 1 && r >= 1 && b >= 1 && workspace, "filter_batch: bad shape");
  FSR_REQUIRE(ctx, u_sparse ? (u_indptr && u_indices && u_values) : (u_dense && ldu >= r),
              "filter_batch: missing U");
  FSR_REQUIRE(ctx, topk >= 0 && topk <= kTopkCap / 4 && topk <= n, "filter_batch: topk must lie in [0, min(n, %d)]",
              kTopkCap / 4);
  FSR_REQUIRE(ctx, X || topk > 0, "filter_batch: nothing to output");
  FSR_REQUIRE(ctx, topk == 0 || (top_idx && top_val), "filter_batch: missing top-k outputs");
  if (dtype == FSR_F64)
    return filter_impl<double>(ctx, n, r, u_sparse, u_indptr, u_indices, (const double*)u_values,
                               (const double*)u_dense, ldu, (const double*)w, eta, b, y_ptr, y_idx,
                               (const double*)y_val, copy_uncovered, workspace, (double*)X, topk, top_idx,
                               (double*)top_val);
  return filter_impl<float>(ctx, n, r, u_sparse, u_indptr, u_indices, (const float*)u_values, (const float*)u_dense,
                            ldu, (const float*)w, eta, b, y_ptr, y_idx, (const float*)y_val, copy_uncovered, workspace,
                            (float*)X, topk, top_idx, (float*)top_val);
}

int fsr_topk_rows(fsr_ctx* ctx, int dtype, int64_t b, int64_t n, const void* X, int64_t ldx, int64_t topk,
                  int64_t* top_idx, void* top_val) {
  FSR_REQUIRE(ctx, b >= 0 && n >= 1 && ldx >= n && topk >= 1 && topk <= n && topk <= kTopkCap / 4,
              "topk_rows: bad args");
  if (!b) return FSR_OK;
  if (dtype == FSR_F64) return launch_topk<double>(ctx, b, n, (const double*)X, ldx, topk, top_idx, (double*)top_val);
  return launch_topk<float>(ctx, b, n, (const float*)X, ldx, topk, top_idx, (float*)top_val);
}

}  // extern "C"
