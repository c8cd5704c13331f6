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

#include <algorithm>
#include <cstdlib>

#include "k9e.cuh"
#include "prune.cuh"
#include "spmm.cuh"
#include "topk.cuh"

namespace {

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
    const T s = w ? w[c] * z[c] : z[c];
    z[c] = s;
    if (Zs) Zs[c * b + j] = s;
  }
}

// Same result as project_kernel<T, true> (rows in query order, entries of a
// row in parallel), but z lives in shared memory and every (col, val) entry of
// the query's rows is prefetched into shared memory first, so the ordered
// accumulation runs at smem latency instead of one HBM round trip per row.
constexpr int kProjCap = 4096;     // prefetched entries
constexpr int kProjMaxRows = 256;  // rows of U~ per query on this path

template <typename T>
__global__ void __launch_bounds__(256) project_smem_kernel(int64_t r, int64_t b, const int64_t* __restrict__ u_indptr,
                                                           const int32_t* __restrict__ u_indices,
                                                           const T* __restrict__ u_values, const T* __restrict__ w,
                                                           const int64_t* __restrict__ y_ptr,
                                                           const int64_t* __restrict__ y_idx,
                                                           const T* __restrict__ y_val, T* __restrict__ Zt,
                                                           T* __restrict__ Zs, __half* __restrict__ Zh = nullptr,
                                                           float2* __restrict__ qp = nullptr,
                                                           int* __restrict__ nflag = nullptr, int64_t zh_ld = 0) {
  extern __shared__ __align__(16) unsigned char dyn[];
  T* z = (T*)dyn;
  T* ev = (T*)(dyn + ((r * sizeof(T) + 15) / 16) * 16);
  int32_t* ec = (int32_t*)(ev + kProjCap);
  __shared__ int64_t offs[kProjMaxRows + 1];
  __shared__ int64_t starts[kProjMaxRows];
  __shared__ T yv[kProjMaxRows];
  const int64_t j = blockIdx.x;
  const int64_t y0 = y_ptr[j], ny = y_ptr[j + 1] - y0;
  // w is read last: pull its lines into L2 now (one 128-byte line per thread)
  if (w)
    for (int64_t c = (int64_t)threadIdx.x * (128 / sizeof(T)); c < r; c += (int64_t)blockDim.x * (128 / sizeof(T)))
      asm volatile("prefetch.global.L2 [%0];" ::"l"(w + c));
  for (int64_t c = threadIdx.x; c < r; c += blockDim.x) z[c] = T(0);
  bool fits = ny <= kProjMaxRows;
  if (fits) {
    for (int64_t e = threadIdx.x; e < ny; e += blockDim.x) {
      const int64_t i = y_idx[y0 + e];
      yv[e] = y_val[y0 + e];
      starts[e] = u_indptr[i];
      offs[e + 1] = u_indptr[i + 1] - u_indptr[i];
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // inclusive scan of the row lengths, 32 at a time
      int64_t carry = 0;
      if (!threadIdx.x) offs[0] = 0;
      for (int64_t e0 = 0; e0 < ny; e0 += 32) {
        const int64_t e = e0 + threadIdx.x;
        int64_t v = e < ny ? offs[e + 1] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int64_t u = __shfl_up_sync(0xffffffffu, v, o);
          if ((int)threadIdx.x >= o) v += u;
        }
        if (e < ny) offs[e + 1] = v + carry;
        carry += __shfl_sync(0xffffffffu, v, 31);
      }
    }
    __syncthreads();
  }
  if (fits) {
    // windows of kProjCap entries, flattened over the query's rows, 8 loads
    // per thread in flight before their shared-memory stores (a row-by-row
    // loop waited one DRAM latency per row: ~50 us for a 50-row query, the
    // whole step at b = 1).  Rows are consumed in query order across windows,
    // so every z[c] sees its contributions in the reference's order.
    const int64_t tot = offs[ny];
    int64_t e_first = 0;  // first row with entries at or after the window start
    for (int64_t w0 = 0; w0 < tot; w0 += kProjCap) {
      const int64_t w1 = min(tot, w0 + (int64_t)kProjCap);
      for (int64_t t0 = w0 + threadIdx.x; t0 < w1; t0 += 8 * (int64_t)blockDim.x) {
        int32_t cc[8];
        T vv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t t = t0 + (int64_t)u * blockDim.x;
          cc[u] = 0;
          vv[u] = T(0);
          if (t < w1) {
            int lo = 0, hi = (int)ny - 1;  // the row of entry t: largest e with offs[e] <= t
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (offs[mid] <= t)
                lo = mid;
              else
                hi = mid - 1;
            }
            FSR_DCHECK(lo >= 0 && lo < ny && offs[lo] <= t && t < offs[lo + 1]);
            const int64_t src = starts[lo] + (t - offs[lo]);
            cc[u] = u_indices[src];
            vv[u] = u_values[src];
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t t = t0 + (int64_t)u * blockDim.x;
          if (t < w1) {
            ec[t - w0] = cc[u];
            ev[t - w0] = vv[u];
          }
        }
      }
      __syncthreads();
      while (e_first < ny && offs[e_first + 1] <= w0) ++e_first;
      for (int64_t e = e_first; e < ny && offs[e] < w1; ++e) {
        const T v = yv[e];
        const int64_t a = max(offs[e], w0), z1 = min(offs[e + 1], w1);
        for (int64_t t = a + threadIdx.x; t < z1; t += blockDim.x) {
          const int32_t c = ec[t - w0];
          FSR_DCHECK(c >= 0 && c < r);
          z[c] = fsr::mul_add_rn(z[c], ev[t - w0], v);
        }
        __syncthreads();
      }
    }
    __syncthreads();
  } else {
    __syncthreads();
    for (int64_t e = 0; e < ny; ++e) {
      const int64_t i = y_idx[y0 + e];
      const T v = y_val[y0 + e];
      for (int64_t s = u_indptr[i] + threadIdx.x; s < u_indptr[i + 1]; s += blockDim.x) {
        const int32_t c = u_indices[s];
        z[c] = fsr::mul_add_rn(z[c], u_values[s], v);
      }
      __syncthreads();
    }
  }
  float amax = 0.f;
  double ss = 0.0;
  for (int64_t c = threadIdx.x; c < r; c += blockDim.x) {
    const T s = w ? w[c] * z[c] : z[c];
    Zt[j * r + c] = s;
    if (Zs) Zs[c * b + j] = s;
    if (Zh) {
      z[c] = s;
      amax = fmaxf(amax, fabsf((float)s));
      ss = fma((double)s, (double)s, ss);
    }
  }
  if constexpr (std::is_same<T, float>::value) {
    // fp16 copy of column j of Zs for the pruned path (prune.cuh zs_half_kernel, fused)
    if (Zh) {
      __shared__ float red_a[8];
      __shared__ double red_s[8];
      __shared__ float sc_s;
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
      }
      if (lane == 0) {
        red_a[wid] = amax;
        red_s[wid] = ss;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
          amax = fmaxf(amax, red_a[k]);
          ss += red_s[k];
        }
        float sc = 1.f, inv = 1.f, zb = 0.f;
        fsr::prune::query_scale(amax, ss, &sc, &inv, &zb);
        sc_s = sc;
        qp[j] = make_float2(inv, zb);
        if (j == 0) {
          nflag[0] = 0;
          nflag[b + 1] = 0;
        }
      }
      __syncthreads();
      const float sc = sc_s;
      if (zh_ld)  // query-major [b][zh_ld] (K9t's K-major GEMM operand): coalesced
        for (int64_t c = threadIdx.x; c < r; c += blockDim.x) Zh[j * zh_ld + c] = __float2half_rn(z[c] * sc);
      else
        for (int64_t c = threadIdx.x; c < r; c += blockDim.x) Zh[c * b + j] = __float2half_rn(z[c] * sc);
    }
  }
}

__global__ void u16_columns_kernel(int64_t nnz, const int32_t* __restrict__ indices, uint16_t* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (uint16_t)indices[e];
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

// K8 for b queries: Zt (b x r) = w .* U[supp y_j]^T y_j (w may be NULL: no
// scaling); also Zs = Zt^T (r x b) when Zs != NULL (sparse U only).
template <typename T>
int launch_project(fsr_ctx* ctx, int64_t r, int64_t b, int u_sparse, const int64_t* u_indptr,
                   const int32_t* u_indices, const T* u_values, const T* u_dense, int64_t ldu, const T* w,
                   const int64_t* y_ptr, const int64_t* y_idx, const T* y_val, T* Zt, T* Zs,
                   __half* Zh = nullptr, float2* qp = nullptr, int* nflag = nullptr, bool* fused = nullptr,
                   int64_t zh_ld = 0) {
  fsr::StageTimer timer(ctx, FSR_STAGE_PROJECT);
  const size_t psmem = ((size_t)r * sizeof(T) + 15) / 16 * 16 + (size_t)kProjCap * (sizeof(T) + 4);
  if (fused) *fused = u_sparse && psmem <= 160 * 1024;
  if (u_sparse && psmem <= 160 * 1024) {
    FSR_TRY(fsr::ensure_smem(ctx, project_smem_kernel<T>, psmem));
    project_smem_kernel<T><<<(unsigned)b, 256, psmem, ctx->stream>>>(r, b, u_indptr, u_indices, u_values, w, y_ptr,
                                                                     y_idx, y_val, Zt, Zs, Zh, qp, nflag, zh_ld);
  } else if (u_sparse)
    project_kernel<T, true><<<(unsigned)b, 256, 0, ctx->stream>>>(r, b, u_indptr, u_indices, u_values, nullptr, 0, w,
                                                                  y_ptr, y_idx, y_val, Zt, Zs);
  else
    project_kernel<T, false><<<(unsigned)b, 256, 0, ctx->stream>>>(r, b, nullptr, nullptr, nullptr, u_dense, ldu, w,
                                                                   y_ptr, y_idx, y_val, Zt, nullptr);
  return fsr::launched(ctx, "project_kernel");
}

inline size_t align256(size_t x) { return (x + 255) / 256 * 256; }

template <int NV, int DEPTH, int ROWS, int MINB, int WARPS = 8>
int launch_k9h(fsr_ctx* ctx, int64_t n, const int64_t* u_indptr, const int32_t* u_indices, const float* u_values,
               int64_t b, const __half* Zh, const float2* qp, float* Xt, float* cb, int* cmax_bits) {
  namespace P = fsr::prune;
  auto kern = P::spmm_T_half_kernel<NV, DEPTH, ROWS, MINB, WARPS>;
  const size_t smem = (size_t)ROWS * (256 * NV + 1) * 4;
  FSR_TRY(fsr::ensure_smem(ctx, kern, smem));
  dim3 grid((unsigned)fsr::ceil_div(n, ROWS), (unsigned)fsr::ceil_div(b, 256 * NV));
  kern<<<grid, 32 * WARPS, smem, ctx->stream>>>(n, u_indptr, u_indices, u_values, b, Zh, b, qp, Xt, n, cb, cmax_bits);
  return fsr::launched(ctx, "spmm_T_half_kernel");
}

// Top-k-only fp32 batch through the certified pruned path (prune.cuh).
int filter_pruned(fsr_ctx* ctx, int64_t n, int64_t r, const int64_t* u_indptr, const int32_t* u_indices,
                  const float* u_values, const float* w, const double* eta, int64_t b, const int64_t* y_ptr,
                  const int64_t* y_idx, const float* y_val, int copy_uncovered, void* workspace, int64_t topk,
                  int64_t* top_idx, float* top_val) {
  namespace P = fsr::prune;
  char* ws = (char*)workspace;
  float* Zt = (float*)ws;
  ws += align256((size_t)b * r * 4);
  float* Zs = (float*)ws;
  ws += align256((size_t)r * b * 4);
  float* Xt = (float*)ws;  // x~ (b x n), then exact rows of flagged queries
  ws += align256((size_t)n * b * 4);
  __half* Zh = (__half*)ws;
  ws += align256((size_t)r * b * 2);
  float2* qp = (float2*)ws;
  ws += align256((size_t)b * 8);
  float* cb = (float*)ws;
  ws += align256((size_t)n * 4);
  int* nflag = (int*)ws;
  int* flags = nflag + 1;
  int* cmax_bits = nflag + b + 1;
  ws += align256((size_t)(b + 2) * 4);
  int32_t* cand = (int32_t*)ws;
  ws += align256((size_t)b * P::kCap * 4);
  int32_t* ccount = (int32_t*)ws;
  ws += align256((size_t)b * 4);
  uint32_t* thr = (uint32_t*)ws;
  ws += align256((size_t)b * 4);
  unsigned* nlow = (unsigned*)ws;
  bool fused = false;
  FSR_TRY(launch_project<float>(ctx, r, b, 1, u_indptr, u_indices, u_values, nullptr, 0, w, y_ptr, y_idx, y_val, Zt,
                                Zs, Zh, qp, nflag, &fused));
  if (!fused) {
    fsr::StageTimer timer(ctx, FSR_STAGE_PROJECT);
    P::zs_half_kernel<<<(unsigned)fsr::ceil_div(b, 32), dim3(32, 8), 0, ctx->stream>>>(r, b, Zs, Zh, qp, nflag);
    FSR_TRY(fsr::launched(ctx, "zs_half_kernel"));
  }
  {
    fsr::StageTimer timer(ctx, FSR_STAGE_FILTER_SPMM);
    FSR_TRY((launch_k9h<1, 4, 32, 4>(ctx, n, u_indptr, u_indices, u_values, b, Zh, qp, Xt, cb, cmax_bits)));
  }
  if (copy_uncovered && eta) {
    fsr::StageTimer timer(ctx, FSR_STAGE_COPY_UNCOVERED);
    copy_uncovered_kernel<float><<<(unsigned)b, 128, 0, ctx->stream>>>(n, y_ptr, y_idx, y_val, eta, Xt, n);
    FSR_TRY(fsr::launched(ctx, "copy_uncovered_kernel"));
  }
  {
    fsr::StageTimer timer(ctx, FSR_STAGE_TOPK);
    const size_t fsmem = (size_t)fsr::topk::kCap * 16;
    FSR_TRY(fsr::ensure_smem(ctx, P::fallback_select_kernel, fsmem));
    static int per_sm = 0;  // occupancy of a smem-free kernel: the same on every B200
    if (!per_sm) {
      FSR_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, P::prune_threshold_kernel, P::kThreads, 0));
      per_sm = std::max(per_sm, 1);
    }
    const int copy = copy_uncovered && eta;
    const int64_t grid = std::min<int64_t>(b, (int64_t)ctx->num_sms * per_sm);
    P::prune_threshold_kernel<<<(unsigned)grid, P::kThreads, 0, ctx->stream>>>(n, b, Xt, n, cb, qp, topk, thr, ccount,
                                                                              nlow, nflag, flags);
    FSR_TRY(fsr::launched(ctx, "prune_threshold_kernel"));
    // segments of the streaming pass: enough CTAs to keep every SM streaming
    const int segs = (int)std::max<int64_t>(1, std::min<int64_t>(16, fsr::ceil_div(4 * ctx->num_sms * 8, b)));
    const int64_t seg_len = fsr::ceil_div(fsr::ceil_div(n, segs), 1024) * 1024;
    P::prune_scan_kernel<<<(unsigned)(b * segs), P::kThreads, 0, ctx->stream>>>(n, segs, seg_len, Xt, n, cb, cmax_bits,
                                                                               qp, thr, cand, ccount, nlow);
    FSR_TRY(fsr::launched(ctx, "prune_scan_kernel"));
    P::prune_finish_kernel<<<(unsigned)b, P::kThreads, 0, ctx->stream>>>(n, Xt, n, cb, qp, cand, ccount, nlow,
                                                                        u_indptr, u_indices, u_values, Zs, b, eta,
                                                                        copy, y_ptr, y_idx, topk, top_idx, top_val,
                                                                        nflag, flags);
    FSR_TRY(fsr::launched(ctx, "prune_finish_kernel"));
    P::fallback_rows_kernel<<<(unsigned)ctx->num_sms * 8, 256, 0, ctx->stream>>>(
        n, Xt, n, u_indptr, u_indices, u_values, Zs, b, eta, copy, y_ptr, y_idx, nflag, flags);
    FSR_TRY(fsr::launched(ctx, "fallback_rows_kernel"));
    P::fallback_select_kernel<<<(unsigned)b, fsr::topk::kThreads, fsmem, ctx->stream>>>(n, Xt, n, topk, top_idx,
                                                                                      top_val, nflag, flags);
    FSR_TRY(fsr::launched(ctx, "fallback_select_kernel"));
  }
  return FSR_OK;
}

template <typename T>
int filter_impl(fsr_ctx* ctx, int64_t n, int64_t r, int u_sparse, const int64_t* u_indptr, const int32_t* u_indices,
                const T* u_values, const T* u_dense, int64_t ldu, const T* w, const double* eta, int64_t b,
                const int64_t* y_ptr, const int64_t* y_idx, const T* y_val, int copy_uncovered, void* workspace,
                T* X, int64_t topk, int64_t* top_idx, T* top_val, const uint16_t* u_cols16 = nullptr,
                const fsr::sell::View* sell = nullptr) {
  if constexpr (std::is_same<T, float>::value) {
    if (u_sparse && !X && topk > 0 && ctx->topk_prune && fsr::prune::applicable(n, b, topk) &&
        fsr::aligned(workspace, 256))
      return filter_pruned(ctx, n, r, u_indptr, u_indices, u_values, w, eta, b, y_ptr, y_idx, y_val, copy_uncovered,
                           workspace, topk, top_idx, top_val);
  }
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

  FSR_TRY(launch_project<T>(ctx, r, b, u_sparse, u_indptr, u_indices, u_values, u_dense, ldu, w, y_ptr, y_idx,
                            y_val, Zt, Zs));

  if (u_sparse) {
    if (b == 1) {
      fsr::StageTimer timer(ctx, FSR_STAGE_FILTER_SPMM);
      bool done = false;
      if constexpr (std::is_same<T, float>::value) {
        if (sell) {  // K9e: sliced-ELL stream, sequential CSR-order sums (k9e.cuh)
          FSR_TRY(fsr::sell::launch_spmv(ctx, n, *sell, u_indptr, u_values, Zs, r, Xout));
          done = true;
        }
      }
      if (done) {
      } else if (u_cols16 && (size_t)r * sizeof(T) <= 160 * 1024)
        FSR_TRY((fsr::launch_spmv_smem<T, uint16_t>(ctx, n, u_indptr, u_cols16, u_values, Zs, r, Xout)));
      else if ((size_t)r * sizeof(T) <= 160 * 1024)
        FSR_TRY(fsr::launch_spmv_smem<T>(ctx, n, u_indptr, u_indices, u_values, Zs, r, Xout));
      else
        FSR_TRY(fsr::launch_spmm<T>(ctx, n, u_indptr, u_indices, u_values, 1, Zs, 1, Xout, 1));
    } else {
      // K9 writes X (b x n) directly: smem-staged transposed tiles, no separate pass
      fsr::StageTimer timer(ctx, FSR_STAGE_FILTER_SPMM);
      bool done = false;
      if constexpr (std::is_same<T, float>::value) {
        if (sell && fsr::sell::batch_applicable(r, b)) {  // K9e, 2 or 4 queries per pass of the sliced-ELL copy
          FSR_TRY(fsr::sell::launch_spmm(ctx, n, *sell, u_indptr, u_values, Zs, r, b, Xout, n));
          done = true;
        }
      }
      if (!done) FSR_TRY(fsr::launch_spmm_T<T>(ctx, n, u_indptr, u_indices, u_values, b, Zs, b, Xout, n));
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
    FSR_TRY(fsr::topk::launch<T>(ctx, b, n, Xout, n, topk, top_idx, top_val));
  }
  return FSR_OK;
}

}  // namespace

namespace fsr {
// K8 for the tensor-core step (k9t.cu): Zt, Zs and the query-major scaled fp16 Zh.
int k9t_project(fsr_ctx* ctx, int64_t r, int64_t b, const int64_t* u_indptr, const int32_t* u_indices,
                const float* u_values, const float* w, const int64_t* y_ptr, const int64_t* y_idx,
                const float* y_val, float* Zt, float* Zs, __half* Zh, int64_t ldzh, float2* qp, int* nflag) {
  bool fused = false;
  const size_t psmem = ((size_t)r * 4 + 15) / 16 * 16 + (size_t)kProjCap * 8;
  FSR_REQUIRE(ctx, psmem <= 160 * 1024, "k9t_project: r = %lld too large for the fused projection", (long long)r);
  FSR_TRY(launch_project<float>(ctx, r, b, 1, u_indptr, u_indices, u_values, nullptr, 0, w, y_ptr, y_idx, y_val, Zt,
                                Zs, Zh, qp, nflag, &fused, ldzh));
  FSR_REQUIRE(ctx, fused, "k9t_project: fused projection unavailable");
  return FSR_OK;
}
}  // namespace fsr

extern "C" {

int64_t fsr_filter_workspace_bytes(int dtype, int64_t n, int64_t r, int64_t b, int need_x) {
  const size_t es = fsr::dtype_size(dtype);
  size_t total = align256((size_t)b * r * es) + align256((size_t)r * b * es);
  if (need_x) total += align256((size_t)n * b * es);
  if (need_x && dtype == FSR_F32) total += fsr::prune::workspace_bytes(n, r, b);
  return (int64_t)total + 256;
}

int fsr_filter_batch(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, int u_sparse, const int64_t* u_indptr,
                     const int32_t* u_indices, const void* u_values, const void* u_dense, int64_t ldu, const void* w,
                     const double* eta, int64_t b, const int64_t* y_ptr, const int64_t* y_idx, const void* y_val,
                     int copy_uncovered, void* workspace, void* X, int64_t topk, int64_t* top_idx, void* top_val) {
  return fsr_filter_batch_u16(ctx, dtype, n, r, u_sparse, u_indptr, u_indices, nullptr, u_values, u_dense, ldu, w, eta,
                              b, y_ptr, y_idx, y_val, copy_uncovered, workspace, X, topk, top_idx, top_val);
}

int fsr_u16_columns(fsr_ctx* ctx, int64_t nnz, const int32_t* indices, uint16_t* out) {
  FSR_REQUIRE(ctx, nnz >= 0 && (nnz == 0 || (indices && out)), "u16_columns: bad args");
  if (!nnz) return FSR_OK;
  u16_columns_kernel<<<fsr::grid_for(nnz, 256, ctx, 8), 256, 0, ctx->stream>>>(nnz, indices, out);
  return fsr::launched(ctx, "u16_columns_kernel");
}

int fsr_filter_batch_u16(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, int u_sparse, const int64_t* u_indptr,
                         const int32_t* u_indices, const uint16_t* u_cols16, const void* u_values, const void* u_dense,
                         int64_t ldu, const void* w, const double* eta, int64_t b, const int64_t* y_ptr,
                         const int64_t* y_idx, const void* y_val, int copy_uncovered, void* workspace, void* X,
                         int64_t topk, int64_t* top_idx, void* top_val) {
  FSR_REQUIRE(ctx, !u_cols16 || (u_sparse && r <= 65536), "filter_batch: 16-bit columns need a sparse U and r <= 65536");
  FSR_REQUIRE(ctx, n >= 1 && r >= 1 && b >= 1 && workspace, "filter_batch: bad shape");
  FSR_REQUIRE(ctx, u_sparse ? (u_indptr && u_indices && u_values) : (u_dense && ldu >= r),
              "filter_batch: missing U");
  FSR_REQUIRE(ctx, topk >= 0 && topk <= fsr::topk::kCap / 4 && topk <= n, "filter_batch: topk must lie in [0, min(n, %d)]",
              fsr::topk::kCap / 4);
  FSR_REQUIRE(ctx, X || topk > 0, "filter_batch: nothing to output");
  FSR_REQUIRE(ctx, topk == 0 || (top_idx && top_val), "filter_batch: missing top-k outputs");
  if (dtype == FSR_F64)
    return filter_impl<double>(ctx, n, r, u_sparse, u_indptr, u_indices, (const double*)u_values,
                               (const double*)u_dense, ldu, (const double*)w, eta, b, y_ptr, y_idx,
                               (const double*)y_val, copy_uncovered, workspace, (double*)X, topk, top_idx,
                               (double*)top_val);
  return filter_impl<float>(ctx, n, r, u_sparse, u_indptr, u_indices, (const float*)u_values, (const float*)u_dense,
                            ldu, (const float*)w, eta, b, y_ptr, y_idx, (const float*)y_val, copy_uncovered, workspace,
                            (float*)X, topk, top_idx, (float*)top_val, u_cols16);
}

int fsr_filter_batch_sell(fsr_ctx* ctx, int64_t n, int64_t r, const int64_t* u_indptr, const int32_t* u_indices,
                          const uint16_t* u_cols16, const float* u_values, const int32_t* sell_perm,
                          const int32_t* sell_lens, const int64_t* sell_slice_ptr, const uint16_t* sell_cols,
                          const float* sell_vals, int64_t n_long, const float* w, const double* eta, int64_t b,
                          const int64_t* y_ptr, const int64_t* y_idx, const float* y_val, int copy_uncovered,
                          void* workspace, float* X, int64_t topk, int64_t* top_idx, float* top_val) {
  FSR_REQUIRE(ctx, n >= 1 && fsr::sell::applicable(r) && workspace && u_indptr && u_indices && u_cols16 && u_values,
              "filter_batch_sell: bad shape (r <= 16384, sparse U with its 16-bit columns)");
  FSR_REQUIRE(ctx, b == 1 || fsr::sell::batch_applicable(r, b),
              "filter_batch_sell: b must lie in [1, %d] (and r <= 12800 for b >= 2)", (int)fsr::sell::kMaxBatch);
  FSR_REQUIRE(ctx, sell_perm && sell_lens && sell_slice_ptr && sell_cols && sell_vals && n_long >= 0 &&
                       n_long % 32 == 0,
              "filter_batch_sell: missing sliced-ELL layout (fsr_sell_plan / fsr_sell_pack)");
  FSR_REQUIRE(ctx, topk >= 0 && topk <= fsr::topk::kCap / 4 && topk <= n, "filter_batch_sell: topk must lie in [0, min(n, %d)]",
              fsr::topk::kCap / 4);
  FSR_REQUIRE(ctx, X || topk > 0, "filter_batch_sell: nothing to output");
  FSR_REQUIRE(ctx, topk == 0 || (top_idx && top_val), "filter_batch_sell: missing top-k outputs");
  fsr::sell::View V;
  V.perm = sell_perm;
  V.lens = sell_lens;
  V.slice_ptr = sell_slice_ptr;
  V.cols = sell_cols;
  V.vals = sell_vals;
  V.n_long = n_long;
  V.csr_cols16 = u_cols16;
  // b <= 64 never takes the pruned branch of filter_impl (prune::applicable needs b >= 256)
  return filter_impl<float>(ctx, n, r, 1, u_indptr, u_indices, u_values, nullptr, 0, w, eta, b, y_ptr, y_idx, y_val,
                            copy_uncovered, workspace, X, topk, top_idx, top_val, u_cols16, &V);
}

int fsr_filter_single_sell(fsr_ctx* ctx, int64_t n, int64_t r, const int64_t* u_indptr, const int32_t* u_indices,
                           const uint16_t* u_cols16, const float* u_values, const int32_t* sell_perm,
                           const int32_t* sell_lens, const int64_t* sell_slice_ptr, const uint16_t* sell_cols,
                           const float* sell_vals, int64_t n_long, const float* w, const double* eta,
                           const int64_t* y_ptr, const int64_t* y_idx, const float* y_val, int copy_uncovered,
                           void* workspace, float* X, int64_t topk, int64_t* top_idx, float* top_val) {
  return fsr_filter_batch_sell(ctx, n, r, u_indptr, u_indices, u_cols16, u_values, sell_perm, sell_lens,
                               sell_slice_ptr, sell_cols, sell_vals, n_long, w, eta, 1, y_ptr, y_idx, y_val,
                               copy_uncovered, workspace, X, topk, top_idx, top_val);
}

int fsr_topk_rows(fsr_ctx* ctx, int dtype, int64_t b, int64_t n, const void* X, int64_t ldx, int64_t topk,
                  int64_t* top_idx, void* top_val) {
  FSR_REQUIRE(ctx, b >= 0 && n >= 1 && ldx >= n && topk >= 1 && topk <= n && topk <= fsr::topk::kCap / 4,
              "topk_rows: bad args");
  if (!b) return FSR_OK;
  if (dtype == FSR_F64) return fsr::topk::launch<double>(ctx, b, n, (const double*)X, ldx, topk, top_idx, (double*)top_val);
  return fsr::topk::launch<float>(ctx, b, n, (const float*)X, ldx, topk, top_idx, (float*)top_val);
}

int fsr_project_batch(fsr_ctx* ctx, int dtype, int64_t n, int64_t r, int u_sparse, const int64_t* u_indptr,
                      const int32_t* u_indices, const void* u_values, const void* u_dense, int64_t ldu,
                      const void* w, int64_t b, const int64_t* y_ptr, const int64_t* y_idx, const void* y_val,
                      void* Zt) {
  FSR_REQUIRE(ctx, n >= 1 && r >= 1 && b >= 0 && Zt, "project_batch: bad shape");
  FSR_REQUIRE(ctx, u_sparse ? (u_indptr && u_indices && u_values) : (u_dense && ldu >= r),
              "project_batch: missing U");
  if (!b) return FSR_OK;
  if (dtype == FSR_F64)
    return launch_project<double>(ctx, r, b, u_sparse, u_indptr, u_indices, (const double*)u_values,
                                  (const double*)u_dense, ldu, (const double*)w, y_ptr, y_idx, (const double*)y_val,
                                  (double*)Zt, nullptr);
  return launch_project<float>(ctx, r, b, u_sparse, u_indptr, u_indices, (const float*)u_values,
                               (const float*)u_dense, ldu, (const float*)w, y_ptr, y_idx, (const float*)y_val,
                               (float*)Zt, nullptr);
}

}  // extern "C"


