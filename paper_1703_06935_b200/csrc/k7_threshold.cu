// K7: keep exactly tau entries of U with the largest |u|, ties in (row, col)
// order (reference spectral.py:269-294: coo_matrix drops zeros, then
// lexsort((col, row, -|u|))[:min(tau, nnz)], CSR build, eta from the kept U).
//
// Instead of an O(nr log nr) sort the device radix-selects the tau-th key of
// |u| (IEEE bits with the sign cleared are monotone in |u|): a few filtered
// digit histograms (one read of U each) pin the threshold key T; a count pass
// gives per-row #(key > T) and #(key == T); ties are taken in global
// (row, col) order via an exclusive scan of the per-row tie counts; a final
// pass compacts the kept entries straight into sorted CSR rows.  The same
// pieces run per row shard with the histogram summed across ranks and a
// per-rank tie offset (multi-GPU).
#include <cub/cub.cuh>

#include "fsr_common.cuh"

namespace {

template <typename T>
__global__ void __launch_bounds__(512) abs_hist_kernel(int64_t n_rows, int64_t r, const T* __restrict__ U,
                                                       int64_t ldu, uint64_t prefix, uint64_t himask, int shift,
                                                       int bits, unsigned long long* __restrict__ hist) {
  extern __shared__ unsigned int sh_hist[];
  const int nb = 1 << bits;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) sh_hist[b] = 0;
  __syncthreads();
  const uint64_t dmask = (uint64_t)nb - 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (ldu == r) {
    const int64_t total = n_rows * r;
    for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total; f += stride) {
      const uint64_t key = fsr::abs_key(U[f]);
      if (key != 0 && (key & himask) == prefix) atomicAdd(&sh_hist[(key >> shift) & dmask], 1u);
    }
  } else {
    const int64_t total = n_rows * r;
    for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total; f += stride) {
      const int64_t i = f / r, j = f - i * r;
      const uint64_t key = fsr::abs_key(U[i * ldu + j]);
      if (key != 0 && (key & himask) == prefix) atomicAdd(&sh_hist[(key >> shift) & dmask], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (sh_hist[b]) atomicAdd(&hist[b], (unsigned long long)sh_hist[b]);
}

template <typename T>
__global__ void __launch_bounds__(256) counts_kernel(int64_t n_rows, int64_t r, const T* __restrict__ U, int64_t ldu,
                                                     uint64_t Tkey, int64_t* __restrict__ gt,
                                                     int64_t* __restrict__ eq) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_rows; i += nwarps) {
    const T* row = U + i * ldu;
    int g = 0, e = 0;
    for (int64_t j = lane; j < r; j += 32) {
      const uint64_t key = fsr::abs_key(row[j]);
      g += key > Tkey;
      e += key == Tkey && key != 0;
    }
    for (int o = 16; o; o >>= 1) {
      g += __shfl_xor_sync(0xffffffffu, g, o);
      e += __shfl_xor_sync(0xffffffffu, e, o);
    }
    if (!lane) {
      gt[i] = g;
      eq[i] = e;
    }
  }
}

__global__ void kept_kernel(int64_t n_rows, const int64_t* __restrict__ gt, const int64_t* __restrict__ eq,
                            const int64_t* __restrict__ tie_base, int64_t tie_offset, int64_t ties_to_take,
                            int64_t* __restrict__ kept) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n_rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n_rows) {
      kept[i] = 0;
      continue;
    }
    int64_t avail = ties_to_take - (tie_offset + tie_base[i]);
    avail = avail < 0 ? 0 : (avail > eq[i] ? eq[i] : avail);
    kept[i] = gt[i] + avail;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) compact_kernel(int64_t n_rows, int64_t r, const T* __restrict__ U, int64_t ldu,
                                                      uint64_t Tkey, const int64_t* __restrict__ tie_base,
                                                      int64_t tie_offset, int64_t ties_to_take,
                                                      const int64_t* __restrict__ indptr,
                                                      int32_t* __restrict__ indices, T* __restrict__ values,
                                                      double* __restrict__ eta) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_rows; i += nwarps) {
    const T* row = U + i * ldu;
    int64_t out = indptr[i];
    const int64_t end = indptr[i + 1];
    int64_t tie = tie_offset + tie_base[i];
    double ss = 0.0;
    for (int64_t j0 = 0; j0 < r && out < end; j0 += 32) {
      const int64_t j = j0 + lane;
      T v = T(0);
      uint64_t key = 0;
      if (j < r) {
        v = row[j];
        key = fsr::abs_key(v);
      }
      const bool is_eq = key == Tkey && key != 0;
      const unsigned eqm = __ballot_sync(0xffffffffu, is_eq);
      const bool take = key > Tkey || (is_eq && tie + __popc(eqm & lt) < ties_to_take);
      const unsigned km = __ballot_sync(0xffffffffu, take);
      if (take) {
        const int64_t pos = out + __popc(km & lt);
        indices[pos] = (int32_t)j;
        values[pos] = v;
        const double d = (double)v;
        ss = fma(d, d, ss);
      }
      out += __popc(km);
      tie += __popc(eqm);
    }
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (!lane && eta) eta[i] = sqrt(ss);
  }
}

}  // namespace

extern "C" {

int fsr_abs_histogram(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t r, const void* U, int64_t ldu,
                      uint64_t prefix, int shift, int bits, uint64_t* hist) {
  FSR_REQUIRE(ctx, n_rows >= 0 && r >= 1 && ldu >= r && bits >= 1 && bits <= 12 && shift >= 0 && shift + bits <= 64,
              "abs_histogram: bad args");
  if (!n_rows) return FSR_OK;
  const uint64_t himask = shift + bits >= 64 ? 0ull : ~((1ull << (shift + bits)) - 1ull);
  const int block = 512;
  const int grid = fsr::grid_for(n_rows * r, block, ctx, 4);
  const size_t smem = (size_t)4 << bits;
  fsr::StageTimer timer(ctx, FSR_STAGE_HISTOGRAM);
  if (dtype == FSR_F64)
    abs_hist_kernel<double><<<grid, block, smem, ctx->stream>>>(n_rows, r, (const double*)U, ldu, prefix & himask,
                                                                 himask, shift, bits, (unsigned long long*)hist);
  else
    abs_hist_kernel<float><<<grid, block, smem, ctx->stream>>>(n_rows, r, (const float*)U, ldu, prefix & himask,
                                                                himask, shift, bits, (unsigned long long*)hist);
  return fsr::launched(ctx, "abs_hist_kernel");
}

int fsr_threshold_counts(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t r, const void* U, int64_t ldu,
                         uint64_t T, int64_t* gt, int64_t* eq) {
  FSR_REQUIRE(ctx, n_rows >= 0 && r >= 1 && ldu >= r, "threshold_counts: bad shape");
  if (!n_rows) return FSR_OK;
  const int grid = fsr::grid_for(n_rows * 32, 256, ctx, 8);
  fsr::StageTimer timer(ctx, FSR_STAGE_COMPACT);
  if (dtype == FSR_F64)
    counts_kernel<double><<<grid, 256, 0, ctx->stream>>>(n_rows, r, (const double*)U, ldu, T, gt, eq);
  else
    counts_kernel<float><<<grid, 256, 0, ctx->stream>>>(n_rows, r, (const float*)U, ldu, T, gt, eq);
  return fsr::launched(ctx, "counts_kernel");
}

int fsr_threshold_compact(fsr_ctx* ctx, int dtype, int64_t n_rows, int64_t r, const void* U, int64_t ldu,
                          uint64_t T, int64_t tie_offset, int64_t ties_to_take, const int64_t* gt,
                          const int64_t* eq, int64_t* indptr_out, int32_t* indices_out, void* values_out,
                          double* eta, int64_t* nnz_host) {
  FSR_REQUIRE(ctx, n_rows >= 0 && r >= 1 && ldu >= r && tie_offset >= 0 && ties_to_take >= 0 && nnz_host,
              "threshold_compact: bad args");
  if (!n_rows) {
    *nnz_host = 0;
    return FSR_OK;
  }
  fsr::StageTimer timer(ctx, FSR_STAGE_COMPACT);
  size_t scan_bytes = 0, scan2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, eq, indptr_out, n_rows, ctx->stream);
  cub::DeviceScan::ExclusiveSum(nullptr, scan2, indptr_out, indptr_out, n_rows + 1, ctx->stream);
  if (scan2 > scan_bytes) scan_bytes = scan2;
  void* buf = nullptr;
  const size_t tie_bytes = (size_t)n_rows * 8;
  FSR_TRY(fsr::scratch(ctx, tie_bytes + scan_bytes + 256, &buf));
  int64_t* tie_base = (int64_t*)buf;
  void* temp = (char*)buf + ((tie_bytes + 255) / 256) * 256;
  FSR_CUDA(ctx, cub::DeviceScan::ExclusiveSum(temp, scan_bytes, eq, tie_base, n_rows, ctx->stream));
  kept_kernel<<<fsr::grid_for(n_rows + 1, 256, ctx), 256, 0, ctx->stream>>>(n_rows, gt, eq, tie_base, tie_offset,
                                                                            ties_to_take, indptr_out);
  FSR_TRY(fsr::launched(ctx, "kept_kernel"));
  FSR_CUDA(ctx, cub::DeviceScan::ExclusiveSum(temp, scan_bytes, indptr_out, indptr_out, n_rows + 1, ctx->stream));
  const int grid = fsr::grid_for(n_rows * 32, 256, ctx, 8);
  if (dtype == FSR_F64)
    compact_kernel<double><<<grid, 256, 0, ctx->stream>>>(n_rows, r, (const double*)U, ldu, T, tie_base, tie_offset,
                                                          ties_to_take, indptr_out, indices_out,
                                                          (double*)values_out, eta);
  else
    compact_kernel<float><<<grid, 256, 0, ctx->stream>>>(n_rows, r, (const float*)U, ldu, T, tie_base, tie_offset,
                                                         ties_to_take, indptr_out, indices_out, (float*)values_out,
                                                         eta);
  FSR_TRY(fsr::launched(ctx, "compact_kernel"));
  FSR_CUDA(ctx, cudaMemcpyAsync(nnz_host, indptr_out + n_rows, 8, cudaMemcpyDeviceToHost, ctx->stream));
  FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FSR_OK;
}

}  // extern "C"
