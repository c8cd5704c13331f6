// K9e layout builder: the sliced-ELL copy of U~ that the single-query filter
// streams (kernel and layout description in k9e.cuh).
#include <cub/cub.cuh>

#include "k9e.cuh"

namespace {

__global__ void row_lens_kernel(int64_t n, const int64_t* __restrict__ indptr, int32_t* __restrict__ lens,
                                int32_t* __restrict__ rows, int* __restrict__ too_long) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = indptr[i + 1] - indptr[i];
    if (l < 0 || l > INT32_MAX) *too_long = 1;
    lens[i] = (int32_t)l;
    rows[i] = (int32_t)i;
  }
}

// widths[s] = 32 * (longest row of slice s, rounded up to even), 0 for the slices of long rows;
// n_long = the sorted positions below the first slice whose longest row fits.
__global__ void slice_widths_kernel(int64_t n, int64_t n_slices, const int32_t* __restrict__ lens_sorted,
                                    int64_t long_len, int64_t* __restrict__ widths) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_slices; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = lens_sorted[s * 32];  // descending: the slice's first row is its longest
    widths[s] = l > long_len ? 0 : 32 * ((l + 1) & ~(int64_t)1);  // even: entries are stored in pairs
  }
}

__global__ void count_long_kernel(int64_t n_slices, const int32_t* __restrict__ lens_sorted, int64_t long_len,
                                  unsigned long long* __restrict__ long_slices) {
  unsigned long long mine = 0;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_slices; s += (int64_t)gridDim.x * blockDim.x)
    mine += lens_sorted[s * 32] > long_len;
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if (!(threadIdx.x & 31) && mine) atomicAdd(long_slices, mine);
}

// One warp per slice: lane = row; the row's entries go to [j / 2][lane][j % 2], the
// padding up to the (even) slice width is (column 0, value 0) and never summed.
__global__ void __launch_bounds__(256) sell_pack_kernel(int64_t n, int64_t n_slices,
                                                        const int64_t* __restrict__ indptr,
                                                        const int32_t* __restrict__ indices,
                                                        const float* __restrict__ values,
                                                        const int32_t* __restrict__ perm,
                                                        const int64_t* __restrict__ slice_ptr,
                                                        uint16_t* __restrict__ cols, float* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n_slices) return;
  const int64_t p0 = slice_ptr[s];
  const int64_t width = (slice_ptr[s + 1] - p0) >> 5;
  if (!width) return;
  const int64_t pos = s * 32 + lane;
  int64_t e0 = 0, len = 0;
  if (pos < n) {
    const int64_t i = perm[pos];
    e0 = indptr[i];
    len = indptr[i + 1] - e0;
  }
  for (int64_t j = 0; j < width; ++j) {
    const bool ok = j < len;
    const int64_t at = p0 + (j >> 1) * 64 + lane * 2 + (j & 1);
    cols[at] = ok ? (uint16_t)indices[e0 + j] : (uint16_t)0;
    vals[at] = ok ? values[e0 + j] : 0.f;
  }
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace

extern "C" {

int64_t fsr_sell_plan_workspace_bytes(int64_t n) {
  if (n < 1) return 256;
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                            (const int32_t*)nullptr, (int32_t*)nullptr, n);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const int64_t*)nullptr, (int64_t*)nullptr, n / 32 + 2);
  return (int64_t)(align256((size_t)n * 4) * 2 + align256((size_t)(n / 32 + 2) * 8) + align256(sort_bytes) +
                   align256(scan_bytes) + 512);
}

int fsr_sell_plan(fsr_ctx* ctx, int64_t n, const int64_t* u_indptr, int64_t long_len, int32_t* perm, int32_t* lens,
                  int64_t* slice_ptr, void* workspace, int64_t* n_long_out, int64_t* total_out) {
  FSR_REQUIRE(ctx, n >= 1 && n <= INT32_MAX && u_indptr && perm && lens && slice_ptr && workspace && n_long_out &&
                       total_out && long_len >= 1,
              "sell_plan: bad args");
  const int64_t n_slices = fsr::ceil_div(n, 32);
  char* ws = (char*)workspace;
  int32_t* lens_in = (int32_t*)ws;
  ws += align256((size_t)n * 4);
  int32_t* rows_in = (int32_t*)ws;
  ws += align256((size_t)n * 4);
  int64_t* widths = (int64_t*)ws;
  ws += align256((size_t)(n / 32 + 2) * 8);
  size_t sort_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                            (const int32_t*)nullptr, (int32_t*)nullptr, n);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const int64_t*)nullptr, (int64_t*)nullptr, n_slices + 1);
  void* sort_tmp = ws;
  ws += align256(sort_bytes);
  void* scan_tmp = ws;
  ws += align256(scan_bytes);
  unsigned long long* d_long = (unsigned long long*)ws;
  int* d_flag = (int*)(d_long + 1);
  FSR_CUDA(ctx, cudaMemsetAsync(d_long, 0, 16, ctx->stream));
  row_lens_kernel<<<fsr::grid_for(n, 256, ctx, 8), 256, 0, ctx->stream>>>(n, u_indptr, lens_in, rows_in, d_flag);
  FSR_TRY(fsr::launched(ctx, "row_lens_kernel"));
  // stable, descending by length: equal lengths keep ascending row order
  FSR_CUDA(ctx, cub::DeviceRadixSort::SortPairsDescending(sort_tmp, sort_bytes, lens_in, lens, rows_in, perm, n, 0, 32,
                                                          ctx->stream));
  ctx->launches++;
  FSR_CUDA(ctx, cudaMemsetAsync(widths, 0, (size_t)(n_slices + 1) * 8, ctx->stream));
  slice_widths_kernel<<<fsr::grid_for(n_slices, 256, ctx, 8), 256, 0, ctx->stream>>>(n, n_slices, lens, long_len,
                                                                                     widths);
  FSR_TRY(fsr::launched(ctx, "slice_widths_kernel"));
  count_long_kernel<<<fsr::grid_for(n_slices, 256, ctx, 8), 256, 0, ctx->stream>>>(n_slices, lens, long_len, d_long);
  FSR_TRY(fsr::launched(ctx, "count_long_kernel"));
  FSR_CUDA(ctx, cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, widths, slice_ptr, n_slices + 1, ctx->stream));
  ctx->launches++;
  void* host = nullptr;
  FSR_TRY(fsr::host_stage(ctx, 32, &host));
  unsigned long long* h = (unsigned long long*)host;
  FSR_CUDA(ctx, cudaMemcpyAsync(h, d_long, 16, cudaMemcpyDeviceToHost, ctx->stream));
  FSR_CUDA(ctx, cudaMemcpyAsync(h + 2, slice_ptr + n_slices, 8, cudaMemcpyDeviceToHost, ctx->stream));
  FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  FSR_REQUIRE(ctx, ((int*)(h + 1))[0] == 0, "sell_plan: a row of U~ is longer than 2^31 entries");
  *n_long_out = (int64_t)h[0] * 32;  // whole slices: may exceed n by < 32
  *total_out = (int64_t)h[2];
  return FSR_OK;
}

int fsr_sell_pack(fsr_ctx* ctx, int64_t n, const int64_t* u_indptr, const int32_t* u_indices, const float* u_values,
                  const int32_t* perm, const int64_t* slice_ptr, uint16_t* cols, float* vals) {
  FSR_REQUIRE(ctx, n >= 1 && u_indptr && u_indices && u_values && perm && slice_ptr && cols && vals,
              "sell_pack: bad args");
  const int64_t n_slices = fsr::ceil_div(n, 32);
  sell_pack_kernel<<<(unsigned)fsr::ceil_div(n_slices * 32, 256), 256, 0, ctx->stream>>>(
      n, n_slices, u_indptr, u_indices, u_values, perm, slice_ptr, cols, vals);
  return fsr::launched(ctx, "sell_pack_kernel");
}

}  // extern "C"
