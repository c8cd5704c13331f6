// K9e: the single-query (b = 1) K9 on a sliced-ELL copy of U~.
//
// Replaces, for one fp32 query, x = U~ zs of specrank.ranking.filter
// (/root/reference/pkg/src/specrank/ranking.py:244-246).  The CSR SpMV spends
// ~0.1 ms at C3 on per-row latency alone (10^6 rows of ~100 entries: row
// pointers -> entries -> warp reduction, one dependent chain per row).  Here
// the rows are sorted by length (descending) and cut into slices of 32 rows;
// a slice stores its entries column-major in pairs ([j / 2][lane][j % 2],
// 16-bit column + fp32 value, padded to the slice's longest row rounded up to
// even), so one warp = one slice, one thread = one row: every load is a
// coalesced 128 + 256 bytes (two entries of each row), there is no row
// pointer chase and no cross-lane reduction, and each x_i is the sequential
// CSR-order fmaf chain -- bitwise the sum of the unpruned wide kernels
// (spmm_rowpanel_T_kernel) and of K9t's exact re-score.  Rows longer than the
// plan's long_len (0.1% of the rows, ~1% of the entries at C3) stay in CSR:
// one warp per row loads 32 entries at a time and runs the same sequential
// chain through shuffles.  Slices are issued longest first, so the hardware
// CTA scheduler balances the skewed row lengths.
#pragma once

#include <type_traits>

#include "fsr_common.cuh"

namespace fsr {
namespace sell {

struct View {
  const int32_t* perm = nullptr;       // sorted position -> row of U~ (n)
  const int32_t* lens = nullptr;       // row length by sorted position (n)
  const int64_t* slice_ptr = nullptr;  // entry offset of slice s (n_slices + 1); long slices are empty
  const uint16_t* cols = nullptr;      // [slice][j / 2][lane][j % 2], slice widths even
  const float* vals = nullptr;
  int64_t n_long = 0;                  // sorted positions [0, n_long) are long rows (a multiple of 32)
  const uint16_t* csr_cols16 = nullptr;  // 16-bit copy of the CSR columns (long rows)
};

constexpr int kDepth = 8;

__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }
__device__ __forceinline__ unsigned short ld_stream(const uint16_t* p) { return __ldcs(p); }
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) { return __ldcs(p); }
__device__ __forceinline__ float2 ld_stream(const float2* p) { return __ldcs(p); }

// grid: ceil(n_long / 8) CTAs of long rows (a warp per row) followed by
// ceil(n_short_slices / 8) CTAs of slices (a warp per slice).
template <int DEPTH>
__global__ void __launch_bounds__(256) sell_spmv_kernel(int64_t n, int64_t n_long, int64_t long_ctas,
                                                        const int32_t* __restrict__ perm,
                                                        const int32_t* __restrict__ lens,
                                                        const int64_t* __restrict__ slice_ptr,
                                                        const uint16_t* __restrict__ cols,
                                                        const float* __restrict__ vals,
                                                        const int64_t* __restrict__ indptr,
                                                        const uint16_t* __restrict__ csr_cols,
                                                        const float* __restrict__ csr_vals,
                                                        const float* __restrict__ z, int64_t r,
                                                        float* __restrict__ x) {
  extern __shared__ __align__(16) float zs[];
  for (int64_t c = threadIdx.x; c < r; c += blockDim.x) zs[c] = z[c];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if ((int64_t)blockIdx.x < long_ctas) {
    const int64_t pos = (int64_t)blockIdx.x * 8 + warp;
    if (pos >= n_long || pos >= n) return;
    const int64_t i = perm[pos];
    const int64_t e0 = __ldg(indptr + i), e1 = __ldg(indptr + i + 1);
    float acc = 0.f;
    constexpr int U = 4;
    for (int64_t base = e0; base < e1; base += 32 * U) {
      float v[U], zz[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = base + 32 * u + lane;
        const bool ok = e < e1;
        const int c = ok ? (int)ld_stream(csr_cols + e) : 0;
        FSR_DCHECK(c < r);
        v[u] = ok ? ld_stream(csr_vals + e) : 0.f;
        zz[u] = ok ? zs[c] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cnt = (int)min((int64_t)32, e1 - (base + 32 * u));
        for (int l = 0; l < cnt; ++l)
          acc = fmaf(__shfl_sync(0xffffffffu, v[u], l), __shfl_sync(0xffffffffu, zz[u], l), acc);
      }
    }
    if (!lane) x[i] = acc;
    return;
  }
  const int64_t s = (n_long >> 5) + ((int64_t)blockIdx.x - long_ctas) * 8 + warp;
  const int64_t pos = s * 32 + lane;
  if (s * 32 >= n) return;
  const int64_t p0 = __ldg(slice_ptr + s);
  const int width = (int)((__ldg(slice_ptr + s + 1) - p0) >> 5);
  const int my_len = pos < n ? __ldg(lens + pos) : 0;
  // entries come in pairs: one 4-byte load = two columns, one 8-byte load = two
  // values of the row (12 bytes in flight per 3 registers instead of per 4)
  const uint32_t* cp = reinterpret_cast<const uint32_t*>(cols + p0) + lane;
  const float2* vp = reinterpret_cast<const float2*>(vals + p0) + lane;
  const int pairs = width >> 1;
  float acc = 0.f;
  int jp = 0;
  for (; jp + DEPTH <= pairs; jp += DEPTH) {
    uint32_t c[DEPTH];
    float2 v[DEPTH];
#pragma unroll
    for (int u = 0; u < DEPTH; ++u) {
      c[u] = ld_stream(cp + (int64_t)(jp + u) * 32);
      v[u] = ld_stream(vp + (int64_t)(jp + u) * 32);
    }
#pragma unroll
    for (int u = 0; u < DEPTH; ++u) {
      const int j = 2 * (jp + u);
      FSR_DCHECK((int)(c[u] & 0xffffu) < r && (int)(c[u] >> 16) < r);
      if (j < my_len) acc = fmaf(v[u].x, zs[c[u] & 0xffffu], acc);
      if (j + 1 < my_len) acc = fmaf(v[u].y, zs[c[u] >> 16], acc);
    }
  }
  for (; jp < pairs; ++jp) {
    const uint32_t c = ld_stream(cp + (int64_t)jp * 32);
    const float2 v = ld_stream(vp + (int64_t)jp * 32);
    if (2 * jp < my_len) acc = fmaf(v.x, zs[c & 0xffffu], acc);
    if (2 * jp + 1 < my_len) acc = fmaf(v.y, zs[c >> 16], acc);
  }
  if (pos < n) x[__ldg(perm + pos)] = acc;
}

// Small batches (2 <= b <= 64): the same layout with NB queries per pass.
// z of the pass's queries sits in shared memory as [column][NB] (one 8- or
// 16-byte read per entry), every thread keeps NB chains; grid.y = the passes.
// X is (b x n) row-major (ldx = n): x[q * ldx + row].
template <int NB, int DEPTH, int THREADS>
__global__ void __launch_bounds__(THREADS) sell_spmm_kernel(int64_t n, int64_t n_long, int64_t long_ctas,
                                                            int64_t n_groups,
                                                            const int32_t* __restrict__ perm,
                                                            const int32_t* __restrict__ lens,
                                                            const int64_t* __restrict__ slice_ptr,
                                                            const uint16_t* __restrict__ cols,
                                                            const float* __restrict__ vals,
                                                            const int64_t* __restrict__ indptr,
                                                            const uint16_t* __restrict__ csr_cols,
                                                            const float* __restrict__ csr_vals,
                                                            const float* __restrict__ Zs, int64_t r, int64_t b,
                                                            float* __restrict__ X, int64_t ldx) {
  constexpr int WARPS = THREADS / 32;
  extern __shared__ __align__(16) float zs[];  // [r][NB]
  const int64_t q0 = (int64_t)blockIdx.y * NB;
  for (int64_t t = threadIdx.x; t < r * NB; t += blockDim.x) {
    const int64_t c = t / NB, jj = t % NB;
    zs[t] = q0 + jj < b ? Zs[c * b + q0 + jj] : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  using ZV = typename std::conditional<NB == 4, float4, float2>::type;
  const ZV* zv = reinterpret_cast<const ZV*>(zs);
  // one group per CTA, or resident CTAs striding over the groups (launch_spmm_nb)
  for (int64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
  float acc[NB];
#pragma unroll
  for (int jj = 0; jj < NB; ++jj) acc[jj] = 0.f;
  if (grp < long_ctas) {
    const int64_t pos = grp * WARPS + warp;
    if (pos >= n_long || pos >= n) continue;
    const int64_t i = perm[pos];
    const int64_t e0 = __ldg(indptr + i), e1 = __ldg(indptr + i + 1);
    for (int64_t base = e0; base < e1; base += 32) {
      const int64_t e = base + lane;
      const bool ok = e < e1;
      const int c = ok ? (int)ld_stream(csr_cols + e) : 0;
      FSR_DCHECK(c < r);
      const float v = ok ? ld_stream(csr_vals + e) : 0.f;
      float zz[NB];
#pragma unroll
      for (int jj = 0; jj < NB; ++jj) zz[jj] = ok ? zs[c * NB + jj] : 0.f;
      const int cnt = (int)min((int64_t)32, e1 - base);
      for (int l = 0; l < cnt; ++l) {
        const float vv = __shfl_sync(0xffffffffu, v, l);
#pragma unroll
        for (int jj = 0; jj < NB; ++jj) acc[jj] = fmaf(vv, __shfl_sync(0xffffffffu, zz[jj], l), acc[jj]);
      }
    }
    if (!lane)
#pragma unroll
      for (int jj = 0; jj < NB; ++jj)
        if (q0 + jj < b) X[(q0 + jj) * ldx + i] = acc[jj];
    continue;
  }
  const int64_t s = (n_long >> 5) + (grp - long_ctas) * WARPS + warp;
  const int64_t pos = s * 32 + lane;
  if (s * 32 >= n) continue;
  const int64_t p0 = __ldg(slice_ptr + s);
  const int width = (int)((__ldg(slice_ptr + s + 1) - p0) >> 5);
  const int my_len = pos < n ? __ldg(lens + pos) : 0;
  const uint32_t* cp = reinterpret_cast<const uint32_t*>(cols + p0) + lane;
  const float2* vp = reinterpret_cast<const float2*>(vals + p0) + lane;
  const int pairs = width >> 1;
  auto step = [&](float vv, uint32_t cc) {
    FSR_DCHECK((int)cc < r);
    const ZV zq = zv[cc];
    const float* zf = reinterpret_cast<const float*>(&zq);
#pragma unroll
    for (int jj = 0; jj < NB; ++jj) acc[jj] = fmaf(vv, zf[jj], acc[jj]);
  };
  constexpr int DP = DEPTH / 2;  // pairs in flight
  int jp = 0;
  for (; jp + DP <= pairs; jp += DP) {
    uint32_t c[DP];
    float2 v[DP];
#pragma unroll
    for (int u = 0; u < DP; ++u) {
      c[u] = ld_stream(cp + (int64_t)(jp + u) * 32);
      v[u] = ld_stream(vp + (int64_t)(jp + u) * 32);
    }
#pragma unroll
    for (int u = 0; u < DP; ++u) {
      const int j = 2 * (jp + u);
      if (j < my_len) step(v[u].x, c[u] & 0xffffu);
      if (j + 1 < my_len) step(v[u].y, c[u] >> 16);
    }
  }
  for (; jp < pairs; ++jp) {
    const uint32_t c = ld_stream(cp + (int64_t)jp * 32);
    const float2 v = ld_stream(vp + (int64_t)jp * 32);
    if (2 * jp < my_len) step(v.x, c & 0xffffu);
    if (2 * jp + 1 < my_len) step(v.y, c >> 16);
  }
  if (pos < n) {
    const int64_t i = __ldg(perm + pos);
#pragma unroll
    for (int jj = 0; jj < NB; ++jj)
      if (q0 + jj < b) X[(q0 + jj) * ldx + i] = acc[jj];
  }
  }
}

inline bool applicable(int64_t r) { return r >= 1 && r <= 16384; }
constexpr int64_t kMaxBatch = 64;  // beyond it the wide kernels / K9t take over
// NB = 4 needs r * 16 bytes of shared memory twice per SM
inline bool batch_applicable(int64_t r, int64_t b) { return applicable(r) && b >= 2 && b <= kMaxBatch && r <= 12800; }

template <int NB, int DEPTH, int THREADS>
int launch_spmm_nb(fsr_ctx* ctx, int64_t n, const View& V, const int64_t* indptr, const float* csr_vals,
                   const float* Zs, int64_t r, int64_t b, float* X, int64_t ldx) {
  constexpr int WARPS = THREADS / 32;
  auto kern = sell_spmm_kernel<NB, DEPTH, THREADS>;
  const size_t smem = (size_t)r * NB * sizeof(float);
  FSR_TRY(fsr::ensure_smem(ctx, kern, smem));
  const int64_t long_ctas = ceil_div(std::min(V.n_long, n), WARPS);
  const int64_t short_slices = ceil_div(n, 32) - (V.n_long >> 5);
  const int64_t n_groups = long_ctas + ceil_div(std::max<int64_t>(short_slices, 0), WARPS);
  if (n_groups <= 0) return FSR_OK;
  int per_sm = 1;
  FSR_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem));
  const int64_t passes = ceil_div(b, NB);
  // up to 4 passes: a CTA per group, issued longest first (measured faster than
  // resident CTAs striding over the groups: C3 2%, b = 4: 0.228 vs 0.295 ms);
  // more passes: resident CTAs, 4 passes side by side so that they share the
  // entry stream through L2 (b = 32: 1.60 vs 1.90 ms)
  const int64_t resident = (int64_t)ctx->num_sms * std::max(per_sm, 1);
  const int64_t gx = passes <= 4 ? n_groups : std::min(n_groups, std::max<int64_t>(1, resident / 4));
  dim3 grid((unsigned)gx, (unsigned)passes);
  kern<<<grid, THREADS, smem, ctx->stream>>>(n, V.n_long, long_ctas, n_groups, V.perm, V.lens, V.slice_ptr, V.cols, V.vals,
                                             indptr, V.csr_cols16, csr_vals, Zs, r, b, X, ldx);
  return launched(ctx, "sell_spmm_kernel");
}

// X (b x n, ld = ldx) = (U~ Zs)^T for 2 <= b <= kMaxBatch; Zs is r x b.
inline int launch_spmm(fsr_ctx* ctx, int64_t n, const View& V, const int64_t* indptr, const float* csr_vals,
                       const float* Zs, int64_t r, int64_t b, float* X, int64_t ldx) {
  if (b > 2 && r <= 6400) return launch_spmm_nb<4, 16, 512>(ctx, n, V, indptr, csr_vals, Zs, r, b, X, ldx);
  return launch_spmm_nb<2, 8, 256>(ctx, n, V, indptr, csr_vals, Zs, r, b, X, ldx);
}

inline int launch_spmv(fsr_ctx* ctx, int64_t n, const View& V, const int64_t* indptr, const float* csr_vals,
                       const float* z, int64_t r, float* x) {
  const size_t smem = (size_t)r * sizeof(float);
  FSR_TRY(fsr::ensure_smem(ctx, sell_spmv_kernel<kDepth>, smem));
  const int64_t long_ctas = ceil_div(std::min(V.n_long, n), 8);
  const int64_t short_slices = ceil_div(n, 32) - (V.n_long >> 5);
  const int64_t grid = long_ctas + ceil_div(std::max<int64_t>(short_slices, 0), 8);
  if (grid <= 0) return FSR_OK;
  sell_spmv_kernel<kDepth><<<(unsigned)grid, 256, smem, ctx->stream>>>(n, V.n_long, long_ctas, V.perm, V.lens, V.slice_ptr,
                                                               V.cols, V.vals, indptr, V.csr_cols16, csr_vals, z, r,
                                                               x);
  return launched(ctx, "sell_spmv_kernel");
}

}  // namespace sell
}  // namespace fsr
