// K2 / K9: CSR x dense-block product, warp per (row, column panel).
//
// Reference call site: spectral.py:170 `block = A @ Q` -> sparsemat.py:63-64 ->
// scipy _sparsetools.csr_matvecs (one thread, float64, y += a*x per nonzero in
// CSR order).  On the device one warp owns one output row-panel: the row's
// (col, val) pairs are loaded 32 at a time with one coalesced load and
// broadcast by shuffle; for each nonzero the warp streams the matching row
// panel of the dense block with 16-byte vector loads (512 B per warp per
// vector for fp32).  Work items are ordered panel-major so the panel of X in
// use (n x panel_width) stays L2-resident while all rows sweep over it.
// Accumulation keeps CSR order per output element; in fp64 the product and
// sum are rounded separately, so the result is bitwise equal to scipy's.
#pragma once

#include <algorithm>
#include <cstdlib>

#include "fsr_common.cuh"

namespace fsr {

template <typename T, int VEC>
struct VecT;
template <>
struct VecT<float, 4> {
  using type = float4;
};
template <>
struct VecT<float, 2> {
  using type = float2;
};
template <>
struct VecT<float, 1> {
  using type = float;
};
template <>
struct VecT<double, 2> {
  using type = double2;
};
template <>
struct VecT<double, 1> {
  using type = double;
};

template <typename T, int VEC>
__device__ __forceinline__ void load_vec(const T* p, T (&v)[VEC]) {
  using V = typename VecT<T, VEC>::type;
  V t = __ldg(reinterpret_cast<const V*>(p));
  const T* s = reinterpret_cast<const T*>(&t);
#pragma unroll
  for (int i = 0; i < VEC; ++i) v[i] = s[i];
}

template <typename T, int VEC>
__device__ __forceinline__ void store_vec(T* p, const T (&v)[VEC]) {
  using V = typename VecT<T, VEC>::type;
  V t;
  T* d = reinterpret_cast<T*>(&t);
#pragma unroll
  for (int i = 0; i < VEC; ++i) d[i] = v[i];
  *reinterpret_cast<V*>(p) = t;
}

// acc + a*x: fp64 keeps the product and the sum separately rounded (scipy's
// sequential y += a*x, bitwise); fp32 has no bitwise target and uses FMA.
__device__ __forceinline__ double axpy1(double acc, double a, double x) { return mul_add_rn(acc, a, x); }
__device__ __forceinline__ float axpy1(float acc, float a, float x) { return fmaf(a, x, acc); }

constexpr int kGatherDepth = 4;  // dense rows gathered before their FMAs (memory-level parallelism)

// Accumulate row i of the CSR matrix against the dense panel columns
// [c0 + u*32*VEC, +VEC) (u < NV) into acc; nonzeros are consumed in CSR order.
// (Broadcasting the (column, value) pairs from shared memory instead of by
// shuffles -- 4.7% faster in the fp16 K9h, prune.cuh -- left this L2-bound
// fp32 K9 unchanged: 19.35 vs 19.34 ms at C3.)
template <typename T, int VEC, int NV, int DEPTH = kGatherDepth>
__device__ __forceinline__ void row_panel_accumulate(int64_t e0, int64_t e1, const int32_t* __restrict__ indices,
                                                     const T* __restrict__ vals, const T* __restrict__ X,
                                                     int64_t ldx, int64_t c0, const bool (&live)[NV],
                                                     T (&acc)[NV][VEC]) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = e0; base < e1; base += 32) {
    const int m = (e1 - base) < 32 ? (int)(e1 - base) : 32;
    int my_col = 0;
    T my_val = T(0);
    if (lane < m) {
      my_col = __ldg(indices + base + lane);
      my_val = __ldg(vals + base + lane);
    }
    int j = 0;
    for (; j + DEPTH <= m; j += DEPTH) {
      int c[DEPTH];
      T a[DEPTH];
#pragma unroll
      for (int g = 0; g < DEPTH; ++g) {
        c[g] = __shfl_sync(0xffffffffu, my_col, j + g);
        a[g] = __shfl_sync(0xffffffffu, my_val, j + g);
      }
      T v[DEPTH][NV][VEC];
#pragma unroll
      for (int g = 0; g < DEPTH; ++g)
#pragma unroll
        for (int u = 0; u < NV; ++u)
          if (live[u]) load_vec<T, VEC>(X + (int64_t)c[g] * ldx + c0 + u * 32 * VEC, v[g][u]);
#pragma unroll
      for (int g = 0; g < DEPTH; ++g)
#pragma unroll
        for (int u = 0; u < NV; ++u)
#pragma unroll
          for (int q = 0; q < VEC; ++q) acc[u][q] = axpy1(acc[u][q], a[g], v[g][u][q]);
    }
    for (; j < m; ++j) {
      const int c = __shfl_sync(0xffffffffu, my_col, j);
      const T a = __shfl_sync(0xffffffffu, my_val, j);
#pragma unroll
      for (int u = 0; u < NV; ++u) {
        if (live[u]) {
          T v[VEC];
          load_vec<T, VEC>(X + (int64_t)c * ldx + c0 + u * 32 * VEC, v);
#pragma unroll
          for (int q = 0; q < VEC; ++q) acc[u][q] = axpy1(acc[u][q], a, v[q]);
        }
      }
    }
  }
}

// One warp per (row, panel); panel width = 32 lanes * VEC * NV columns.
template <typename T, int VEC, int NV>
__global__ void __launch_bounds__(256) spmm_rowpanel_kernel(int64_t n_rows, const int64_t* __restrict__ indptr,
                                                            const int32_t* __restrict__ indices,
                                                            const T* __restrict__ vals, int64_t ncols,
                                                            const T* __restrict__ X, int64_t ldx,
                                                            T* __restrict__ Y, int64_t ldy, int64_t n_panels) {
  constexpr int PW = 32 * VEC * NV;
  const int lane = threadIdx.x & 31;
  const int64_t total = n_rows * n_panels;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < total; w += nwarps) {
    const int64_t p = w / n_rows;
    const int64_t i = w - p * n_rows;
    const int64_t c0 = p * PW + (int64_t)lane * VEC;
    T acc[NV][VEC];
#pragma unroll
    for (int u = 0; u < NV; ++u)
#pragma unroll
      for (int q = 0; q < VEC; ++q) acc[u][q] = T(0);
    bool live[NV];
#pragma unroll
    for (int u = 0; u < NV; ++u) live[u] = c0 + u * 32 * VEC < ncols;
    row_panel_accumulate<T, VEC, NV>(__ldg(indptr + i), __ldg(indptr + i + 1), indices, vals, X, ldx, c0, live, acc);
    T* yr = Y + i * ldy + c0;
#pragma unroll
    for (int u = 0; u < NV; ++u)
      if (live[u]) store_vec<T, VEC>(yr + u * 32 * VEC, acc[u]);
  }
}

// K9 variant with a transposed output: CTA = ROWS consecutive rows x one panel;
// warps take the rows one at a time from a shared counter, the ROWS x PW tile
// is staged in shared memory (padded) and written as Y^T (ldy = n): 128-byte
// coalesced column segments.
template <typename T, int VEC, int NV, int DEPTH = kGatherDepth, int ROWS = 32>
__global__ void __launch_bounds__(256) spmm_rowpanel_T_kernel(int64_t n_rows, const int64_t* __restrict__ indptr,
                                                              const int32_t* __restrict__ indices,
                                                              const T* __restrict__ vals, int64_t ncols,
                                                              const T* __restrict__ X, int64_t ldx,
                                                              T* __restrict__ Yt, int64_t ldy) {
  constexpr int PW = 32 * VEC * NV;
  extern __shared__ __align__(16) unsigned char dyn_tile[];
  T(*tile)[PW + 1] = reinterpret_cast<T(*)[PW + 1]>(dyn_tile);  // ROWS x (PW + 1)
  __shared__ int next_row;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row0 = (int64_t)blockIdx.x * ROWS;
  const int64_t p0 = (int64_t)blockIdx.y * PW;
  const int64_t c0 = p0 + (int64_t)lane * VEC;
  bool live[NV];
#pragma unroll
  for (int u = 0; u < NV; ++u) live[u] = c0 + u * 32 * VEC < ncols;
  // rows are handed out dynamically, longest first: U~'s row lengths are
  // skewed (median 54, max > 2000 at C3), so a static 4-rows-per-warp split
  // leaves warps idle, and short rows handed out last keep the warps'
  // finishing times close (fewer idle warps at the end-of-block barrier)
  static_assert(ROWS == 32, "one lane per row ranks the block's rows");
  __shared__ int order_s[ROWS];
  if (warp == 0) {
    const int64_t i = row0 + lane;
    const int64_t len = i < n_rows ? __ldg(indptr + i + 1) - __ldg(indptr + i) : 0;
    int rank = 0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const int64_t lk = __shfl_sync(0xffffffffu, len, k);
      rank += (lk > len) || (lk == len && k < lane);
    }
    order_s[rank] = lane;
  }
  if (threadIdx.x == 0) next_row = 8;
  __syncthreads();
  for (int pos = warp; pos < ROWS;) {
    const int rr = order_s[pos];
    const int64_t i = row0 + rr;
    T acc[NV][VEC];
#pragma unroll
    for (int u = 0; u < NV; ++u)
#pragma unroll
      for (int q = 0; q < VEC; ++q) acc[u][q] = T(0);
    if (i < n_rows)
      row_panel_accumulate<T, VEC, NV, DEPTH>(__ldg(indptr + i), __ldg(indptr + i + 1), indices, vals, X, ldx, c0,
                                              live, acc);
#pragma unroll
    for (int u = 0; u < NV; ++u)
#pragma unroll
      for (int q = 0; q < VEC; ++q) tile[rr][lane * VEC + u * 32 * VEC + q] = acc[u][q];
    int nr = 0;
    if (lane == 0) nr = atomicAdd(&next_row, 1);
    pos = __shfl_sync(0xffffffffu, nr, 0);
  }
  __syncthreads();
  for (int c = warp; c < PW; c += 8) {
    const int64_t col = p0 + c;
#pragma unroll
    for (int h = 0; h < ROWS / 32; ++h) {
      const int64_t i = row0 + h * 32 + lane;
      if (col < ncols && i < n_rows) Yt[col * ldy + i] = tile[h * 32 + lane][c];
    }
  }
}

// Single dense column (SpMV): warp per row, lanes over nonzeros, tree reduce.
template <typename T>
__global__ void __launch_bounds__(256) spmv_kernel(int64_t n_rows, const int64_t* __restrict__ indptr,
                                                   const int32_t* __restrict__ indices,
                                                   const T* __restrict__ vals, const T* __restrict__ x,
                                                   T* __restrict__ y, int64_t ldy) {
  // Half-warp per row (two rows in flight per warp), 4 nonzeros per lane per
  // iteration: the index/value streams are the HBM traffic, the gathers of x
  // hit L1/L2; short load chains keep many rows in flight per SM.
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const int64_t nhalves = ((int64_t)gridDim.x * blockDim.x) >> 4;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 4; i - half < n_rows; i += nhalves) {
    T acc = T(0);
    if (i < n_rows) {
      const int64_t e0 = __ldg(indptr + i), e1 = __ldg(indptr + i + 1);
      for (int64_t base = e0 + hl; base < e1; base += 64) {
        int c[4];
        T a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t e = base + 16 * u;
          c[u] = e < e1 ? (int)__ldg(indices + e) : -1;
          a[u] = e < e1 ? __ldg(vals + e) : T(0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c[u] >= 0) acc = axpy1(acc, a[u], __ldg(x + c[u]));
      }
    }
#pragma unroll
    for (int o = 8; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (!hl && i < n_rows) y[i * ldy] = acc;
  }
}

// Narrow dense blocks (ncols <= LPR * VEC): one warp per row (no divergence
// across rows of different lengths); the warp's lanes form 32/LPR groups of
// LPR column lanes, group g taking nonzeros g, g+G, g+2G, ... of the row; the
// G partial rows are summed by shuffles at the end.  Output Y^T (ldy = n) via
// a padded shared tile, like the wide kernel.
template <typename T, int VEC, int LPR, bool TRANS = true>
__global__ void __launch_bounds__(256) spmm_narrow_T_kernel(int64_t n_rows, const int64_t* __restrict__ indptr,
                                                            const int32_t* __restrict__ indices,
                                                            const T* __restrict__ vals, int64_t ncols,
                                                            const T* __restrict__ X, int64_t ldx,
                                                            T* __restrict__ Yt, int64_t ldy) {
  constexpr int PW = LPR * VEC;
  constexpr int G = 32 / LPR;  // nonzero groups per row
  __shared__ T tile[64][PW + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / LPR, sl = lane % LPR;
  const int64_t row0 = (int64_t)blockIdx.x * 64;
  const int64_t p0 = (int64_t)blockIdx.y * PW;  // column panel (row-major output mode)
  const int64_t c0 = p0 + (int64_t)sl * VEC;
  const bool live = c0 < ncols;
  // rows are handed out dynamically (as in the wide kernel), longest first:
  // a warp that drew short rows takes more of them instead of idling at the
  // barrier, and the rows handed out last are the short ones
  __shared__ int next_row;
  __shared__ int order_s[64];
  if (warp == 0) {
    int64_t len[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = row0 + h * 32 + lane;
      len[h] = i < n_rows ? __ldg(indptr + i + 1) - __ldg(indptr + i) : 0;
    }
    int rank[2] = {0, 0};
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const int64_t lk = __shfl_sync(0xffffffffu, len[g], k);
#pragma unroll
        for (int h = 0; h < 2; ++h) rank[h] += (lk > len[h]) || (lk == len[h] && g * 32 + k < h * 32 + lane);
      }
    order_s[rank[0]] = lane;
    order_s[rank[1]] = 32 + lane;
  }
  if (threadIdx.x == 0) next_row = 8;
  __syncthreads();
  for (int pos = warp; pos < 64;) {
    const int rr = order_s[pos];
    const int64_t i = row0 + rr;
    T acc[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) acc[q] = T(0);
    if (i < n_rows) {
      const int64_t e0 = __ldg(indptr + i), e1 = __ldg(indptr + i + 1);
      for (int64_t base = e0; base < e1; base += 32) {
        const int m = (e1 - base) < 32 ? (int)(e1 - base) : 32;
        int my_col = 0;
        T my_val = T(0);
        if (lane < m) {
          my_col = __ldg(indices + base + lane);
          my_val = __ldg(vals + base + lane);
        }
        // group grp consumes chunk entries grp, grp+G, ... (4 in flight)
        for (int j0 = 0; j0 < m; j0 += 4 * G) {
          int c[4];
          T a[4], v[4][VEC];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = j0 + u * G + grp;
            c[u] = __shfl_sync(0xffffffffu, my_col, j & 31);
            a[u] = __shfl_sync(0xffffffffu, my_val, j & 31);
            if (j >= m) a[u] = T(0), c[u] = -1;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (live && c[u] >= 0) load_vec<T, VEC>(X + (int64_t)c[u] * ldx + c0, v[u]);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c[u] >= 0)
#pragma unroll
              for (int q = 0; q < VEC; ++q) acc[q] = axpy1(acc[q], a[u], v[u][q]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < VEC; ++q)
#pragma unroll
      for (int o = LPR; o < 32; o <<= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
    if (TRANS) {
      if (grp == 0)
#pragma unroll
        for (int q = 0; q < VEC; ++q) tile[rr][sl * VEC + q] = acc[q];
    } else if (grp == 0 && live && i < n_rows) {
      store_vec<T, VEC>(Yt + i * ldy + c0, acc);  // row-major Y, this panel's columns
    }
    int nr = 0;
    if (lane == 0) nr = atomicAdd(&next_row, 1);
    pos = __shfl_sync(0xffffffffu, nr, 0);
  }
  if (!TRANS) return;
  __syncthreads();
  for (int t = threadIdx.x; t < 64 * PW; t += blockDim.x) {
    const int c = t / 64, rr = t % 64;
    const int64_t i = row0 + rr;
    if (c < ncols && i < n_rows) Yt[(int64_t)c * ldy + i] = tile[rr][c];
  }
}

// L2-resident column panels (row-major output): a group of LPR lanes owns one
// output row and VEC*LPR columns of one panel, so a warp advances 32/LPR rows
// at once with no cross-lane reduction; each group keeps DEPTH dense-row
// gathers in flight and prefetches the next DEPTH (col, val) pairs while they
// land.  Blocks are ordered panel-major (blockIdx.x = row block), so the whole
// GPU sweeps one n x PW panel of X at a time; sized to fit one die's share
// of L2, the panel is read from DRAM once and every gather after the first
// hits L2.  The CSR stream is re-read once per panel.  Accumulation keeps CSR
// order per output element (fp64: bitwise equal to scipy).
template <typename T, int VEC, int LPR, int DEPTH>
__global__ void __launch_bounds__(256) spmm_l2panel_kernel(int64_t n_rows, const int64_t* __restrict__ indptr,
                                                           const int32_t* __restrict__ indices,
                                                           const T* __restrict__ vals, int64_t ncols,
                                                           const T* __restrict__ X, int64_t ldx,
                                                           T* __restrict__ Y, int64_t ldy) {
  constexpr int G = 32 / LPR;  // rows per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / LPR, sl = lane % LPR;
  const int64_t i = ((int64_t)blockIdx.x * 8 + warp) * G + grp;
  const int64_t c0 = (int64_t)blockIdx.y * (LPR * VEC) + (int64_t)sl * VEC;
  if (i >= n_rows || c0 >= ncols) return;
  const int64_t e0 = __ldg(indptr + i), e1 = __ldg(indptr + i + 1);
  T acc[VEC];
#pragma unroll
  for (int q = 0; q < VEC; ++q) acc[q] = T(0);
  int c[DEPTH];
  T a[DEPTH];
#pragma unroll
  for (int g = 0; g < DEPTH; ++g) {
    const bool ok = e0 + g < e1;
    c[g] = ok ? __ldg(indices + e0 + g) : -1;
    a[g] = ok ? __ldg(vals + e0 + g) : T(0);
  }
  for (int64_t e = e0; e < e1; e += DEPTH) {
    T v[DEPTH][VEC];
#pragma unroll
    for (int g = 0; g < DEPTH; ++g)
      if (c[g] >= 0) load_vec<T, VEC>(X + (int64_t)c[g] * ldx + c0, v[g]);
    T an[DEPTH];
    int cn[DEPTH];
#pragma unroll
    for (int g = 0; g < DEPTH; ++g) {
      const bool ok = e + DEPTH + g < e1;
      cn[g] = ok ? __ldg(indices + e + DEPTH + g) : -1;
      an[g] = ok ? __ldg(vals + e + DEPTH + g) : T(0);
    }
#pragma unroll
    for (int g = 0; g < DEPTH; ++g)
      if (c[g] >= 0)
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = axpy1(acc[q], a[g], v[g][q]);
#pragma unroll
    for (int g = 0; g < DEPTH; ++g) {
      c[g] = cn[g];
      a[g] = an[g];
    }
  }
  store_vec<T, VEC>(Y + i * ldy + c0, acc);
}

// SpMV with the dense vector staged in shared memory: random 4-byte gathers
// from L1 cost one wavefront per distinct 128B line (~32 per warp access);
// from shared memory they cost a few bank cycles.  Warp per row, 4 nonzeros
// per lane in flight.  (Tried: a warp owning 32 consecutive rows with one
// coalesced row-pointer load and 1-4 rows in flight -- faster on uniform
// rows, but 3-25% slower on the bench's U~, whose row lengths are very
// skewed: rows of small clusters keep hundreds of entries, rows of large
// clusters few.  Grid-stride warp-per-row balances that best.  A software-
// pipelined version -- next row's pointers and first 128 entries in flight
// while the current row is summed -- measured 10-15% slower on that U~:
// 0.171/0.217/0.401 vs 0.150/0.189/0.377 ms at 1/2/5%, tools/b1_probe.py.
// A merge-style streaming SpMV -- warp per 32-row group streaming the group's
// entries in 256-entry windows of 16-byte loads, per-row sums by a thread-
// local pass plus a segmented warp scan, next window prefetched -- measured
// 0.142/0.225/0.479 ms: the per-entry row-boundary bookkeeping makes it
// issue-bound before it is HBM-bound.)
// I = int32_t (the CSR's columns) or uint16_t (a packed copy for r <= 65536:
// 6 instead of 8 bytes per entry streamed; same sums, bit for bit).
template <typename T, typename I = int32_t>
__global__ void __launch_bounds__(256) spmv_smem_kernel(int64_t n_rows, const int64_t* __restrict__ indptr,
                                                        const I* __restrict__ indices,
                                                        const T* __restrict__ vals, const T* __restrict__ x,
                                                        int64_t x_len, T* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char dyn[];
  T* xs = (T*)dyn;
  for (int64_t c = threadIdx.x; c < x_len; c += blockDim.x) xs[c] = x[c];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_rows; i += nwarps) {
    T acc = T(0);
    const int64_t e0 = __ldg(indptr + i), e1 = __ldg(indptr + i + 1);
    for (int64_t base = e0 + lane; base < e1; base += 128) {
      int c[4];
      T a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t e = base + 32 * u;
        c[u] = e < e1 ? (int)__ldg(indices + e) : -1;
        FSR_DCHECK(c[u] < x_len);
        a[u] = e < e1 ? __ldg(vals + e) : T(0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c[u] >= 0) acc = axpy1(acc, a[u], xs[c[u]]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (!lane) y[i] = acc;
  }
}

inline bool aligned(const void* p, int bytes) { return ((uintptr_t)p % bytes) == 0; }

template <typename T, typename I = int32_t>
int launch_spmv_smem(fsr_ctx* ctx, int64_t n_rows, const int64_t* indptr, const I* indices, const T* vals,
                     const T* x, int64_t x_len, T* y) {
  const size_t smem = (size_t)x_len * sizeof(T);
  FSR_TRY(fsr::ensure_smem(ctx, spmv_smem_kernel<T, I>, smem));
  // full occupancy (8 blocks x 8 warps per SM); each block re-stages x (L2 hits)
  const int grid = (int)std::min<int64_t>(ceil_div(n_rows * 32, 256), (int64_t)ctx->num_sms * 8);
  spmv_smem_kernel<T, I><<<grid, 256, smem, ctx->stream>>>(n_rows, indptr, indices, vals, x, x_len, y);
  return launched(ctx, sizeof(I) == 2 ? "spmv_smem_u16_kernel" : "spmv_smem_kernel");
}

template <typename T, int VEC, int NV, int ROWS>
int launch_rowpanel_T(fsr_ctx* ctx, int64_t n_rows, const int64_t* indptr, const int32_t* indices, const T* vals,
                      int64_t ncols, const T* X, int64_t ldx, T* Yt, int64_t ldy) {
  constexpr int PW = 32 * VEC * NV;
  const size_t smem = (size_t)ROWS * (PW + 1) * sizeof(T);
  FSR_TRY(fsr::ensure_smem(ctx, spmm_rowpanel_T_kernel<T, VEC, NV, kGatherDepth, ROWS>, smem));
  dim3 grid((unsigned)ceil_div(n_rows, ROWS), (unsigned)ceil_div(ncols, PW));
  spmm_rowpanel_T_kernel<T, VEC, NV, kGatherDepth, ROWS><<<grid, 256, smem, ctx->stream>>>(
      n_rows, indptr, indices, vals, ncols, X, ldx, Yt, ldy);
  return FSR_OK;
}

// Y^T (ncols x n_rows, ld = ldy) = A X for ncols >= 2 (online K9 output layout).
template <typename T>
int launch_spmm_T(fsr_ctx* ctx, int64_t n_rows, const int64_t* indptr, const int32_t* indices, const T* vals,
                  int64_t ncols, const T* X, int64_t ldx, T* Yt, int64_t ldy) {
  if (n_rows <= 0 || ncols <= 0) return FSR_OK;
  constexpr int VW = sizeof(T) == 4 ? 4 : 2;
  const bool vec_ok = ncols % VW == 0 && ldx % VW == 0 && aligned(X, 16);
  dim3 block(256);
  if (vec_ok && ncols <= 8 * VW) {
    dim3 grid((unsigned)ceil_div(n_rows, 64));
    spmm_narrow_T_kernel<T, VW, 8><<<grid, block, 0, ctx->stream>>>(n_rows, indptr, indices, vals, ncols, X, ldx, Yt,
                                                                     ldy);
    return launched(ctx, "spmm_narrow_T_kernel");
  }
  if (vec_ok && ncols <= 16 * VW) {
    dim3 grid((unsigned)ceil_div(n_rows, 64));
    spmm_narrow_T_kernel<T, VW, 16><<<grid, block, 0, ctx->stream>>>(n_rows, indptr, indices, vals, ncols, X, ldx,
                                                                      Yt, ldy);
    return launched(ctx, "spmm_narrow_T_kernel");
  }
  // Schedule variants measured on B200 (tools/k9_micro.py, C3 shape, b = 1024):
  // NV=2 (256 columns, 80 registers, 3 CTAs/SM) 20.9 ms; NV=1 22.2 ms; NV=1
  // depth 8 22.7 ms; NV=2 capped at 64 registers (4 CTAs/SM) 45.7 ms; NV=1 at
  // 6 CTAs/SM 30.4 ms -- all bitwise identical.  Letting NV=2 grow to 96
  // registers (2 CTAs/SM) cost 30% on the bench's U~ (skewed row lengths).
  // The kernel streams ~19.6 TB/s of L2->SM gathers.
  if (vec_ok && ncols > 32 * VW) {
    // 32-row blocks: 64-row blocks (same occupancy) measured 22.4 vs 21.0 ms at C3
    constexpr int NV = 2;
    FSR_TRY((launch_rowpanel_T<T, VW, NV, 32>(ctx, n_rows, indptr, indices, vals, ncols, X, ldx, Yt, ldy)));
  } else if (vec_ok) {
    FSR_TRY((launch_rowpanel_T<T, VW, 1, 32>(ctx, n_rows, indptr, indices, vals, ncols, X, ldx, Yt, ldy)));
  } else {
    FSR_TRY((launch_rowpanel_T<T, 1, 1, 32>(ctx, n_rows, indptr, indices, vals, ncols, X, ldx, Yt, ldy)));
  }
  return launched(ctx, "spmm_rowpanel_T_kernel");
}

template <typename T>
int launch_spmm(fsr_ctx* ctx, int64_t n_rows, const int64_t* indptr, const int32_t* indices, const T* vals,
                int64_t ncols, const T* X, int64_t ldx, T* Y, int64_t ldy) {
  if (n_rows <= 0 || ncols <= 0) return FSR_OK;
  const int block = 256;
  if (ncols == 1) {
    spmv_kernel<T><<<grid_for(n_rows * 32, block, ctx, 8), block, 0, ctx->stream>>>(n_rows, indptr, indices,
                                                                                      vals, X, Y, ldy);
    return launched(ctx, "spmv_kernel");
  }
  constexpr int VW = sizeof(T) == 4 ? 4 : 2;  // 16-byte vectors
  const bool vec_ok = ncols % VW == 0 && ldx % VW == 0 && ldy % VW == 0 && aligned(X, 16) && aligned(Y, 16);
  // L2-resident column panels (FSR_OPT_SPMM_PANEL_BYTES = 32 | 64 | 128 bytes
  // of each dense row per panel); 0 = the wide row-panel kernel below.
  // Measured on B200 (tools/spmm_micro.py, n = 1e6, k = 5500, 29 nnz/row of
  // random columns): wide 107 ms (gathers stream at 5.95 TB/s from DRAM);
  // 32/64/128-byte panels 443/236/177 ms.  Panels strided across the 22 GB
  // block touch every page on every pass (TLB reach); even a contiguous
  // panel copy (n x 8/16/32 columns) extrapolates to 145/121/129 ms, because
  // 32-128 byte gathers from L2 run at a lower request efficiency than the
  // wide kernel's DRAM stream.  So the wide kernel stays the default.
  const int panel_bytes = ctx->spmm_panel_bytes;
  if (panel_bytes > 0 && vec_ok) {
    constexpr int D = 8;
    const int lpr = panel_bytes / 16;  // 16-byte vectors per row segment
    const int64_t pw = (int64_t)lpr * VW;
    dim3 grid((unsigned)ceil_div(n_rows, 8 * (32 / lpr)), (unsigned)ceil_div(ncols, pw));
    if (lpr == 2)
      spmm_l2panel_kernel<T, VW, 2, D><<<grid, block, 0, ctx->stream>>>(n_rows, indptr, indices, vals, ncols, X, ldx,
                                                                         Y, ldy);
    else if (lpr == 4)
      spmm_l2panel_kernel<T, VW, 4, D><<<grid, block, 0, ctx->stream>>>(n_rows, indptr, indices, vals, ncols, X, ldx,
                                                                         Y, ldy);
    else
      spmm_l2panel_kernel<T, VW, 8, D><<<grid, block, 0, ctx->stream>>>(n_rows, indptr, indices, vals, ncols, X, ldx,
                                                                         Y, ldy);
    return launched(ctx, "spmm_l2panel_kernel");
  }
  if (vec_ok) {
    constexpr int NV = 2;
    constexpr int PW = 32 * VW * NV;
    if (ncols > PW / 2) {
      const int64_t panels = ceil_div(ncols, PW);
      spmm_rowpanel_kernel<T, VW, NV><<<grid_for(n_rows * panels * 32, block, ctx, 8), block, 0, ctx->stream>>>(
          n_rows, indptr, indices, vals, ncols, X, ldx, Y, ldy, panels);
    } else {
      const int64_t panels = ceil_div(ncols, 32 * VW);
      spmm_rowpanel_kernel<T, VW, 1><<<grid_for(n_rows * panels * 32, block, ctx, 8), block, 0, ctx->stream>>>(
          n_rows, indptr, indices, vals, ncols, X, ldx, Y, ldy, panels);
    }
  } else {
    const int64_t panels = ceil_div(ncols, 32);
    spmm_rowpanel_kernel<T, 1, 1><<<grid_for(n_rows * panels * 32, block, ctx, 8), block, 0, ctx->stream>>>(
        n_rows, indptr, indices, vals, ncols, X, ldx, Y, ldy, panels);
  }
  return launched(ctx, "spmm_rowpanel_kernel");
}

}  // namespace fsr
