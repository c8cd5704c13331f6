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
template <typename T, int VEC, int NV>
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
    for (; j + kGatherDepth <= m; j += kGatherDepth) {
      int c[kGatherDepth];
      T a[kGatherDepth];
#pragma unroll
      for (int g = 0; g < kGatherDepth; ++g) {
        c[g] = __shfl_sync(0xffffffffu, my_col, j + g);
        a[g] = __shfl_sync(0xffffffffu, my_val, j + g);
      }
      T v[kGatherDepth][NV][VEC];
#pragma unroll
      for (int g = 0; g < kGatherDepth; ++g)
#pragma unroll
        for (int u = 0; u < NV; ++u)
          if (live[u]) load_vec<T, VEC>(X + (int64_t)c[g] * ldx + c0 + u * 32 * VEC, v[g][u]);
#pragma unroll
      for (int g = 0; g < kGatherDepth; ++g)
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

// K9 variant with a transposed output: CTA = 32 consecutive rows x one panel;
// each warp computes 4 rows, the 32 x PW tile is staged in shared memory
// (padded) and written as Y^T (ldy = n): 128-byte coalesced column segments.
template <typename T, int VEC, int NV>
__global__ void __launch_bounds__(256) spmm_rowpanel_T_kernel(int64_t n_rows, const int64_t* __restrict__ indptr,
                                                              const int32_t* __restrict__ indices,
                                                              const T* __restrict__ vals, int64_t ncols,
                                                              const T* __restrict__ X, int64_t ldx,
                                                              T* __restrict__ Yt, int64_t ldy) {
  constexpr int PW = 32 * VEC * NV;
  __shared__ T tile[32][PW + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row0 = (int64_t)blockIdx.x * 32;
  const int64_t p0 = (int64_t)blockIdx.y * PW;
  const int64_t c0 = p0 + (int64_t)lane * VEC;
  bool live[NV];
#pragma unroll
  for (int u = 0; u < NV; ++u) live[u] = c0 + u * 32 * VEC < ncols;
  for (int rr = warp; rr < 32; rr += 8) {
    const int64_t i = row0 + rr;
    T acc[NV][VEC];
#pragma unroll
    for (int u = 0; u < NV; ++u)
#pragma unroll
      for (int q = 0; q < VEC; ++q) acc[u][q] = T(0);
    if (i < n_rows)
      row_panel_accumulate<T, VEC, NV>(__ldg(indptr + i), __ldg(indptr + i + 1), indices, vals, X, ldx, c0, live,
                                       acc);
#pragma unroll
    for (int u = 0; u < NV; ++u)
#pragma unroll
      for (int q = 0; q < VEC; ++q) tile[rr][lane * VEC + u * 32 * VEC + q] = acc[u][q];
  }
  __syncthreads();
  const int64_t i = row0 + lane;
  for (int c = warp; c < PW; c += 8) {
    const int64_t col = p0 + c;
    if (col < ncols && i < n_rows) Yt[col * ldy + i] = tile[lane][c];
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
          c[u] = e < e1 ? __ldg(indices + e) : -1;
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
  for (int rr = warp; rr < 64; rr += 8) {
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
  }
  if (!TRANS) return;
  __syncthreads();
  for (int t = threadIdx.x; t < 64 * PW; t += blockDim.x) {
    const int c = t / 64, rr = t % 64;
    const int64_t i = row0 + rr;
    if (c < ncols && i < n_rows) Yt[(int64_t)c * ldy + i] = tile[rr][c];
  }
}

// SpMV with the dense vector staged in shared memory: random 4-byte gathers
// from L1 cost one wavefront per distinct 128B line (~32 per warp access);
// from shared memory they cost a few bank cycles.  Warp per row, 4 nonzeros
// per lane in flight.
template <typename T>
__global__ void __launch_bounds__(256) spmv_smem_kernel(int64_t n_rows, const int64_t* __restrict__ indptr,
                                                        const int32_t* __restrict__ indices,
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
        c[u] = e < e1 ? __ldg(indices + e) : -1;
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

template <typename T>
int launch_spmv_smem(fsr_ctx* ctx, int64_t n_rows, const int64_t* indptr, const int32_t* indices, const T* vals,
                     const T* x, int64_t x_len, T* y) {
  const size_t smem = (size_t)x_len * sizeof(T);
  static size_t configured[2] = {0, 0};
  if (configured[sizeof(T) == 8] < smem) {
    FSR_CUDA(ctx, cudaFuncSetAttribute(spmv_smem_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[sizeof(T) == 8] = smem;
  }
  // full occupancy (8 blocks x 8 warps per SM); each block re-stages x (L2 hits)
  const int grid = (int)std::min<int64_t>(ceil_div(n_rows * 32, 256), (int64_t)ctx->num_sms * 8);
  spmv_smem_kernel<T><<<grid, 256, smem, ctx->stream>>>(n_rows, indptr, indices, vals, x, x_len, y);
  return launched(ctx, "spmv_smem_kernel");
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
  if (vec_ok && ncols > 32 * VW) {
    constexpr int NV = 2, PW = 32 * VW * NV;
    dim3 grid((unsigned)ceil_div(n_rows, 32), (unsigned)ceil_div(ncols, PW));
    spmm_rowpanel_T_kernel<T, VW, NV><<<grid, block, 0, ctx->stream>>>(n_rows, indptr, indices, vals, ncols, X, ldx,
                                                                        Yt, ldy);
  } else if (vec_ok) {
    dim3 grid((unsigned)ceil_div(n_rows, 32), (unsigned)ceil_div(ncols, 32 * VW));
    spmm_rowpanel_T_kernel<T, VW, 1><<<grid, block, 0, ctx->stream>>>(n_rows, indptr, indices, vals, ncols, X, ldx,
                                                                       Yt, ldy);
  } else {
    dim3 grid((unsigned)ceil_div(n_rows, 32), (unsigned)ceil_div(ncols, 32));
    spmm_rowpanel_T_kernel<T, 1, 1><<<grid, block, 0, ctx->stream>>>(n_rows, indptr, indices, vals, ncols, X, ldx,
                                                                      Yt, ldy);
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
  // Large dense blocks: the wide panel (256 fp32 / 128 fp64 columns of all n
  // rows) would not stay L2-resident while every row gathers from it, so use
  // narrow panels (16 or 32 columns, warp per row) whose n x panel slice fits L2;
  // W is re-streamed once per panel instead.
  // Narrow row-major panels (warp per row, nonzero groups): an experiment knob
  // (FSR_K2_PANEL = 16 | 32 | 64 | 128 columns).  Measured on B200 at C3
  // (n = 1e6, r_hat = 5500): 16/32-column panels 241 ms vs 107 ms for the wide
  // kernel, which streams its gathers at ~6.5 TB/s of DRAM; the default stays wide.
  static const int k2_panel = [] {
    const char* e = getenv("FSR_K2_PANEL");
    return e ? atoi(e) : 0;
  }();
  if (k2_panel > 0 && vec_ok && ncols >= 16) {
    dim3 grid((unsigned)ceil_div(n_rows, 64), (unsigned)ceil_div(ncols, k2_panel));
    if (k2_panel == 16)
      spmm_narrow_T_kernel<T, VW, 16 / VW, false><<<grid, block, 0, ctx->stream>>>(n_rows, indptr, indices, vals, ncols,
                                                                                   X, ldx, Y, ldy);
    else if (k2_panel == 32)
      spmm_narrow_T_kernel<T, VW, 32 / VW, false><<<grid, block, 0, ctx->stream>>>(n_rows, indptr, indices, vals, ncols,
                                                                                   X, ldx, Y, ldy);
    else if (k2_panel == 64)
      spmm_narrow_T_kernel<T, VW, 64 / VW, false><<<grid, block, 0, ctx->stream>>>(n_rows, indptr, indices, vals, ncols,
                                                                                   X, ldx, Y, ldy);
    else
      spmm_narrow_T_kernel<T, VW, 32, false><<<dim3(grid.x, (unsigned)ceil_div(ncols, 32 * VW)), block, 0,
                                                ctx->stream>>>(n_rows, indptr, indices, vals, ncols, X, ldx, Y, ldy);
    return launched(ctx, "spmm_narrow_rowmajor_kernel");
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
