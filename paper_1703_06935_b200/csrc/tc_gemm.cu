// Tensor-core (tcgen05, kind::tf32) dense stages of CholeskyQR2 and
// Rayleigh-Ritz for float32 blocks, FP32-accurate by 3xTF32 splitting.
//
// Reference call sites these replace (all float64 LAPACK/BLAS there):
//   spectral.py:165-169  np.linalg.qr (+ Q^T Q check)  -> Gram B^T B + Q = B R^-1
//   spectral.py:186      C = Q^T B                      -> cross product
//   spectral.py:190      U = Q V                        -> lift
//
// Precision scheme: every fp32 operand x is split into hi = x with the low 13
// mantissa bits cleared (exact in TF32) and lo = x - hi; a product uses
// hi*hi + hi*lo + lo*hi (3 tcgen05.mma per k-step), which recovers ~fp32
// accuracy.  The first CholeskyQR pass may use 1 product (its Gram only
// needs to be well enough conditioned, span(Q) is exact either way).
//
// Kernel shapes (one CTA per SM, 192 threads: warp 0 = TMA producer, warp 1 =
// tcgen05 issuer + TMEM owner, warps 2-5 = epilogue):
//  * gram: D[128 x 256] = sum over rows of A[r, i] B[r, j]; both operands are
//    row-major n x k blocks, i.e. MN-major for the MMA.  The K loop runs over
//    a split of the rows; fp32 TMEM accumulators are flushed into fp64 every
//    `flush_iters` k-iterations (double-buffered TMEM, 2 x 256 columns) so the
//    long reduction over n rows keeps fp64 accuracy.  Symmetric Grams skip
//    tiles strictly below the diagonal.  Per-split fp64 partials are reduced
//    in fixed order: deterministic.
//  * apply: Out[128 x N] = A[rows, :] M[:, cols] with A K-major (row-major
//    n x K) and the small M (K x N2) MN-major.
// Operands are staged by TMA (SWIZZLE_128B boxes of 32 fp32 x rows) through
// an mbarrier ring; tcgen05.commit releases stages and hands accumulators to
// the epilogue.
#include <cuda.h>

#include <algorithm>
#include <mutex>

#include "fsr_common.cuh"
#include "tc_common.cuh"

namespace {

using namespace fsr::tc;

constexpr int kThreads = 192;

// ------------------------------------------------------------------ split --
// hi/lo (fp32, ld_out) from a row-major (or column-major if col_major) source.
template <typename Tin>
__global__ void split_tf32_kernel(int64_t rows, int64_t cols, const Tin* __restrict__ in, int64_t ld_in,
                                  int col_major, float* __restrict__ hi, float* __restrict__ lo, int64_t ld_out,
                                  int64_t pad_cols) {
  const int64_t total = rows * pad_cols;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = f / pad_cols, j = f - i * pad_cols;
    float h = 0.f, l = 0.f;
    if (j < cols) {
      const Tin x = col_major ? in[j * ld_in + i] : in[i * ld_in + j];
      const float xf = (float)x;
      h = __uint_as_float(__float_as_uint(xf) & 0xFFFFE000u);
      l = (float)(x - (Tin)h);
    }
    hi[i * ld_out + j] = h;
    if (lo) lo[i * ld_out + j] = l;
  }
}

// --------------------------------------------------------------- gram/cross --
template <int NPROD, int BK, int STAGES>
struct GramCfg {
  static constexpr int A_BYTES = 4 * BK * 128;  // 128 (M) x BK rows of fp32
  static constexpr int B_BYTES = 8 * BK * 128;  // 256 (N) x BK
  static constexpr int STAGE_BYTES = (NPROD == 1 ? 1 : 2) * (A_BYTES + B_BYTES);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int NPROD, int BK, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gram_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                   const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl, int64_t n,
                   int ka, int kb, int tiles_n, int64_t rows_per_split, int flush_iters, double* __restrict__ P,
                   int symmetric) {
  using Cfg = GramCfg<NPROD, BK, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int ti = blockIdx.x / tiles_n, tj = blockIdx.x % tiles_n;
  const int i0 = ti * 128, j0 = tj * 256;
  if (symmetric && j0 + 255 < i0) return;  // tile strictly below the diagonal: mirrored later
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = min(n, r0 + rows_per_split);
  const int iters = r1 > r0 ? (int)((r1 - r0 + BK - 1) / BK) : 0;
  const int nchunks = (iters + flush_iters - 1) / flush_iters;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mAh);
    tma_prefetch(&mBh);
    if (NPROD == 3) {
      tma_prefetch(&mAl);
      tma_prefetch(&mBl);
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    for (int it = 0; it < iters; ++it) {
      const int s = it % STAGES;
      mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
      if (lane == 0) {
        uint8_t* st = smem + s * Cfg::STAGE_BYTES;
        mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
        const int row = (int)(r0 + (int64_t)it * BK);
#pragma unroll
        for (int mb = 0; mb < 4; ++mb) tma_load_2d(st + mb * BK * 128, &mAh, &full[s], i0 + 32 * mb, row);
#pragma unroll
        for (int nb = 0; nb < 8; ++nb)
          tma_load_2d(st + Cfg::A_BYTES + nb * BK * 128, &mBh, &full[s], j0 + 32 * nb, row);
        if (NPROD == 3) {
          uint8_t* lo = st + Cfg::A_BYTES + Cfg::B_BYTES;
#pragma unroll
          for (int mb = 0; mb < 4; ++mb) tma_load_2d(lo + mb * BK * 128, &mAl, &full[s], i0 + 32 * mb, row);
#pragma unroll
          for (int nb = 0; nb < 8; ++nb)
            tma_load_2d(lo + Cfg::A_BYTES + nb * BK * 128, &mBl, &full[s], j0 + 32 * nb, row);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- tcgen05 issuer
    constexpr uint32_t idesc = idesc_tf32(128, 256, true, true);
    for (int it = 0; it < iters; ++it) {
      const int c = it / flush_iters, buf = c & 1;
      const bool first = (it % flush_iters) == 0;
      if (first) {
        mbar_wait(&tempty[buf], ((c >> 1) & 1) ^ 1);
        tc_fence_after();
      }
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t base = smem_u32(smem + s * Cfg::STAGE_BYTES);
        const uint32_t aH = base, bH = base + Cfg::A_BYTES;
        const uint32_t aL = base + Cfg::A_BYTES + Cfg::B_BYTES, bL = aL + Cfg::A_BYTES;
        const uint32_t d = tmem + buf * 256;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint64_t ad = smem_desc_sw128(aH + ks * 1024, BK * 128, 1024);
          const uint64_t bd = smem_desc_sw128(bH + ks * 1024, BK * 128, 1024);
          mma_tf32(d, ad, bd, idesc, (first && ks == 0) ? 0u : 1u);
          if (NPROD == 3) {
            mma_tf32(d, ad, smem_desc_sw128(bL + ks * 1024, BK * 128, 1024), idesc, 1u);
            mma_tf32(d, smem_desc_sw128(aL + ks * 1024, BK * 128, 1024), bd, idesc, 1u);
          }
        }
        mma_commit(&empty[s]);
        if ((it % flush_iters) == flush_iters - 1 || it == iters - 1) mma_commit(&tfull[buf]);
      }
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: TMEM fp32 -> fp64 partial in global memory
    const int q = warp & 3;
    const int row = i0 + 32 * q + lane;
    double* prow = P + ((int64_t)blockIdx.y * ka + row) * (int64_t)kb;
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1;
      mbar_wait(&tfull[buf], (c >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < 8; ++cc) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + buf * 256 + cc * 32, v);
        if (row < ka) {
          const int cbase = j0 + cc * 32;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            if (cbase + t < kb) prow[cbase + t] = (c == 0 ? 0.0 : prow[cbase + t]) + (double)v[t];
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[buf]);
    }
    if (nchunks == 0 && row < ka)
      for (int t = j0; t < min(kb, j0 + 256); ++t) prow[t] = 0.0;
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// C (ka x kb row-major fp64) (+)= sum_s P[s]; symmetric: mirror the upper part.
__global__ void gram_reduce_kernel(int ka, int kb, int splits, const double* __restrict__ P, double* __restrict__ C,
                                   int accumulate, int symmetric) {
  const int64_t total = (int64_t)ka * kb;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = f / kb, j = f - i * kb;
    int64_t src = f;
    if (symmetric && i > j) src = j * kb + i;
    double s = 0.0;
    for (int p = 0; p < splits; ++p) s += P[(int64_t)p * total + src];
    C[f] = accumulate ? C[f] + s : s;
  }
}

// ---------------------------------------------------------------- apply ----
template <int N, int STAGES>
struct ApplyCfg {
  static constexpr int BK = 32;
  static constexpr int A_BYTES = 128 * 128;          // 128 rows x 32 fp32 (K-major)
  static constexpr int B_BYTES = (N / 32) * BK * 128;  // N x 32 K-rows (MN-major)
  static constexpr int STAGE_BYTES = 2 * (A_BYTES + B_BYTES);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int N, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    tc_apply_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                    const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl, int64_t n,
                    int K, int N2, float* __restrict__ Out, int64_t ldo) {
  using Cfg = ApplyCfg<N, STAGES>;
  constexpr int BK = Cfg::BK;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = (uint32_t*)(tfull + 1);

  const int n0 = blockIdx.x * N;
  const int m0 = blockIdx.y * 128;
  const int iters = (K + BK - 1) / BK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mAh);
    tma_prefetch(&mAl);
    tma_prefetch(&mBh);
    tma_prefetch(&mBl);
  }
  constexpr uint32_t kCols = N < 32 ? 32 : N;
  if (warp == 1) tmem_alloc(tmem_slot, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % STAGES;
      mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
      if (lane == 0) {
        uint8_t* st = smem + s * Cfg::STAGE_BYTES;
        mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
        const int kk = it * BK;
        tma_load_2d(st, &mAh, &full[s], kk, m0);
        tma_load_2d(st + Cfg::A_BYTES, &mAl, &full[s], kk, m0);
        uint8_t* b = st + 2 * Cfg::A_BYTES;
#pragma unroll
        for (int nb = 0; nb < N / 32; ++nb) {
          tma_load_2d(b + nb * BK * 128, &mBh, &full[s], n0 + 32 * nb, kk);
          tma_load_2d(b + Cfg::B_BYTES + nb * BK * 128, &mBl, &full[s], n0 + 32 * nb, kk);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_tf32(128, N, false, true);
    for (int it = 0; it < iters; ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t base = smem_u32(smem + s * Cfg::STAGE_BYTES);
        const uint32_t aH = base, aL = base + Cfg::A_BYTES;
        const uint32_t bH = base + 2 * Cfg::A_BYTES, bL = bH + Cfg::B_BYTES;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {
          const uint64_t adh = smem_desc_sw128(aH + ks * 32, 16, 1024);
          const uint64_t adl = smem_desc_sw128(aL + ks * 32, 16, 1024);
          const uint64_t bdh = smem_desc_sw128(bH + ks * 1024, BK * 128, 1024);
          const uint64_t bdl = smem_desc_sw128(bL + ks * 1024, BK * 128, 1024);
          mma_tf32(tmem, adh, bdh, idesc, (it == 0 && ks == 0) ? 0u : 1u);
          mma_tf32(tmem, adh, bdl, idesc, 1u);
          mma_tf32(tmem, adl, bdh, idesc, 1u);
        }
        mma_commit(&empty[s]);
        if (it == iters - 1) mma_commit(&tfull[0]);
      }
      __syncwarp();
    }
  } else {
    const int q = warp & 3;
    const int64_t row = (int64_t)m0 + 32 * q + lane;
    mbar_wait(&tfull[0], 0);
    tc_fence_after();
    float* orow = Out + row * ldo;
#pragma unroll 1
    for (int cc = 0; cc < N / 32; ++cc) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + cc * 32, v);
      const int cbase = n0 + cc * 32;
      if (row < n) {
        if (cbase + 32 <= N2 && (ldo % 4) == 0 && (((uintptr_t)orow) % 16) == 0) {
#pragma unroll
          for (int t = 0; t < 32; t += 4)
            *reinterpret_cast<float4*>(orow + cbase + t) = make_float4(v[t], v[t + 1], v[t + 2], v[t + 3]);
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t)
            if (cbase + t < N2) orow[cbase + t] = v[t];
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kCols);
  }
}

// ------------------------------------------------------------ host side ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  return fn;
}

// 2-D fp32 map over a row-major (rows x cols, ld) block; box = 32 columns x box_rows.
int make_map(fsr_ctx* ctx, CUtensorMap* m, const float* base, int64_t rows, int64_t cols, int64_t ld,
             int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fsr::set_error(ctx, FSR_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fsr::set_error(ctx, FSR_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return FSR_OK;
}

inline int64_t pad4(int64_t x) { return (x + 3) / 4 * 4; }

template <typename Tin>
int split(fsr_ctx* ctx, int64_t rows, int64_t cols, const Tin* in, int64_t ld_in, int col_major, float* hi,
          float* lo, int64_t ld_out) {
  const int64_t total = rows * ld_out;
  split_tf32_kernel<Tin><<<fsr::grid_for(total, 256, ctx, 16), 256, 0, ctx->stream>>>(rows, cols, in, ld_in,
                                                                                       col_major, hi, lo, ld_out,
                                                                                       ld_out);
  return fsr::launched(ctx, "split_tf32_kernel");
}

template <typename K>
int set_smem(fsr_ctx* ctx, K kernel, int bytes) {
  FSR_CUDA(ctx, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return FSR_OK;
}

constexpr size_t kChunkBudget = (size_t)6 << 30;  // bytes of hi/lo staging per row chunk

}  // namespace

namespace fsr {

// C (ka x kb, fp64 row-major) (+)= A^T B over n rows of fp32 row-major blocks.
int tc_gram(fsr_ctx* ctx, int64_t n, int64_t ka, const float* A, int64_t lda, int64_t kb, const float* B,
            int64_t ldb, double* C, int accumulate, int nprod, int symmetric) {
  const bool same = (A == B) && lda == ldb && ka == kb;
  const int64_t pa = pad4(ka), pb = pad4(kb);
  const int64_t per_row = (nprod == 3 ? 2 : 1) * 4 * (pa + (same ? 0 : pb));
  int64_t chunk = std::max<int64_t>(256, std::min<int64_t>(n, (int64_t)(kChunkBudget / per_row)));
  const int tiles_m = (int)ceil_div(ka, 128), tiles_n = (int)ceil_div(kb, 256);
  int tiles_eff = 0;
  for (int ti = 0; ti < tiles_m; ++ti)
    for (int tj = 0; tj < tiles_n; ++tj) tiles_eff += !(symmetric && tj * 256 + 255 < ti * 128);
  const int bk = nprod == 3 ? 16 : 32;
  int splits = (int)std::max<int64_t>(1, ceil_div(2 * ctx->num_sms, tiles_eff));
  splits = (int)std::min<int64_t>(splits, std::max<int64_t>(1, ceil_div(chunk, 64 * bk)));
  const size_t stage_bytes = (size_t)chunk * per_row;
  const size_t p_bytes = (size_t)splits * ka * kb * 8;
  void* buf = nullptr;
  FSR_TRY(scratch(ctx, stage_bytes + p_bytes + 4096, &buf));
  double* P = (double*)buf;
  float* ah = (float*)((char*)buf + ((p_bytes + 1023) / 1024) * 1024);
  float* al = nprod == 3 ? ah + chunk * pa : nullptr;
  float* bh = same ? ah : (nprod == 3 ? al : ah) + chunk * pa;
  float* bl = same ? al : (nprod == 3 ? bh + chunk * pb : nullptr);
  const int flush_iters = nprod == 3 ? 2048 / bk : 4096 / bk;
  static bool attr_done[2] = {false, false};
  for (int64_t s0 = 0; s0 < n; s0 += chunk) {
    const int64_t rows = std::min(chunk, n - s0);
    FSR_TRY(split<float>(ctx, rows, ka, A + s0 * lda, lda, 0, ah, al, pa));
    if (!same) FSR_TRY(split<float>(ctx, rows, kb, B + s0 * ldb, ldb, 0, bh, bl, pb));
    CUtensorMap mAh, mAl, mBh, mBl;
    FSR_TRY(make_map(ctx, &mAh, ah, rows, ka, pa, bk));
    FSR_TRY(make_map(ctx, &mBh, bh, rows, kb, pb, bk));
    if (nprod == 3) {
      FSR_TRY(make_map(ctx, &mAl, al, rows, ka, pa, bk));
      FSR_TRY(make_map(ctx, &mBl, bl, rows, kb, pb, bk));
    } else {
      mAl = mAh;
      mBl = mBh;
    }
    const int64_t rps = ceil_div(rows, splits);
    dim3 grid((unsigned)(tiles_m * tiles_n), (unsigned)ceil_div(rows, rps));
    if (nprod == 3) {
      using Cfg = GramCfg<3, 16, 4>;
      if (!attr_done[0]) {
        FSR_TRY(set_smem(ctx, tc_gram_kernel<3, 16, 4>, Cfg::SMEM));
        attr_done[0] = true;
      }
      tc_gram_kernel<3, 16, 4><<<grid, kThreads, Cfg::SMEM, ctx->stream>>>(
          mAh, mAl, mBh, mBl, rows, (int)ka, (int)kb, tiles_n, rps, flush_iters, P, symmetric);
    } else {
      using Cfg = GramCfg<1, 32, 4>;
      if (!attr_done[1]) {
        FSR_TRY(set_smem(ctx, tc_gram_kernel<1, 32, 4>, Cfg::SMEM));
        attr_done[1] = true;
      }
      tc_gram_kernel<1, 32, 4><<<grid, kThreads, Cfg::SMEM, ctx->stream>>>(
          mAh, mAl, mBh, mBl, rows, (int)ka, (int)kb, tiles_n, rps, flush_iters, P, symmetric);
    }
    FSR_TRY(launched(ctx, "tc_gram_kernel"));
    const int acc = (s0 > 0) || accumulate;
    gram_reduce_kernel<<<grid_for(ka * kb, 256, ctx, 8), 256, 0, ctx->stream>>>(
        (int)ka, (int)kb, (int)grid.y, P, C, acc, symmetric);
    FSR_TRY(launched(ctx, "gram_reduce_kernel"));
  }
  return FSR_OK;
}

// Out (n x N2 fp32) = A (n x K fp32) * M (K x N2, fp64; column-major if m_col_major).
int tc_apply(fsr_ctx* ctx, int64_t n, int64_t K, const float* A, int64_t lda, int64_t N2, const double* M,
             int64_t ldm, int m_col_major, float* Out, int64_t ldo) {
  const int64_t pk = pad4(K), pn = pad4(N2);
  const size_t m_bytes = (size_t)2 * K * pn * 4;
  const int64_t per_row = 2 * 4 * pk;
  int64_t chunk = std::max<int64_t>(128, std::min<int64_t>(n, (int64_t)(kChunkBudget / per_row)));
  chunk = (chunk + 127) / 128 * 128;
  void* buf = nullptr;
  FSR_TRY(scratch(ctx, m_bytes + (size_t)chunk * per_row + 4096, &buf));
  float* mh = (float*)buf;
  float* ml = mh + K * pn;
  float* ah = (float*)((char*)buf + ((m_bytes + 1023) / 1024) * 1024);
  float* al = ah + chunk * pk;
  FSR_TRY(split<double>(ctx, K, N2, M, ldm, m_col_major, mh, ml, pn));
  CUtensorMap mBh, mBl;
  FSR_TRY(make_map(ctx, &mBh, mh, K, N2, pn, 32));
  FSR_TRY(make_map(ctx, &mBl, ml, K, N2, pn, 32));
  constexpr int N = 256, STAGES = 2;
  using Cfg = ApplyCfg<N, STAGES>;
  static bool attr_done = false;
  if (!attr_done) {
    FSR_TRY(set_smem(ctx, tc_apply_kernel<N, STAGES>, Cfg::SMEM));
    attr_done = true;
  }
  for (int64_t s0 = 0; s0 < n; s0 += chunk) {
    const int64_t rows = std::min(chunk, n - s0);
    FSR_TRY(split<float>(ctx, rows, K, A + s0 * lda, lda, 0, ah, al, pk));
    CUtensorMap mAh, mAl;
    FSR_TRY(make_map(ctx, &mAh, ah, rows, K, pk, 128));
    FSR_TRY(make_map(ctx, &mAl, al, rows, K, pk, 128));
    dim3 grid((unsigned)ceil_div(N2, N), (unsigned)ceil_div(rows, 128));
    tc_apply_kernel<N, STAGES><<<grid, kThreads, Cfg::SMEM, ctx->stream>>>(mAh, mAl, mBh, mBl, rows, (int)K,
                                                                           (int)N2, Out + s0 * ldo, ldo);
    FSR_TRY(launched(ctx, "tc_apply_kernel"));
  }
  return FSR_OK;
}

}  // namespace fsr
