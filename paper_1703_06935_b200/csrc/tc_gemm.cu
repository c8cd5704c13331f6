// Tensor-core (tcgen05, kind::i8) dense stages of CholeskyQR2 and
// Rayleigh-Ritz for float32 blocks: an Ozaki-style fixed-point splitting with
// EXACT int32 accumulation.
//
// Reference call sites these replace (all float64 LAPACK/BLAS there):
//   spectral.py:165-169  np.linalg.qr (+ Q^T Q check)  -> Gram B^T B + Q = B R^-1
//   spectral.py:186      C = Q^T B                      -> cross product
//   spectral.py:190      U = Q V                        -> lift
//
// Why int8 and not 3xTF32: the sm_100 tensor-core fp32 accumulator truncates
// on every accumulation (measured: relative error -2^-24 per MMA step, linear
// in K; tools/tc_debug.cu), so a 1e6-row Gram cannot reach fp32 accuracy with
// fp32 accumulation.  Integer accumulation is exact.
//
// Scheme: for a reduction over index r, every value x of an operand gets an
// exponent e shared along r (per column of a Gram operand, per row of the big
// apply operand, per column of the small matrix) with |x| < 2^e, and is written
// as x = 2^(e-6) (s1 + s2/2^7 + s3/2^14 + s4/2^21 + eps), s_t = rint slices in
// [-64, 64] (int8), |eps| <= 2^-22: 28 bits of fixed point below 2^e, rounding
// unbiased.  A product keeps the 10 slice pairs with level t+u <= 3 (0-based),
// each level summed in its own int32 TMEM accumulator (|term| <= 2^12 and at
// most 4 terms per level, so int32 is exact for K <= 2^17); the epilogue forms
// 2^(e+e'-12) sum_l L_l / 2^(7 l) in fp64.  21 bits (3 slices) were measured
// NOT to be fp32-accurate on incoherent sums (C1 ranking vectors ~1e-4 vs
// 9e-7 for cuBLAS fp32; tools/precision_probe.py).
// LEVELS = 1 (one 7-bit slice, one product) serves the first CholeskyQR pass,
// whose R only preconditions (span(B R^-1) = span(B) for any R).
//
// Kernel (one CTA per SM, 192 threads: warp 0 = TMA producer, warp 1 = MMA
// issuer + TMEM owner, warps 2-5 = epilogue): D[128 x N] over a K range, both
// operands K-major int8 slice planes staged by TMA (SWIZZLE_64B, 64 bytes of K
// per row per stage) through an mbarrier ring; tcgen05.commit frees stages and
// hands the accumulators to the epilogue.  Gram mode writes a per-split fp64
// partial (reduced later in fixed order: deterministic); apply mode writes
// fp32 output rows.
#include <cuda.h>

#include <algorithm>
#include <mutex>

#include "fsr_common.cuh"
#include "tc_common.cuh"

namespace {

using namespace fsr::tc;

constexpr int kThreads = 192;
// K bytes (int8 elements) per stage = one 64B swizzle atom.  Measured
// alternative (tools/dense_micro.py, C3 shapes): 32-byte stages (SWIZZLE_32B)
// with twice the stages were 20-30% slower on every dense stage.
constexpr int kBK = 64;
constexpr int kSlices = 4;         // slice planes produced
constexpr int64_t kMaxK = 65536;   // reduction length per launch (int32-exact bound: 131072)
// column tiles per L2-resident group in the apply raster.  Measured at C3
// (k = 5500): 4 .. 43 all within 3% (apply 239-246 ms) although DRAM reads
// differ ~5x: the int8 MMA stream runs at the board power limit (ncu: Gram
// 94% tensor-busy at 1.55 GHz, apply 74% at 1.85 GHz), not at a feed limit.
constexpr int kApplyGroup = 32;

// --------------------------------------------------------------- exponents --
__device__ __forceinline__ int exp_above(double m) {
  // smallest e with m < 2^e (m >= 0); zero vectors get 0
  if (!(m > 0.0)) return 0;
  int e;
  frexp(m, &e);  // m = f 2^e, f in [0.5, 1)
  return e;
}

template <typename T>
__global__ void exp_of_cols_kernel(int64_t rows, int64_t cols, const T* __restrict__ A, int64_t lda,
                                   int* __restrict__ e) {
  // block (32 x 8): 32 columns, rows strided; max reduce then atomicMax on the exponent
  __shared__ double sm[8][33];
  const int64_t c = (int64_t)blockIdx.x * 32 + threadIdx.x;
  double m = 0.0;
  if (c < cols)
    for (int64_t r = (int64_t)blockIdx.y * 8 + threadIdx.y; r < rows; r += (int64_t)gridDim.y * 8)
      m = fmax(m, fabs((double)A[r * lda + c]));
  sm[threadIdx.y][threadIdx.x] = m;
  __syncthreads();
  if (threadIdx.y == 0 && c < cols) {
    for (int t = 1; t < 8; ++t) m = fmax(m, sm[t][threadIdx.x]);
    atomicMax(&e[c], exp_above(m) + 2048);  // biased so the initial 0 never wins
  }
}

// per "row" exponent of a logical rows x cols matrix read row-major (or transposed)
template <typename T>
__global__ void exp_of_rows_kernel(int64_t rows, int64_t cols, const T* __restrict__ A, int64_t lda, int transposed,
                                   int* __restrict__ e) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nwarps) {
    double m = 0.0;
    for (int64_t c = lane; c < cols; c += 32) m = fmax(m, fabs((double)(transposed ? A[c * lda + r] : A[r * lda + c])));
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (!lane) e[r] = exp_above(m) + 2048;
  }
}

__device__ __forceinline__ void slice4(double x, int e, int8_t (&s)[kSlices]) {
  double y = ldexp(x, 6 - e);  // |y| < 64
#pragma unroll
  for (int t = 0; t < kSlices; ++t) {
    const double a = rint(y);
    s[t] = (int8_t)a;
    y = (y - a) * 128.0;
  }
}

__device__ __forceinline__ uint32_t pack4(int8_t a, int8_t b, int8_t c, int8_t d) {
  return (uint32_t)(uint8_t)a | ((uint32_t)(uint8_t)b << 8) | ((uint32_t)(uint8_t)c << 16) |
         ((uint32_t)(uint8_t)d << 24);
}

// Gram operand: a 128-row x 32-column tile is read coalesced, transposed
// through shared memory, and every thread emits 16 consecutive rows of one
// column as one 16-byte store per slice plane.  Output plane p: cols x ld_out
// int8, the rows (reduction index) contiguous (K-major for the MMA).
// Requires ld_out % 16 == 0; rows beyond `rows` become zero slices.
__global__ void __launch_bounds__(256) slice_T_packed_kernel(int64_t rows, int64_t cols, const float* __restrict__ in,
                                                             int64_t ld_in, const int* __restrict__ ecol,
                                                             int8_t* __restrict__ S, int64_t ld_out) {
  __shared__ float tile[32][129];
  // column blocks vary fastest: neighbouring CTAs read neighbouring 128-byte
  // segments of the same rows (DRAM row locality; the other order measured
  // ~1 ms per 65536-row chunk at k = 5500, 2.8 TB/s)
  const int64_t r0 = (int64_t)blockIdx.y * 128, c0 = (int64_t)blockIdx.x * 32;
#pragma unroll 4
  for (int k = 0; k < 16; ++k) {
    const int idx = threadIdx.x + k * 256;
    const int r = idx >> 5, c = idx & 31;
    const int64_t gr = r0 + r, gc = c0 + c;
    tile[c][r] = (gr < rows && gc < cols) ? __ldg(in + gr * ld_in + gc) : 0.f;
  }
  __syncthreads();
  const int c = threadIdx.x >> 3, g = threadIdx.x & 7;
  const int64_t gc = c0 + c;
  const int64_t gr = r0 + 16 * g;
  if (gc >= cols || gr >= ld_out) return;
  const int e = ecol[gc] - 2048;
  uint32_t w[kSlices][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int8_t s[4][kSlices];
#pragma unroll
    for (int u = 0; u < 4; ++u) slice4((double)tile[c][16 * g + 4 * q + u], e, s[u]);
#pragma unroll
    for (int p = 0; p < kSlices; ++p) w[p][q] = pack4(s[0][p], s[1][p], s[2][p], s[3][p]);
  }
  const int64_t plane = cols * ld_out;
#pragma unroll
  for (int p = 0; p < kSlices; ++p)
    *reinterpret_cast<uint4*>(S + p * plane + gc * ld_out + gr) = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
}

// Apply operand, fused: warp per row, pass 1 finds the row exponent, pass 2
// (row still in L1/L2) slices four values per lane into packed 4-byte stores.
// Requires ld_out % 4 == 0; columns in [cols, ld_out) are zero slices.
__global__ void __launch_bounds__(256) slice_rows_fused_kernel(int64_t rows, int64_t cols, const float* __restrict__ in,
                                                               int64_t ld_in, int* __restrict__ erow,
                                                               int8_t* __restrict__ S, int64_t ld_out) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t plane = rows * ld_out;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nwarps) {
    const float* row = in + r * ld_in;
    float m = 0.f;
    for (int64_t c = lane; c < cols; c += 32) m = fmaxf(m, fabsf(row[c]));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const int e = exp_above((double)m);
    if (!lane) erow[r] = e + 2048;
    for (int64_t c = 4 * lane; c < ld_out; c += 128) {
      int8_t s[4][kSlices];
#pragma unroll
      for (int u = 0; u < 4; ++u) slice4((double)((c + u < cols) ? row[c + u] : 0.f), e, s[u]);
#pragma unroll
      for (int p = 0; p < kSlices; ++p)
        *reinterpret_cast<uint32_t*>(S + p * plane + r * ld_out + c) = pack4(s[0][p], s[1][p], s[2][p], s[3][p]);
    }
  }
}

// Small operands (the r_hat x r_hat / r_hat x r matrices, fp64): logical rows x
// cols read row-major or transposed, per-row exponent, planes rows x ld_out.
template <typename T>
__global__ void slice_rows_kernel(int64_t rows, int64_t cols, const T* __restrict__ in, int64_t ld_in, int transposed,
                                  const int* __restrict__ erow, int8_t* __restrict__ S, int64_t ld_out) {
  const int64_t total = rows * ld_out, plane = rows * ld_out;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = f / ld_out, c = f - r * ld_out;
    int8_t s[kSlices] = {0, 0, 0, 0};
    if (c < cols) slice4((double)(transposed ? in[c * ld_in + r] : in[r * ld_in + c]), erow[r] - 2048, s);
#pragma unroll
    for (int p = 0; p < kSlices; ++p) S[p * plane + f] = s[p];
  }
}

// ------------------------------------------------------------------ kernel --
template <int N, int STAGES, int LEVELS, int BPL, int BK>
struct OzCfg {
  static constexpr int APLANES = LEVELS;    // level l needs A slices 0..l
  static constexpr int BPLANES = BPL;       // B slices kept (1: B is a 7-bit matrix)
  static constexpr int A_PLANE = 128 * BK;  // 128 rows x BK K bytes
  static constexpr int B_PLANE = N * BK;
  static constexpr int STAGE_BYTES = APLANES * A_PLANE + BPLANES * B_PLANE;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 512;  // alignment slack + barriers
  static constexpr uint32_t TMEM_COLS = LEVELS * N <= 128 ? 128 : (LEVELS * N <= 256 ? 256 : 512);
  static_assert(LEVELS * N <= 512, "accumulators exceed TMEM");
  static_assert(SMEM <= 227 * 1024, "stages exceed shared memory");
};

// kind::i8, signed x signed, s32 accumulate, both K-major
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// K-major swizzled matrix descriptor: 8-row x BK-byte atoms (SBO = 8 * BK),
// SWIZZLE_64B for BK = 64, SWIZZLE_32B for BK = 32.
template <int BK>
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr) {
  static_assert(BK == 64 || BK == 32, "one swizzle atom of K per stage");
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;                // LBO (ignored for swizzled K-major) = 16 B
  d |= (uint64_t)((8 * BK) >> 4) << 32;  // SBO
  d |= (uint64_t)1 << 46;                // descriptor version (sm_100)
  d |= (uint64_t)(BK == 64 ? 4 : 6) << 61;
  return d;
}

// x * 2^k: an exact multiply by a constructed power of two in the normal
// range, ldexp (with its range handling) otherwise
__device__ __forceinline__ double scale_pow2(double x, int k) {
  if (k >= -1022 && k <= 1023) return x * __hiloint2double((k + 1023) << 20, 0);
  return ldexp(x, k);
}

__device__ __forceinline__ void tmem_ld32_i(uint32_t taddr, int (&v)[32]) {
  float f[32];
  tmem_ld32(taddr, f);
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __float_as_int(f[i]);
}

// MODE 0 (Gram/cross): D[i, j] over K rows [k_begin, k_end) of the split, A
//   rows = output rows i (ka of them), B rows = output cols j; result written
//   to the fp64 partial P[split] (ka x kb).
// MODE 1 (apply): D[r, j] = sum_K A[r, :] B[j, :] over the full K; fp32 out.
template <int MODE, int N, int STAGES, int LEVELS, int BPL, bool WIDE, int BK>
__global__ void __launch_bounds__(kThreads, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, int rowsA,
                   int rowsB, int64_t planeA_rows, int64_t planeB_rows, int64_t K, int tiles_n, int64_t k_per_split,
                   const int* __restrict__ eA, const int* __restrict__ eB, int symmetric, double* __restrict__ P,
                   float* __restrict__ Out, int64_t ldo, int vec_out, int group) {
  using Cfg = OzCfg<N, STAGES, LEVELS, BPL, BK>;
  static_assert(!WIDE || (LEVELS == 4 && BPL == 4 && N == 128), "wide MMAs pair 128-column levels");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 1);

  // Persistent over output tiles (MODE 1: grid = #SMs; MODE 0: one tile per
  // CTA): the TMA warp runs ahead into the next tile while the epilogue
  // drains TMEM, and setup is paid once per CTA.
  const int tiles_m = (int)((rowsA + 127) / 128);
  const int total = tiles_m * tiles_n;
  const int64_t kb0 = (int64_t)blockIdx.y * k_per_split;
  const int64_t kb1 = min(K, kb0 + k_per_split);
  const int iters = kb1 > kb0 ? (int)((kb1 - kb0 + BK - 1) / BK) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // tile index -> (row tile, column tile); false if the tile is skipped
  auto tile_of = [&](int idx, int& ti, int& tj) -> bool {
    if (MODE == 1) {
      // column tiles in groups of kApplyGroup, all row tiles swept per group:
      // the group's B slices stay L2-resident while A row blocks stream; tj
      // fastest inside a group so an A block is reused by neighbouring tiles
      const int per_group = tiles_m * group;
      const int g = idx / per_group, rr = idx % per_group;
      const int gw = min(group, tiles_n - g * group);
      ti = rr / gw;
      tj = g * group + rr % gw;
      return true;
    }
    ti = idx / tiles_n;
    tj = idx % tiles_n;
    return !(symmetric && tj * N + N - 1 < ti * 128);  // strictly below the diagonal: mirrored later
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], 4);  // one arrive per epilogue warp
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mA);
    tma_prefetch(&mB);
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    int g = 0;  // stage-ring position across tiles
    for (int idx = blockIdx.x; idx < total; idx += gridDim.x) {
      int ti, tj;
      if (!tile_of(idx, ti, tj)) continue;
      const int i0 = ti * 128, j0 = tj * N;
      for (int it = 0; it < iters; ++it, ++g) {
        const int s = g % STAGES;
        mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
        if (lane == 0) {
          uint8_t* st = smem + s * Cfg::STAGE_BYTES;
          mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
          const int kk = (int)(kb0 + (int64_t)it * BK);
#pragma unroll
          for (int p = 0; p < Cfg::APLANES; ++p)
            tma_load_2d(st + p * Cfg::A_PLANE, &mA, &full[s], kk, (int)(p * planeA_rows + i0));
#pragma unroll
          for (int p = 0; p < Cfg::BPLANES; ++p)
            tma_load_2d(st + Cfg::APLANES * Cfg::A_PLANE + p * Cfg::B_PLANE, &mB, &full[s], kk,
                        (int)(p * planeB_rows + j0));
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_i8(128, N);
    constexpr uint32_t idesc_w = idesc_i8(128, WIDE ? 2 * N : N);
    int g = 0, tcount = 0;
    for (int idx = blockIdx.x; idx < total; idx += gridDim.x) {
      int ti, tj;
      if (!tile_of(idx, ti, tj)) continue;
      if (tcount > 0) {  // the epilogue has drained the previous tile's accumulators
        mbar_wait(&tempty[0], (tcount - 1) & 1);
        tc_fence_after();
      }
      for (int it = 0; it < iters; ++it, ++g) {
        const int s = g % STAGES;
        mbar_wait(&full[s], (g / STAGES) & 1);
        tc_fence_after();
        // descriptors are warp-uniform (computed by the whole warp, so they can
        // live in uniform registers); one elected lane issues the MMAs.  A
        // descriptor's start-address field is addr >> 4, so an offset is a
        // 64-bit add of (offset >> 4) while the field does not overflow.
        const uint64_t d0 = desc_kmajor<BK>(smem_u32(smem + s * Cfg::STAGE_BYTES));
        if (lane == 0) {
#pragma unroll
          for (int ks = 0; ks < BK / 32; ++ks) {
            uint64_t a[Cfg::APLANES], b[Cfg::BPLANES];
#pragma unroll
            for (int p = 0; p < Cfg::APLANES; ++p) a[p] = d0 + (uint64_t)((p * Cfg::A_PLANE + ks * 32) >> 4);
#pragma unroll
            for (int p = 0; p < Cfg::BPLANES; ++p)
              b[p] = d0 + (uint64_t)((Cfg::APLANES * Cfg::A_PLANE + p * Cfg::B_PLANE + ks * 32) >> 4);
            const uint32_t acc = (it == 0 && ks == 0) ? 0u : 1u;
            if (WIDE) {
              // 4 x 4 planes: B planes u, u+1 are adjacent in shared memory
              // (one 2N-row operand) and levels l, l+1 are adjacent in TMEM,
              // so A_t [B_u | B_u+1] is ONE N = 2*128 MMA into levels t+u and
              // t+u+1: the 10 slice pairs become 4 wide + 2 narrow MMAs, and
              // the A tile is read from shared memory 6 times instead of 10.
              mma_i8(tmem + 0 * N, a[0], b[0], idesc_w, acc);  // L0 += A0B0, L1 += A0B1
              mma_i8(tmem + 2 * N, a[0], b[2], idesc_w, acc);  // L2 += A0B2, L3 += A0B3
              mma_i8(tmem + 1 * N, a[1], b[0], idesc_w, 1u);   // L1 += A1B0, L2 += A1B1
              mma_i8(tmem + 3 * N, a[1], b[2], idesc, 1u);     // L3 += A1B2
              mma_i8(tmem + 2 * N, a[2], b[0], idesc_w, 1u);   // L2 += A2B0, L3 += A2B1
              mma_i8(tmem + 3 * N, a[3], b[0], idesc, 1u);     // L3 += A3B0
            } else {
              // level l accumulates the kept slice pairs (t, l - t); the first
              // product issued into each accumulator starts it (acc == 0)
#pragma unroll
              for (int l = 0; l < LEVELS; ++l) {
                const int t0 = l - (Cfg::BPLANES - 1) > 0 ? l - (Cfg::BPLANES - 1) : 0;
#pragma unroll
                for (int t = t0; t <= l; ++t) mma_i8(tmem + l * N, a[t], b[l - t], idesc, t == t0 ? acc : 1u);
              }
            }
          }
          mma_commit(&empty[s]);
          if (it == iters - 1) mma_commit(&tfull[0]);
        }
        __syncwarp();
      }
      ++tcount;
    }
  } else {
    const int q = warp & 3;
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
    int tcount = 0;
    for (int idx = blockIdx.x; idx < total; idx += gridDim.x) {
      int ti, tj;
      if (!tile_of(idx, ti, tj)) continue;
      const int i0 = ti * 128, j0 = tj * N;
      const int row = i0 + 32 * q + lane;
      const bool row_ok = row < rowsA;
      const int ea = row_ok ? eA[row] - 2048 : 0;
      if (iters > 0) {
        mbar_wait(&tfull[0], tcount & 1);
        tc_fence_after();
      }
#pragma unroll 1
      for (int cc = 0; cc < N / 32; ++cc) {
        double v[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) v[t] = 0.0;
        if (iters > 0) {
          double scale = 1.0;
#pragma unroll
          for (int l = 0; l < LEVELS; ++l) {
            int acc[32];
            tmem_ld32_i(tl + l * N + cc * 32, acc);
#pragma unroll
            for (int t = 0; t < 32; ++t) v[t] += (double)acc[t] * scale;
            scale *= 0x1p-7;
          }
        }
        if (!row_ok) continue;
        const int cbase = j0 + cc * 32;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const int col = cbase + t < rowsB ? cbase + t : rowsB - 1;
          v[t] = scale_pow2(v[t], ea + eB[col] - 2048 - 12);
        }
        // 16-byte stores when the whole 32-column chunk is in range and aligned
        // (a warp writes 32 different rows: wide stores cut sector traffic 4x/2x)
        const bool full_chunk = vec_out && cbase + 32 <= rowsB;
        if (MODE == 0) {
          double* prow = P + ((int64_t)blockIdx.y * rowsA + row) * (int64_t)rowsB + cbase;
          if (full_chunk) {
#pragma unroll
            for (int t = 0; t < 32; t += 2) *reinterpret_cast<double2*>(prow + t) = make_double2(v[t], v[t + 1]);
          } else {
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (cbase + t < rowsB) prow[t] = v[t];
          }
        } else {
          float* orow = Out + (int64_t)row * ldo + cbase;
          if (full_chunk) {
#pragma unroll
            for (int t = 0; t < 32; t += 4)
              *reinterpret_cast<float4*>(orow + t) =
                  make_float4((float)v[t], (float)v[t + 1], (float)v[t + 2], (float)v[t + 3]);
          } else {
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (cbase + t < rowsB) orow[t] = (float)v[t];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[0]);
      ++tcount;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, Cfg::TMEM_COLS);
  }
}

// C (ka x kb row-major fp64) (+)= sum_s P[s]; symmetric: mirror the upper part.
__global__ void gram_reduce_kernel(int ka, int kb, int splits, const double* __restrict__ P, double* __restrict__ C,
                                   int accumulate, int symmetric) {
  const int64_t total = (int64_t)ka * kb;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = f / kb, j = f - i * kb;
    const int64_t src = (symmetric && i > j) ? j * kb + i : f;
    double s = 0.0;
    for (int p = 0; p < splits; ++p) s += P[(int64_t)p * total + src];
    C[f] = accumulate ? C[f] + s : s;
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

// 2-D byte map over rows x cols int8 (row pitch ld bytes), box = bk bytes x box_rows, bk-byte swizzle.
int make_map_u8(fsr_ctx* ctx, CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld,
                int box_rows, int bk) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fsr::set_error(ctx, FSR_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)bk, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, bk == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fsr::set_error(ctx, FSR_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return FSR_OK;
}

inline int64_t pad_to(int64_t x, int64_t m) { return (x + m - 1) / m * m; }


constexpr size_t kChunkBudget = (size_t)6 << 30;  // bytes of slice staging per row chunk

// tile width / pipeline depth per variant (A slice planes = LEVELS, B planes = BPL)
template <int LEVELS, int BPL, int BK>
struct Variant;
template <>
struct Variant<4, 4, 64> {  // 4 x 128 TMEM columns; 3 stages of 4 x (128 + 128) x 64 B
  static constexpr int N = 128, STAGES = 3;
};
template <>
struct Variant<4, 1, 64> {  // 4 x 128 TMEM columns; 5 stages of (4 x 128 + 128) x 64 B
  static constexpr int N = 128, STAGES = 5;
};
template <>
struct Variant<1, 1, 64> {  // 160 TMEM columns; 8 stages of (128 + 160) x 64 B
  static constexpr int N = 160, STAGES = 8;
};

template <int MODE, int LEVELS, int BPL = LEVELS>
int launch_oz(fsr_ctx* ctx, dim3 grid, const CUtensorMap& mA, const CUtensorMap& mB, int rowsA, int rowsB,
              int64_t pA, int64_t pB, int64_t K, int tiles_n, int64_t kps, const int* eA, const int* eB, int sym,
              double* P, float* Out, int64_t ldo) {
  constexpr int BK = kBK;
  constexpr int N = Variant<LEVELS, BPL, BK>::N, STAGES = Variant<LEVELS, BPL, BK>::STAGES;
  constexpr bool kWide = LEVELS == 4 && BPL == 4;
  using Cfg = OzCfg<N, STAGES, LEVELS, BPL, BK>;
  FSR_TRY(fsr::ensure_smem(ctx, oz_gemm_kernel<MODE, N, STAGES, LEVELS, BPL, kWide, BK>, Cfg::SMEM));
  // 16-byte epilogue stores need 16-byte aligned rows
  const int vec_out = MODE == 0 ? (rowsB % 2 == 0 && ((uintptr_t)P & 15) == 0)
                                : (ldo % 4 == 0 && ((uintptr_t)Out & 15) == 0);
  oz_gemm_kernel<MODE, N, STAGES, LEVELS, BPL, kWide, BK><<<grid, kThreads, Cfg::SMEM, ctx->stream>>>(
      mA, mB, rowsA, rowsB, pA, pB, K, tiles_n, kps, eA, eB, sym, P, Out, ldo, vec_out, kApplyGroup);
  return fsr::launched(ctx, MODE == 0 ? "oz_gram_kernel" : "oz_apply_kernel");
}

}  // namespace

namespace fsr {

// C (ka x kb, fp64 row-major) (+)= A^T B over n rows of fp32 row-major blocks.
// levels == 1: one-slice preconditioner Gram; otherwise the full 28-bit scheme.
int tc_gram(fsr_ctx* ctx, int64_t n, int64_t ka, const float* A, int64_t lda, int64_t kb, const float* B,
            int64_t ldb, double* C, int accumulate, int levels, int symmetric) {
  const bool same = (A == B) && lda == ldb && ka == kb;
  // symmetric: compute the upper triangle only and mirror it (A == B, or a
  // caller that knows A^T B is symmetric up to rounding, fsr_cross_sym)
  symmetric = symmetric && ka == kb;
  const int NT = levels == 1 ? Variant<1, 1, 64>::N : Variant<4, 4, 64>::N;
  const int64_t per_row = kSlices * (ka + (same ? 0 : kb));
  int64_t chunk = std::max<int64_t>(128, std::min<int64_t>({n, kMaxK, (int64_t)(kChunkBudget / per_row)}));
  chunk = pad_to(chunk, 128);
  const int tiles_m = (int)ceil_div(ka, 128), tiles_n = (int)ceil_div(kb, NT);
  int tiles_eff = 0;
  for (int ti = 0; ti < tiles_m; ++ti)
    for (int tj = 0; tj < tiles_n; ++tj) tiles_eff += !(symmetric && tj * NT + NT - 1 < ti * 128);
  int splits = (int)std::max<int64_t>(1, ceil_div(2 * ctx->num_sms, tiles_eff));
  splits = (int)std::min<int64_t>(splits, std::max<int64_t>(1, chunk / (8 * kBK)));
  const size_t p_bytes = (size_t)splits * ka * kb * 8;
  const size_t e_bytes = (size_t)(ka + kb) * 4 + 256;
  const size_t s_bytes = (size_t)chunk * per_row;
  void* buf = nullptr;
  FSR_TRY(scratch(ctx, p_bytes + e_bytes + s_bytes + 4096, &buf));
  double* P = (double*)buf;
  int* eA = (int*)((char*)buf + pad_to(p_bytes, 256));
  int* eB = same ? eA : eA + ka;
  int8_t* sA = (int8_t*)((char*)buf + pad_to(p_bytes + e_bytes, 1024));
  int8_t* sB = same ? sA : sA + kSlices * ka * chunk;
  for (int64_t s0 = 0; s0 < n; s0 += chunk) {
    const int64_t rows = std::min(chunk, n - s0);
    const int64_t ldT = pad_to(rows, 128);
    // exponents per column over this chunk, then transposed slice planes
    FSR_CUDA(ctx, cudaMemsetAsync(eA, 0, (ka + (same ? 0 : kb)) * 4, ctx->stream));
    {
      dim3 g((unsigned)ceil_div(ka, 32), (unsigned)std::min<int64_t>(ceil_div(rows, 8), 256)), b(32, 8);
      exp_of_cols_kernel<float><<<g, b, 0, ctx->stream>>>(rows, ka, A + s0 * lda, lda, eA);
      FSR_TRY(launched(ctx, "exp_of_cols_kernel"));
      dim3 gs((unsigned)ceil_div(ka, 32), (unsigned)ceil_div(ldT, 128));
      slice_T_packed_kernel<<<gs, 256, 0, ctx->stream>>>(rows, ka, A + s0 * lda, lda, eA, sA, ldT);
      FSR_TRY(launched(ctx, "slice_T_packed_kernel"));
    }
    if (!same) {
      dim3 g((unsigned)ceil_div(kb, 32), (unsigned)std::min<int64_t>(ceil_div(rows, 8), 256)), b(32, 8);
      exp_of_cols_kernel<float><<<g, b, 0, ctx->stream>>>(rows, kb, B + s0 * ldb, ldb, eB);
      FSR_TRY(launched(ctx, "exp_of_cols_kernel"));
      dim3 gs((unsigned)ceil_div(kb, 32), (unsigned)ceil_div(ldT, 128));
      slice_T_packed_kernel<<<gs, 256, 0, ctx->stream>>>(rows, kb, B + s0 * ldb, ldb, eB, sB, ldT);
      FSR_TRY(launched(ctx, "slice_T_packed_kernel"));
    }
    CUtensorMap mA, mB;
    FSR_TRY(make_map_u8(ctx, &mA, sA, kSlices * ka, ldT, ldT, 128, kBK));
    FSR_TRY(make_map_u8(ctx, &mB, sB, kSlices * kb, ldT, ldT, NT, kBK));
    const int64_t kps = pad_to(ceil_div(ldT, splits), kBK);
    dim3 grid((unsigned)(tiles_m * tiles_n), (unsigned)ceil_div(ldT, kps));
    if (levels == 1)
      FSR_TRY((launch_oz<0, 1>(ctx, grid, mA, mB, (int)ka, (int)kb, ka, kb, ldT, tiles_n, kps, eA, eB, symmetric,
                               P, nullptr, 0)));
    else
      FSR_TRY((launch_oz<0, 4>(ctx, grid, mA, mB, (int)ka, (int)kb, ka, kb, ldT, tiles_n, kps, eA, eB, symmetric,
                               P, nullptr, 0)));
    const int acc = (s0 > 0) || accumulate;
    gram_reduce_kernel<<<grid_for(ka * kb, 256, ctx, 8), 256, 0, ctx->stream>>>((int)ka, (int)kb, (int)grid.y, P,
                                                                                C, acc, symmetric);
    FSR_TRY(launched(ctx, "gram_reduce_kernel"));
  }
  return FSR_OK;
}

// Out (n x N2 fp32) = A (n x K fp32) * M (K x N2, fp64; column-major if m_col_major).
// Out may alias A (row chunks are sliced before they are overwritten).
// m_slices = 1: M enters as its 7-bit first slice M' (4 products instead of
// 10); the product A M' is still 28-bit accurate in A.  For the first
// CholeskyQR pass that is all that matters: span(A M') = span(A) for any
// invertible M', and the second pass orthonormalises A M' exactly.
int tc_apply(fsr_ctx* ctx, int64_t n, int64_t K, const float* A, int64_t lda, int64_t N2, const double* M,
             int64_t ldm, int m_col_major, float* Out, int64_t ldo, int m_slices) {
  if (K > kMaxK) return set_error(ctx, FSR_EINVAL, "tc_apply: K=%lld exceeds the int32-exact bound", (long long)K);
  constexpr int NT = Variant<4, 4, 64>::N;
  static_assert(Variant<4, 1, 64>::N == NT, "apply variants share the output tile width");
  const int64_t pk = pad_to(K, 128);
  const size_t m_bytes = (size_t)kSlices * N2 * pk;
  const int64_t per_row = kSlices * pk;
  int64_t chunk = std::max<int64_t>(128, std::min<int64_t>(n, (int64_t)(kChunkBudget / per_row)));
  chunk = pad_to(chunk, 128);
  const size_t e_bytes = (size_t)(N2 + chunk) * 4 + 256;
  void* buf = nullptr;
  FSR_TRY(scratch(ctx, pad_to(m_bytes, 1024) + pad_to(e_bytes, 1024) + (size_t)chunk * per_row + 4096, &buf));
  int8_t* sM = (int8_t*)buf;  // M^T slices: N2 rows x pk
  int* eM = (int*)((char*)buf + pad_to(m_bytes, 1024));
  int* eR = eM + N2;
  int8_t* sR = (int8_t*)((char*)buf + pad_to(m_bytes, 1024) + pad_to(e_bytes, 1024));
  // M^T row j = column j of M: row-major M is read transposed; column-major M is already M^T
  const int tr = m_col_major ? 0 : 1;
  exp_of_rows_kernel<double><<<grid_for(N2 * 32, 256, ctx, 8), 256, 0, ctx->stream>>>(N2, K, M, ldm, tr, eM);
  FSR_TRY(launched(ctx, "exp_of_rows_kernel"));
  slice_rows_kernel<double><<<grid_for(N2 * pk, 256, ctx, 16), 256, 0, ctx->stream>>>(N2, K, M, ldm, tr, eM, sM, pk);
  FSR_TRY(launched(ctx, "slice_rows_kernel"));
  CUtensorMap mB;
  FSR_TRY(make_map_u8(ctx, &mB, sM, kSlices * N2, pk, pk, NT, kBK));
  const int tiles_n = (int)ceil_div(N2, NT);
  for (int64_t s0 = 0; s0 < n; s0 += chunk) {
    const int64_t rows = std::min(chunk, n - s0);
    slice_rows_fused_kernel<<<grid_for(rows * 32, 256, ctx, 8), 256, 0, ctx->stream>>>(rows, K, A + s0 * lda, lda,
                                                                                       eR, sR, pk);
    FSR_TRY(launched(ctx, "slice_rows_fused_kernel"));
    CUtensorMap mA;
    FSR_TRY(make_map_u8(ctx, &mA, sR, kSlices * rows, pk, pk, 128, kBK));
    // persistent: one CTA per SM walks the tiles (see oz_gemm_kernel)
    dim3 grid((unsigned)std::min<int64_t>(ceil_div(rows, 128) * tiles_n, ctx->num_sms), 1);
    if (m_slices == 1)
      FSR_TRY((launch_oz<1, 4, 1>(ctx, grid, mA, mB, (int)rows, (int)N2, rows, N2, pk, tiles_n, pk, eR, eM, 0,
                                  nullptr, Out + s0 * ldo, ldo)));
    else
      FSR_TRY((launch_oz<1, 4>(ctx, grid, mA, mB, (int)rows, (int)N2, rows, N2, pk, tiles_n, pk, eR, eM, 0, nullptr,
                               Out + s0 * ldo, ldo)));
  }
  return FSR_OK;
}

}  // namespace fsr
