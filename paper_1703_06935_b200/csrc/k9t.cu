// K9t: the online ranked-query step (top-K of x_q = U~ h(Lambda) U~^T y_q for
// a batch of b queries, reference ranking.py:229-255 + rank ranking.py:390-395)
// on the 5th-generation tensor cores, certified to return bit for bit the
// top-K of the unpruned fp32 path.
//
// Why a dense GEMM for a 2%-dense U~.  The sparse K9/K9h kernels gather one
// b-wide row of the projected queries per nonzero of U~ (tau * b * 2 bytes =
// 205 GB of L2 -> SM traffic per 1024-query batch at C3) and are bound by the
// loaded L2 latency of those gathers (K9h 11.6 ms, 88% of the random-row L2
// probe; staging the rows in shared memory only moves the bound to shared
// memory bandwidth, tools/fma_rate.cu).  The same product as a dense fp16 GEMM
// (M = n, N = b, K = r: 1.02e16 flop at C3) runs at tensor-core rate, and the
// dense fp16 U~ (n x r x 2 bytes = 10 GB at C3, independent of tau) streams
// from HBM once per batch.  Both fp16 operands make the products approximate,
// so -- exactly as in the K9h pruned path (prune.cuh) -- a rigorous per-row
// bound selects the rows that can still be in the top K and only those are
// re-scored in fp32 in the unpruned kernel's order.
//
// Bound (row i with m_i stored entries, query q; prune.cuh has the fp16
// rounding part): |x_fp32 - x~| <= c_i * Zb_q with
//   c_i = 1.01 (||u_i||_2 (2^-10 + 2.01 m_i 2^-24 + m_i 2^-21 + sqrt(m_i) 2^-38) + sqrt(m_i) 2^-25).
// The new term m_i 2^-21 covers the tensor-core accumulation: products of two
// fp16 values are exact in fp32; the accumulator is modelled as aligning each
// MMA step's addends to the largest and truncating (at most one unit in the
// 23rd bit per addend, <= 2 * 2^-22 relative per step with a nonzero
// product; steps whose products are all zero leave it unchanged).  A row has
// at most m_i steps with a nonzero product.  The measured behaviour (a
// -2^-24 relative drift per MMA step, tools/tc_debug.cu) is 8x inside it.
//
// Step (one CUDA graph):
//   K8 project (k8_online.cu, fp32 Zs + fp16 Zh[b][ldr] with a per-query
//      power-of-two scale);
//   k9t_gemm<0> on every 32nd 128-row tile (sample) -> lower keys;
//   k9t_threshold: per query t = the sample's target-th largest lower key
//      (any t with >= K rows of lower >= t satisfies t <= x_(K));
//   k9t_gemm<1> on all tiles: the epilogue drains TMEM, counts rows with
//      lower >= t and appends rows with upper >= t (and their x~) to the
//      query's candidate list -- x~ (b x n) is never written;
//   k9t_finish: adds copied uncovered rows (eta = 0, ranking.py:248-254),
//      lambda_K = K-th largest lower, keeps upper >= lambda_K, exact fp32
//      re-score in the unpruned K9's order, sort by (-x, index);
//   k9t_empty: queries with z = 0 (empty observation, FilterGraph padding);
//   fallback (flagged queries only): exact scores of every row + exact select.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <mutex>

#include "fsr_common.cuh"
#include "prune.cuh"
#include "tc_common.cuh"
#include "topk.cuh"

namespace fsr {
namespace k9t {

using namespace fsr::tc;

constexpr int kThreads = 192;   // warp 0 TMA, warp 1 MMA + TMEM owner, warps 2-5 epilogue
constexpr int BM = 128;         // rows of U~ per tile (TMEM lanes)
constexpr int BN = 256;         // queries per tile (TMEM columns per accumulator)
constexpr int BK = 64;          // fp16 K elements per stage = 128 bytes = one SWIZZLE_128B row
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;
// per query-tile width TN (256 for b > 128; 128 / 64 for smaller batches, so
// the MMA does not multiply padding queries): stage / shared-memory / TMEM sizes
template <int TN>
struct TileCfg {
  static_assert(TN == 64 || TN == 128 || TN == 256, "query tile of 64, 128 or 256");
  static constexpr int B_BYTES = TN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256 + 2 * TN * 16 + 2 * TN * 4 + TN * 4;
  static constexpr uint32_t TMEM_COLS = 2 * TN;  // double-buffered accumulators (a power of two >= 32)
};
constexpr int SMEM = TileCfg<BN>::SMEM;
constexpr int kSampleStride = 32;  // threshold sample: every 32nd row tile
constexpr int kCap = 4096;         // candidates per query (row << 12 | slot packs into int64)
constexpr int kFinishThreads = 256;
constexpr int kEmpty = -2;         // ccount marker: z = 0 query, answered by k9t_empty
static_assert(SMEM <= 227 * 1024, "stages exceed shared memory");

__host__ __device__ constexpr int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t ld_of(int64_t r) { return round_up(r, 8); }  // 16-byte rows for TMA

// kind::f16: A, B fp16 (format 0), D fp32 (format 1), both K-major.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void epi_barrier() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// ---- thread-block cluster (B tile split across the cluster, TMA multicast) --
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-D TMA load written to the same smem offset (and signalling the same
// mbarrier offset) in every CTA of `mask`
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                               int32_t c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
// arrive once on the mbarrier at this offset in every CTA of `mask` when this
// thread's previously issued MMAs complete
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// per-row bound factor (see the file comment); m entries, ss = sum of squares (rounded up)
__device__ __forceinline__ float row_bound(double m, float ss) {
  const double f = 0x1p-10 + 2.01 * m * 0x1p-24 + m * 0x1p-21 + sqrt(m) * 0x1p-38;
  return __double2float_ru((__dsqrt_ru((double)ss) * f + sqrt(m) * 0x1p-25) * 1.01);
}

// ---------------------------------------------------------------- layout --
// Dense fp16 copy of U~ (n x ldr, zeros off the support) + c_i + max_i c_i.
// Warp per row: scatter the row's entries, bound factor from the fp32 row.
__global__ void __launch_bounds__(256) densify_kernel(int64_t n, int64_t ldr, const int64_t* __restrict__ indptr,
                                                      const int32_t* __restrict__ indices,
                                                      const float* __restrict__ vals, __half* __restrict__ Ud,
                                                      float* __restrict__ cb, int* __restrict__ cmax_bits) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int cmax = 0;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    const int64_t e0 = indptr[i], e1 = indptr[i + 1];
    float ss = 0.f;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const float v = vals[e];
      ss = __fmaf_ru(v, v, ss);
      FSR_DCHECK(indices[e] >= 0 && indices[e] < ldr);
      Ud[i * ldr + indices[e]] = __float2half_rn(v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss = __fadd_ru(ss, __shfl_xor_sync(0xffffffffu, ss, o));
    if (lane == 0) {
      const float c = e1 > e0 ? row_bound((double)(e1 - e0), ss) : 0.f;
      cb[i] = c;
      cmax = max(cmax, __float_as_int(c));
    }
  }
  if (lane == 0) atomicMax(cmax_bits, cmax);
}

// ------------------------------------------------------------------ GEMM --
// MODE 0 (sample): row tiles kSampleStride * s, writes the lower keys of the
//   sampled rows, Ks[q * ns + s * BM + row-in-tile].
// MODE 1 (select): all row tiles; counts lower >= t (nlow) and appends rows
//   with upper >= t to cand / cval.
struct QParam {
  float tf_pre;  // conservative round-to-nearest pre-filter of t (NaN: skip the query)
  float inv;     // 1 / s_q
  float cz;      // max_i c_i * Zb_q (1 + 2^-20)
  float zb;      // Zb_q
};

// CL CTAs (consecutive blockIdx.x) form a cluster working on CL consecutive
// row tiles of the same query tile: each loads its own A tile and 1/CL of the
// B tile, multicast into every member's stage -- the L2 -> SM traffic per tile
// drops from A + B to A + B / CL (ncu at CL = 1: L2 throughput 72%, tensor
// pipe 48% -- L2-fed).  A stage is refilled only after every member's MMAs
// consumed it (the commits are multicast: empty barriers count CL arrivals).
template <int MODE, int CL, int TN, bool M2 = false>
__global__ void __launch_bounds__(kThreads, 1)
    k9t_gemm_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, int n, int b,
                    int r, int tiles_n, int band, int total, const float* __restrict__ cb,
                    const float2* __restrict__ qp,
                    const QParam* __restrict__ qpar, const uint32_t* __restrict__ thr, uint32_t* __restrict__ Ks,
                    int64_t ns, int32_t* __restrict__ cand, float* __restrict__ cval, int32_t* __restrict__ ccount,
                    unsigned* __restrict__ nlow) {
  using Cfg = TileCfg<TN>;
  constexpr int STAGE_BYTES = Cfg::STAGE_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  float4* spar = (float4*)(smem + STAGES * STAGE_BYTES + 256);  // [2][TN]
  uint32_t* sthr = (uint32_t*)(spar + 2 * TN);                  // [2][TN]
  unsigned* scnt = sthr + 2 * TN;                               // [TN]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int iters = (r + BK - 1) / BK;
  const int rank = CL > 1 ? (int)cluster_rank() : 0;
  const int cluster = blockIdx.x / CL, nclusters = gridDim.x / CL;
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1);
  constexpr int PART_ROWS = TN / CL, PART_BYTES = PART_ROWS * BK * 2;
  // M2 (2-D multicast, CL = 4, rank = 2 rq + rr): the cluster is 2 row tiles x
  // 2 query tiles; each CTA loads half its A tile, multicast to the CTA with
  // the same row tile (rank ^ 2), and half its B tile, multicast to the CTA
  // with the same query tile (rank ^ 1).  A stage of CTA x is written by x,
  // x ^ 1 and x ^ 2, so its empty barrier waits for those three consumers.
  static_assert(!M2 || CL == 4, "2-D multicast needs 4-CTA clusters");
  const int rr = rank & 1, rq = rank >> 1;
  const uint16_t maskA = (uint16_t)((1u << rank) | (1u << (rank ^ 2)));
  const uint16_t maskB = (uint16_t)((1u << rank) | (1u << (rank ^ 1)));
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], M2 ? 3 : CL);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mA);
    tma_prefetch(&mB);
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  for (int t = threadIdx.x; t < TN; t += blockDim.x) scnt[t] = 0;
  tc_fence_before();
  if (CL > 1)
    cluster_sync();  // every member's barriers exist before any multicast lands
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // work item idx (per cluster) -> this CTA's (row tile, query tile)
  // Raster: query tiles in bands of `band` (their fp16 Zh, band x TN x r x 2
  // bytes, stays L2-resident), row tiles within a band, the band's query
  // tiles fastest -- so the clusters in flight share row tiles of A (L2 hits)
  // and a large batch does not re-read its whole Zh from DRAM per row tile
  // (b = 10000: 40 query tiles, 100 MB of Zh).  band = tiles_n: one band.
  const int row_groups = total / tiles_n;  // row-tile groups (of CL tiles) per query tile
  auto tile_of = [&](int idx, int& ti, int& tj) {
    if (M2) {  // the same raster over query-tile pairs
      const int tiles_np = tiles_n / 2, bandp = max(1, band / 2), rgp = total / tiles_np;
      const int bnd = idx / (bandp * rgp);
      const int rem = idx - bnd * bandp * rgp;
      const int gw = min(bandp, tiles_np - bnd * bandp);
      ti = (rem / gw) * 2 + rr;
      tj = (bnd * bandp + rem % gw) * 2 + rq;
      if (MODE == 0) ti *= kSampleStride;
      return;
    }
    const int bnd = idx / (band * row_groups);
    const int rem = idx - bnd * band * row_groups;
    const int gw = min(band, tiles_n - bnd * band);  // the last band may be narrower
    ti = (rem / gw) * CL + rank;
    tj = bnd * band + rem % gw;
    if (MODE == 0) ti *= kSampleStride;
  };

  if (warp == 0) {
    int g = 0;
    for (int idx = cluster; idx < total; idx += nclusters) {
      int ti, tj;
      tile_of(idx, ti, tj);
      for (int it = 0; it < iters; ++it, ++g) {
        const int s = g % STAGES;
        mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
        if (lane == 0) {
          uint8_t* st = smem + s * STAGE_BYTES;
          mbar_expect_tx(&full[s], STAGE_BYTES);
          if (M2) {
            tma_load_2d_mc(st + rq * (A_BYTES / 2), &mA, &full[s], it * BK, ti * BM + rq * (BM / 2), maskA);
            tma_load_2d_mc(st + A_BYTES + rr * (Cfg::B_BYTES / 2), &mB, &full[s], it * BK, tj * TN + rr * (TN / 2),
                           maskB);
          } else {
          tma_load_2d(st, &mA, &full[s], it * BK, ti * BM);
          if (CL == 1)
            tma_load_2d(st + A_BYTES, &mB, &full[s], it * BK, tj * TN);
          else
            tma_load_2d_mc(st + A_BYTES + rank * PART_BYTES, &mB, &full[s], it * BK, tj * TN + rank * PART_ROWS,
                           kMask);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_f16(BM, TN);
    int g = 0, tcount = 0;
    for (int idx = cluster; idx < total; idx += nclusters, ++tcount) {
      const int ab = tcount & 1, use = tcount >> 1;
      if (use > 0) {  // the epilogue has drained this accumulator's previous tile
        mbar_wait(&tempty[ab], (use - 1) & 1);
        tc_fence_after();
      }
      const uint32_t d = tmem + ab * TN;
      for (int it = 0; it < iters; ++it, ++g) {
        const int s = g % STAGES;
        mbar_wait(&full[s], (g / STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * STAGE_BYTES);
        const uint64_t da = smem_desc_sw128(sa, 16, 1024), db = smem_desc_sw128(sa + A_BYTES, 16, 1024);
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // K = 16 per MMA: +32 bytes inside the 128-byte swizzle row
            mma_f16(d, da + (uint64_t)(2 * k), db + (uint64_t)(2 * k), idesc, (it | k) ? 1u : 0u);
          if (CL == 1)
            mma_commit(&empty[s]);
          else if (M2)
            mma_commit_mc(&empty[s], (uint16_t)(maskA | maskB));  // this CTA's A and B writers
          else
            mma_commit_mc(&empty[s], kMask);  // the stage holds every member's B part
          if (it == iters - 1) mma_commit(&tfull[ab]);
        }
        __syncwarp();
      }
    }
  } else {
    const int q4 = warp & 3;  // TMEM lane quarter this warp may access
    const int et = threadIdx.x - 64;  // 0..127 among the epilogue threads
    int tcount = 0;
    for (int idx = cluster; idx < total; idx += nclusters, ++tcount) {
      int ti, tj;
      tile_of(idx, ti, tj);
      const int ab = tcount & 1, use = tcount >> 1, pb = tcount & 1;
      const int j0 = tj * TN;
      // per-query parameters of this tile's columns
      for (int t = et; t < TN; t += 128) {
        const int q = j0 + t;
        float4 p = make_float4(__int_as_float(0x7fffffff), 1.f, 0.f, 0.f);
        uint32_t tk = 0xffffffffu;
        if (q < b) {
          if (MODE == 0) {
            const float2 v = qp[q];
            p = make_float4(0.f, v.x, 0.f, v.y);
          } else {
            const QParam v = qpar[q];
            p = make_float4(v.tf_pre, v.inv, v.cz, v.zb);
            tk = thr[q];
          }
        }
        spar[pb * TN + t] = p;
        sthr[pb * TN + t] = tk;
      }
      const int row = ti * BM + 32 * q4 + lane;
      const bool row_ok = row < n;
      const float c = row_ok ? __ldg(cb + row) : 0.f;
      mbar_wait(&tfull[ab], use & 1);
      tc_fence_after();
      epi_barrier();
      const uint32_t tl = tmem + ((uint32_t)(32 * q4) << 16) + ab * TN;
#pragma unroll 1
      for (int cc = 0; cc < TN / 32; ++cc) {
        float v[32];
        tmem_ld32(tl + cc * 32, v);
        if (!row_ok) continue;
        if (MODE == 0) {
          const int64_t srow = (int64_t)(ti / kSampleStride) * BM + 32 * q4 + lane;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int jj = cc * 32 + t;
            if (j0 + jj < b) {
              const float4 p = spar[pb * TN + jj];
              const float x = v[t] * p.y;
              Ks[(int64_t)(j0 + jj) * ns + srow] = prune::key32(__fsub_rd(x, prune::bound_of(c, p.w)));
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int jj = cc * 32 + t;
            const float4 p = spar[pb * TN + jj];
            const float x = v[t] * p.y;
            if (x + p.z >= p.x) {  // rare: within reach of the threshold
              const float bd = prune::bound_of(c, p.w);
              const uint32_t tk = sthr[pb * TN + jj];
              if (prune::key32(__fsub_rd(x, bd)) >= tk) atomicAdd(&scnt[jj], 1u);
              if (prune::key32(__fadd_ru(x, bd)) >= tk) {
                FSR_DCHECK(j0 + jj < b && row < n);
                const int slot = atomicAdd(ccount + j0 + jj, 1);
                if (slot < kCap) {
                  cand[(int64_t)(j0 + jj) * kCap + slot] = row;
                  cval[(int64_t)(j0 + jj) * kCap + slot] = x;
                }
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      if (MODE == 1) {
        epi_barrier();
        for (int t = et; t < TN; t += 128) {
          const unsigned k = scnt[t];
          if (k) {
            atomicAdd(nlow + j0 + t, k);
            scnt[t] = 0;
          }
        }
      }
    }
  }
  if (CL > 1)
    cluster_sync();  // no member exits while a peer may still signal its barriers
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, Cfg::TMEM_COLS);
  }
}


// ---------------------------------------------------- 2-SM (cta_group::2) --
// The same main pass with CTA-pair MMAs: a cluster of 4 = 2 pairs; pair p
// multiplies a 256-row tile of U~ (CTA h of the pair holds rows h*128..+128)
// by query tile 2 qp + p (each CTA holds half the tile's 256 queries), with
// `tcgen05.mma.cta_group::2` M = 256 N = 256 issued by the pair's even CTA.
// Per CTA and K-step the stage is A 16 KB + B 16 KB (instead of A + a whole
// B tile), so 6 stages fit where 4 did; the A rows are also shared across
// the two pairs (each CTA loads half and multicasts it to its counterpart,
// rank ^ 2).  Barriers: full[s] lives in each pair's even CTA and counts the
// pair's 64 KB (the odd CTA's TMA loads signal it, peer bit cleared);
// empty[s] of every CTA waits for both pairs' MMA commits (its A half is in
// the other pair's stage too); tempty[] of the even CTA counts the epilogue
// warps of both CTAs.
namespace sm2 {
constexpr int STAGES2 = 6;
constexpr int BM2 = 256;                          // rows per pair tile
constexpr int A_HALF = 128 * BK * 2;              // 16 KB: this CTA's 128 rows
constexpr int B_HALF = 128 * BK * 2;              // 16 KB: this CTA's 128 queries
constexpr int STAGE2 = A_HALF + B_HALF;
constexpr int TN2 = 256;
constexpr int SMEM2 = STAGES2 * STAGE2 + 1024 + 256 + 2 * TN2 * 16 + 2 * TN2 * 4 + TN2 * 4;
constexpr int kSample2 = kSampleStride;           // every 32nd 256-row tile: the same 1/32 of the rows
static_assert(SMEM2 <= 227 * 1024, "stages exceed shared memory");

__host__ __device__ constexpr uint32_t idesc_f16_m256(int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
__device__ __forceinline__ void mma2_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit2_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// 2-D TMA into this CTA's smem, completion counted on the pair's even CTA's barrier
__device__ __forceinline__ void tma2_load(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma2_load_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0, int32_t c1,
                                             uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
// arrive on the pair's even CTA's barrier (this CTA's copy at the same offset)
__device__ __forceinline__ void mbar_arrive_pair0(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & 0xFEFFFFFFu) : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    k9t_gemm2sm_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, int n, int b,
                       int r, int tiles_np, int total, const float* __restrict__ cb, const float2* __restrict__ qp,
                       const QParam* __restrict__ qpar, const uint32_t* __restrict__ thr, uint32_t* __restrict__ Ks,
                       int64_t ns, int32_t* __restrict__ cand, float* __restrict__ cval,
                       int32_t* __restrict__ ccount, unsigned* __restrict__ nlow) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + STAGES2 * STAGE2);
  uint64_t* empty = full + STAGES2;
  uint64_t* tfull = empty + STAGES2;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  float4* spar = (float4*)(smem + STAGES2 * STAGE2 + 256);  // [2][TN2]
  uint32_t* sthr = (uint32_t*)(spar + 2 * TN2);              // [2][TN2]
  unsigned* scnt = sthr + 2 * TN2;                           // [TN2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int iters = (r + BK - 1) / BK;
  const int rank = (int)cluster_rank();
  const int h = rank & 1, p = rank >> 1;  // half within the pair, pair index
  const bool lead = h == 0;
  const int cluster = blockIdx.x / 4, nclusters = gridDim.x / 4;
  const uint16_t maskA = (uint16_t)((1u << rank) | (1u << (rank ^ 2)));
  const uint16_t maskPair = (uint16_t)(3u << (2 * p));
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);   // the even CTA's producer arrives (with the pair's 64 KB of tx)
      mbar_init(&empty[s], 2);  // both pairs' MMA commits
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps in each CTA of the pair
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mA);
    tma_prefetch(&mB);
  }
  if (warp == 1) tmem_alloc2(tmem_slot, 512);
  for (int t = threadIdx.x; t < TN2; t += blockDim.x) scnt[t] = 0;
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // item -> (256-row tile, query-tile pair); this CTA's query tile is 2 qp + p
  auto tile_of = [&](int idx, int& t2, int& tj) {
    t2 = idx / tiles_np;
    tj = (idx % tiles_np) * 2 + p;
    if (MODE == 0) t2 *= kSample2;
  };

  if (warp == 0) {
    int g = 0;
    for (int idx = cluster; idx < total; idx += nclusters) {
      int t2, tj;
      tile_of(idx, t2, tj);
      for (int it = 0; it < iters; ++it, ++g) {
        const int s = g % STAGES2;
        mbar_wait(&empty[s], ((g / STAGES2) & 1) ^ 1);
        if (lane == 0) {
          uint8_t* st = smem + s * STAGE2;
          if (lead) mbar_expect_tx(&full[s], 2 * STAGE2);
          // A: 64 of this CTA's 128 rows (half p of them), multicast to the other pair's CTA h
          tma2_load_mc(st + p * (A_HALF / 2), &mA, &full[s], it * BK, t2 * BM2 + h * 128 + p * 64, maskA);
          // B: this CTA's 128 of the query tile's 256 queries
          tma2_load(st + A_HALF, &mB, &full[s], it * BK, tj * TN2 + h * 128);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    if (lead) {
      constexpr uint32_t idesc = idesc_f16_m256(TN2);
      int g = 0, tcount = 0;
      for (int idx = cluster; idx < total; idx += nclusters, ++tcount) {
        const int ab = tcount & 1, use = tcount >> 1;
        if (use > 0) {
          mbar_wait(&tempty[ab], (use - 1) & 1);
          tc_fence_after();
        }
        const uint32_t d = tmem + ab * TN2;
        for (int it = 0; it < iters; ++it, ++g) {
          const int s = g % STAGES2;
          mbar_wait(&full[s], (g / STAGES2) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * STAGE2);
          const uint64_t da = smem_desc_sw128(sa, 16, 1024), db = smem_desc_sw128(sa + A_HALF, 16, 1024);
          if (lane == 0) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma2_f16(d, da + (uint64_t)(2 * k), db + (uint64_t)(2 * k), idesc, (it | k) ? 1u : 0u);
            commit2_mc(&empty[s], 0xF);  // every CTA: both pairs read the A halves it wrote
            if (it == iters - 1) commit2_mc(&tfull[ab], maskPair);
          }
          __syncwarp();
        }
      }
    }
  } else {
    const int q4 = warp & 3;
    const int et = threadIdx.x - 64;
    int tcount = 0;
    for (int idx = cluster; idx < total; idx += nclusters, ++tcount) {
      int t2, tj;
      tile_of(idx, t2, tj);
      const int ab = tcount & 1, use = tcount >> 1, pb = tcount & 1;
      const int j0 = tj * TN2;
      for (int t = et; t < TN2; t += 128) {
        const int q = j0 + t;
        float4 pp = make_float4(__int_as_float(0x7fffffff), 1.f, 0.f, 0.f);
        uint32_t tk = 0xffffffffu;
        if (q < b) {
          if (MODE == 0) {
            const float2 v = qp[q];
            pp = make_float4(0.f, v.x, 0.f, v.y);
          } else {
            const QParam v = qpar[q];
            pp = make_float4(v.tf_pre, v.inv, v.cz, v.zb);
            tk = thr[q];
          }
        }
        spar[pb * TN2 + t] = pp;
        sthr[pb * TN2 + t] = tk;
      }
      const int row = t2 * BM2 + h * 128 + 32 * q4 + lane;
      const bool row_ok = row < n;
      const float c = row_ok ? __ldg(cb + row) : 0.f;
      mbar_wait(&tfull[ab], use & 1);
      tc_fence_after();
      epi_barrier();
      const uint32_t tl = tmem + ((uint32_t)(32 * q4) << 16) + ab * TN2;
#pragma unroll 1
      for (int cc = 0; cc < TN2 / 32; ++cc) {
        float v[32];
        tmem_ld32(tl + cc * 32, v);
        if (!row_ok) continue;
        if (MODE == 0) {
          const int64_t srow = (int64_t)(t2 / kSample2) * BM2 + h * 128 + 32 * q4 + lane;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int jj = cc * 32 + t;
            if (j0 + jj < b) {
              const float4 pp = spar[pb * TN2 + jj];
              const float x = v[t] * pp.y;
              Ks[(int64_t)(j0 + jj) * ns + srow] = prune::key32(__fsub_rd(x, prune::bound_of(c, pp.w)));
            }
          }
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int jj = cc * 32 + t;
            const float4 pp = spar[pb * TN2 + jj];
            const float x = v[t] * pp.y;
            if (x + pp.z >= pp.x) {
              const float bd = prune::bound_of(c, pp.w);
              const uint32_t tk = sthr[pb * TN2 + jj];
              if (prune::key32(__fsub_rd(x, bd)) >= tk) atomicAdd(&scnt[jj], 1u);
              if (prune::key32(__fadd_ru(x, bd)) >= tk) {
                FSR_DCHECK(j0 + jj < b && row < n);
                const int slot = atomicAdd(ccount + j0 + jj, 1);
                if (slot < kCap) {
                  cand[(int64_t)(j0 + jj) * kCap + slot] = row;
                  cval[(int64_t)(j0 + jj) * kCap + slot] = x;
                }
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_pair0(&tempty[ab]);  // the pair's MMA issuer may reuse this accumulator
      if (MODE == 1) {
        epi_barrier();
        for (int t = et; t < TN2; t += 128) {
          const unsigned k = scnt[t];
          if (k) {
            atomicAdd(nlow + j0 + t, k);
            scnt[t] = 0;
          }
        }
      }
    }
  }
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem, 512);
  }
}

}  // namespace sm2

// ------------------------------------------------------------- threshold --
// Per query: t = the target-th largest lower key of the sample (two 12-bit
// digits), the QParam of the main pass, zeroed counters.  z = 0 queries are
// marked kEmpty; non-finite z, and thresholds at or below the smallest normal
// (fewer than ~target positive sampled scores), are flagged for the exact
// fallback.
__global__ void __launch_bounds__(256) k9t_threshold_kernel(int64_t b, int64_t ns, int64_t n_valid_s,
                                                            const uint32_t* __restrict__ Ks,
                                                            const float2* __restrict__ qp,
                                                            const int* __restrict__ cmax_bits, int64_t target,
                                                            uint32_t* __restrict__ thr, QParam* __restrict__ qpar,
                                                            int32_t* __restrict__ ccount, unsigned* __restrict__ nlow,
                                                            int* __restrict__ nflag, int* __restrict__ flags,
                                                            const int32_t* __restrict__ n_valid_dev) {
  constexpr int KB = 32, HB = topk::kHistBits, nb = 1 << HB;
  if (n_valid_dev) n_valid_s = *n_valid_dev;  // the streaming path's sample size lives on the device
  __shared__ unsigned hist[nb];
  __shared__ unsigned found_bin;
  __shared__ unsigned long long above;
  const float nanf_ = __int_as_float(0x7fffffff);
  for (int64_t q = blockIdx.x; q < b; q += gridDim.x) {
    const float2 p = qp[q];
    const float zb = p.y;
    if (zb == 0.f || !(zb <= FLT_MAX)) {
      if (threadIdx.x == 0) {
        qpar[q] = QParam{nanf_, p.x, 0.f, zb};
        if (zb == 0.f) {
          ccount[q] = kEmpty;
        } else {
          ccount[q] = -1;
          flags[atomicAdd(nflag, 1)] = (int)q;
        }
      }
      continue;
    }
    const uint32_t* kq = Ks + q * ns;
    uint32_t prefix = 0;
    unsigned long long above0 = 0;
    for (int level = 0; level < 2; ++level) {
      for (int t = threadIdx.x; t < nb; t += blockDim.x) hist[t] = 0;
      __syncthreads();
      // 8 keys per thread in flight before their atomics (a small batch runs
      // one CTA per query: a load-then-atomic loop was DRAM-latency bound)
      for (int64_t e0 = (int64_t)threadIdx.x; e0 < n_valid_s; e0 += 8 * (int64_t)blockDim.x) {
        uint32_t kk[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t e = e0 + (int64_t)u * blockDim.x;
          kk[u] = e < n_valid_s ? kq[e] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (e0 + (int64_t)u * blockDim.x >= n_valid_s) break;
          const uint32_t k = kk[u];
          if (level == 0)
            atomicAdd(&hist[k >> (KB - HB)], 1u);
          else if ((k >> (KB - HB)) == prefix)
            atomicAdd(&hist[(k >> (KB - 2 * HB)) & (nb - 1)], 1u);
        }
      }
      __syncthreads();
      topk::find_bin_t<256>(hist, nb, level == 0 ? target : target - above0, &found_bin, &above);
      FSR_DCHECK(found_bin < (unsigned)nb);
      if (level == 0) above0 = above;
      prefix = (prefix << HB) | found_bin;
      __syncthreads();
    }
    const uint32_t t_lo = prefix << (KB - 2 * HB);
    if (threadIdx.x == 0) {
      const float tf = prune::key_to_float((uint64_t)t_lo);
      if (!(tf >= FLT_MIN)) {  // t <= 0: zero-valued rows would all be candidates
        qpar[q] = QParam{nanf_, p.x, 0.f, zb};
        ccount[q] = -1;
        flags[atomicAdd(nflag, 1)] = (int)q;
      } else {
        thr[q] = t_lo;
        ccount[q] = 0;
        nlow[q] = 0;
        const float cz = __int_as_float(*cmax_bits) * zb * (1.f + 0x1p-20f);
        qpar[q] = QParam{tf - fabsf(tf) * 0x1p-20f - 0x1p-126f, p.x, cz, zb};
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- finish --
// x_i of the unpruned fp32 path for a row with no stored product to re-score:
// the copied y_i of an uncovered observed row (ranking.py:248-254), else 0.
__device__ __forceinline__ bool copied_value(int64_t i, int64_t q, const double* __restrict__ eta, int copy,
                                             const int64_t* __restrict__ y_ptr, const int64_t* __restrict__ y_idx,
                                             const float* __restrict__ y_val, float* v) {
  if (!(copy && eta && eta[i] == 0.0)) return false;
  for (int64_t t = y_ptr[q]; t < y_ptr[q + 1]; ++t)
    if (y_idx[t] == i) {
      *v = y_val[t];
      return true;
    }
  return false;
}

// The exact fp32 score of row i (thread-sequential, the unpruned K9's order).
__device__ __forceinline__ float exact_row(int64_t i, int64_t q, const int64_t* __restrict__ indptr,
                                           const int32_t* __restrict__ indices, const float* __restrict__ vals,
                                           const float* __restrict__ Zs, int64_t ldz, const double* __restrict__ eta,
                                           int copy, const int64_t* __restrict__ y_ptr,
                                           const int64_t* __restrict__ y_idx, const float* __restrict__ y_val) {
  float v;
  if (copied_value(i, q, eta, copy, y_ptr, y_idx, y_val, &v)) return v;
  float acc = 0.f;
  for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e)
    acc = fmaf(__ldg(vals + e), __ldg(Zs + (int64_t)__ldg(indices + e) * ldz + q), acc);
  return acc;
}

// The same for one row by a G-lane group (uniform result): copied rows first,
// then the grouped sequential sum of prune.cuh (bitwise the thread version).
template <int G>
__device__ __forceinline__ float exact_row_group(int64_t i, int64_t q, const int64_t* __restrict__ indptr,
                                                 const int32_t* __restrict__ indices, const float* __restrict__ vals,
                                                 const float* __restrict__ Zs, int64_t ldz,
                                                 const double* __restrict__ eta, int copy,
                                                 const int64_t* __restrict__ y_ptr, const int64_t* __restrict__ y_idx,
                                                 const float* __restrict__ y_val, unsigned mask) {
  float v;
  if (copied_value(i, q, eta, copy, y_ptr, y_idx, y_val, &v)) return v;
  if (indptr[i] == indptr[i + 1]) return 0.f;
  return prune::exact_score_group<G>(i, q, Zs /* unused: the row is not empty */, indptr, indices, vals, Zs, ldz,
                                     nullptr, 0, y_ptr, y_idx, mask);
}

// Small batches: the finish kernel is one CTA per query, so its exact
// re-score (~100-400 rows of ~100 dependent entries) would run on a handful of
// SMs.  This kernel re-scores every candidate of every query instead, one
// 8-lane group per (query, slot), spread over the GPU; finish then only reads
// the values.  Same sequential fp32 order (exact_row_group).
__global__ void __launch_bounds__(256) k9t_rescore_kernel(
    int64_t b, const int32_t* __restrict__ cand, const int32_t* __restrict__ ccount,
    const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, const float* __restrict__ vals,
    const float* __restrict__ Zs, int64_t ldz, const double* __restrict__ eta, int copy,
    const int64_t* __restrict__ y_ptr, const int64_t* __restrict__ y_idx, const float* __restrict__ y_val,
    float* __restrict__ pre);

constexpr int kKeep = 1024;  // rows re-scored exactly per query (upper >= lambda_K); more -> fallback
// Candidates a finish CTA holds in shared memory (C3: at most 1365 per query;
// a query with more takes the exact fallback).
constexpr int kFinishCap = 2048;
// Shared memory of a finish CTA: the radix histogram, later the kept rows'
// sort keys and indices (16 KB); lower keys, later the kept rows' entry
// offsets (8 KB); rows, later the kept rows' lengths (8 KB); scores (8 KB);
// then the query's fp32 zs column (r floats) when it fits kZsSmemMax.
constexpr size_t kFinishSmem = (size_t)kKeep * 16 + (size_t)kFinishCap * 12;
static_assert((size_t)(1 << topk::kHistBits) * 4 <= (size_t)kKeep * 16, "histogram aliases the kept keys");
constexpr int64_t kZsSmemMax = 24576;  // r up to this: zs_q staged in shared memory (96 KB)
inline size_t finish_smem(int64_t r) { return kFinishSmem + (r <= kZsSmemMax ? (size_t)r * 4 : 0); }

// The sequential fp32 sum of `len` entries from e0 by a G-lane group, the
// query's zs in shared memory (zsm) or strided in global memory (Zs[c * ldz]):
// all R loads per lane of a 64-entry round in flight, then the dependent FMA
// chain in CSR order on broadcast values -- bitwise exact_row / exact_row_group.
template <int G, bool SMEM>
__device__ __forceinline__ float seq_sum_group(int64_t e0, int len, const int32_t* __restrict__ indices,
                                               const float* __restrict__ vals, const float* __restrict__ zsm,
                                               const float* __restrict__ Zs, int64_t ldz, unsigned mask) {
  constexpr int R = 64 / G;
  const int gl = threadIdx.x & (G - 1);
  float acc = 0.f;
  for (int base = 0; base < len; base += G * R) {
    const int m = len - base < G * R ? len - base : G * R;
    float a[R], z[R];
    int c[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int t = k * G + gl;
      c[k] = t < m ? __ldg(indices + e0 + base + t) : 0;
      a[k] = t < m ? __ldg(vals + e0 + base + t) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) z[k] = SMEM ? zsm[c[k]] : (k * G + gl < m ? __ldg(Zs + (int64_t)c[k] * ldz) : 0.f);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int mk = m - k * G < G ? m - k * G : G;
      if (mk <= 0) break;
      if (mk == G) {
#pragma unroll
        for (int e = 0; e < G; ++e)
          acc = fmaf(__shfl_sync(mask, a[k], e, G), __shfl_sync(mask, z[k], e, G), acc);
      } else {
        for (int e = 0; e < mk; ++e) acc = fmaf(__shfl_sync(mask, a[k], e, G), __shfl_sync(mask, z[k], e, G), acc);
      }
    }
  }
  return acc;
}

__global__ void __launch_bounds__(256) k9t_rescore_kernel(
    int64_t b, const int32_t* __restrict__ cand, const int32_t* __restrict__ ccount,
    const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, const float* __restrict__ vals,
    const float* __restrict__ Zs, int64_t ldz, const double* __restrict__ eta, int copy,
    const int64_t* __restrict__ y_ptr, const int64_t* __restrict__ y_idx, const float* __restrict__ y_val,
    float* __restrict__ pre) {
  constexpr int G = 8;
  const int lane = threadIdx.x & 31, gl = threadIdx.x & (G - 1);
  const unsigned gmask = 0xffu << (lane & ~(G - 1));
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; g < b * kCap; g += ngroups) {
    const int64_t q = g / kCap;
    const int slot = (int)(g - q * kCap);
    const int cnt = ccount[q];
    if (cnt < 0 || cnt > kCap || slot >= cnt) continue;  // group-uniform
    FSR_DCHECK(cand[g] >= 0);
    const float v = exact_row_group<G>(cand[g], q, indptr, indices, vals, Zs, ldz, eta, copy, y_ptr, y_idx, y_val,
                                       gmask);
    if (gl == 0) pre[g] = v;
  }
}

__global__ void __launch_bounds__(kFinishThreads) k9t_finish_kernel(
    const float* __restrict__ cb, const QParam* __restrict__ qpar, const uint32_t* __restrict__ thr,
    const int32_t* __restrict__ cand, const float* __restrict__ cval, const int32_t* __restrict__ ccount,
    const unsigned* __restrict__ nlow, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
    const float* __restrict__ vals, const float* __restrict__ Zs, int64_t ldz, const float* __restrict__ Zt,
    int64_t r, const double* __restrict__ eta, int copy, const int64_t* __restrict__ y_ptr,
    const int64_t* __restrict__ y_idx, const float* __restrict__ y_val, int64_t K, int64_t* __restrict__ out_idx,
    float* __restrict__ out_val, int* __restrict__ nflag, int* __restrict__ flags, int2* __restrict__ stats,
    const float* __restrict__ pre) {
  constexpr int HB = topk::kHistBits, NB = 1 << HB;
  extern __shared__ __align__(16) unsigned char dyn[];
  uint64_t* kkey = (uint64_t*)dyn;             // [kKeep] exact order keys of the kept rows
  int64_t* kidx = (int64_t*)(kkey + kKeep);    // [kKeep] row << 12 | slot
  unsigned* hist = (unsigned*)dyn;             // [NB], before kkey / kidx are written
  uint32_t* lkey = (uint32_t*)(kidx + kKeep);  // [kFinishCap] lower-bound keys by slot
  int64_t* ke0 = (int64_t*)lkey;               // [kKeep] after the keep pass: entry offset of kept row t
  int32_t* crow = (int32_t*)(lkey + kFinishCap);  // [kFinishCap] rows by slot
  int32_t* klen = crow;                           // [kKeep] after the keep pass: its length (-1: no re-score)
  float* cv = (float*)(crow + kFinishCap);        // [kFinishCap] x~, then exact scores, by slot
  float* zsm = cv + kFinishCap;                   // [r] zs_q when r <= kZsSmemMax
  __shared__ unsigned n_extra, n_extra_ge, n_keep, n_next, found_bin;
  __shared__ unsigned long long above;
  const int64_t q = blockIdx.x;
  const int cnt0 = ccount[q];
  if (cnt0 < 0) return;  // flagged (fallback) or empty observation (k9t_empty)
  const bool zs_smem = pre == nullptr && r <= kZsSmemMax;
  if (zs_smem) {  // zs_q (= Zt row q, the same fp32 values as Zs[:, q]) in flight while the candidates load
    const float* src = Zt + q * r;
    for (int64_t c = threadIdx.x; c < r; c += blockDim.x) {
      const unsigned dst = (unsigned)__cvta_generic_to_shared(zsm + c);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src + c) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  const int cnt = min(cnt0, kFinishCap);
  const uint32_t tk = thr[q];
  const float zb = qpar[q].zb;
  if (threadIdx.x == 0) n_extra = n_extra_ge = n_keep = 0;
  __syncthreads();
  // main candidates (rows with upper >= t) and their lower-bound keys
  for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
    const int32_t i = cand[q * kCap + t];
    const float x = cval[q * kCap + t];
    crow[t] = i;
    cv[t] = x;
    lkey[t] = prune::key32(__fsub_rd(x, prune::bound_of(cb[i], zb)));
  }
  // copied uncovered rows of this query: exact value y_i (the main pass saw 0 < t)
  if (copy && eta) {
    for (int64_t t = y_ptr[q] + threadIdx.x; t < y_ptr[q + 1]; t += blockDim.x) {
      const int64_t i = y_idx[t];
      if (eta[i] != 0.0) continue;
      const float v = y_val[t];
      const unsigned s = atomicAdd(&n_extra, 1u);
      if (prune::key32(v) >= tk) atomicAdd(&n_extra_ge, 1u);
      const int slot = cnt + (int)s;
      if (slot < kFinishCap) {
        crow[slot] = (int32_t)i;
        cv[slot] = v;
        lkey[slot] = prune::key32(v);
      }
    }
  }
  __syncthreads();
  const int total = cnt + (int)n_extra;
  if (cnt0 > kFinishCap || total > kFinishCap ||
      (unsigned long long)nlow[q] + n_extra_ge < (unsigned long long)K) {
    if (threadIdx.x == 0) flags[atomicAdd(nflag, 1)] = (int)q;  // overflow, or the sampled t was too high
    if (zs_smem) asm volatile("cp.async.wait_all;\n" ::: "memory");
    return;
  }
  // lambda' <= lambda_K (the K-th largest lower bound): two 12-bit radix
  // digits of the candidates' lower keys, the low end of the K-th key's bucket
  uint32_t prefix = 0;
  unsigned long long above0 = 0;
  for (int level = 0; level < 2; ++level) {
    for (int t = threadIdx.x; t < NB; t += blockDim.x) hist[t] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const uint32_t k = lkey[t];
      if (level == 0)
        atomicAdd(&hist[k >> (32 - HB)], 1u);
      else if ((k >> (32 - HB)) == prefix)
        atomicAdd(&hist[(k >> (32 - 2 * HB)) & (NB - 1)], 1u);
    }
    __syncthreads();
    topk::find_bin_t<kFinishThreads>(hist, NB, level == 0 ? (unsigned long long)K : K - above0, &found_bin, &above);
    if (level == 0) above0 = above;
    prefix = (prefix << HB) | found_bin;
    __syncthreads();
  }
  const uint32_t lam = prefix << (32 - 2 * HB);
  FSR_DCHECK(total <= kFinishCap && cnt <= kFinishCap);
  // keep upper >= lambda' (copied rows: exact, upper == lower)
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int32_t i = crow[t];
    const bool keep = t >= cnt ? lkey[t] >= lam
                               : prune::key32(__fadd_ru(cv[t], prune::bound_of(cb[i], zb))) >= lam;
    if (keep) {
      const unsigned k = atomicAdd(&n_keep, 1u);
      if (k < (unsigned)kKeep) kidx[k] = ((int64_t)i << 12) | t;
    }
  }
  __syncthreads();
  const unsigned keep = n_keep;
  FSR_DCHECK(keep >= (unsigned)K || keep > (unsigned)kKeep || total < K);
  if (threadIdx.x == 0) stats[q] = make_int2(total, (int)keep);
  if (keep > (unsigned)kKeep) {
    if (threadIdx.x == 0) flags[atomicAdd(nflag, 1)] = (int)q;
    if (zs_smem) asm volatile("cp.async.wait_all;\n" ::: "memory");
    return;
  }
  if (pre) {  // small batches: every candidate was re-scored by k9t_rescore_kernel
    for (unsigned t = threadIdx.x; t < keep; t += blockDim.x) {
      const int slot = (int)(kidx[t] & 4095);
      if (slot < cnt) cv[slot] = pre[q * kCap + slot];
    }
  } else {
    // exact re-score of the kept main candidates.  First every kept row's
    // extent (and the copied value of an uncovered observed row) with all
    // loads in flight at once, then 4-lane groups sum the rows sequentially
    // against zs_q in shared memory.
    for (unsigned t = threadIdx.x; t < keep; t += blockDim.x) {
      const int64_t packed = kidx[t];
      const int slot = (int)(packed & 4095);
      const int64_t i = packed >> 12;
      int len = -1;
      if (slot < cnt) {
        float v;
        if (copied_value(i, q, eta, copy, y_ptr, y_idx, y_val, &v)) {
          cv[slot] = v;
        } else {
          const int64_t e0 = indptr[i], e1 = indptr[i + 1];
          if (e0 == e1) {
            cv[slot] = 0.f;
          } else {
            ke0[t] = e0;
            len = (int)(e1 - e0);
          }
        }
      }
      klen[t] = len;
    }
    if (zs_smem) asm volatile("cp.async.wait_all;\n" ::: "memory");
    constexpr int G = 4;
    const int lane = threadIdx.x & 31, grp = threadIdx.x / G, gl = threadIdx.x & (G - 1);
    const unsigned gmask = 0xfu << (lane & ~(G - 1));
    if (threadIdx.x == 0) n_next = kFinishThreads / G;
    __syncthreads();
    for (unsigned t = grp; t < keep;) {
      const int len = klen[t];
      if (len > 0) {
        const float v = zs_smem ? seq_sum_group<G, true>(ke0[t], len, indices, vals, zsm, nullptr, 0, gmask)
                                : seq_sum_group<G, false>(ke0[t], len, indices, vals, nullptr, Zs + q, ldz, gmask);
        if (gl == 0) cv[kidx[t] & 4095] = v;
      }
      unsigned nt = 0;
      if (gl == 0) nt = atomicAdd(&n_next, 1u);
      t = __shfl_sync(gmask, nt, 0, G);
    }
  }
  __syncthreads();
  for (unsigned t = threadIdx.x; t < keep; t += blockDim.x) kkey[t] = topk::order_key(cv[kidx[t] & 4095]);
  __syncthreads();
  topk::bitonic_sort(kkey, kidx, (int)keep);
  for (int64_t m = threadIdx.x; m < K; m += blockDim.x) {
    const int64_t packed = kidx[m];
    out_idx[q * K + m] = packed >> 12;
    out_val[q * K + m] = cv[packed & 4095];
  }
}

// ------------------------------------------------------------------ empty --
// z = 0: every summed row scores +0; copied uncovered rows carry y_i.  Top K
// by (key desc, index asc): the positive copies sorted, then the zero-valued
// rows in index order (a copied +-0 keeps its own bits).  Copies of more than
// kCap rows are flagged for the fallback.
__global__ void __launch_bounds__(256) k9t_empty_kernel(int64_t n, const int32_t* __restrict__ ccount,
                                                        const double* __restrict__ eta, int copy,
                                                        const int64_t* __restrict__ y_ptr,
                                                        const int64_t* __restrict__ y_idx,
                                                        const float* __restrict__ y_val, int64_t K,
                                                        int64_t* __restrict__ out_idx, float* __restrict__ out_val,
                                                        int* __restrict__ nflag, int* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char dyn[];
  uint64_t* pkey = (uint64_t*)dyn;          // positives: key, row
  int64_t* prow = (int64_t*)(pkey + kCap);
  uint64_t* zkey = (uint64_t*)(prow + kCap);  // all copies by row: key = ~row (ascending row), value bits
  int64_t* zval = (int64_t*)(zkey + kCap);
  __shared__ unsigned npos, ncop;
  const int64_t q = blockIdx.x;
  if (ccount[q] != kEmpty) return;
  if (threadIdx.x == 0) npos = ncop = 0;
  __syncthreads();
  if (copy && eta)
    for (int64_t t = y_ptr[q] + threadIdx.x; t < y_ptr[q + 1]; t += blockDim.x) {
      const int64_t i = y_idx[t];
      if (eta[i] != 0.0) continue;
      const float v = y_val[t];
      const unsigned s = atomicAdd(&ncop, 1u);
      if (s < (unsigned)kCap) {
        zkey[s] = ~(uint64_t)i;  // bitonic_sort is descending in key: ~row gives ascending rows
        zval[s] = (int64_t)__float_as_uint(v);
      }
      if (topk::order_key(v) > topk::order_key(0.f)) {
        const unsigned p = atomicAdd(&npos, 1u);
        if (p < (unsigned)kCap) {
          pkey[p] = topk::order_key(v);
          prow[p] = i;
        }
      }
    }
  __syncthreads();
  if (ncop > (unsigned)kCap) {
    if (threadIdx.x == 0) flags[atomicAdd(nflag, 1)] = (int)q;
    return;
  }
  const int np = (int)npos, nc = (int)ncop;
  topk::bitonic_sort(pkey, prow, np);
  topk::bitonic_sort(zkey, zval, nc);
  for (int64_t m = threadIdx.x; m < (np < K ? (int64_t)np : K); m += blockDim.x) {
    out_idx[q * K + m] = prow[m];
    out_val[q * K + m] = prune::key_to_float(pkey[m]);
  }
  if (threadIdx.x == 0) {
    // zero-valued rows in index order, skipping the positive copies; copies
    // are walked in ascending row order alongside
    int c = 0;
    int64_t i = 0;
    for (int64_t m = np; m < K && i < n; ++i) {
      while (c < nc && (int64_t)~zkey[c] < i) ++c;
      float v = 0.f;
      if (c < nc && (int64_t)~zkey[c] == i) {
        v = __uint_as_float((uint32_t)zval[c]);
        if (topk::order_key(v) != topk::order_key(0.f)) continue;  // a positive (or negative) copy
      }
      out_idx[q * K + m] = i;
      out_val[q * K + m] = v;
      ++m;
    }
  }
}

// --------------------------------------------------------------- fallback --
__global__ void __launch_bounds__(256) k9t_fallback_rows_kernel(
    int64_t n, float* __restrict__ Xt, int64_t ldx, const int64_t* __restrict__ indptr,
    const int32_t* __restrict__ indices, const float* __restrict__ vals, const float* __restrict__ Zs, int64_t ldz,
    const double* __restrict__ eta, int copy, const int64_t* __restrict__ y_ptr, const int64_t* __restrict__ y_idx,
    const float* __restrict__ y_val, const int* __restrict__ nflag, const int* __restrict__ flags) {
  const int nf = *nflag;
  if (!nf) return;
  const int64_t nblk = (n + 255) / 256;
  for (int64_t item = blockIdx.x; item < nf * nblk; item += gridDim.x) {
    const int64_t q = flags[item / nblk];
    const int64_t i = (item % nblk) * 256 + threadIdx.x;
    if (i < n) Xt[q * ldx + i] = exact_row(i, q, indptr, indices, vals, Zs, ldz, eta, copy, y_ptr, y_idx, y_val);
  }
}

// ------------------------------------------------------------ host side --
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  return fn;
}

// rows x cols fp16 (row pitch ld elements), box = 64 x box_rows, SWIZZLE_128B; OOB reads zero
int make_map_f16(fsr_ctx* ctx, CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld,
                 int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return set_error(ctx, FSR_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult res = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)base, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (res != CUDA_SUCCESS) return set_error(ctx, FSR_ECUDA, "cuTensorMapEncodeTiled (fp16) failed (%d)", (int)res);
  return FSR_OK;
}

inline size_t al256(size_t x) { return (x + 255) / 256 * 256; }

struct DenseLayout {
  __half* Ud;
  float* cb;
  int* cmax_bits;
};
inline DenseLayout dense_layout(void* base, int64_t n, int64_t r) {
  char* p = (char*)base;
  DenseLayout L;
  L.Ud = (__half*)p;
  p += al256((size_t)n * ld_of(r) * 2);
  L.cb = (float*)p;
  p += al256((size_t)n * 4);
  L.cmax_bits = (int*)p;
  return L;
}
inline size_t dense_bytes(int64_t n, int64_t r) { return al256((size_t)n * ld_of(r) * 2) + al256((size_t)n * 4) + 256; }

constexpr int kCluster = 4;  // CTAs per cluster sharing a query tile (B multicast)

inline int64_t sample_rows(int64_t n) {
  const int64_t tiles_m = (n + BM - 1) / BM;
  const int64_t s_tiles = (tiles_m + kSampleStride - 1) / kSampleStride;
  const int64_t rows1 = (s_tiles + kCluster - 1) / kCluster * kCluster * BM;  // whole clusters of sampled tiles
  // the 2-SM pass samples 256-row tiles
  const int64_t tiles_m2 = (n + sm2::BM2 - 1) / sm2::BM2;
  const int64_t rows2 = (tiles_m2 + sm2::kSample2 - 1) / sm2::kSample2 * sm2::BM2;
  return std::max(rows1, rows2);
}

// persistent grid: as many whole clusters as fit at once (1 CTA per SM)
template <int CL, int TN, bool M2 = false>
int cluster_grid(fsr_ctx* ctx) {
  static int cached[64] = {0};
  int& g = cached[ctx->device & 63];
  constexpr int SMEM = TileCfg<TN>::SMEM;
  if (g) return g;
  if (ensure_smem(ctx, k9t_gemm_kernel<1, CL, TN, M2>, SMEM) != FSR_OK) return -1;
  if (ensure_smem(ctx, k9t_gemm_kernel<0, CL, TN, M2>, SMEM) != FSR_OK) return -1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ctx->num_sms / CL * CL));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = SMEM;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, k9t_gemm_kernel<1, CL, TN, M2>, &cfg) != cudaSuccess ||
      nclusters < 1) {
    cudaGetLastError();
    nclusters = ctx->num_sms / CL;
  }
  g = nclusters * CL;
  return g;
}

template <int MODE, int CL, int TN, bool M2 = false>
int launch_gemm(fsr_ctx* ctx, int grid, const CUtensorMap& mA, const CUtensorMap& mB, int n, int b, int r,
                int tiles_n, int band, int total, const float* cb, const float2* qp, const QParam* qpar,
                const uint32_t* thr, uint32_t* Ks, int64_t ns, int32_t* cand, float* cval, int32_t* ccount,
                unsigned* nlow) {
  constexpr int SMEM = TileCfg<TN>::SMEM;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FSR_CUDA(ctx, cudaLaunchKernelEx(&cfg, k9t_gemm_kernel<MODE, CL, TN, M2>, mA, mB, n, b, r, tiles_n, band, total, cb, qp,
                                   qpar, thr, Ks, ns, cand, cval, ccount, nlow));
  return launched(ctx, MODE == 0 ? "k9t_gemm_sample" : "k9t_gemm_select");
}

struct Work {
  int* nflag;  // [0] = flagged count, [1 .. b] = flagged queries (first, so the host can read it)
  float* Zt;
  float* Zs;
  __half* Zh;
  float2* qp;
  QParam* qpar;
  uint32_t* Ks;
  uint32_t* thr;
  int32_t* ccount;
  unsigned* nlow;
  int32_t* cand;
  float* cval;
  float* cex;   // small batches: exact scores of every candidate, computed by k9t_rescore_kernel (else null)
  int2* stats;  // per query (candidates, rows re-scored): diagnostics
  float* Xt;
};
constexpr int64_t kPreScoreMaxB = 64;  // batches up to this size re-score all candidates on many CTAs (b = 1024: 1.0 ms vs finish 0.46 ms)
// ks_rows: sample keys per query (K9t: sample_rows(n); the streaming path: n)
inline size_t work_bytes(int64_t n, int64_t r, int64_t b, Work* w, void* base, int64_t ks_rows) {
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* q = p ? p + off : nullptr;
    off += al256(bytes);
    return q;
  };
  Work W;
  W.nflag = (int*)take((size_t)(b + 2) * 4);
  W.stats = (int2*)take((size_t)b * 8);
  W.Zt = (float*)take((size_t)b * r * 4);
  W.Zs = (float*)take((size_t)r * b * 4);
  W.Zh = (__half*)take((size_t)b * ld_of(r) * 2);
  W.qp = (float2*)take((size_t)b * 8);
  W.qpar = (QParam*)take((size_t)b * sizeof(QParam));
  W.thr = (uint32_t*)take((size_t)b * 4);
  W.ccount = (int32_t*)take((size_t)b * 4);
  W.nlow = (unsigned*)take((size_t)b * 4);
  W.cand = (int32_t*)take((size_t)b * kCap * 4);
  W.cval = (float*)take((size_t)b * kCap * 4);
  W.cex = b <= kPreScoreMaxB ? (float*)take((size_t)b * kCap * 4) : nullptr;
  W.Ks = (uint32_t*)take((size_t)b * ks_rows * 4);  // sample keys: last but one (their count differs by path)
  W.Xt = (float*)take((size_t)n * b * 4);
  if (w) *w = W;
  return off + 256;
}

// sample GEMM -> threshold -> selecting GEMM, with CL-CTA clusters (M2: the
// 2-D multicast 2 x 2 clusters; needs an even number of query tiles)
template <int CL, int TN, bool M2 = false>
int tc_gemms(fsr_ctx* ctx, const DenseLayout& L, const Work& Wk, int64_t n, int64_t r, int64_t b, int64_t topk) {
  const int64_t ldr = ld_of(r);
  CUtensorMap mA, mB;
  FSR_TRY(make_map_f16(ctx, &mA, L.Ud, n, r, ldr, M2 ? BM / 2 : BM));
  FSR_TRY(make_map_f16(ctx, &mB, Wk.Zh, b, r, ldr, M2 ? TN / 2 : TN / CL));
  const int grid = cluster_grid<CL, TN, M2>(ctx);
  if (grid <= 0) return set_error(ctx, FSR_ECUDA, "filter_topk_tc: no co-resident %d-CTA clusters", CL);
  const int tiles_m = (int)((n + BM - 1) / BM), tiles_n = (int)((b + TN - 1) / TN);
  // query tiles per raster band: their fp16 Zh within ~32 MB of L2
  const int band = (int)std::max<int64_t>(1, std::min<int64_t>(tiles_n, (32ll << 20) / ((int64_t)TN * ldr * 2)));
  const int64_t ns = sample_rows(n);
  const int s_tiles = (tiles_m + kSampleStride - 1) / kSampleStride;
  {
    StageTimer timer(ctx, FSR_STAGE_TOPK);
    // work items per cluster
    const int total0 = M2 ? (s_tiles + 1) / 2 * (tiles_n / 2) : (s_tiles + CL - 1) / CL * tiles_n;
    FSR_TRY((launch_gemm<0, CL, TN, M2>(ctx, grid, mA, mB, (int)n, (int)b, (int)r, tiles_n, band, total0, L.cb, Wk.qp,
                                    nullptr, nullptr, Wk.Ks, ns, nullptr, nullptr, nullptr, nullptr)));
    // rows of the last sampled tile beyond n hold no key: count only valid rows
    const int64_t last_tile = (int64_t)(s_tiles - 1) * kSampleStride;
    const int64_t n_valid_s = (int64_t)(s_tiles - 1) * BM + std::min<int64_t>(BM, n - last_tile * BM);
    const int64_t target = (2 * topk + kSampleStride - 1) / kSampleStride + 8;
    k9t_threshold_kernel<<<(unsigned)std::min<int64_t>(b, (int64_t)ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        b, ns, n_valid_s, Wk.Ks, Wk.qp, L.cmax_bits, target, Wk.thr, Wk.qpar, Wk.ccount, Wk.nlow, Wk.nflag,
        Wk.nflag + 1, nullptr);
    FSR_TRY(launched(ctx, "k9t_threshold_kernel"));
  }
  {
    StageTimer timer(ctx, FSR_STAGE_FILTER_SPMM);
    const int total1 = M2 ? (tiles_m + 1) / 2 * (tiles_n / 2) : (tiles_m + CL - 1) / CL * tiles_n;
    FSR_TRY((launch_gemm<1, CL, TN, M2>(ctx, grid, mA, mB, (int)n, (int)b, (int)r, tiles_n, band, total1, L.cb, Wk.qp,
                                    Wk.qpar, Wk.thr, nullptr, 0, Wk.cand, Wk.cval, Wk.ccount, Wk.nlow)));
  }
  return FSR_OK;
}

// 2-SM main pass (sm2::k9t_gemm2sm_kernel): 4-CTA clusters = 2 CTA pairs
template <int MODE>
int launch_gemm2sm(fsr_ctx* ctx, int grid, const CUtensorMap& mA, const CUtensorMap& mB, int n, int b, int r,
                   int tiles_np, int total, const float* cb, const float2* qp, const QParam* qpar,
                   const uint32_t* thr, uint32_t* Ks, int64_t ns, int32_t* cand, float* cval, int32_t* ccount,
                   unsigned* nlow) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sm2::SMEM2;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 4;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  FSR_CUDA(ctx, cudaLaunchKernelEx(&cfg, sm2::k9t_gemm2sm_kernel<MODE>, mA, mB, n, b, r, tiles_np, total, cb, qp, qpar,
                                   thr, Ks, ns, cand, cval, ccount, nlow));
  return launched(ctx, MODE == 0 ? "k9t_gemm2sm_sample" : "k9t_gemm2sm_select");
}

inline int grid2sm(fsr_ctx* ctx) {
  static int cached[64] = {0};
  int& g = cached[ctx->device & 63];
  if (g) return g;
  if (ensure_smem(ctx, sm2::k9t_gemm2sm_kernel<1>, sm2::SMEM2) != FSR_OK) return -1;
  if (ensure_smem(ctx, sm2::k9t_gemm2sm_kernel<0>, sm2::SMEM2) != FSR_OK) return -1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ctx->num_sms / 4 * 4));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sm2::SMEM2;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 4;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, sm2::k9t_gemm2sm_kernel<1>, &cfg) != cudaSuccess || nclusters < 1) {
    cudaGetLastError();
    nclusters = ctx->num_sms / 4;
  }
  g = nclusters * 4;
  return g;
}

// sample GEMM -> threshold -> selecting GEMM on the 2-SM pass (an even number of 256-query tiles)
inline int tc_gemms_2sm(fsr_ctx* ctx, const DenseLayout& L, const Work& Wk, int64_t n, int64_t r, int64_t b,
                        int64_t topk) {
  using namespace sm2;
  const int64_t ldr = ld_of(r);
  CUtensorMap mA, mB;
  FSR_TRY(make_map_f16(ctx, &mA, L.Ud, n, r, ldr, 64));
  FSR_TRY(make_map_f16(ctx, &mB, Wk.Zh, b, r, ldr, 128));
  const int grid = grid2sm(ctx);
  if (grid <= 0) return set_error(ctx, FSR_ECUDA, "filter_topk_tc: no co-resident 4-CTA clusters (2-SM)");
  const int tiles_m2 = (int)((n + BM2 - 1) / BM2), tiles_np = (int)((b + TN2 - 1) / TN2) / 2;
  const int64_t ns = sample_rows(n);
  const int s_tiles2 = (tiles_m2 + kSample2 - 1) / kSample2;
  {
    StageTimer timer(ctx, FSR_STAGE_TOPK);
    FSR_TRY((launch_gemm2sm<0>(ctx, grid, mA, mB, (int)n, (int)b, (int)r, tiles_np, s_tiles2 * tiles_np, L.cb, Wk.qp,
                               nullptr, nullptr, Wk.Ks, ns, nullptr, nullptr, nullptr, nullptr)));
    const int64_t last_tile = (int64_t)(s_tiles2 - 1) * kSample2;
    const int64_t n_valid_s = (int64_t)(s_tiles2 - 1) * BM2 + std::min<int64_t>(BM2, n - last_tile * BM2);
    const int64_t target = (2 * topk + kSampleStride - 1) / kSampleStride + 8;
    k9t_threshold_kernel<<<(unsigned)std::min<int64_t>(b, (int64_t)ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        b, ns, n_valid_s, Wk.Ks, Wk.qp, L.cmax_bits, target, Wk.thr, Wk.qpar, Wk.ccount, Wk.nlow, Wk.nflag,
        Wk.nflag + 1, nullptr);
    FSR_TRY(launched(ctx, "k9t_threshold_kernel"));
  }
  {
    StageTimer timer(ctx, FSR_STAGE_FILTER_SPMM);
    FSR_TRY((launch_gemm2sm<1>(ctx, grid, mA, mB, (int)n, (int)b, (int)r, tiles_np, tiles_m2 * tiles_np, L.cb, Wk.qp,
                               Wk.qpar, Wk.thr, nullptr, 0, Wk.cand, Wk.cval, Wk.ccount, Wk.nlow)));
  }
  return FSR_OK;
}

// FSR_K9T_CLUSTER = 1 / 2 / 4 CTAs per cluster (B-tile multicast), 22 = 2 x 2
// clusters with A and B multicast, 42 = 2-SM CTA pairs (cta_group::2) in
// 4-CTA clusters with A multicast across the pairs (default; an odd number of
// 256-query tiles falls back to 2).  C3 b = 1024, same box back to back: 2
// 8.87 ms, 2 x 2 8.41 ms (DRAM reads 26 -> 13 GB per launch, the power cap
// then allows 1.75 instead of 1.41 GHz), 2-SM 7.49 ms (6 stages instead of 4:
// the MMA issuer waited on data ~20% of the time).
inline int cluster_choice() {
  static int c = [] {
    const char* e = getenv("FSR_K9T_CLUSTER");
    const int v = e ? atoi(e) : 42;
    return (v == 1 || v == 2 || v == 4 || v == 22 || v == 42) ? v : 42;
  }();
  return c;
}


// ------------------------------------------------------ small-batch stream --
// K9s: the same certified top-K for batches too small to feed the tensor
// cores (b < 128: K9t would stream the whole 10 GB fp16 U~ for a handful of
// queries; the exact sparse K9 gathers 4-byte fp32 Zs values).  U~ is
// re-packed once per decomposition into 4 bytes per entry -- fp16 value << 16
// | column (r <= 65536): 0.4 GB at C3 2% instead of the 0.8 GB fp32 CSR --
// and streamed from HBM by warp-per-row passes at full occupancy (the b = 1
// exact kernel's shape, spmv_smem_kernel, which reaches ~3 TB/s on the fp32
// CSR).  The NB-query slice of the scaled fp16 Zh sits in shared memory as
// [column][query] (NB r 2 bytes); each entry costs NB fma.rn.f32.f16, the
// warp's partial sums meet in a butterfly reduce-scatter.  The sums differ
// from K9t's only in order, which the bound's gamma_m term covers, and the
// per-row factor c_i is K9t's (it also covers tensor-core accumulation, so it
// is conservative here).  Threshold (on a 1/32 sample of 128-row tiles),
// finish, empty and fallback are K9t's kernels: the top-K is the unpruned
// sequential fp32 top-K bit for bit.
// (A TMA-bulk chunk pipeline with a producer warp was measured slower here:
// one CTA per SM cannot keep enough rows in flight.)
namespace stream {

constexpr int kThreads = 256;
constexpr int kTile = 128;         // sample unit: 128 consecutive rows
constexpr int kSampleStride = 32;  // every 32nd tile

inline int64_t sample_tiles(int64_t n) { return ((n + kTile - 1) / kTile + kSampleStride - 1) / kSampleStride; }
inline int64_t sample_slots(int64_t n) { return sample_tiles(n) * kTile; }
inline int64_t sample_valid(int64_t n) {
  const int64_t st = sample_tiles(n), last = (st - 1) * kSampleStride;
  return (st - 1) * kTile + std::min<int64_t>(kTile, n - last * kTile);
}
inline size_t smem_bytes(int nb, int64_t r) { return (size_t)round_up((int64_t)nb * r * 2, 16) + (size_t)nb * 24; }

struct Layout {
  uint32_t* pk;    // [nnz + 16] fp16 value << 16 | column
  float* cb;       // [n] per-row bound factor (K9t's row_bound)
  int* cmax_bits;  // max c_i (as int bits)
};
inline Layout layout(void* base, int64_t n, int64_t nnz) {
  char* p = (char*)base;
  Layout L;
  L.pk = (uint32_t*)p;
  p += al256((size_t)(nnz + 16) * 4);
  L.cb = (float*)p;
  p += al256((size_t)n * 4);
  L.cmax_bits = (int*)p;
  return L;
}
inline size_t layout_bytes(int64_t n, int64_t nnz) { return al256((size_t)(nnz + 16) * 4) + al256((size_t)n * 4) + 256; }

// warp per row: packed entries + the bound factor of densify_kernel
__global__ void __launch_bounds__(256) pack_kernel(int64_t n, const int64_t* __restrict__ indptr,
                                                   const int32_t* __restrict__ indices, const float* __restrict__ vals,
                                                   uint32_t* __restrict__ pk, float* __restrict__ cb,
                                                   int* __restrict__ cmax_bits) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int cmax = 0;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    const int64_t e0 = indptr[i], e1 = indptr[i + 1];
    float ss = 0.f;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const float v = vals[e];
      ss = __fmaf_ru(v, v, ss);
      pk[e] = ((uint32_t)__half_as_ushort(__float2half_rn(v)) << 16) | (uint32_t)indices[e];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss = __fadd_ru(ss, __shfl_xor_sync(0xffffffffu, ss, o));
    if (lane == 0) {
      const float c = e1 > e0 ? row_bound((double)(e1 - e0), ss) : 0.f;
      cb[i] = c;
      cmax = max(cmax, __float_as_int(c));
    }
  }
  if (lane == 0) atomicMax(cmax_bits, cmax);
}

// acc[q] += u * zh[col][q] for the NB queries (fp16 x fp16 -> fp32, one FHFMA each)
template <int NB>
__device__ __forceinline__ void entry_fma(uint32_t w, const __half* __restrict__ zh, float (&acc)[NB]) {
  const uint16_t u = (uint16_t)(w >> 16);
  const uint32_t col = w & 0xffffu;
  if constexpr (NB == 1) {
    const uint16_t z = __half_as_ushort(zh[col]);
    asm("{ .reg .f16 a, z; mov.b16 a, %1; mov.b16 z, %2; fma.rn.f32.f16 %0, a, z, %0; }"
        : "+f"(acc[0])
        : "h"(u), "h"(z));
  } else if constexpr (NB == 2) {
    prune::fhfma2(reinterpret_cast<const uint32_t*>(zh)[col], u, acc[0], acc[1]);
  } else if constexpr (NB == 4) {
    const uint2 z = reinterpret_cast<const uint2*>(zh)[col];
    prune::fhfma2(z.x, u, acc[0], acc[1]);
    prune::fhfma2(z.y, u, acc[2], acc[3]);
  } else {
    static_assert(NB == 8, "NB in {1, 2, 4, 8}");
    const uint4 z = reinterpret_cast<const uint4*>(zh)[col];
    prune::fhfma2(z.x, u, acc[0], acc[1]);
    prune::fhfma2(z.y, u, acc[2], acc[3]);
    prune::fhfma2(z.z, u, acc[4], acc[5]);
    prune::fhfma2(z.w, u, acc[6], acc[7]);
  }
}

// Butterfly reduce-scatter of M per-lane partial sums over the warp: returns
// the warp sum of output oidx(lane) (lane bits 4, 3, ... most significant first).
template <int M>
__device__ __forceinline__ float reduce_scatter(float (&a)[M], int lane) {
  static_assert(M >= 1 && M <= 32 && (M & (M - 1)) == 0, "M a power of two <= 32");
#pragma unroll
  for (int h = M / 2, off = 16; h >= 1; h >>= 1, off >>= 1) {
    const bool upper = lane & off;
#pragma unroll
    for (int j = 0; j < h; ++j) {
      const float send = upper ? a[j] : a[j + h];
      const float keep = upper ? a[j + h] : a[j];
      a[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
#pragma unroll
  for (int off = 16 / M; off >= 1; off >>= 1) a[0] += __shfl_xor_sync(0xffffffffu, a[0], off);
  return a[0];
}
template <int M>
__device__ __forceinline__ int oidx(int lane) {
  int o = 0;
#pragma unroll
  for (int t = 0, b = 4; (1 << t) < M; ++t, --b) o = (o << 1) | ((lane >> b) & 1);
  return o;
}

// rows summed together per warp step (R rows x NB queries partial sums, one reduce-scatter)
template <int NB>
constexpr int rows_per_step() { return NB <= 2 ? 4 : 2; }  // R = 8 for NB = 1 measured slower (0.33 vs 0.23 ms)

// MODE 0 (sample): the rows of every 32nd 128-row tile, lower keys into
//   Ks[q * ns + slot] (slot = sampled tile * 128 + row in tile).
// MODE 1 (select): every row; counts lower >= t, appends rows with upper >= t.
// Queries q0 .. q0 + nq - 1 (nq <= NB).  A warp takes 32 consecutive rows:
// their indptr / c_i in one coalesced load, then R rows at a time with all
// their entries' loads in flight before any is used (the per-row dependent
// global loads of a warp-per-row loop left it latency-bound at ~1.4 TB/s).
template <int MODE, int NB>
__global__ void __launch_bounds__(kThreads)
    stream_kernel(const uint32_t* __restrict__ pk, const int64_t* __restrict__ indptr, int64_t n, int r,
                  const __half* __restrict__ Zh, int64_t ldzh, int q0, int nq, const float* __restrict__ cb,
                  const float2* __restrict__ qp, const QParam* __restrict__ qpar, const uint32_t* __restrict__ thr,
                  uint32_t* __restrict__ Ks, int64_t ns, int32_t* __restrict__ cand, float* __restrict__ cval,
                  int32_t* __restrict__ ccount, unsigned* __restrict__ nlow) {
  constexpr int R = rows_per_step<NB>(), M = R * NB;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __half* zh = (__half*)smem_raw;                                                   // [r][NB]
  float4* sp = (float4*)(smem_raw + round_up((int64_t)NB * r * 2, 16));            // [NB]
  uint32_t* sthr = (uint32_t*)(sp + NB);                                           // [NB]
  unsigned* scnt = sthr + NB;                                                      // [NB]
  // the queries' fp16 Zh slice as [column][query] (padding queries zero) and their parameters
  for (int64_t t = threadIdx.x; t < (int64_t)r * NB; t += kThreads) {
    const int q = (int)(t % NB);
    const int64_t col = t / NB;
    zh[t] = q < nq ? Zh[(int64_t)(q0 + q) * ldzh + col] : __float2half_rn(0.f);
  }
  if (threadIdx.x < NB) {
    const int q = threadIdx.x;
    float4 p = make_float4(__int_as_float(0x7fffffff), 1.f, 0.f, 0.f);
    uint32_t tk = 0xffffffffu;
    if (q < nq) {
      if (MODE == 0) {
        const float2 v = qp[q0 + q];
        p = make_float4(0.f, v.x, 0.f, v.y);
      } else {
        const QParam v = qpar[q0 + q];
        p = make_float4(v.tf_pre, v.inv, v.cz, v.zb);
        tk = thr[q0 + q];
      }
    }
    sp[q] = p;
    sthr[q] = tk;
    scnt[q] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int my = oidx<M>(lane);  // this lane's output after the reduce-scatter: row my / NB, query my % NB
  const int my_r = my / NB, my_q = my % NB;
  const bool leader = (lane & (32 / M - 1)) == 0 && my_q < nq;
  // rows per warp block: 32 for the main pass; 8 for the sample pass (1/32 of
  // the rows -- smaller blocks keep enough warps in flight)
  constexpr int RB = MODE == 0 ? 8 : 32;
  const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
  const int64_t blocks = ((MODE == 0 ? ns : n) + RB - 1) / RB;
  auto first_row = [&](int64_t blk) {
    const int64_t t0 = blk * RB;  // MODE 0: sample slot of the block's first row
    return MODE == 0 ? (t0 / kTile) * kSampleStride * kTile + t0 % kTile : t0;
  };
  // the block's indptr / c_i, loaded one block ahead (their latency overlaps the current block's rows)
  int64_t lo_n = 0;
  int len_n = 0;
  float cl_n = 0.f;
  auto fetch = [&](int64_t blk) {
    lo_n = 0;
    len_n = 0;
    cl_n = 0.f;
    const int64_t il = first_row(blk) + lane;
    if (blk < blocks && lane < RB && il < n) {
      lo_n = __ldg(indptr + il);
      len_n = (int)(__ldg(indptr + il + 1) - lo_n);
      cl_n = __ldg(cb + il);
    }
  };
  fetch(((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5);
  for (int64_t blk = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5; blk < blocks; blk += nw) {
    const int64_t t0 = blk * RB;
    const int64_t i0 = first_row(blk);
    const int64_t lo = lo_n;
    const int len_l = len_n;
    const float cl = cl_n;
    fetch(blk + nw);
    if (i0 >= n) continue;  // warp-uniform: the last sampled tile's rows past n
#pragma unroll 1
    for (int jj = 0; jj < RB && i0 + jj < n; jj += R) {
      const uint32_t* rp[R];
      int len[R];
      int maxlen = 0;
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        rp[rr] = pk + __shfl_sync(0xffffffffu, lo, jj + rr);
        len[rr] = __shfl_sync(0xffffffffu, len_l, jj + rr);  // 0 for rows past n
        maxlen = max(maxlen, len[rr]);
      }
      float acc[M];
#pragma unroll
      for (int m = 0; m < M; ++m) acc[m] = 0.f;
      for (int off = lane; off < maxlen; off += 64) {  // two entries per row per lane in flight
        uint32_t w0[R], w1[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          w0[rr] = off < len[rr] ? __ldg(rp[rr] + off) : 0u;
          w1[rr] = off + 32 < len[rr] ? __ldg(rp[rr] + off + 32) : 0u;
        }
#pragma unroll
        for (int rr = 0; rr < R; ++rr) {
          FSR_DCHECK(!(off < len[rr]) || (int)(w0[rr] & 0xffffu) < r);
          FSR_DCHECK(!(off + 32 < len[rr]) || (int)(w1[rr] & 0xffffu) < r);
          if (off < len[rr]) entry_fma<NB>(w0[rr], zh, *reinterpret_cast<float(*)[NB]>(acc + rr * NB));
          if (off + 32 < len[rr]) entry_fma<NB>(w1[rr], zh, *reinterpret_cast<float(*)[NB]>(acc + rr * NB));
        }
      }
      float c_my = 0.f;
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        const float c = __shfl_sync(0xffffffffu, cl, jj + rr);
        if (rr == my_r) c_my = c;
      }
      const float v = reduce_scatter<M>(acc, lane);
      const int64_t i = i0 + jj + my_r;
      if (leader && jj + my_r < RB && i < n) {
        const float4 p = sp[my_q];
        const float x = v * p.y;
        if (MODE == 0) {
          FSR_DCHECK(t0 + jj + my_r < ns);
          Ks[(int64_t)(q0 + my_q) * ns + t0 + jj + my_r] = prune::key32(__fsub_rd(x, prune::bound_of(c_my, p.w)));
        } else if (x + p.z >= p.x) {  // rare: within reach of the threshold
          const float bd = prune::bound_of(c_my, p.w);
          const uint32_t tk = sthr[my_q];
          if (prune::key32(__fsub_rd(x, bd)) >= tk) atomicAdd(&scnt[my_q], 1u);
          if (prune::key32(__fadd_ru(x, bd)) >= tk) {
            const int slot = atomicAdd(ccount + q0 + my_q, 1);
            if (slot < kCap) {
              cand[(int64_t)(q0 + my_q) * kCap + slot] = (int32_t)i;
              cval[(int64_t)(q0 + my_q) * kCap + slot] = x;
            }
          }
        }
      }
    }
  }
  __syncthreads();
  if (MODE == 1 && threadIdx.x < nq && scnt[threadIdx.x]) atomicAdd(nlow + q0 + threadIdx.x, scnt[threadIdx.x]);
}

// queries per pass: FSR_K9S_NB (1/2/4/8) or the largest NB <= b, at most 8, whose Zh slice fits
inline int pick_nb(int64_t b, int64_t r) {
  static int forced = [] {
    const char* e = getenv("FSR_K9S_NB");
    const int v = e ? atoi(e) : 0;
    return (v == 1 || v == 2 || v == 4 || v == 8) ? v : 0;
  }();
  for (int nb = 8; nb >= 1; nb >>= 1)
    if ((forced ? nb <= forced : nb <= b || nb == 1) && smem_bytes(nb, r) <= 200 * 1024) return nb;
  return 0;
}

template <int MODE, int NB>
int launch(fsr_ctx* ctx, const Layout& L, const Work& Wk, const int64_t* indptr, int64_t n, int64_t r, int q0,
           int nq) {
  const size_t smem = smem_bytes(NB, r);
  FSR_TRY(ensure_smem(ctx, stream_kernel<MODE, NB>, smem));
  static int per_sm[2][9] = {};
  int& occ = per_sm[MODE][NB];
  if (!occ) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stream_kernel<MODE, NB>, kThreads, smem) != cudaSuccess ||
        occ < 1) {
      cudaGetLastError();
      occ = 1;
    }
  }
  const int64_t ns = sample_slots(n);
  const int64_t rows = MODE == 0 ? ns : n;
  const int rows_per_cta = (MODE == 0 ? 8 : 32) * (kThreads / 32);
  const int grid =
      (int)std::max<int64_t>(1, std::min<int64_t>((rows + rows_per_cta - 1) / rows_per_cta, (int64_t)ctx->num_sms * occ));
  stream_kernel<MODE, NB><<<grid, kThreads, smem, ctx->stream>>>(L.pk, indptr, n, (int)r, Wk.Zh, ld_of(r), q0, nq,
                                                                 L.cb, Wk.qp, Wk.qpar, Wk.thr, Wk.Ks, ns, Wk.cand,
                                                                 Wk.cval, Wk.ccount, Wk.nlow);
  return launched(ctx, MODE == 0 ? "k9s_stream_sample" : "k9s_stream_select");
}

template <int MODE>
int launch_groups(fsr_ctx* ctx, const Layout& L, const Work& Wk, const int64_t* indptr, int64_t n, int64_t r,
                  int64_t b) {
  const int nb = pick_nb(b, r);
  for (int64_t q0 = 0; q0 < b; q0 += nb) {
    const int nq = (int)std::min<int64_t>(nb, b - q0);
    if (nb == 8)
      FSR_TRY((launch<MODE, 8>(ctx, L, Wk, indptr, n, r, (int)q0, nq)));
    else if (nb == 4)
      FSR_TRY((launch<MODE, 4>(ctx, L, Wk, indptr, n, r, (int)q0, nq)));
    else if (nb == 2)
      FSR_TRY((launch<MODE, 2>(ctx, L, Wk, indptr, n, r, (int)q0, nq)));
    else
      FSR_TRY((launch<MODE, 1>(ctx, L, Wk, indptr, n, r, (int)q0, nq)));
  }
  return FSR_OK;
}

}  // namespace stream


// finish (exact re-score of the kept candidates, sort), empty observations,
// fallback: shared by K9t and the streaming path
inline int finish_stage(fsr_ctx* ctx, const float* cb, const Work& Wk, int64_t n, int64_t r, int64_t b, const int64_t* u_indptr,
                        const int32_t* u_indices, const float* u_values, const double* eta, int copy,
                        const int64_t* y_ptr, const int64_t* y_idx, const float* y_val, int64_t topk,
                        int64_t* top_idx, float* top_val) {
  {
    StageTimer timer(ctx, FSR_STAGE_TOPK);
    const size_t fsm = finish_smem(r);
    FSR_TRY(ensure_smem(ctx, k9t_finish_kernel, fsm));
    if (Wk.cex) {
      k9t_rescore_kernel<<<(unsigned)std::min<int64_t>((b * kCap * 8 + 255) / 256, (int64_t)ctx->num_sms * 8), 256,
                           0, ctx->stream>>>(b, Wk.cand, Wk.ccount, u_indptr, u_indices, u_values, Wk.Zs, b, eta,
                                             copy, y_ptr, y_idx, y_val, Wk.cex);
      FSR_TRY(launched(ctx, "k9t_rescore_kernel"));
    }
    k9t_finish_kernel<<<(unsigned)b, kFinishThreads, fsm, ctx->stream>>>(
        cb, Wk.qpar, Wk.thr, Wk.cand, Wk.cval, Wk.ccount, Wk.nlow, u_indptr, u_indices, u_values, Wk.Zs, b, Wk.Zt,
        r, eta, copy, y_ptr, y_idx, y_val, topk, top_idx, top_val, Wk.nflag, Wk.nflag + 1, Wk.stats, Wk.cex);
    FSR_TRY(launched(ctx, "k9t_finish_kernel"));
    const size_t esm = (size_t)kCap * 32;
    FSR_TRY(ensure_smem(ctx, k9t_empty_kernel, esm));
    k9t_empty_kernel<<<(unsigned)b, 256, esm, ctx->stream>>>(n, Wk.ccount, eta, copy, y_ptr, y_idx, y_val, topk,
                                                           top_idx, top_val, Wk.nflag, Wk.nflag + 1);
    FSR_TRY(launched(ctx, "k9t_empty_kernel"));
    k9t_fallback_rows_kernel<<<(unsigned)ctx->num_sms * 8, 256, 0, ctx->stream>>>(
        n, Wk.Xt, n, u_indptr, u_indices, u_values, Wk.Zs, b, eta, copy, y_ptr, y_idx, y_val, Wk.nflag,
        Wk.nflag + 1);
    FSR_TRY(launched(ctx, "k9t_fallback_rows_kernel"));
    const size_t fsmem = (size_t)topk::kCap * 16;
    FSR_TRY(ensure_smem(ctx, prune::fallback_select_kernel, fsmem));
    prune::fallback_select_kernel<<<(unsigned)b, topk::kThreads, fsmem, ctx->stream>>>(
        n, Wk.Xt, n, topk, top_idx, top_val, Wk.nflag, Wk.nflag + 1);
    FSR_TRY(launched(ctx, "fallback_select_kernel"));
  }
  return FSR_OK;
}

}  // namespace k9t

// K8 with the fp16 query-major Zh (k8_online.cu)
int k9t_project(fsr_ctx* ctx, int64_t r, int64_t b, const int64_t* u_indptr, const int32_t* u_indices,
                const float* u_values, const float* w, const int64_t* y_ptr, const int64_t* y_idx,
                const float* y_val, float* Zt, float* Zs, __half* Zh, int64_t ldzh, float2* qp, int* nflag);

}  // namespace fsr

using namespace fsr;

extern "C" {

int64_t fsr_dense_u_bytes(int64_t n, int64_t r) { return (int64_t)k9t::dense_bytes(n, r); }

int fsr_dense_u_build(fsr_ctx* ctx, int64_t n, int64_t r, const int64_t* indptr, const int32_t* indices,
                      const float* values, void* out) {
  FSR_REQUIRE(ctx, n >= 1 && r >= 1 && indptr && indices && values && out, "dense_u_build: bad args");
  FSR_REQUIRE(ctx, aligned(out, 256), "dense_u_build: out must be 256-byte aligned");
  k9t::DenseLayout L = k9t::dense_layout(out, n, r);
  FSR_CUDA(ctx, cudaMemsetAsync(out, 0, k9t::dense_bytes(n, r), ctx->stream));
  k9t::densify_kernel<<<grid_for(n * 32, 256, ctx, 8), 256, 0, ctx->stream>>>(n, k9t::ld_of(r), indptr, indices,
                                                                             values, L.Ud, L.cb, L.cmax_bits);
  return launched(ctx, "densify_kernel");
}

int64_t fsr_filter_tc_workspace_bytes(int64_t n, int64_t r, int64_t b) {
  return (int64_t)k9t::work_bytes(n, r, b, nullptr, nullptr, k9t::sample_rows(n));
}

int fsr_filter_tc_applicable(int64_t n, int64_t r, int64_t b, int64_t topk) {
  return n >= 8 * k9t::BM * k9t::kSampleStride && n < ((int64_t)1 << 31) - 4096 && r >= 1 && r <= 32768 && b >= 1 &&
         topk >= 1 && topk <= k9t::kCap / 8 && topk <= n;
}

int fsr_filter_topk_tc(fsr_ctx* ctx, int64_t n, int64_t r, const int64_t* u_indptr, const int32_t* u_indices,
                       const float* u_values, const void* dense_u, const float* w, const double* eta, int64_t b,
                       const int64_t* y_ptr, const int64_t* y_idx, const float* y_val, int copy_uncovered,
                       void* workspace, int64_t topk, int64_t* top_idx, float* top_val) {
  using namespace k9t;
  FSR_REQUIRE(ctx, fsr_filter_tc_applicable(n, r, b, topk), "filter_topk_tc: shape outside the tensor-core path");
  FSR_REQUIRE(ctx, u_indptr && u_indices && u_values && dense_u && workspace && top_idx && top_val,
              "filter_topk_tc: missing argument");
  FSR_REQUIRE(ctx, aligned(dense_u, 256) && aligned(workspace, 256), "filter_topk_tc: buffers must be 256-aligned");
  const DenseLayout L = dense_layout(const_cast<void*>(dense_u), n, r);
  Work Wk;
  work_bytes(n, r, b, &Wk, workspace, sample_rows(n));
  const int64_t ldr = ld_of(r);
  const int copy = copy_uncovered && eta;
  // K8: Zt, Zs (fp32) and the query-major fp16 Zh with per-query scale
  FSR_TRY(k9t_project(ctx, r, b, u_indptr, u_indices, u_values, w, y_ptr, y_idx, y_val, Wk.Zt, Wk.Zs, Wk.Zh, ldr,
                      Wk.qp, Wk.nflag));
  const int cl = cluster_choice();
  const int tn = b <= 64 ? 64 : b <= 128 ? 128 : 256;  // query tile: no MMA work on padding queries
  if (tn == 64)
    FSR_TRY((cl == 1 ? tc_gemms<1, 64>(ctx, L, Wk, n, r, b, topk)
             : cl == 2 || cl == 22 || cl == 42 ? tc_gemms<2, 64>(ctx, L, Wk, n, r, b, topk)
                                   : tc_gemms<4, 64>(ctx, L, Wk, n, r, b, topk)));
  else if (tn == 128)
    FSR_TRY((cl == 1   ? tc_gemms<1, 128>(ctx, L, Wk, n, r, b, topk)
             : cl == 2 || cl == 22 || cl == 42 ? tc_gemms<2, 128>(ctx, L, Wk, n, r, b, topk)
                       : tc_gemms<4, 128>(ctx, L, Wk, n, r, b, topk)));
  else if (cl == 42 && ((b + 255) / 256) % 2 == 0)
    FSR_TRY(tc_gemms_2sm(ctx, L, Wk, n, r, b, topk));
  else if ((cl == 22 || cl == 42) && ((b + 255) / 256) % 2 == 0)
    FSR_TRY((tc_gemms<4, 256, true>(ctx, L, Wk, n, r, b, topk)));
  else
    FSR_TRY((cl == 1   ? tc_gemms<1, 256>(ctx, L, Wk, n, r, b, topk)
             : cl == 2 || cl == 22 || cl == 42 ? tc_gemms<2, 256>(ctx, L, Wk, n, r, b, topk)
                       : tc_gemms<4, 256>(ctx, L, Wk, n, r, b, topk)));
  return finish_stage(ctx, L.cb, Wk, n, r, b, u_indptr, u_indices, u_values, eta, copy, y_ptr, y_idx, y_val, topk,
                      top_idx, top_val);
}

int fsr_filter_tc_stats(fsr_ctx* ctx, int64_t n, int64_t r, int64_t b, const void* workspace, int32_t* out) {
  FSR_REQUIRE(ctx, workspace && out && b >= 1, "filter_tc_stats: bad args");
  k9t::Work Wk;
  k9t::work_bytes(n, r, b, &Wk, const_cast<void*>(workspace), 0);  // stats precede the sample keys
  FSR_CUDA(ctx, cudaMemcpyAsync(out, Wk.stats, (size_t)b * 8, cudaMemcpyDeviceToHost, ctx->stream));
  FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FSR_OK;
}

int fsr_filter_tc_fallback_count(fsr_ctx* ctx, const void* workspace, int* out) {
  FSR_REQUIRE(ctx, workspace && out, "filter_tc_fallback_count: bad args");
  FSR_CUDA(ctx, cudaMemcpyAsync(out, workspace, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FSR_OK;
}

// ---- small-batch streaming path (K9s) ----
int64_t fsr_stream_u_bytes(int64_t n, int64_t r, int64_t nnz) {
  (void)r;
  return (int64_t)k9t::stream::layout_bytes(n, nnz);
}

int fsr_stream_u_build(fsr_ctx* ctx, int64_t n, int64_t r, int64_t nnz, const int64_t* indptr,
                       const int32_t* indices, const float* values, void* out) {
  using namespace k9t::stream;
  FSR_REQUIRE(ctx, n >= 1 && r >= 1 && r <= 65536 && nnz >= 0 && indptr && out && (nnz == 0 || (indices && values)),
              "stream_u_build: bad args (r <= 65536)");
  FSR_REQUIRE(ctx, n < ((int64_t)1 << 31) - 1, "stream_u_build: n >= 2^31 - 1");
  FSR_REQUIRE(ctx, aligned(out, 256), "stream_u_build: out must be 256-byte aligned");
  const Layout L = layout(out, n, nnz);
  FSR_CUDA(ctx, cudaMemsetAsync(out, 0, layout_bytes(n, nnz), ctx->stream));
  pack_kernel<<<grid_for(n * 32, 256, ctx, 8), 256, 0, ctx->stream>>>(n, indptr, indices, values, L.pk, L.cb,
                                                                      L.cmax_bits);
  return launched(ctx, "stream_pack_kernel");
}

int fsr_filter_stream_applicable(int64_t n, int64_t r, int64_t nnz, int64_t b, int64_t topk) {
  return n >= 1 && n < ((int64_t)1 << 31) - 1 && r >= 1 && r <= 65536 && nnz >= 0 && b >= 1 && topk >= 1 &&
         topk <= k9t::kCap / 8 && topk <= n && k9t::stream::pick_nb(b, r) > 0 &&
         (size_t)r * 4 + 16 + (size_t)4096 * 8 <= 160 * 1024;  // k9t_project (k8_online.cu, kProjCap = 4096)
}

int64_t fsr_filter_stream_workspace_bytes(int64_t n, int64_t r, int64_t b) {
  return (int64_t)k9t::work_bytes(n, r, b, nullptr, nullptr, k9t::stream::sample_slots(n));
}

int fsr_filter_topk_stream(fsr_ctx* ctx, int64_t n, int64_t r, int64_t nnz, const int64_t* u_indptr,
                           const int32_t* u_indices, const float* u_values, const void* stream_u, const float* w,
                           const double* eta, int64_t b, const int64_t* y_ptr, const int64_t* y_idx,
                           const float* y_val, int copy_uncovered, void* workspace, int64_t topk, int64_t* top_idx,
                           float* top_val) {
  using namespace k9t;
  FSR_REQUIRE(ctx, fsr_filter_stream_applicable(n, r, nnz, b, topk), "filter_topk_stream: shape outside the path");
  FSR_REQUIRE(ctx, u_indptr && stream_u && workspace && top_idx && top_val && (nnz == 0 || (u_indices && u_values)),
              "filter_topk_stream: missing argument");
  FSR_REQUIRE(ctx, aligned(stream_u, 256) && aligned(workspace, 256),
              "filter_topk_stream: buffers must be 256-aligned");
  const stream::Layout L = stream::layout(const_cast<void*>(stream_u), n, nnz);
  Work Wk;
  work_bytes(n, r, b, &Wk, workspace, stream::sample_slots(n));
  const int copy = copy_uncovered && eta;
  FSR_TRY(k9t_project(ctx, r, b, u_indptr, u_indices, u_values, w, y_ptr, y_idx, y_val, Wk.Zt, Wk.Zs, Wk.Zh,
                      ld_of(r), Wk.qp, Wk.nflag));
  {
    StageTimer timer(ctx, FSR_STAGE_TOPK);
    FSR_TRY(stream::launch_groups<0>(ctx, L, Wk, u_indptr, n, r, b));
    const int64_t target = (2 * topk + stream::kSampleStride - 1) / stream::kSampleStride + 8;
    k9t_threshold_kernel<<<(unsigned)std::min<int64_t>(b, (int64_t)ctx->num_sms * 8), 256, 0, ctx->stream>>>(
        b, stream::sample_slots(n), stream::sample_valid(n), Wk.Ks, Wk.qp, L.cmax_bits, target, Wk.thr, Wk.qpar,
        Wk.ccount, Wk.nlow, Wk.nflag, Wk.nflag + 1, nullptr);
    FSR_TRY(launched(ctx, "k9t_threshold_kernel"));
  }
  {
    StageTimer timer(ctx, FSR_STAGE_FILTER_SPMM);
    FSR_TRY(stream::launch_groups<1>(ctx, L, Wk, u_indptr, n, r, b));
  }
  return finish_stage(ctx, L.cb, Wk, n, r, b, u_indptr, u_indices, u_values, eta, copy, y_ptr, y_idx, y_val, topk,
                      top_idx, top_val);
}

}  // extern "C"
