// Certified top-k for the online step (K9 + select), fp32 only.
//
// The ranked-query step returns the top K of every x_q = U~ Zs[:, q] in the
// reference's rank order (ranking.py:390-395).  K9 is bound by the L2 -> SM
// gathers of Zs rows (4 bytes per column per nonzero), so
// the pruned path gathers Zs rounded to fp16 (per-query power-of-two scale,
// half the bytes), and then re-scores only the rows that can still be in the
// top K with the fp32 data, in the same order as the unpruned fp32 K9.  The
// returned top-K indices and values are therefore the ones the unpruned fp32
// path returns, bit for bit; fp16 values are never returned.
//
// Bound (row i with m_i entries, query q, rounding unit u = 2^-24): K9h
// multiplies u~ = fp16(u) by zs~ = fp16(zs s_q) / s_q with fp32 accumulation
// (FHFMA), so with du = u~ - u, dz = zs~ - zs,
//   |x_fp32 - x~_fp32| <= sum_j (|u_ij||dz_j| + |du_ij||zs~_j|) + gamma_m (sum |u||zs| + sum |u~||zs~|)
//                      <= ||u_i||_2 ||zs_q||_2 (2 * 2^-11 + 2.01 m_i u) + sqrt(m_i) ||u_i||_2 2^-25 / s_q
//                         + sqrt(m_i) 2^-25 ||zs~_q||_2                        (all to first order)
//                      <= c_i * Zb_q,
//   c_i  = (||u_i||_2 (2^-10 + 2.01 m_i 2^-24 + sqrt(m_i) 2^-38) + sqrt(m_i) 2^-25) * 1.01
//          (K9h, from the row it streams; 1.01 covers the second-order terms)
//   Zb_q = max(||zs_q||_2, 2^13 / s_q)                           (K8 / zs_half_kernel)
// (fp16 rounding is relative 2^-11 for normal values and absolute 2^-25 below
// the normal range; Cauchy-Schwarz bounds every sum.)  With
// lower_i = x~_i - c_i Zb and upper_i = x~_i + c_i Zb (directed rounding), any
// threshold t such that at least K rows have lower >= t satisfies t <= x_(K),
// so {i : upper_i >= t} contains every exact top-K row and every tie at the
// K-th value.  t comes from a 1/16 sample of the lower keys and is verified
// by counting on the full pass; when the count falls short or the candidates
// overflow shared memory the query is flagged and recomputed exactly by the
// fallback kernels (launched always, they exit at once when nothing is
// flagged, so the step stays one CUDA graph).
#pragma once

#include <cuda_fp16.h>

#include <cfloat>


#include "spmm.cuh"
#include "topk.cuh"

namespace fsr {
namespace prune {

constexpr int kExactRows = 1 << 30;  // flag bit: the query's x~ row is exact (z = 0), no recompute
constexpr int kThreads = 256;  // prune_select_kernel: several CTAs per SM overlap their serial phases
constexpr int kCap = 2048;     // candidates per query (typical ~3.7K + band, max seen 844 at C3); more -> fallback

// Scale of one query column from its max |zs| and sum of squares:
// s = 2^(14 - e) with amax < 2^e, 1/s, and Zb = max(||zs||_2 rounded up, 2^13 / s);
// an all-zero column keeps s = 1 and Zb = 0 (its x~ is exact).
__device__ __forceinline__ void query_scale(float amax, double ss, float* s, float* inv, float* zb) {
  *s = 1.f;
  *inv = 1.f;
  *zb = 0.f;
  if (!(amax <= FLT_MAX) || !(ss <= DBL_MAX)) {  // inf / NaN in zs: no bound, exact fallback
    *zb = __int_as_float(0x7fffffff);
    return;
  }
  if (amax > 0.f) {
    int e;
    frexpf(amax, &e);  // amax = f 2^e, f in [0.5, 1)
    const int k = max(-120, min(120, 14 - e));
    *s = ldexpf(1.f, k);
    *inv = ldexpf(1.f, -k);
    const float zn = __double2float_ru(__dsqrt_ru(ss) * (1.0 + 0x1p-40));
    *zb = fmaxf(zn, ldexpf(1.f, 13 - k));
  }
}

// Per query column q of Zs (r x b, ld b): amax, ||zs_q||_2 and the scale
// s_q = 2^(14 - e) with amax < 2^e (so |zs * s| < 2^14); Zh = half(Zs * s).
// qp[q] = {1 / s_q, Zb_q}.  Also clears the fallback counter and max c_i.
static __global__ void __launch_bounds__(256) zs_half_kernel(int64_t r, int64_t b, const float* __restrict__ Zs,
                                                      __half* __restrict__ Zh, float2* __restrict__ qp,
                                                      int* __restrict__ nflag) {
  __shared__ float smax[8][33];
  __shared__ double sss[8][33];
  __shared__ float sscale[32];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t col = (int64_t)blockIdx.x * 32 + tx;
  float amax = 0.f;
  double ss = 0.0;
  if (col < b)
    for (int64_t j = ty; j < r; j += 8) {
      const float v = Zs[j * b + col];
      amax = fmaxf(amax, fabsf(v));
      ss = fma((double)v, (double)v, ss);
    }
  smax[ty][tx] = amax;
  sss[ty][tx] = ss;
  __syncthreads();
  if (ty == 0) {
    for (int k = 1; k < 8; ++k) {
      amax = fmaxf(amax, smax[k][tx]);
      ss += sss[k][tx];
    }
    float s = 1.f, inv = 1.f, zb = 0.f;
    query_scale(amax, ss, &s, &inv, &zb);
    sscale[tx] = s;
    if (col < b) qp[col] = make_float2(inv, zb);
  }
  __syncthreads();
  const float s = sscale[tx];
  if (col < b)
    for (int64_t j = ty; j < r; j += 8) Zh[j * b + col] = __float2half_rn(Zs[j * b + col] * s);
  if (blockIdx.x == 0 && tx == 0 && ty == 0) {
    nflag[0] = 0;
    nflag[b + 1] = 0;  // max_i c_i (float bits), raised by K9h
  }
}

// acc0 += a * lo(pair), acc1 += a * hi(pair): fp32 accumulation of fp16
// products (FHFMA, one instruction per column; no fp16 -> fp32 conversions).
__device__ __forceinline__ void fhfma2(uint32_t pair, uint16_t a, float& acc0, float& acc1) {
  asm("{ .reg .f16 lo, hi, ah; mov.b32 {lo, hi}, %2; mov.b16 ah, %3;\n\t"
      "fma.rn.f32.f16 %0, ah, lo, %0; fma.rn.f32.f16 %1, ah, hi, %1; }"
      : "+f"(acc0), "+f"(acc1)
      : "r"(pair), "h"(a));
}

// 16-byte gather of an fp16 Zs row segment (read-only path; L1-allocating:
// ld.global.nc.L1::no_allocate measured 10% slower, 16.0 vs 14.5 ms at C3).
__device__ __forceinline__ uint4 ld_gather(const __half* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
// The same at base + c * ldxb bytes: one IMAD.WIDE.U32 per address (a 32-bit
// element offset scaled by sizeof(half) afterwards compiled to six integer
// instructions per gather).
__device__ __forceinline__ uint4 ld_gather(const char* base, uint32_t c, uint32_t ldxb) {
  return __ldg(reinterpret_cast<const uint4*>(base + (uint64_t)c * ldxb));
}

// K9h: Xt~ (ncols x n_rows, ld ldy) = (A Zh) .* inv_s over column panels of
// PW = 256 NV columns (8 halves = 16 bytes per lane per vector); the same
// CTA layout as spmm_rowpanel_T_kernel (ROWS rows handed to 8 warps from a
// shared counter, longest first; transposed tile in shared memory).  Panel 0
// also writes the row bound factor c_i and raises max_i c_i.  Requires
// ncols % 8 == 0 and 16-byte aligned Zh rows.
// Measured at C3 2%, b = 1024: NV = 1 (256-column
// panels), DEPTH 8, 4 CTAs/SM (64 registers) 14.8 ms, then 14.5 with the next
// 32 entries prefetched, 13.7 with the rows handed out longest first, 13.1
// with the entries broadcast from shared memory, 11.9 with FHFMA (fp16 u):
// DEPTH 4 at 4 CTAs/SM (64 registers, no spills) 11.90 -- kept -- and DEPTH 8
// at 3 CTAs/SM 11.92, then 11.64 with one IMAD.WIDE.U32 per gather address
// (6 -> 2 integer instructions; 17.6 TB/s of gathers, 88% of the random-row
// L2 probe, so fewer L2 bytes is the remaining lever; with it DEPTH 6 / 8 at
// 4 CTAs/SM still spill, DEPTH 8 at 3 CTAs/SM spills 64 B: 13.74); DEPTH 8 / 10 / 12 spilling at 64-80 registers 14.7 /
// 15.2 / 23.3, DEPTH 16 at 2 CTAs/SM 13.8; DEPTH 4 at 4 / 5 / 6 CTAs/SM 15.7 / 16.4 / 18.1; DEPTH 6 at 5 CTAs/SM
// 16.6; NV = 2 DEPTH 4 at 2 or 3 CTAs/SM 20.5 / 16.5; a barrier-free variant
// (warp-owned 8-row items, persistent grid, per-warp transposes) 19.1-19.4;
// a one-row lookahead in the hand-out 16.5; gathers landing in shared memory
// (cp.async, per-warp rings of 16-32 512-byte slots, up to 224 KB in flight
// per SM, 4-byte direct output writes) 33-41.  FFMA2 on converted half pairs
// and 32-bit row offsets (one IMAD.WIDE per gather) took it from 18.7 to 16.8
// ms on a synthetic U~.  Neither L2 (62%) nor issue (68%) is saturated (ncu,
// profiles/r01/k9h_ncu_full.json): the bytes in flight per SM over the loaded
// L2 latency bound it.  64-row blocks (8 or 16 warps) and 4-warp blocks at 6
// CTAs/SM measured 14.7-15.0 ms; DEPTH 10 / 12 / 16 at 3 CTAs/SM 15.3 / 17.4 /
// 14.6 ms; a predicated last round per chunk (instead of single gathers) spilled
// at 64 registers: 22.5 ms.
template <int NV, int DEPTH, int ROWS, int MINB, int WARPS = 8>
__global__ void __launch_bounds__(32 * WARPS, MINB) spmm_T_half_kernel(int64_t n_rows, const int64_t* __restrict__ indptr,
                                                          const int32_t* __restrict__ indices,
                                                          const float* __restrict__ vals, int64_t ncols,
                                                          const __half* __restrict__ Zh, int64_t ldx,
                                                          const float2* __restrict__ qp, float* __restrict__ Yt,
                                                          int64_t ldy, float* __restrict__ cbound,
                                                          int* __restrict__ cmax_bits) {
  constexpr int PW = 256 * NV;
  extern __shared__ __align__(16) unsigned char dyn_tile[];
  float(*tile)[PW + 1] = reinterpret_cast<float(*)[PW + 1]>(dyn_tile);
  __shared__ int next_row;
  __shared__ int cmax_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row0 = (int64_t)blockIdx.x * ROWS;
  const int64_t p0 = (int64_t)blockIdx.y * PW;
  if (threadIdx.x == 0) cmax_s = 0;
  const int64_t c0 = p0 + (int64_t)lane * 8;
  bool live[NV];
#pragma unroll
  for (int u = 0; u < NV; ++u) live[u] = c0 + u * 256 < ncols;
  // Rows are handed out from a shared counter longest first (row lengths are
  // skewed; handing out the short rows last keeps the warps' finishing times
  // close -- the end-of-block barrier held 21% of the stall samples with the
  // rows in index order).  Within a row the next 32 entries are in flight
  // while the current 32 are summed.
  static_assert(NV == 1, "row loop is written for one 256-column vector per lane");
  static_assert(DEPTH % 2 == 0, "entries are read in pairs");
  static_assert(ROWS % 32 == 0 && ROWS <= 128, "lanes of warp 0 rank the block's rows, ROWS / 32 each");
  constexpr int RPL = ROWS / 32;
  __shared__ int order_s[ROWS];
  __shared__ int64_t start_s[ROWS];
  __shared__ int len_s[ROWS];
  if (warp == 0) {
    int len[RPL];
#pragma unroll
    for (int h = 0; h < RPL; ++h) {
      const int64_t i = row0 + h * 32 + lane;
      int64_t a = 0, z = 0;
      if (i < n_rows) {
        a = __ldg(indptr + i);
        z = __ldg(indptr + i + 1);
      }
      len[h] = (int)(z - a);
      start_s[h * 32 + lane] = a;
      len_s[h * 32 + lane] = len[h];
    }
    int rank[RPL];
#pragma unroll
    for (int h = 0; h < RPL; ++h) rank[h] = 0;
#pragma unroll
    for (int g = 0; g < RPL; ++g)
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const int lk = __shfl_sync(0xffffffffu, len[g], k);
#pragma unroll
        for (int h = 0; h < RPL; ++h)
          rank[h] += (lk > len[h]) || (lk == len[h] && g * 32 + k < h * 32 + lane);
      }
#pragma unroll
    for (int h = 0; h < RPL; ++h) order_s[rank[h]] = h * 32 + lane;
  }
  if (threadIdx.x == 0) next_row = WARPS;
  __syncthreads();
  // per-lane base of its 8 columns; 32-bit column index times the byte stride: one IMAD.WIDE.U32 per gather
  const char* zl = reinterpret_cast<const char*>(Zh + c0);
  const uint32_t ldxb = (uint32_t)ldx * (uint32_t)sizeof(__half);
  __shared__ __align__(16) int2 ent_s[32 * WARPS];
  int2* ent = ent_s + warp * 32;
  int pos = warp;
  int rr = order_s[pos];
  int64_t e0 = start_s[rr], e1 = e0 + len_s[rr];
  int cc = 0;
  float cv = 0.f;
  if (lane < e1 - e0) {
    cc = __ldg(indices + e0 + lane);
    cv = __ldg(vals + e0 + lane);
  }
  while (pos < ROWS) {
    const int64_t i = row0 + rr;
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.f;
    float ss = 0.f;  // sum of squares, rounded up (an upper bound of ||u_i||^2)
    for (int64_t base = e0; base < e1; base += 32) {
      const int m = (e1 - base) < 32 ? (int)(e1 - base) : 32;
      int pc = 0;
      float pv = 0.f;
      if (lane < e1 - base - 32) {
        pc = __ldg(indices + base + 32 + lane);
        pv = __ldg(vals + base + 32 + lane);
      }
      ss = __fmaf_ru(cv, cv, ss);
      // the chunk's (column, value) pairs go through shared memory: one
      // broadcast LDS.128 yields two entries (instead of four shuffles)
      __syncwarp();
      ent[lane] = make_int2(cc, (int)__half_as_ushort(__float2half_rn(cv)));  // u~ = fp16(u)
      __syncwarp();
      int j = 0;
      for (; j + DEPTH <= m; j += DEPTH) {
        uint32_t c[DEPTH];
        uint16_t a[DEPTH];
#pragma unroll
        for (int g = 0; g < DEPTH; g += 2) {
          const int4 p2 = *reinterpret_cast<const int4*>(&ent[j + g]);
          c[g] = (uint32_t)p2.x;
          a[g] = (uint16_t)p2.y;
          c[g + 1] = (uint32_t)p2.z;
          a[g + 1] = (uint16_t)p2.w;
        }
        uint4 raw[DEPTH];
#pragma unroll
        for (int g = 0; g < DEPTH; ++g)
          if (live[0]) raw[g] = ld_gather(zl, c[g], ldxb);
#pragma unroll
        for (int g = 0; g < DEPTH; ++g) {
          if (!live[0]) continue;
          fhfma2(raw[g].x, a[g], acc[0], acc[1]);
          fhfma2(raw[g].y, a[g], acc[2], acc[3]);
          fhfma2(raw[g].z, a[g], acc[4], acc[5]);
          fhfma2(raw[g].w, a[g], acc[6], acc[7]);
        }
      }
      for (; j < m; ++j) {
        const int2 p1 = ent[j];
        const uint32_t c = (uint32_t)p1.x;
        const uint16_t ah = (uint16_t)p1.y;
        if (live[0]) {
          const uint4 t = ld_gather(zl, c, ldxb);
          fhfma2(t.x, ah, acc[0], acc[1]);
          fhfma2(t.y, ah, acc[2], acc[3]);
          fhfma2(t.z, ah, acc[4], acc[5]);
          fhfma2(t.w, ah, acc[6], acc[7]);
        }
      }
      cc = pc;
      cv = pv;
    }
    if (blockIdx.y == 0 && i < n_rows) {
#pragma unroll
      for (int o = 16; o; o >>= 1) ss = __fadd_ru(ss, __shfl_xor_sync(0xffffffffu, ss, o));
      if (lane == 0) {
        const double m = (double)(e1 - e0);
        // u and zs both rounded to fp16 (2^-11 relative each), fp32 sums, subnormal fp16 u
        const double f = 2.0 * 0x1p-11 + 2.01 * m * 0x1p-24 + sqrt(m) * 0x1p-38;
        const float c = __double2float_ru((__dsqrt_ru((double)ss) * f + sqrt(m) * 0x1p-25) * 1.01);
        cbound[i] = c;
        atomicMax(&cmax_s, __float_as_int(c));  // c >= 0: int order == float order
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) tile[rr][lane * 8 + q] = acc[q];
    int nr = 0;
    if (lane == 0) nr = atomicAdd(&next_row, 1);
    pos = __shfl_sync(0xffffffffu, nr, 0);
    e0 = e1 = 0;
    if (pos < ROWS) {
      rr = order_s[pos];
      e0 = start_s[rr];
      e1 = e0 + len_s[rr];
    }
    cc = 0;
    cv = 0.f;
    if (pos < ROWS && lane < e1 - e0) {
      cc = __ldg(indices + e0 + lane);
      cv = __ldg(vals + e0 + lane);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.y == 0) atomicMax(cmax_bits, cmax_s);
  for (int c = warp; c < PW; c += WARPS) {
    const int64_t col = p0 + c;
#pragma unroll
    for (int h = 0; h < ROWS / 32; ++h) {
      const int64_t i = row0 + h * 32 + lane;
      if (col < ncols && i < n_rows) Yt[col * ldy + i] = tile[h * 32 + lane][c] * qp[col].x;
    }
  }
}

__device__ __forceinline__ float bound_of(float c, float zb) { return __fadd_ru(__fmul_ru(c, zb), 1.401298464e-45f); }

// 32-bit order key of a float (-0 folded onto +0): key order == value order.
__device__ __forceinline__ uint32_t key32(float x) {
  if (x == 0.0f) x = 0.0f;
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ float key_to_float(uint64_t k) {
  return __uint_as_float((k & 0x80000000ull) ? (uint32_t)(k & 0x7fffffffull) : (uint32_t)~k);
}

// Visit (e, x[e]) for e in [0, m) (m < 2^31) with 16-byte loads, U vectors in
// flight per thread, 32-bit indexing.
template <int U, typename F>
__device__ __forceinline__ void for_each_x32(const float* __restrict__ x, int m, F&& f) {
  if (((uintptr_t)x & 15) != 0) {
    for (int e = threadIdx.x; e < m; e += blockDim.x) f(e, x[e]);
    return;
  }
  const float4* xv = reinterpret_cast<const float4*>(x);
  const int mv = m / 4, step = blockDim.x * U;
  for (int base = threadIdx.x; base < mv; base += step) {
    float4 xa[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * blockDim.x;
      if (i < mv) xa[u] = __ldg(xv + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * blockDim.x;
      if (i < mv) {
        f(4 * i, xa[u].x);
        f(4 * i + 1, xa[u].y);
        f(4 * i + 2, xa[u].z);
        f(4 * i + 3, xa[u].w);
      }
    }
  }
  for (int e = mv * 4 + threadIdx.x; e < m; e += blockDim.x) f(e, x[e]);
}

// The exact fp32 score of row i for query q, in the unpruned K9's order
// (sequential FMAs over the row's entries from 0), computed by one warp
// (lanes load and gather, the chain runs on broadcast values), or the stored
// value for rows the unpruned path does not sum (empty rows; copied uncovered
// rows).  Uniform across the warp.
template <int G>
__device__ __forceinline__ float exact_score_group(int64_t i, int64_t q, const float* __restrict__ xt_row,
                                                   const int64_t* __restrict__ indptr,
                                                   const int32_t* __restrict__ indices,
                                                   const float* __restrict__ vals, const float* __restrict__ Zs,
                                                   int64_t ldz, const double* __restrict__ eta, int copy,
                                                   const int64_t* __restrict__ y_ptr,
                                                   const int64_t* __restrict__ y_idx, unsigned mask) {
  const int gl = threadIdx.x & (G - 1);
  const int64_t e0 = indptr[i], e1 = indptr[i + 1];
  if (e0 == e1) return xt_row[i];
  if (copy && eta && eta[i] == 0.0) {
    bool hit = false;
    for (int64_t t = y_ptr[q] + gl; t < y_ptr[q + 1]; t += G) hit |= y_idx[t] == i;
    if (__any_sync(mask, hit)) return xt_row[i];
  }
  // R entries per lane per round: all loads of a round in flight together
  // (larger rounds measured no faster: a round is bound by the dependent
  // DRAM latencies indptr -> entries -> Zs of the candidate's row)
  constexpr int R = 64 / G;
  float acc = 0.f;
  for (int64_t base = e0; base < e1; base += G * R) {
    const int m = e1 - base < G * R ? (int)(e1 - base) : G * R;
    float a[R], z[R];
    int c[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int t = k * G + gl;
      c[k] = t < m ? __ldg(indices + base + t) : 0;
      a[k] = t < m ? __ldg(vals + base + t) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) z[k] = k * G + gl < m ? __ldg(Zs + (int64_t)c[k] * ldz + q) : 0.f;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int mk = m - k * G < G ? m - k * G : G;
      int e = 0;
      // groups of 8: the 16 shuffles are issued ahead of the dependent FMA chain
      for (; e + 8 <= mk; e += 8) {
        float av[8], zv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          av[u] = __shfl_sync(mask, a[k], e + u, G);
          zv[u] = __shfl_sync(mask, z[k], e + u, G);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = fmaf(av[u], zv[u], acc);
      }
      for (; e < mk; ++e) acc = fmaf(__shfl_sync(mask, a[k], e, G), __shfl_sync(mask, z[k], e, G), acc);
    }
  }
  return acc;
}

// Thread-sequential form of the same score (fallback_rows_kernel).
__device__ __forceinline__ float exact_score(int64_t i, int64_t q, const float* __restrict__ xt_row,
                                             const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                             const float* __restrict__ vals, const float* __restrict__ Zs,
                                             int64_t ldz, const double* __restrict__ eta, int copy,
                                             const int64_t* __restrict__ y_ptr, const int64_t* __restrict__ y_idx) {
  const int64_t e0 = indptr[i], e1 = indptr[i + 1];
  if (e0 == e1) return xt_row[i];
  if (copy && eta && eta[i] == 0.0) {
    for (int64_t t = y_ptr[q]; t < y_ptr[q + 1]; ++t)
      if (y_idx[t] == i) return xt_row[i];
  }
  float acc = 0.f;
  for (int64_t e = e0; e < e1; ++e)
    acc = fmaf(__ldg(vals + e), __ldg(Zs + (int64_t)__ldg(indices + e) * ldz + q), acc);
  return acc;
}

// Selection in three kernels:
// prune_threshold_kernel -- per query (persistent CTAs): t = threshold on the
//    lower keys from a 1/16 sample (two 12-bit digits); zeroes the query's
//    counters; z = 0 queries are flagged for the exact select at once.
// prune_scan_kernel -- per (query, segment), b x segs CTAs so every SM keeps
//    streaming (one persistent CTA per query left the DRAM at 53%): one pass
//    counts lower >= t and collects the rows with upper >= t into cand[q]
//    through per-query global counters.
// prune_finish_kernel -- per query: flags the query when count < K or the
//    candidates overflow; else lambda_K = K-th largest lower among the
//    candidates (they hold every row with lower >= t), keep upper >= lambda_K,
//    exact re-score of those (8-lane group per row, from a counter), bitonic
//    sort, top K out.
struct SelShared {
  unsigned int hist[1 << topk::kHistBits];
  unsigned int count;
  unsigned int found_bin;
  unsigned long long above;
  unsigned long long n_lower;
  unsigned int n_keep;
};

static __global__ void __launch_bounds__(kThreads) prune_threshold_kernel(int64_t n, int64_t b, const float* __restrict__ Xt,
                                                                    int64_t ldx, const float* __restrict__ cb,
                                                                    const float2* __restrict__ qp, int64_t K,
                                                                    uint32_t* __restrict__ thr,
                                                                    int32_t* __restrict__ ccount,
                                                                    unsigned* __restrict__ nlow,
                                                                    int* __restrict__ nflag, int* __restrict__ flags) {
  constexpr int KB = 32;
  constexpr int nb = 1 << topk::kHistBits;
  __shared__ SelShared sh;
  const int lane = threadIdx.x & 31;
  const int64_t nblk = (n + topk::kSampleChunk - 1) / topk::kSampleChunk;
  const unsigned long long target = (unsigned long long)((2 * K + topk::kSampleEvery - 1) / topk::kSampleEvery) + 8;
  for (int64_t q = blockIdx.x; q < b; q += gridDim.x) {
    const float* xr = Xt + q * ldx;
    const float zb = qp[q].y;
    if (zb == 0.f) {  // z = 0 (empty observation): x~ is exact (zeros and copied y); exact select only
      if (!threadIdx.x) {
        ccount[q] = -1;
        flags[atomicAdd(nflag, 1)] = (int)q | kExactRows;
      }
      continue;
    }
    if (!(zb <= FLT_MAX)) {  // non-finite zs: no bound; exact recompute + select (as the unpruned path)
      if (!threadIdx.x) {
        ccount[q] = -1;
        flags[atomicAdd(nflag, 1)] = (int)q;
      }
      continue;
    }
    const bool vec_ok = ((((uintptr_t)xr) | ((uintptr_t)cb)) & 15) == 0;
    // 1. sampled threshold on the lower keys
    uint32_t prefix = 0;
    unsigned long long above0 = 0;
    for (int level = 0; level < 2; ++level) {
      for (int t = threadIdx.x; t < nb; t += blockDim.x) sh.hist[t] = 0;
      __syncthreads();
      auto add = [&](float x, float c) {
        const uint32_t k = key32(__fsub_rd(x, bound_of(c, zb)));
        if (level == 0)
          atomicAdd(&sh.hist[k >> (KB - topk::kHistBits)], 1u);
        else if ((k >> (KB - topk::kHistBits)) == prefix)
          atomicAdd(&sh.hist[(k >> (KB - 2 * topk::kHistBits)) & (nb - 1)], 1u);
      };
      if (vec_ok) {
        // sampled blocks = every kSampleEvery-th block of kSampleChunk elements (whole blocks only)
        constexpr int VPB = topk::kSampleChunk / 4;  // float4 per block
        const int nsb = (int)((n / topk::kSampleChunk + topk::kSampleEvery - 1) / topk::kSampleEvery);
        const int nvec = nsb * VPB;
        const float4* xv = reinterpret_cast<const float4*>(xr);
        const float4* cv = reinterpret_cast<const float4*>(cb);
        for (int v0 = threadIdx.x; v0 < nvec; v0 += 2 * blockDim.x) {
          float4 xa[2], ca[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int v = v0 + u * blockDim.x;
            if (v < nvec) {
              const int off = (v / VPB) * topk::kSampleEvery * VPB + v % VPB;
              xa[u] = __ldg(xv + off);
              ca[u] = __ldg(cv + off);
            }
          }
#pragma unroll
          for (int u = 0; u < 2; ++u)
            if (v0 + u * blockDim.x < nvec) {
              add(xa[u].x, ca[u].x);
              add(xa[u].y, ca[u].y);
              add(xa[u].z, ca[u].z);
              add(xa[u].w, ca[u].w);
            }
        }
      } else {
        for (int64_t bk = 0; bk < nblk; bk += topk::kSampleEvery) {
          const int64_t e0 = bk * topk::kSampleChunk, e1 = min(n, e0 + (int64_t)topk::kSampleChunk);
          for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) add(xr[e], __ldg(cb + e));
        }
      }
      __syncthreads();
      topk::find_bin_t<kThreads>(sh.hist, nb, level == 0 ? target : target - above0, &sh.found_bin, &sh.above);
      if (level == 0) above0 = sh.above;
      prefix = (prefix << topk::kHistBits) | sh.found_bin;
      __syncthreads();
    }
    const uint32_t t_lo = prefix << (KB - 2 * topk::kHistBits);
    if (!threadIdx.x) {
      thr[q] = t_lo;
      ccount[q] = 0;
      nlow[q] = 0;
    }
    __syncthreads();
  }
}

// One streaming pass over a segment of one query's x~ row (grid = b x segs):
// count lower >= t and collect the rows with upper >= t into cand[q] through
// per-query global counters (a round-to-nearest pre-filter with max_i c_i
// skips the directed-rounding work, and the read of c_i, far below t).
static __global__ void __launch_bounds__(kThreads) prune_scan_kernel(int64_t n, int segs, int64_t seg_len,
                                                               const float* __restrict__ Xt, int64_t ldx,
                                                               const float* __restrict__ cb,
                                                               const int* __restrict__ cmax_bits,
                                                               const float2* __restrict__ qp,
                                                               const uint32_t* __restrict__ thr,
                                                               int32_t* __restrict__ cand, int32_t* __restrict__ ccount,
                                                               unsigned* __restrict__ nlow) {
  __shared__ unsigned red[kThreads / 32];
  const int64_t q = blockIdx.x / segs;
  const int64_t s0 = (blockIdx.x % segs) * seg_len, s1 = min(n, s0 + seg_len);
  if (ccount[q] < 0 || s0 >= s1) return;  // z = 0: answered by the exact select
  const uint32_t t_lo = thr[q];
  const float zb = qp[q].y;
  const float tf = key_to_float((uint64_t)t_lo);
  const float tf_pre = tf - fabsf(tf) * 0x1p-20f - 0x1p-126f;  // conservative round-to-nearest pre-filter
  const float cz_max = __int_as_float(*cmax_bits) * zb * (1.f + 0x1p-20f);
  const float* xr = Xt + q * ldx + s0;
  int32_t* cq = cand + q * kCap;
  unsigned mine = 0;
  for_each_x32<8>(xr, (int)(s1 - s0), [&](int e, float x) {
    if (x + cz_max >= tf_pre) {
      const int64_t i = s0 + e;
      const float bd = bound_of(__ldg(cb + i), zb);
      mine += key32(__fsub_rd(x, bd)) >= t_lo;
      if (key32(__fadd_ru(x, bd)) >= t_lo) {
        const int slot = atomicAdd(ccount + q, 1);
        if (slot < kCap) cq[slot] = (int32_t)i;
      }
    }
  });
#pragma unroll
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned tot = 0;
    for (int w = 0; w < kThreads / 32; ++w) tot += red[w];
    if (tot) atomicAdd(nlow + q, tot);
  }
}

static __global__ void __launch_bounds__(kThreads) prune_finish_kernel(
    int64_t n, const float* __restrict__ Xt, int64_t ldx, const float* __restrict__ cb, const float2* __restrict__ qp,
    const int32_t* __restrict__ cand, const int32_t* __restrict__ ccount, const unsigned* __restrict__ nlow,
    const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, const float* __restrict__ vals,
    const float* __restrict__ Zs, int64_t ldz, const double* __restrict__ eta, int copy,
    const int64_t* __restrict__ y_ptr, const int64_t* __restrict__ y_idx, int64_t K, int64_t* __restrict__ out_idx,
    float* __restrict__ out_val, int* __restrict__ nflag, int* __restrict__ flags) {
  __shared__ uint64_t ckey[kCap];
  __shared__ int64_t cidx[kCap];
  __shared__ unsigned n_keep, n_next;
  const int64_t q = blockIdx.x;
  const int cnt = ccount[q];
  if (cnt < 0) return;  // z = 0: flagged by the threshold kernel, answered by the exact select
  if (nlow[q] < (unsigned long long)K || cnt > kCap) {  // sampled threshold too high, or overflow
    if (threadIdx.x == 0) flags[atomicAdd(nflag, 1)] = (int)q;
    return;
  }
  const int lane = threadIdx.x & 31;
  const float* xr = Xt + q * ldx;
  const float zb = qp[q].y;
  const int32_t* cq = cand + q * kCap;
  if (!threadIdx.x) n_keep = 0;
  // 3. lambda_K among the candidates
  for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
    const int64_t i = cq[t];
    cidx[t] = i;
    ckey[t] = topk::order_key(__fsub_rd(xr[i], bound_of(cb[i], zb)));
  }
  __syncthreads();
  topk::bitonic_sort(ckey, cidx, cnt);  // (lower key desc, index asc)
  const uint64_t lam = ckey[K - 1];
  __syncthreads();
  // compaction in place: the writes of one round land below the reads of the next
  for (int base = 0; base < cnt; base += blockDim.x) {
    const int t = base + threadIdx.x;
    int64_t i = 0;
    bool keep = false;
    if (t < cnt) {
      i = cidx[t];
      keep = topk::order_key(__fadd_ru(xr[i], bound_of(cb[i], zb))) >= lam;
    }
    __syncthreads();
    if (keep) cidx[atomicAdd(&n_keep, 1u)] = i;
  }
  __syncthreads();
  const unsigned keep = n_keep;
  // 4. exact re-score (warp per row; rows handed out from a counter, their
  //    lengths differ by 10x and more), sort, output
  //    8-lane groups take the rows, four rows per warp in flight (a warp per
  //    row: +0.07 ms, half-warps: +0.03 ms at C3).
  constexpr int G = 8;
  const int grp = threadIdx.x / G, gl = threadIdx.x & (G - 1);
  const unsigned gmask = 0xffu << (lane & ~(G - 1));
  if (threadIdx.x == 0) n_next = kThreads / G;
  __syncthreads();
  for (unsigned t = grp; t < keep;) {
    const float v = exact_score_group<G>(cidx[t], q, xr, indptr, indices, vals, Zs, ldz, eta, copy, y_ptr, y_idx,
                                         gmask);
    unsigned nt = 0;
    if (gl == 0) {
      ckey[t] = topk::order_key(v);
      nt = atomicAdd(&n_next, 1u);
    }
    t = __shfl_sync(gmask, nt, 0, G);
  }
  __syncthreads();
  topk::bitonic_sort(ckey, cidx, (int)keep);
  for (int64_t m = threadIdx.x; m < K; m += blockDim.x) {
    out_idx[q * K + m] = cidx[m];
    float v = key_to_float(ckey[m]);
    // the key folds -0 onto +0 (they tie); return the score's own bits, as the
    // unpruned path does (the thread-sequential sum is bitwise the group's)
    if (v == 0.f) v = exact_score(cidx[m], q, xr, indptr, indices, vals, Zs, ldz, eta, copy, y_ptr, y_idx);
    out_val[q * K + m] = v;
  }
}

// ---- fallback for flagged queries (exit at once when nothing is flagged) ----

// Exact fp32 scores of every summed row of the flagged queries, written over
// the pruned values (persistent grid over (flagged query, 256-row block)).
static __global__ void __launch_bounds__(256) fallback_rows_kernel(int64_t n, float* __restrict__ Xt, int64_t ldx,
                                                            const int64_t* __restrict__ indptr,
                                                            const int32_t* __restrict__ indices,
                                                            const float* __restrict__ vals,
                                                            const float* __restrict__ Zs, int64_t ldz,
                                                            const double* __restrict__ eta, int copy,
                                                            const int64_t* __restrict__ y_ptr,
                                                            const int64_t* __restrict__ y_idx,
                                                            const int* __restrict__ nflag,
                                                            const int* __restrict__ flags) {
  const int nf = *nflag;
  if (!nf) return;
  const int64_t nblk = (n + 255) / 256;
  for (int64_t item = blockIdx.x; item < nf * nblk; item += gridDim.x) {
    const int f = flags[item / nblk];
    if (f & kExactRows) continue;  // x~ is already exact for this query
    const int64_t q = f;
    const int64_t i = (item % nblk) * 256 + threadIdx.x;
    if (i < n) {
      float* xr = Xt + q * ldx;
      xr[i] = exact_score(i, q, xr, indptr, indices, vals, Zs, ldz, eta, copy, y_ptr, y_idx);
    }
  }
}

// Exact top K of the (now exact) rows of the flagged queries.
static __global__ void __launch_bounds__(topk::kThreads) fallback_select_kernel(int64_t n, const float* __restrict__ Xt,
                                                                         int64_t ldx, int64_t K,
                                                                         int64_t* __restrict__ out_idx,
                                                                         float* __restrict__ out_val,
                                                                         const int* __restrict__ nflag,
                                                                         const int* __restrict__ flags) {
  if ((int)blockIdx.x >= *nflag) return;
  extern __shared__ __align__(16) unsigned char dyn[];
  uint64_t* ckey = (uint64_t*)dyn;
  int64_t* cidx = (int64_t*)(ckey + topk::kCap);
  __shared__ topk::Shared sh;
  const int64_t q = flags[blockIdx.x] & ~kExactRows;
  topk::Range<float, false> R{Xt + q * ldx, nullptr, n, 0};
  topk::select_exact<float, false>(R, K, sh, ckey, cidx);
  __syncthreads();
  for (int64_t m = threadIdx.x; m < K; m += blockDim.x) {
    const int64_t i = cidx[m];
    out_idx[q * K + m] = i;
    out_val[q * K + m] = R.v[i];
  }
}

// Workspace of the pruned path beyond the unpruned one.
inline size_t workspace_bytes(int64_t n, int64_t r, int64_t b) {
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  return al((size_t)r * b * 2) + al((size_t)b * 8) + al((size_t)n * 4) + al((size_t)(b + 2) * 4) +
         al((size_t)b * kCap * 4) + al((size_t)b * 4) + al((size_t)b * 4) + al((size_t)b * 4);
}

// b >= 256: a narrow variant for 64 <= b < 256 (64-column panels, 8-lane
// groups per row) measured K9 1.95 vs 2.05 ms at b = 64 but 0.40 vs 0.17 ms of
// selection -- slower overall -- and b <= 64's exact kernel sums a row in two
// interleaved halves, so its values are not the sequential order re-scored here.
inline bool applicable(int64_t n, int64_t b, int64_t K) {
  return n >= (int64_t)topk::kSampleChunk * topk::kSampleEvery * 8 && n < ((int64_t)1 << 31) && b >= 256 && b % 8 == 0 && K >= 1 &&
         K <= kCap / 8;
}

}  // namespace prune
}  // namespace fsr
