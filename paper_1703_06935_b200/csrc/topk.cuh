// Exact top-k per row in the reference's rank order (ranking.py:390-395:
// descending score, ties by ascending index), for b rows of length n.
//
// One CTA selects the top K of a contiguous range of a row:
//  * order keys: IEEE bits mapped to unsigned so that key order == value order
//    (-0 folded onto +0, numpy compares values);
//  * long ranges: a 1/16 block sample (two 12-bit digit histograms) proposes a
//    threshold key, ONE pass over the range collects every key >= threshold
//    into shared memory, a bitonic sort on (key desc, index asc) finishes;
//  * short ranges, and whenever the sampled threshold yields fewer than K or
//    more than kCap candidates: the exact path -- a digit histogram pins the
//    K-th key bin, candidates >= that bin are collected (or, if that overflows,
//    the exact threshold key T is pinned digit by digit and the ties at T are
//    taken in index order).
// Few rows (b small) are split into segments: stage 1 emits each segment's
// top K (sorted, so equal keys stay in index order), stage 2 selects from the
// per-row candidate lists with their explicit indices.
#pragma once

#include <cub/cub.cuh>

#include <algorithm>
#include <type_traits>

#include "fsr_common.cuh"

namespace fsr {
namespace topk {

constexpr int kThreads = 512;
constexpr int kCap = 4096;  // candidates held in shared memory
constexpr int kHistBits = 12;
constexpr int kSampleChunk = 1024;  // elements per sampled block
constexpr int kSampleEvery = 16;    // one block of every 16 is sampled

__device__ __forceinline__ uint64_t order_key(float x) {
  if (x == 0.0f) x = 0.0f;
  const uint32_t u = __float_as_uint(x);
  return (uint64_t)((u & 0x80000000u) ? ~u : (u | 0x80000000u));
}
__device__ __forceinline__ uint64_t order_key(double x) {
  if (x == 0.0) x = 0.0;
  const uint64_t u = (uint64_t)__double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

struct Shared {
  unsigned int hist[1 << kHistBits];
  unsigned int count;
  unsigned int found_bin;
  unsigned long long above;
  unsigned long long warp_sums[kThreads / 32];
};

// The bin (scanning from the top) where the running count first reaches `need`
// (or the lowest bin if the total is smaller): *found_bin, *above (count
// strictly above).  NT = threads per block.
template <int NT>
__device__ void find_bin_t(const unsigned int* hist, int nb, unsigned long long need, unsigned int* found_bin,
                           unsigned long long* above) {
  typedef cub::BlockScan<unsigned long long, NT> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;
  const int per = nb / NT > 0 ? nb / NT : 1;
  unsigned long long mine = 0;
  const int hi = nb - 1 - (int)threadIdx.x * per;
  for (int q = 0; q < per; ++q) {
    const int bin = hi - q;
    if (bin >= 0) mine += hist[bin];
  }
  if (threadIdx.x == 0) {
    *found_bin = 0;
    *above = 0;
  }
  __syncthreads();
  unsigned long long before = 0, total = 0;
  Scan(scan_tmp).ExclusiveSum(mine, before, total);
  unsigned long long run = before;
  for (int q = 0; q < per; ++q) {
    const int bin = hi - q;
    if (bin < 0) break;
    const unsigned long long h = hist[bin];
    if (run < need && run + h >= need) {
      *found_bin = (unsigned)bin;
      *above = run;
    }
    run += h;
  }
  if (total < need && threadIdx.x == 0) *above = total;  // everything qualifies; bin 0
  __syncthreads();
}

__device__ __forceinline__ void find_bin(Shared& sh, int nb, unsigned long long need) {
  find_bin_t<kThreads>(sh.hist, nb, need, &sh.found_bin, &sh.above);
}

__device__ __forceinline__ bool before_in_rank(uint64_t ka, int64_t ia, uint64_t kb, int64_t ib) {
  return ka > kb || (ka == kb && ia < ib);
}

__device__ inline void bitonic_sort(uint64_t* key, int64_t* idx, int count) {
  int P = 1;
  while (P < count) P <<= 1;
  for (int t = count + threadIdx.x; t < P; t += blockDim.x) {
    key[t] = 0;
    idx[t] = INT64_MAX;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < P / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const bool swap = up ? before_in_rank(key[hi], idx[hi], key[lo], idx[lo])
                             : before_in_rank(key[lo], idx[lo], key[hi], idx[hi]);
        if (swap) {
          const uint64_t tk = key[lo];
          key[lo] = key[hi];
          key[hi] = tk;
          const int64_t ti = idx[lo];
          idx[lo] = idx[hi];
          idx[hi] = ti;
        }
      }
      __syncthreads();
    }
  }
}

// Range view: element e (0 <= e < m) is value v[e] with index ix(e).
template <typename T, bool EXPLICIT>
struct Range {
  const T* v;
  const int64_t* ix;
  int64_t m;
  int64_t base;  // implicit index of element 0
  __device__ __forceinline__ int64_t index(int64_t e) const { return EXPLICIT ? ix[e] : base + e; }
};

// Exact selection of the top K of a range (keys, indices into ckey/cidx, sorted).
template <typename T, bool EXPLICIT>
__device__ void select_exact(const Range<T, EXPLICIT>& R, int64_t K, Shared& sh, uint64_t* ckey, int64_t* cidx) {
  constexpr int KB = sizeof(T) * 8;
  constexpr int nb = 1 << kHistBits;
  for (int t = threadIdx.x; t < nb; t += blockDim.x) sh.hist[t] = 0;
  if (!threadIdx.x) sh.count = 0;
  __syncthreads();
  for (int64_t e = threadIdx.x; e < R.m; e += blockDim.x)
    atomicAdd(&sh.hist[order_key(R.v[e]) >> (KB - kHistBits)], 1u);
  __syncthreads();
  find_bin(sh, nb, (unsigned long long)K);
  uint64_t prefix = sh.found_bin;
  int pbits = kHistBits;
  const unsigned long long above = sh.above;
  const unsigned long long in_bin = sh.hist[prefix];
  __syncthreads();
  if (above + in_bin <= (unsigned long long)kCap) {
    for (int64_t e = threadIdx.x; e < R.m; e += blockDim.x) {
      const uint64_t k = order_key(R.v[e]);
      if ((k >> (KB - kHistBits)) >= prefix) {
        const unsigned slot = atomicAdd(&sh.count, 1u);
        ckey[slot] = k;
        cidx[slot] = R.index(e);
      }
    }
    __syncthreads();
    bitonic_sort(ckey, cidx, (int)sh.count);
    return;
  }
  // pin the exact threshold key, then take ties in position (= index) order
  unsigned long long need = (unsigned long long)K - above;
  while (pbits < KB) {
    const int d = KB - pbits < kHistBits ? KB - pbits : kHistBits;
    const int shift = KB - pbits - d;
    for (int t = threadIdx.x; t < nb; t += blockDim.x) sh.hist[t] = 0;
    __syncthreads();
    for (int64_t e = threadIdx.x; e < R.m; e += blockDim.x) {
      const uint64_t k = order_key(R.v[e]);
      if ((k >> (KB - pbits)) == prefix) atomicAdd(&sh.hist[(k >> shift) & ((1u << d) - 1u)], 1u);
    }
    __syncthreads();
    find_bin(sh, 1 << d, need);
    need -= sh.above;
    prefix = (prefix << d) | sh.found_bin;
    pbits += d;
    __syncthreads();
  }
  const uint64_t Tk = prefix;
  const unsigned long long gt_total = (unsigned long long)K - need;
  for (int64_t e = threadIdx.x; e < R.m; e += blockDim.x) {
    const uint64_t k = order_key(R.v[e]);
    if (k > Tk) {
      const unsigned slot = atomicAdd(&sh.count, 1u);
      ckey[slot] = k;
      cidx[slot] = R.index(e);
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long taken = 0;
  for (int64_t base = 0; base < R.m && taken < need; base += blockDim.x) {
    const int64_t e = base + threadIdx.x;
    const bool tie = e < R.m && order_key(R.v[e]) == Tk;
    const unsigned msk = __ballot_sync(0xffffffffu, tie);
    if (!lane) sh.warp_sums[wid] = __popc(msk);
    __syncthreads();
    unsigned long long off = 0, tot = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      if (w < wid) off += sh.warp_sums[w];
      tot += sh.warp_sums[w];
    }
    const unsigned long long rnk = taken + off + __popc(msk & ((1u << lane) - 1u));
    if (tie && rnk < need) {
      ckey[gt_total + rnk] = Tk;
      cidx[gt_total + rnk] = R.index(e);
    }
    taken += tot;
    __syncthreads();
  }
  bitonic_sort(ckey, cidx, (int)K);
}

// Visit element values of a range with 16-byte vector loads, U vectors in
// flight per thread (fp32 rows are HBM-streamed: one CTA per row must keep
// enough bytes in flight); f(e, v) is called for every element e in [0, m).
// Falls back to scalar loads when the range start is not 16-byte aligned.
template <typename T, int U, typename F>
__device__ __forceinline__ void for_each_vec(const T* __restrict__ v, int64_t m, F&& f) {
  constexpr int W = 16 / sizeof(T);
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  if (((uintptr_t)v & 15) != 0) {
    for (int64_t e = threadIdx.x; e < m; e += blockDim.x) f(e, v[e]);
    return;
  }
  const V* vv = reinterpret_cast<const V*>(v);
  const int64_t mv = m / W;
  const int64_t step = (int64_t)blockDim.x * U;
  for (int64_t base = threadIdx.x; base < mv; base += step) {
    V x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x;
      if (i < mv) x[u] = __ldg(vv + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (int64_t)u * blockDim.x;
      if (i < mv) {
        const T* xs = reinterpret_cast<const T*>(&x[u]);
#pragma unroll
        for (int c = 0; c < W; ++c) f(i * W + c, xs[c]);
      }
    }
  }
  for (int64_t e = mv * W + threadIdx.x; e < m; e += blockDim.x) f(e, v[e]);
}

// Sampled single-pass selection; returns false when the caller must fall back.
template <typename T>
__device__ bool select_sampled(const Range<T, false>& R, int64_t K, Shared& sh, uint64_t* ckey, int64_t* cidx) {
  constexpr int KB = sizeof(T) * 8;
  constexpr int nb = 1 << kHistBits;
  // sample: two digit levels over blocks 0, 16, 32, ... of kSampleChunk elements
  const int64_t nblk = (R.m + kSampleChunk - 1) / kSampleChunk;
  const unsigned long long target = (unsigned long long)((3 * K + kSampleEvery - 1) / kSampleEvery) + 4;
  uint64_t prefix = 0;
  unsigned long long above0 = 0;
  for (int level = 0; level < 2; ++level) {
    for (int t = threadIdx.x; t < nb; t += blockDim.x) sh.hist[t] = 0;
    __syncthreads();
    for (int64_t b = 0; b < nblk; b += kSampleEvery) {
      const int64_t e0 = b * kSampleChunk, e1 = min(R.m, e0 + kSampleChunk);
      for_each_vec<T, 1>(R.v + e0, e1 - e0, [&](int64_t, T x) {
        const uint64_t k = order_key(x);
        if (level == 0)
          atomicAdd(&sh.hist[k >> (KB - kHistBits)], 1u);
        else if ((k >> (KB - kHistBits)) == prefix)
          atomicAdd(&sh.hist[(k >> (KB - 2 * kHistBits)) & (nb - 1)], 1u);
      });
    }
    __syncthreads();
    find_bin(sh, nb, level == 0 ? target : target - above0);
    if (level == 0) above0 = sh.above;
    prefix = (prefix << kHistBits) | sh.found_bin;
    __syncthreads();
  }
  const uint64_t T_lo = prefix << (KB - 2 * kHistBits);  // candidates: key >= T_lo
  if (!threadIdx.x) sh.count = 0;
  __syncthreads();
  const int64_t base = R.base;
  for_each_vec<T, 4>(R.v, R.m, [&](int64_t e, T x) {
    const uint64_t k = order_key(x);
    if (k >= T_lo) {
      const unsigned slot = atomicAdd(&sh.count, 1u);
      if (slot < (unsigned)kCap) {
        ckey[slot] = k;
        cidx[slot] = base + e;
      }
    }
  });
  __syncthreads();
  const unsigned c = sh.count;
  if (c < (unsigned)K || c > (unsigned)kCap) return false;
  bitonic_sort(ckey, cidx, (int)c);
  return true;
}

// grid.x = rows * segs; row q = blockIdx.x / segs, segment s = blockIdx.x % segs.
// Input element e of (q, s): src[q * ld + s * seg + e] (e < len - s * seg, <= seg),
// index = EXPLICIT ? isrc[same] : s * seg + e.  Output: K (value, index) pairs at
// out_*[blockIdx.x * K], sorted in rank order; padded with (-inf, INT64_MAX).
template <typename T, bool EXPLICIT>
__global__ void __launch_bounds__(kThreads) select_kernel(const T* __restrict__ src, const int64_t* __restrict__ isrc,
                                                          int64_t ld, int64_t len, int64_t seg, int segs, int64_t K,
                                                          int use_sample, T* __restrict__ out_val,
                                                          int64_t* __restrict__ out_idx) {
  extern __shared__ __align__(16) unsigned char dyn[];
  uint64_t* ckey = (uint64_t*)dyn;
  int64_t* cidx = (int64_t*)(ckey + kCap);
  __shared__ Shared sh;
  const int64_t q = blockIdx.x / segs, s = blockIdx.x % segs;
  const int64_t b0 = s * seg, b1 = min(len, b0 + seg);
  Range<T, EXPLICIT> R{src + q * ld + b0, EXPLICIT ? isrc + q * ld + b0 : nullptr, b1 > b0 ? b1 - b0 : 0, b0};
  const int64_t Kr = min(K, R.m);
  bool done = false;
  if (!EXPLICIT && use_sample && R.m >= (int64_t)kSampleChunk * kSampleEvery * 4 && Kr == K)
    done = select_sampled<T>(*reinterpret_cast<const Range<T, false>*>(&R), K, sh, ckey, cidx);
  __syncthreads();
  if (!done && Kr > 0) select_exact<T, EXPLICIT>(R, Kr, sh, ckey, cidx);
  __syncthreads();
  for (int64_t m = threadIdx.x; m < K; m += blockDim.x) {
    const int64_t o = (int64_t)blockIdx.x * K + m;
    if (m < Kr) {
      const int64_t i = cidx[m];
      out_idx[o] = i;
      out_val[o] = EXPLICIT ? T(0) : R.v[i - b0];
    } else {
      out_idx[o] = INT64_MAX;
      out_val[o] = -INFINITY;
    }
  }
  if (EXPLICIT) {
    // values: recover from the key order (search the candidate list for the index)
    __syncthreads();
    for (int64_t m = threadIdx.x; m < Kr; m += blockDim.x) {
      const uint64_t k = ckey[m];
      const uint64_t u = (k & (1ull << (sizeof(T) * 8 - 1))) ? (k & ~(1ull << (sizeof(T) * 8 - 1))) : ~k;
      T v;
      if (sizeof(T) == 4) {
        const uint32_t u32 = (uint32_t)u;
        memcpy(&v, &u32, 4);
      } else {
        memcpy(&v, &u, 8);
      }
      out_val[(int64_t)blockIdx.x * K + m] = v;
    }
  }
}

// ---- few rows (b < #SMs), fp32: two grid-wide passes -------------------------
// The segmented path above selects K per segment and merges b * segs * K
// candidates in one CTA per row (b = 1, n = 1e6: 22 + 35 us).  Here every CTA
// of a row adds its segment to ONE 12-bit key histogram of the row
// (hist_kernel), and in the second pass reads that histogram, finds the bin
// of the K-th key and appends its segment's keys at or above that bin to the
// row's candidate list; the row's last CTA to finish sorts the candidates by
// (key desc, index asc) and writes the top K.  More than kCap candidates
// (masses of keys sharing 12 bits, e.g. a row of zeros) fall back to
// select_exact over the whole row in that last CTA.  The state (histograms,
// counters, candidate lists) lives in the context and is left zeroed by the
// last CTA, so a call needs no memset.
struct FewRows {
  unsigned* hist;    // rows x 2^kHistBits
  unsigned* count;   // rows
  unsigned* ticket;  // rows
  uint64_t* ckey;    // rows x kCap
  int64_t* cidx;     // rows x kCap
};

inline size_t few_rows_bytes(int rows) {
  return (size_t)rows * ((size_t)(1 << kHistBits) * 4 + 8 + (size_t)kCap * 16) + 256;
}

inline int few_rows_state(fsr_ctx* ctx, FewRows* st) {
  const int rows = ctx->num_sms;
  if (!ctx->topk_state) {
    const size_t bytes = few_rows_bytes(rows);
    cudaError_t e = cudaMalloc(&ctx->topk_state, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      ctx->topk_state = nullptr;
      return set_error(ctx, FSR_ENOMEM, "top-k state alloc of %zu bytes failed", bytes);
    }
    e = cudaMemsetAsync(ctx->topk_state, 0, bytes, ctx->stream);
    if (e != cudaSuccess) return cuda_status(ctx, e, "top-k state memset");
  }
  char* p = (char*)ctx->topk_state;
  st->ckey = (uint64_t*)p;
  p += (size_t)rows * kCap * 8;
  st->cidx = (int64_t*)p;
  p += (size_t)rows * kCap * 8;
  st->hist = (unsigned*)p;
  p += (size_t)rows * (1 << kHistBits) * 4;
  st->count = (unsigned*)p;
  st->ticket = st->count + rows;
  return FSR_OK;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) few_rows_hist_kernel(const T* __restrict__ X, int64_t ld, int64_t n,
                                                                 int64_t seg, unsigned* __restrict__ ghist) {
  constexpr int nb = 1 << kHistBits;
  __shared__ unsigned h[nb];
  for (int t = threadIdx.x; t < nb; t += blockDim.x) h[t] = 0;
  __syncthreads();
  const int64_t q = blockIdx.y, b0 = (int64_t)blockIdx.x * seg, b1 = min(n, b0 + seg);
  if (b1 > b0)
    for_each_vec<T, 4>(X + q * ld + b0, b1 - b0,
                       [&](int64_t, T x) { atomicAdd(&h[order_key(x) >> (sizeof(T) * 8 - kHistBits)], 1u); });
  __syncthreads();
  for (int t = threadIdx.x; t < nb; t += blockDim.x)
    if (h[t]) atomicAdd(&ghist[q * nb + t], h[t]);
}

template <typename T>
__global__ void __launch_bounds__(kThreads) few_rows_select_kernel(const T* __restrict__ X, int64_t ld, int64_t n,
                                                                   int64_t seg, int64_t K, FewRows st,
                                                                   T* __restrict__ out_val,
                                                                   int64_t* __restrict__ out_idx) {
  constexpr int nb = 1 << kHistBits;
  constexpr int KB = sizeof(T) * 8;
  extern __shared__ __align__(16) unsigned char dyn[];
  uint64_t* ckey = (uint64_t*)dyn;
  int64_t* cidx = (int64_t*)(ckey + kCap);
  __shared__ Shared sh;
  const int64_t q = blockIdx.y, b0 = (int64_t)blockIdx.x * seg, b1 = min(n, b0 + seg);
  unsigned* ghist = st.hist + q * nb;
  for (int t = threadIdx.x; t < nb; t += blockDim.x) sh.hist[t] = __ldcg(ghist + t);
  __syncthreads();
  find_bin(sh, nb, (unsigned long long)K);
  const uint64_t bin = sh.found_bin;
  uint64_t* gkey = st.ckey + q * kCap;
  int64_t* gidx = st.cidx + q * kCap;
  if (b1 > b0)
    for_each_vec<T, 4>(X + q * ld + b0, b1 - b0, [&](int64_t e, T x) {
      const uint64_t k = order_key(x);
      if ((k >> (KB - kHistBits)) >= bin) {
        const unsigned slot = atomicAdd(&st.count[q], 1u);
        if (slot < (unsigned)kCap) {
          gkey[slot] = k;
          gidx[slot] = b0 + e;
        }
      }
    });
  __threadfence();
  __syncthreads();
  if (!threadIdx.x) sh.count = atomicAdd(&st.ticket[q], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!sh.count) return;
  __threadfence();
  const unsigned c = __ldcg(&st.count[q]);
  __syncthreads();
  bool written = false;
  if (c <= (unsigned)kCap) {
    for (unsigned t = threadIdx.x; t < c; t += blockDim.x) {
      ckey[t] = __ldcg(gkey + t);
      cidx[t] = __ldcg(gidx + t);
    }
    __syncthreads();
    if (c <= 512u) {
      // few candidates: the rank of each one by counting those before it (the
      // order is total: indices are distinct) -- c^2 / 512 broadcast reads per
      // thread instead of the bitonic network's ~45 block-wide rounds
      for (unsigned t = threadIdx.x; t < c; t += blockDim.x) {
        const uint64_t k = ckey[t];
        const int64_t i = cidx[t];
        unsigned rank = 0;
        for (unsigned s2 = 0; s2 < c; ++s2) rank += before_in_rank(ckey[s2], cidx[s2], k, i) ? 1u : 0u;
        if (rank < (unsigned)K) {
          out_idx[q * K + rank] = i;
          out_val[q * K + rank] = X[q * ld + i];
        }
      }
      written = true;
    } else {
      bitonic_sort(ckey, cidx, (int)c);
    }
  } else {
    Range<T, false> R{X + q * ld, nullptr, n, 0};
    select_exact<T, false>(R, K, sh, ckey, cidx);
  }
  __syncthreads();
  if (!written)
    for (int64_t m = threadIdx.x; m < K; m += blockDim.x) {
      const int64_t i = cidx[m];
      out_idx[q * K + m] = i;
      out_val[q * K + m] = X[q * ld + i];
    }
  for (int t = threadIdx.x; t < nb; t += blockDim.x) ghist[t] = 0;
  if (!threadIdx.x) {
    st.count[q] = 0;
    st.ticket[q] = 0;
  }
}

inline bool few_rows_applicable(fsr_ctx* ctx, int64_t b, int64_t n, int64_t K) {
  if (!(ctx->topk_segments == 0 && b < ctx->num_sms && n >= 65536 && K <= n && K <= kCap / 4)) return false;
  if (!ctx->topk_state) {
    // the state is allocated on first use; not while the stream is being captured into a graph
    // (callers warm up before capturing; otherwise the segmented path serves the captured call)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(ctx->stream, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return false;
    }
  }
  return true;
}

inline int launch_few_rows(fsr_ctx* ctx, int64_t b, int64_t n, const float* X, int64_t ldx, int64_t K, int64_t* top_idx,
                           float* top_val) {
  FewRows st;
  FSR_TRY(few_rows_state(ctx, &st));
  const size_t smem = (size_t)kCap * 16;
  FSR_TRY(ensure_smem(ctx, few_rows_select_kernel<float>, smem));
  int64_t segs = std::max<int64_t>(1, std::min<int64_t>(ceil_div(2 * ctx->num_sms, b), n / 4096));
  const int64_t seg = ceil_div(ceil_div(n, segs), 1024) * 1024;  // 16-byte aligned segment starts
  segs = ceil_div(n, seg);
  dim3 grid((unsigned)segs, (unsigned)b);
  few_rows_hist_kernel<float><<<grid, kThreads, 0, ctx->stream>>>(X, ldx, n, seg, st.hist);
  FSR_TRY(launched(ctx, "topk_few_rows_hist_kernel"));
  few_rows_select_kernel<float><<<grid, kThreads, smem, ctx->stream>>>(X, ldx, n, seg, K, st, top_val, top_idx);
  return launched(ctx, "topk_few_rows_select_kernel");
}

template <typename T>
int launch(fsr_ctx* ctx, int64_t b, int64_t n, const T* X, int64_t ldx, int64_t K, int64_t* top_idx, T* top_val) {
  if constexpr (std::is_same<T, float>::value) {
    if (few_rows_applicable(ctx, b, n, K)) return launch_few_rows(ctx, b, n, X, ldx, K, top_idx, top_val);
  }
  const size_t smem = (size_t)kCap * 16;
  FSR_TRY(ensure_smem(ctx, select_kernel<T, false>, smem));
  FSR_TRY(ensure_smem(ctx, select_kernel<T, true>, smem));
  int segs = 1;
  if (b < ctx->num_sms) {
    segs = (int)std::min<int64_t>(ceil_div(2 * ctx->num_sms, b), std::max<int64_t>(1, n / (8 * K)));
    if (ctx->topk_segments > 0) segs = (int)std::min<int64_t>(ctx->topk_segments, std::max<int64_t>(1, n / (8 * K)));
    segs = std::max(segs, 1);
  }
  if (segs == 1) {
    select_kernel<T, false><<<(unsigned)b, kThreads, smem, ctx->stream>>>(X, nullptr, ldx, n, n, 1, K, 1, top_val,
                                                                          top_idx);
    return launched(ctx, "topk_select_kernel");
  }
  const int64_t seg = ceil_div(n, segs);
  void* buf = nullptr;
  const size_t cand = (size_t)b * segs * K;
  FSR_TRY(scratch(ctx, cand * (sizeof(T) + 8) + 256, &buf));
  int64_t* cidx = (int64_t*)buf;
  T* cval = (T*)(cidx + cand);
  select_kernel<T, false><<<(unsigned)(b * segs), kThreads, smem, ctx->stream>>>(X, nullptr, ldx, n, seg, segs, K, 1,
                                                                                 cval, cidx);
  FSR_TRY(launched(ctx, "topk_select_kernel"));
  select_kernel<T, true><<<(unsigned)b, kThreads, smem, ctx->stream>>>(cval, cidx, segs * K, segs * K, segs * K, 1, K,
                                                                       0, top_val, top_idx);
  return launched(ctx, "topk_merge_kernel");
}

}  // namespace topk
}  // namespace fsr
