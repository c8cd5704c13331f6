// K0: the seeded Gaussian start block (reference spectral.py:55-65) and
// K1: degree / symmetric normalisation of the adjacency (graph.py:118-139).
//
// K0 regenerates numpy's Generator(Philox(seed)).random() stream on the device:
// uniform m comes from Philox4x64-10 block (counter = m/4 + 1, key) word m%4 as
// (x >> 11) * 2^-53.  With half = ceil(rows*cols/2), flat element f of the block
// is sqrt(-2 ln(1-U[i])) * {cos | sin}(2*pi*U[half+i]) with i = f (cos, f < half)
// or i = f - half (sin).  Every rank can therefore generate exactly its own row
// shard without communication.  Each thread produces 4 consecutive i (one
// Philox block for the radii) and both of their outputs.
#include "fsr_common.cuh"

namespace {

constexpr uint64_t kM0 = 0xD2E7470EE14C6C93ull;
constexpr uint64_t kM1 = 0xCA5A826395121157ull;
constexpr uint64_t kW0 = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kW1 = 0xBB67AE8584CAA73Bull;

struct U4 {
  uint64_t v[4];
};

__device__ __forceinline__ U4 philox4x64_10(uint64_t ctr0, uint64_t k0, uint64_t k1) {
  uint64_t c0 = ctr0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    if (round) {
      k0 += kW0;
      k1 += kW1;
    }
    const uint64_t lo0 = kM0 * c0, hi0 = __umul64hi(kM0, c0);
    const uint64_t lo1 = kM1 * c2, hi1 = __umul64hi(kM1, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return U4{{c0, c1, c2, c3}};
}

__device__ __forceinline__ double to_unit(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

template <typename T>
__global__ void gaussian_kernel(int64_t count, int64_t half, int64_t f0, int64_t f1, int64_t segA_lo,
                                int64_t segA_len, int64_t segB_lo, int64_t segB_len, uint64_t k0,
                                uint64_t k1, T* __restrict__ out) {
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t groupsA = (segA_len + 3) / 4, groupsB = (segB_len + 3) / 4;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < groupsA + groupsB;
       t += nthreads) {
    // i0: first of 4 consecutive radius indices, aligned down to a Philox block
    int64_t i0 = t < groupsA ? segA_lo + 4 * t : segB_lo + 4 * (t - groupsA);
    i0 &= ~int64_t(3);
    const U4 rad_blk = philox4x64_10((uint64_t)(i0 / 4) + 1, k0, k1);
    const int64_t a0 = half + i0;  // first angle uniform index
    const U4 ang_lo = philox4x64_10((uint64_t)(a0 / 4) + 1, k0, k1);
    U4 ang_hi = ang_lo;
    if (a0 % 4) ang_hi = philox4x64_10((uint64_t)(a0 / 4) + 2, k0, k1);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = i0 + q;
      if (i >= half) break;
      const int64_t fc = i, fs = half + i;
      const bool want_c = fc >= f0 && fc < f1;
      const bool want_s = fs >= f0 && fs < f1 && fs < count;
      if (!want_c && !want_s) continue;
      const int am = (int)((a0 + q) & 3);
      const uint64_t araw = ((a0 % 4) + q) < 4 ? ang_lo.v[am] : ang_hi.v[am];
      const double radius = sqrt(-2.0 * log(1.0 - to_unit(rad_blk.v[q])));
      const double angle = 6.283185307179586 * to_unit(araw);  // (2.0*np.pi)*u2
      if (want_c) out[fc - f0] = (T)(radius * cos(angle));
      if (want_s) out[fs - f0] = (T)(radius * sin(angle));
    }
  }
}

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum): < 8 terms sequential from 0; <= 128 terms eight strided
// accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a
// sequential tail; longer runs split at n/2 rounded down to a multiple of 8.
__device__ double pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_sum(a, n2), pairwise_sum(a + n2, n - n2));
}

// Degrees exactly as the reference computes them: W.sum(axis=1) on a CSR
// matrix reduces each nonempty row with np.add.reduceat, i.e. a[0] +
// pairwise_sum(a[1:]) (graph.py:121 -> scipy _cs_matrix.sum/_minor_reduce).
__global__ void row_sums_kernel(int64_t n_rows, const int64_t* __restrict__ indptr,
                                const double* __restrict__ data, double* __restrict__ deg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = indptr[i], len = indptr[i + 1] - e0;
    deg[i] = len ? __dadd_rn(data[e0], pairwise_sum(data + e0 + 1, len - 1)) : 0.0;
  }
}

__device__ __forceinline__ double inv_sqrt_or_zero(double d) { return d > 0.0 ? 1.0 / sqrt(d) : 0.0; }

template <typename T>
__global__ void normalize_kernel(int64_t n_rows, int64_t row_offset, const int64_t* __restrict__ indptr,
                                 const int32_t* __restrict__ indices, const double* __restrict__ data,
                                 const double* __restrict__ deg, T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n_rows; i += warps) {
    const double si = inv_sqrt_or_zero(deg[row_offset + i]);
    for (int64_t e = indptr[i] + lane; e < indptr[i + 1]; e += 32) {
      const double sj = inv_sqrt_or_zero(deg[indices[e]]);
      out[e] = (T)__dmul_rn(__dmul_rn(data[e], si), sj);
    }
  }
}

template <typename T>
__global__ void convert_kernel(int64_t n, const double* __restrict__ in, T* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (T)in[i];
}

}  // namespace

extern "C" {

int fsr_gaussian_block(fsr_ctx* ctx, int dtype, int64_t total_rows, int64_t cols, int64_t row_begin,
                       int64_t row_end, uint64_t key0, uint64_t key1, void* out) {
  FSR_REQUIRE(ctx, total_rows >= 0 && cols >= 0 && 0 <= row_begin && row_begin <= row_end &&
                       row_end <= total_rows,
              "gaussian_block: bad shape");
  const int64_t count = total_rows * cols, half = (count + 1) / 2;
  const int64_t f0 = row_begin * cols, f1 = row_end * cols;
  if (f1 <= f0) return FSR_OK;
  // radius indices needed: cos part [f0, min(f1, half)), sin part [max(f0,half)-half, f1-half)
  int64_t aLo = f0, aHi = f1 < half ? f1 : half;
  int64_t bLo = (f0 > half ? f0 : half) - half, bHi = f1 - half;
  if (aHi < aLo) aHi = aLo;
  if (bHi < bLo) bHi = bLo;
  // merge overlapping ranges so no group is emitted twice
  if (aHi > aLo && bHi > bLo && bLo <= aHi && aLo <= bHi) {
    aLo = aLo < bLo ? aLo : bLo;
    aHi = aHi > bHi ? aHi : bHi;
    bLo = bHi = 0;
  }
  // align each segment start down to 4 (kernel re-aligns), extend length accordingly
  const int64_t aLen = (aHi > aLo) ? aHi - (aLo & ~int64_t(3)) : 0;
  const int64_t bLen = (bHi > bLo) ? bHi - (bLo & ~int64_t(3)) : 0;
  const int64_t groups = (aLen + 3) / 4 + (bLen + 3) / 4;
  const int block = 256;
  const int grid = fsr::grid_for(groups, block, ctx, 32);
  fsr::StageTimer timer(ctx, FSR_STAGE_GAUSSIAN);
  if (dtype == FSR_F64)
    gaussian_kernel<double><<<grid, block, 0, ctx->stream>>>(count, half, f0, f1, aLo & ~int64_t(3), aLen,
                                                             bLo & ~int64_t(3), bLen, key0, key1,
                                                             (double*)out);
  else
    gaussian_kernel<float><<<grid, block, 0, ctx->stream>>>(count, half, f0, f1, aLo & ~int64_t(3), aLen,
                                                            bLo & ~int64_t(3), bLen, key0, key1,
                                                            (float*)out);
  return fsr::launched(ctx, "gaussian_kernel");
}

int fsr_csr_row_sums(fsr_ctx* ctx, int64_t n_rows, const int64_t* indptr, const double* data, double* deg) {
  FSR_REQUIRE(ctx, n_rows >= 0, "row_sums: bad shape");
  if (!n_rows) return FSR_OK;
  fsr::StageTimer timer(ctx, FSR_STAGE_NORMALIZE);
  row_sums_kernel<<<fsr::grid_for(n_rows, 256, ctx), 256, 0, ctx->stream>>>(n_rows, indptr, data, deg);
  return fsr::launched(ctx, "row_sums_kernel");
}

int fsr_csr_normalize(fsr_ctx* ctx, int dtype_out, int64_t n_rows, int64_t row_offset, const int64_t* indptr,
                      const int32_t* indices, const double* data, const double* deg, void* out) {
  FSR_REQUIRE(ctx, n_rows >= 0 && row_offset >= 0, "normalize: bad shape");
  if (!n_rows) return FSR_OK;
  const int grid = fsr::grid_for(n_rows * 32, 256, ctx);
  fsr::StageTimer timer(ctx, FSR_STAGE_NORMALIZE);
  if (dtype_out == FSR_F64)
    normalize_kernel<double><<<grid, 256, 0, ctx->stream>>>(n_rows, row_offset, indptr, indices, data, deg,
                                                            (double*)out);
  else
    normalize_kernel<float><<<grid, 256, 0, ctx->stream>>>(n_rows, row_offset, indptr, indices, data, deg,
                                                           (float*)out);
  return fsr::launched(ctx, "normalize_kernel");
}

int fsr_convert_from_f64(fsr_ctx* ctx, int dtype, int64_t n, const double* in, void* out) {
  if (n <= 0) return FSR_OK;
  if (dtype == FSR_F64) {
    if ((const void*)in == out) return FSR_OK;
    FSR_CUDA(ctx, cudaMemcpyAsync(out, in, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    return FSR_OK;
  }
  convert_kernel<float><<<fsr::grid_for(n, 256, ctx), 256, 0, ctx->stream>>>(n, in, (float*)out);
  return fsr::launched(ctx, "convert_kernel");
}

}  // extern "C"
