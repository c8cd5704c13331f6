// K2 schedule probe: L2-resident column panels x source-row slabs (B200, sm_100a).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/k2_slab tools/k2_slab.cu
//   tools/k2_slab [n] [k]        -> JSON lines
//
// B = S Q with S a random CSR of the C3 graph's shape (n rows, 8..50 sorted
// random columns per row), Q dense n x k fp32.  Q is held panel-major
// ([k/W][n][W]); a pass handles one W-column panel and one slab of source
// rows (columns [h n/H, (h+1) n/H) of S), so the slab's n/H x W block of Q
// (<= 64 MB) stays in L2 while every nonzero of the slab gathers from it.
// Slabs after the first continue from the partial sums in B, so every output
// element is still the sequential CSR-order sum (bitwise the reference).
// Entries are staged per warp through shared memory from a slab-major packed
// (column, value) copy of S, so index loads cost one L1 wavefront per 128
// bytes instead of one per row of the warp.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_hint(const float4* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int2 ld_stream2(const int2* p, uint64_t pol) {
  int2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_stream4(float4* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}

// One warp = G = 32 / LPR consecutive rows; lane sl of a row's group owns 4
// columns of the W = 4 LPR wide panel.  ptr: slab CSR row pointers (n + 1),
// ent: packed (column - slab base, value bits).  Xs: the slab's block of the
// panel (rows x W, contiguous).  Y: row-major output, ldy floats per row.
template <int LPR, int DEPTH, int CAP, bool HINTS, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) slab_kernel(int64_t n_rows, const int64_t* __restrict__ ptr,
                                                   const int2* __restrict__ ent, const float4* __restrict__ Xs,
                                                   float* __restrict__ Y, int64_t ldy, int64_t c0, int accumulate,
                                                   int64_t xs4 = LPR) {
  constexpr int G = 32 / LPR;
  __shared__ int2 stage[8][CAP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / LPR, sl = lane % LPR;
  const int64_t r0 = ((int64_t)blockIdx.x * 8 + warp) * G;
  if (r0 >= n_rows) return;
  const int64_t i = r0 + grp;
  const bool live = i < n_rows;
  const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
  // row pointers of the warp's rows: lanes 0..G load ptr[r0 + lane]
  int64_t my_ptr = 0;
  if (lane <= G) my_ptr = __ldg(ptr + min(r0 + lane, n_rows));
  const int64_t p0 = __shfl_sync(0xffffffffu, my_ptr, 0);
  const int64_t p1 = __shfl_sync(0xffffffffu, my_ptr, G);
  const int64_t e0 = __shfl_sync(0xffffffffu, my_ptr, grp);
  const int64_t e1 = __shfl_sync(0xffffffffu, my_ptr, grp + 1);
  float4* yp = reinterpret_cast<float4*>(Y + i * ldy + c0) + sl;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (accumulate && live) acc = *yp;
  int2* st = stage[warp];
  for (int64_t base = p0; base < p1; base += CAP) {
    const int cnt = (int)min((int64_t)CAP, p1 - base);
    __syncwarp();
    for (int t = lane; t < cnt; t += 32) st[t] = HINTS ? ld_stream2(ent + base + t, pol_stream) : __ldg(ent + base + t);
    __syncwarp();
    const int lo = (int)max(e0 - base, (int64_t)0);
    const int hi = (int)min(e1 - base, (int64_t)cnt);
    for (int j = lo; j < hi; j += DEPTH) {
      int2 cv[DEPTH];
      float4 v[DEPTH];
#pragma unroll
      for (int g = 0; g < DEPTH; ++g) cv[g] = st[min(j + g, hi - 1)];
#pragma unroll
      for (int g = 0; g < DEPTH; ++g) {
        const float4* p = Xs + (int64_t)cv[g].x * xs4 + sl;
        v[g] = HINTS ? ld_hint(p, pol_keep) : __ldg(p);
      }
#pragma unroll
      for (int g = 0; g < DEPTH; ++g) {
        if (j + g < hi) {
          const float a = __int_as_float(cv[g].y);
          acc.x = fmaf(a, v[g].x, acc.x);
          acc.y = fmaf(a, v[g].y, acc.y);
          acc.z = fmaf(a, v[g].z, acc.z);
          acc.w = fmaf(a, v[g].w, acc.w);
        }
      }
    }
  }
  if (live) {
    if (HINTS)
      st_stream4(yp, acc, pol_stream);
    else
      *yp = acc;
  }
}


// ---- pipelined variant: a producer warp stages (row pointers, entries) of
// 8-row blocks into a shared-memory ring with bulk async copies; 7 consumer
// warps gather.  Consumers never wait for their index stream.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int LPR, int DEPTH, int RB, int CAP, int NS>
__global__ void __launch_bounds__(256) slab_pipe_kernel(int64_t n_rows, const int64_t* __restrict__ ptr,
                                                        const int2* __restrict__ ent, const float4* __restrict__ Xs,
                                                        float* __restrict__ Y, int64_t ldy, int64_t c0, int accumulate) {
  constexpr int G = 32 / LPR;    // rows in flight per warp
  constexpr int NC = 7;          // consumer warps
  constexpr int PW = RB + 2;     // staged row pointers (80 bytes for RB = 8)
  extern __shared__ __align__(16) unsigned char dyn[];
  int2* s_ent = reinterpret_cast<int2*>(dyn);                                  // [NS][CAP]
  int64_t* s_ptr = reinterpret_cast<int64_t*>(dyn + (size_t)NS * CAP * 8);    // [NS][PW]
  uint64_t* full = reinterpret_cast<uint64_t*>(s_ptr + NS * PW);
  uint64_t* empty = full + NS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t n_blocks = (n_rows + RB - 1) / RB;
  const int64_t my_blocks = blockIdx.x < n_blocks ? (n_blocks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (warp == 0) {
    for (int64_t q0 = 0; q0 < my_blocks; q0 += 32) {
      const int64_t q = q0 + lane;
      int64_t p0 = 0, p1 = 0, r0 = 0;
      if (q < my_blocks) {
        r0 = ((int64_t)blockIdx.x + q * gridDim.x) * RB;
        p0 = __ldg(ptr + r0);
        p1 = __ldg(ptr + min(r0 + RB, n_rows));
      }
      const int cnt = (int)min((int64_t)32, my_blocks - q0);
      for (int l = 0; l < cnt; ++l) {
        const int64_t b0 = __shfl_sync(0xffffffffu, p0, l), b1 = __shfl_sync(0xffffffffu, p1, l);
        const int64_t rr = __shfl_sync(0xffffffffu, r0, l);
        if (lane == 0) {
          const int64_t qq = q0 + l;
          const int slot = (int)(qq % NS);
          mbar_wait(&empty[slot], (uint32_t)(((qq / NS) & 1) ^ 1));
          const int64_t a0 = b0 & ~(int64_t)1;
          const uint32_t eb = (uint32_t)((((b1 - a0) * 8) + 15) & ~(int64_t)15);
          mbar_expect_tx(&full[slot], eb + PW * 8);
          bulk_g2s(s_ptr + slot * PW, ptr + rr, PW * 8, &full[slot]);
          if (eb) bulk_g2s(s_ent + (size_t)slot * CAP, ent + a0, eb, &full[slot]);
        }
      }
    }
    return;
  }
  const int cw = warp - 1;
  const int grp = lane / LPR, sl = lane % LPR;
  for (int64_t q = cw; q < my_blocks; q += NC) {
    const int slot = (int)(q % NS);
    const int64_t r0 = ((int64_t)blockIdx.x + q * gridDim.x) * RB;
    mbar_wait(&full[slot], (uint32_t)((q / NS) & 1));
    const int64_t* sp = s_ptr + slot * PW;
    const int2* st = s_ent + (size_t)slot * CAP;
    const int64_t a0 = sp[0] & ~(int64_t)1;
    int row = grp;
    int j = (int)(sp[row] - a0), e = (int)(sp[row + 1] - a0);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (accumulate && r0 + row < n_rows) acc = *(reinterpret_cast<const float4*>(Y + (r0 + row) * ldy + c0) + sl);
    while (true) {
      while (row < RB && j >= e) {
        if (r0 + row < n_rows) *(reinterpret_cast<float4*>(Y + (r0 + row) * ldy + c0) + sl) = acc;
        row += G;
        if (row < RB) {
          j = (int)(sp[row] - a0);
          e = (int)(sp[row + 1] - a0);
          acc = make_float4(0.f, 0.f, 0.f, 0.f);
          if (accumulate && r0 + row < n_rows) acc = *(reinterpret_cast<const float4*>(Y + (r0 + row) * ldy + c0) + sl);
        }
      }
      const bool active = row < RB;
      if (!__any_sync(0xffffffffu, active)) break;
      const int cnt = active ? min(DEPTH, e - j) : 0;
      int2 cv[DEPTH];
      float4 v[DEPTH];
#pragma unroll
      for (int g = 0; g < DEPTH; ++g) cv[g] = g < cnt ? st[j + g] : make_int2(0, 0);
#pragma unroll
      for (int g = 0; g < DEPTH; ++g)
        if (g < cnt) v[g] = __ldg(Xs + (int64_t)cv[g].x * LPR + sl);
#pragma unroll
      for (int g = 0; g < DEPTH; ++g) {
        if (g < cnt) {
          const float a = __int_as_float(cv[g].y);
          acc.x = fmaf(a, v[g].x, acc.x);
          acc.y = fmaf(a, v[g].y, acc.y);
          acc.z = fmaf(a, v[g].z, acc.z);
          acc.w = fmaf(a, v[g].w, acc.w);
        }
      }
      j += cnt;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
}

template <int LPR, int DEPTH, int RB, int CAP, int NS>
static float run_pipe(int H, int64_t n, int n_panels_timed, const std::vector<int64_t*>& d_ptr,
                      const std::vector<int2*>& d_ent, const float* d_Xp, float* d_Y, int64_t ldy, int reps) {
  constexpr int W = 4 * LPR;
  const int64_t slab_rows = (n + H - 1) / H;
  const size_t smem = (size_t)NS * CAP * 8 + (size_t)NS * (RB + 2) * 8 + (size_t)NS * 16;
  auto kern = slab_pipe_kernel<LPR, DEPTH, RB, CAP, NS>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
  const unsigned grid = 148u * (unsigned)std::max(per_sm, 1);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto pass = [&](int p) {
    for (int h = 0; h < H; ++h) {
      const float4* Xs = reinterpret_cast<const float4*>(d_Xp + ((int64_t)p * n + (int64_t)h * slab_rows) * W);
      if (getenv("K2_YPANEL"))
        kern<<<grid, 256, smem>>>(n, d_ptr[h], d_ent[h], Xs, d_Y + (int64_t)p * n * W, W, 0, h > 0);
      else
        kern<<<grid, 256, smem>>>(n, d_ptr[h], d_ent[h], Xs, d_Y, ldy, (int64_t)p * W, h > 0);
    }
  };
  pass(0);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r)
    for (int p = 0; p < n_panels_timed; ++p) pass(p);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / (reps * n_panels_timed);
}


// ---- block variant: a warp owns RBW consecutive rows; their entries (one
// contiguous range of the slab CSR) are staged with one round of coalesced
// loads, then every LPR-lane group walks its rows (grp, grp + G, ...) on its
// own -- no lock step between the groups' rows, start-up paid once per RBW rows.
template <int LPR, int DEPTH, int RBW, int CAP>
__global__ void __launch_bounds__(256) slab_block_kernel(int64_t n_rows, const int64_t* __restrict__ ptr,
                                                         const int2* __restrict__ ent, const float4* __restrict__ Xs,
                                                         float* __restrict__ Y, int64_t ldy, int64_t c0, int accumulate) {
  constexpr int G = 32 / LPR;
  extern __shared__ __align__(16) unsigned char dyn[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int2* st = reinterpret_cast<int2*>(dyn) + (size_t)warp * CAP;
  int64_t* sp = reinterpret_cast<int64_t*>(dyn + (size_t)8 * CAP * 8) + warp * (RBW + 1);
  const int grp = lane / LPR, sl = lane % LPR;
  const int64_t r0 = ((int64_t)blockIdx.x * 8 + warp) * RBW;
  if (r0 >= n_rows) return;
  for (int t = lane; t <= RBW; t += 32) sp[t] = __ldg(ptr + min(r0 + t, n_rows));
  __syncwarp();
  const int64_t p0 = sp[0], p1 = sp[RBW];
  int row = grp;
  int64_t j = sp[row], e = sp[row + 1];
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (accumulate && r0 + row < n_rows) acc = *(reinterpret_cast<const float4*>(Y + (r0 + row) * ldy + c0) + sl);
  for (int64_t base = p0;; base += CAP) {
    const int64_t wend = min(p1, base + CAP);
    __syncwarp();
    for (int64_t t = base + lane; t < wend; t += 32) st[t - base] = __ldg(ent + t);
    __syncwarp();
    while (true) {
      while (row < RBW && j >= e) {
        if (r0 + row < n_rows) *(reinterpret_cast<float4*>(Y + (r0 + row) * ldy + c0) + sl) = acc;
        row += G;
        if (row < RBW) {
          j = sp[row];
          e = sp[row + 1];
          acc = make_float4(0.f, 0.f, 0.f, 0.f);
          if (accumulate && r0 + row < n_rows)
            acc = *(reinterpret_cast<const float4*>(Y + (r0 + row) * ldy + c0) + sl);
        }
      }
      const bool active = row < RBW && j < wend;
      if (!__any_sync(0xffffffffu, active)) break;
      const int cnt = active ? (int)min((int64_t)DEPTH, min(e, wend) - j) : 0;
      const int o = (int)(j - base);
      int2 cv[DEPTH];
      float4 v[DEPTH];
#pragma unroll
      for (int g = 0; g < DEPTH; ++g) cv[g] = g < cnt ? st[o + g] : make_int2(0, 0);
#pragma unroll
      for (int g = 0; g < DEPTH; ++g)
        if (g < cnt) v[g] = __ldg(Xs + (int64_t)cv[g].x * LPR + sl);
#pragma unroll
      for (int g = 0; g < DEPTH; ++g) {
        if (g < cnt) {
          const float a = __int_as_float(cv[g].y);
          acc.x = fmaf(a, v[g].x, acc.x);
          acc.y = fmaf(a, v[g].y, acc.y);
          acc.z = fmaf(a, v[g].z, acc.z);
          acc.w = fmaf(a, v[g].w, acc.w);
        }
      }
      j += cnt;
    }
    if (wend >= p1) break;
  }
}

template <int LPR, int DEPTH, int RBW, int CAP>
static float run_block(int H, int64_t n, int n_panels_timed, const std::vector<int64_t*>& d_ptr,
                       const std::vector<int2*>& d_ent, const float* d_Xp, float* d_Y, int64_t ldy, int reps) {
  constexpr int W = 4 * LPR;
  const int64_t slab_rows = (n + H - 1) / H;
  const size_t smem = (size_t)8 * CAP * 8 + (size_t)8 * (RBW + 1) * 8;
  auto kern = slab_block_kernel<LPR, DEPTH, RBW, CAP>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned grid = (unsigned)((n + 8 * RBW - 1) / (8 * RBW));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto pass = [&](int p) {
    for (int h = 0; h < H; ++h) {
      const float4* Xs = reinterpret_cast<const float4*>(d_Xp + ((int64_t)p * n + (int64_t)h * slab_rows) * W);
      if (getenv("K2_YPANEL"))
        kern<<<grid, 256, smem>>>(n, d_ptr[h], d_ent[h], Xs, d_Y + (int64_t)p * n * W, W, 0, h > 0);
      else
        kern<<<grid, 256, smem>>>(n, d_ptr[h], d_ent[h], Xs, d_Y, ldy, (int64_t)p * W, h > 0);
    }
  };
  pass(0);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r)
    for (int p = 0; p < n_panels_timed; ++p) pass(p);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / (reps * n_panels_timed);
}

// Reference: thread per (row, column), CSR order, fmaf.
__global__ void ref_kernel(int64_t n, const int64_t* ptr, const int32_t* cols, const float* vals, const float* Xp,
                           int W, float* Yref) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * W) return;
  const int64_t i = t / W;
  const int c = (int)(t % W);
  float acc = 0.f;
  for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) acc = fmaf(vals[e], Xp[(int64_t)cols[e] * W + c], acc);
  Yref[t] = acc;
}

__global__ void cmp_kernel(int64_t n, int W, const float* Y, int64_t ldy, int64_t c0, const float* Yref,
                           unsigned long long* bad) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * W) return;
  const int64_t i = t / W;
  const int c = (int)(t % W);
  if (__float_as_uint(Y[i * ldy + c0 + c]) != __float_as_uint(Yref[t])) atomicAdd(bad, 1ull);
}

__global__ void fill_kernel(float* p, int64_t n, uint64_t seed) {
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += nt) {
    uint64_t s = (t + 1) * 0x9E3779B97F4A7C15ull + seed;
    s ^= s >> 29;
    s *= 0xBF58476D1CE4E5B9ull;
    s ^= s >> 32;
    p[t] = (float)((double)(s & 0xffffff) / 16777216.0 - 0.5);
  }
}

static uint64_t rng_state = 88172645463325252ull;
static inline uint64_t xr() {
  rng_state ^= rng_state << 13;
  rng_state ^= rng_state >> 7;
  rng_state ^= rng_state << 17;
  return rng_state;
}

__global__ void fill_kernel(float* p, int64_t n, uint64_t seed);

template <int LPR, int DEPTH, int CAP, bool HINTS, int MINB = 1>
static float run_cfg(int H, int64_t n, int n_panels_timed, const std::vector<int64_t*>& d_ptr,
                     const std::vector<int2*>& d_ent, const float* d_Xp, float* d_Y, int64_t ldy, int reps) {
  constexpr int W = 4 * LPR, G = 32 / LPR;
  const int64_t slab_rows = (n + H - 1) / H;
  const unsigned grid = (unsigned)((n + 8 * G - 1) / (8 * G));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  static float* d_Xr = nullptr;  // K2_XROW: X row-major (n x ldy floats), gathers strided by ldy
  if (getenv("K2_XROW")) {
    if (!d_Xr) {
      CK(cudaMalloc(&d_Xr, (size_t)n * ldy * 4));
      fill_kernel<<<148 * 8, 256>>>(d_Xr, n * ldy, 11);
    }
    CK(cudaMemcpy2D(d_Xr, (size_t)ldy * 4, d_Xp, (size_t)W * 4, (size_t)W * 4, (size_t)n, cudaMemcpyDeviceToDevice));
  }
  auto pass = [&](int p) {
    for (int h = 0; h < H; ++h) {
      const float4* Xs = reinterpret_cast<const float4*>(d_Xp + ((int64_t)p * n + (int64_t)h * slab_rows) * W);
      if (d_Xr && getenv("K2_XROW")) {
        const float4* Xr = reinterpret_cast<const float4*>(d_Xr + (int64_t)h * slab_rows * ldy + (int64_t)p * W);
        slab_kernel<LPR, DEPTH, CAP, HINTS, MINB><<<grid, 256>>>(n, d_ptr[h], d_ent[h], Xr, d_Y, ldy, (int64_t)p * W, h > 0,
                                                                 ldy / 4);
      } else if (getenv("K2_YPANEL"))  // panel-major output: panel p at d_Y + p n W, W floats per row
        slab_kernel<LPR, DEPTH, CAP, HINTS, MINB><<<grid, 256>>>(n, d_ptr[h], d_ent[h], Xs, d_Y + (int64_t)p * n * W, W, 0, h > 0);
      else
        slab_kernel<LPR, DEPTH, CAP, HINTS, MINB><<<grid, 256>>>(n, d_ptr[h], d_ent[h], Xs, d_Y, ldy, (int64_t)p * W, h > 0);
    }
  };
  pass(0);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r)
    for (int p = 0; p < n_panels_timed; ++p) pass(p);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / (reps * n_panels_timed);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 1000000;
  const int64_t k = argc > 2 ? atoll(argv[2]) : 5500;
  const int lo = 8, hi = 50;
  // host CSR
  std::vector<int64_t> ptr(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) ptr[i + 1] = ptr[i] + lo + (int64_t)(xr() % (hi - lo + 1));
  const int64_t nnz = ptr[n];
  std::vector<int32_t> cols(nnz);
  std::vector<float> vals(nnz);
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) cols[e] = (int32_t)(xr() % n);
    std::sort(cols.begin() + ptr[i], cols.begin() + ptr[i + 1]);
    for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) vals[e] = (float)((xr() & 0xffff) / 65536.0);
  }
  printf("{\"n\": %lld, \"k\": %lld, \"nnz\": %lld}\n", (long long)n, (long long)k, (long long)nnz);
  fflush(stdout);
  int64_t *d_ptr0;
  int32_t* d_cols;
  float* d_vals;
  CK(cudaMalloc(&d_ptr0, (n + 1) * 8));
  CK(cudaMalloc(&d_cols, nnz * 4));
  CK(cudaMalloc(&d_vals, nnz * 4));
  CK(cudaMemcpy(d_ptr0, ptr.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_cols, cols.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_vals, vals.data(), nnz * 4, cudaMemcpyHostToDevice));
  const int P = 8;           // panels of 64 columns' worth of X held (rotated so each pass starts cold)
  const int64_t XW = 64 * P;  // floats per row held
  float* d_Xp;
  CK(cudaMalloc(&d_Xp, n * XW * 4));
  fill_kernel<<<148 * 8, 256>>>(d_Xp, n * XW, 7);
  const int64_t ldy = (k + 3) / 4 * 4;
  float* d_Y;
  CK(cudaMalloc(&d_Y, n * ldy * 4));
  CK(cudaMemset(d_Y, 0, n * ldy * 4));
  float* d_ref;
  CK(cudaMalloc(&d_ref, n * 64 * 4));
  unsigned long long* d_bad;
  CK(cudaMalloc(&d_bad, 8));

  for (int H : {1, 2, 4}) {
    // slab-major packed copies
    const int64_t slab_rows = (n + H - 1) / H;
    std::vector<std::vector<int64_t>> sp(H, std::vector<int64_t>(n + 1 + 16, 0));
    std::vector<std::vector<int2>> se(H);
    for (int h = 0; h < H; ++h) se[h].reserve(nnz / H + n);
    for (int64_t i = 0; i < n; ++i) {
      for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
        const int h = (int)(cols[e] / slab_rows);
        int2 x;
        x.x = (int)(cols[e] - h * slab_rows);
        memcpy(&x.y, &vals[e], 4);
        se[h].push_back(x);
      }
      for (int h = 0; h < H; ++h) sp[h][i + 1] = (int64_t)se[h].size();
    }
    for (int h = 0; h < H; ++h)
      for (int t = 1; t <= 16; ++t) sp[h][n + t] = sp[h][n];  // padding the bulk copies may read
    std::vector<int64_t*> d_ptr(H);
    std::vector<int2*> d_ent(H);
    for (int h = 0; h < H; ++h) {
      CK(cudaMalloc(&d_ptr[h], (n + 1 + 16) * 8));
      CK(cudaMalloc(&d_ent[h], (se[h].size() + 4) * 8));
      CK(cudaMemcpy(d_ptr[h], sp[h].data(), (n + 1 + 16) * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(d_ent[h], se[h].data(), se[h].size() * 8, cudaMemcpyHostToDevice));
    }
    auto report = [&](const char* name, int W, float ms) {
      // check panel 0 bitwise against the reference kernel (panel 0 of width W)
      ref_kernel<<<(unsigned)((n * W + 255) / 256), 256>>>(n, d_ptr0, d_cols, d_vals, d_Xp, W, d_ref);
      CK(cudaMemset(d_bad, 0, 8));
      cmp_kernel<<<(unsigned)((n * W + 255) / 256), 256>>>(n, W, d_Y, getenv("K2_YPANEL") ? W : ldy, 0, d_ref, d_bad);
      unsigned long long bad = 0;
      CK(cudaMemcpy(&bad, d_bad, 8, cudaMemcpyDeviceToHost));
      const double passes = (double)((k + W - 1) / W);
      printf("{\"cfg\": \"%s\", \"H\": %d, \"W\": %d, \"ms_per_panel\": %.4f, \"extrapolated_ms\": %.2f, "
             "\"gather_TBs\": %.2f, \"mismatches\": %llu}\n",
             name, H, W, ms, ms * passes, (double)nnz * W * 4 / ms / 1e9, bad);
      fflush(stdout);
    };
    const int reps = 3;
#define RUN(LPR, DEPTH, CAP, HINTS, NAME)                                                                      \
  {                                                                                                            \
    const int npan = (int)(XW / (4 * LPR));                                                                    \
    const float ms = run_cfg<LPR, DEPTH, CAP, HINTS>(H, n, npan, d_ptr, d_ent, d_Xp, d_Y, ldy, reps);        \
    report(NAME, 4 * LPR, ms);                                                                                 \
  }
    if (H == 1) {
      RUN(2, 8, 512, true, "w8_d8_hint");
      RUN(4, 8, 256, true, "w16_d8_hint");
      RUN(4, 8, 256, false, "w16_d8_nohint");
      RUN(4, 4, 256, true, "w16_d4_hint");
    }
#define RUNP(LPR, DEPTH, RB, CAP, NS, NAME)                                                                   \
  {                                                                                                            \
    const int npan = (int)(XW / (4 * LPR));                                                                    \
    const float ms = run_pipe<LPR, DEPTH, RB, CAP, NS>(H, n, npan, d_ptr, d_ent, d_Xp, d_Y, ldy, reps);      \
    report(NAME, 4 * LPR, ms);                                                                                 \
  }
#define RUNB(LPR, DEPTH, RBW, CAP, NAME)                                                                      \
  {                                                                                                            \
    const int npan = (int)(XW / (4 * LPR));                                                                    \
    const float ms = run_block<LPR, DEPTH, RBW, CAP>(H, n, npan, d_ptr, d_ent, d_Xp, d_Y, ldy, reps);        \
    report(NAME, 4 * LPR, ms);                                                                                 \
  }
    if (H == 1) {
      RUNB(4, 4, 32, 1024, "block_w16_d4_r32");
      RUNB(4, 8, 32, 1024, "block_w16_d8_r32");
      RUNB(4, 4, 16, 512, "block_w16_d4_r16");
    }
#define RUNM(LPR, DEPTH, CAP, MINB, NAME)                                                                     \
  {                                                                                                            \
    const int npan = (int)(XW / (4 * LPR));                                                                    \
    const float ms = run_cfg<LPR, DEPTH, CAP, false, MINB>(H, n, npan, d_ptr, d_ent, d_Xp, d_Y, ldy, reps); \
    report(NAME, 4 * LPR, ms);                                                                                 \
  }
    if (H == 2) {
      RUNM(8, 4, 128, 8, "w32_d4_occ8");
      RUNM(8, 4, 128, 6, "w32_d4_occ6");
      RUNM(8, 2, 128, 8, "w32_d2_occ8");
      RUNM(8, 6, 128, 6, "w32_d6_occ6");
      RUNM(8, 3, 128, 8, "w32_d3_occ8");
    }
    if (H == 1) {
      RUNM(4, 4, 256, 8, "w16_d4_occ8");
      RUNM(4, 6, 256, 6, "w16_d6_occ6");
    }
    if (H == 2) {
      RUNB(8, 4, 32, 1024, "block_w32_d4_r32");
      RUNB(8, 8, 32, 1024, "block_w32_d8_r32");
      RUNB(8, 4, 16, 512, "block_w32_d4_r16");
      RUNB(8, 4, 32, 512, "block_w32_d4_r32_c512");
      RUNB(8, 2, 32, 1024, "block_w32_d2_r32");
    }
    if (H == 1) {
      RUNP(4, 4, 8, 512, 14, "pipe_w16_d4");
      RUNP(4, 8, 8, 512, 14, "pipe_w16_d8");
    }
    if (H == 2) {
      RUNP(8, 4, 8, 512, 14, "pipe_w32_d4");
      RUNP(8, 8, 8, 512, 14, "pipe_w32_d8");
      RUNP(8, 8, 8, 512, 28, "pipe_w32_d8_ns28");
    }
    if (H == 2) {
      RUN(4, 8, 256, true, "w16_d8_hint");
      RUN(8, 8, 128, true, "w32_d8_hint");
      RUN(8, 8, 128, false, "w32_d8_nohint");
      RUN(8, 4, 128, true, "w32_d4_hint");
    }
    if (H == 4) {
      RUN(8, 8, 128, true, "w32_d8_hint");
      RUN(16, 8, 64, true, "w64_d8_hint");
      RUN(16, 4, 64, true, "w64_d4_hint");
    }
    for (int h = 0; h < H; ++h) {
      cudaFree(d_ptr[h]);
      cudaFree(d_ent[h]);
    }
  }
  return 0;
}
