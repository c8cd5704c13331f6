// Raw tcgen05 kind::i8 issue-rate probe: one CTA (or CTA pair) per SM issues
// back-to-back MMAs from shared memory into TMEM, no TMA, no epilogue, and the
// achieved int8 TOPS are printed for M x N x 32 shapes with cta_group::1 and
// cta_group::2.  Operand contents are irrelevant (zeros): only the rate is
// measured.  This is the ceiling the Ozaki kernels in tc_gemm.cu run against.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu -lcuda
//   tools/mma_rate
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

template <int CG>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (CG == 1)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

// M = 128 * CG rows of the MMA (each CTA holds 128), N columns, K = 32 bytes.
template <int CG, int N>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  // A: 128 x 64 bytes x 4 buffers; B: N/CG x 64 bytes x 4 buffers
  for (int i = threadIdx.x; i < (4 * 128 * 64 + 4 * N * 64) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = idesc_i8(128 * CG, N);
  const uint64_t a0 = desc_sw64(su32(base)), b0 = desc_sw64(su32(base + 4 * 128 * 64));
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0 && rank == 0) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        // two K=32 halves of a 64-byte swizzle atom per buffer
        mma<CG>(tmem + (u & 1) * 256 % 512, a0 + (uint64_t)((u * 128 * 64) >> 4),
                b0 + (uint64_t)((u * (N / CG) * 64) >> 4), idesc, 1u);
        mma<CG>(tmem + (u & 1) * 256 % 512, a0 + (uint64_t)((u * 128 * 64 + 32) >> 4),
                b0 + (uint64_t)((u * (N / CG) * 64 + 32) >> 4), idesc, 1u);
      }
    }
    if (CG == 1)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                   : "memory");
    else
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              su32(&bar)),
          "h"((uint16_t)3)
          : "memory");
  }
  __syncwarp();
  if (threadIdx.x == 0 && (CG == 2 || rank == 0)) {
    uint32_t done = 0;
    do {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(su32(&bar))
          : "memory");
    } while (!done);
    t1 = clock64();
    if (rank == 0) cycles[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int CG, int N>
void run(int sms, int iters) {
  const int smem = 4 * 128 * 64 + 4 * N * 64 + 1024;
  cudaFuncSetAttribute(rate_kernel<CG, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  cudaMemset(cyc, 0, sms * sizeof(unsigned long long));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, rate_kernel<CG, N>, iters / 10, cyc);  // warm-up
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, rate_kernel<CG, N>, iters, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[1024] = {0};
  cudaMemcpy(h, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double macs = (double)sms / CG * iters * 8 * (128.0 * CG) * N * 32;
  const double mma_per_sm_cycle = (double)iters * 8 / mx;  // MMAs per issuing-CTA cycle
  printf("{\"cg\": %d, \"M\": %d, \"N\": %d, \"K\": 32, \"ctas\": %d, \"err\": \"%s\", \"ms\": %.3f, \"tops\": %.1f, "
         "\"cycles_per_mma\": %.2f, \"macs_per_sm_cycle\": %.0f}\n",
         CG, 128 * CG, N, sms, cudaGetErrorString(err), ms, 2 * macs / (ms * 1e-3) / 1e12, 1.0 / mma_per_sm_cycle,
         (128.0 * CG * N * 32) * mma_per_sm_cycle / CG);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  run<1, 64>(sms, iters);
  run<1, 128>(sms, iters);
  run<1, 256>(sms, iters);
  run<2, 128>(sms, iters);
  run<2, 256>(sms, iters);
  return 0;
}
