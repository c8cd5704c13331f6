// Raw tcgen05 kind::f16 issue-rate probe, dense against 2:4 structured-sparse
// (tcgen05.mma.sp): one CTA per SM issues back-to-back MMAs from shared memory
// into TMEM, no TMA, no epilogue.  Operand contents and the sparsity metadata
// are irrelevant to the rate (zeros / whatever TMEM holds): the question is
// whether a sparse M x N x 32 step costs what a dense M x N x 16 step costs,
// i.e. whether K9t's main pass could halve its MMA time (next levers).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_sp_rate tools/mma_sp_rate.cu -lcuda
//   tools/mma_sp_rate
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// kind::f16: A, B fp16, D fp32, K-major; bit 2 = sparse A
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, bool sparse) {
  return (sparse ? 4u : 0u) | (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
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

template <int SP>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, uint32_t meta) {
  if (SP == 0)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(meta)
        : "memory");
}

// M = 128 rows, N columns; dense: K = 16 fp16 (32 bytes of A and of B per row); sparse: K = 32
// (32 bytes of compressed A, 64 bytes of B per row).  SP = 0 dense, 1 sparse.
template <int SP, int N>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  constexpr int CG = 1;
  const uint32_t rank = 0;
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
  constexpr uint32_t idesc = idesc_f16(128, N, SP != 0);
  const uint64_t a0 = desc_sw64(su32(base)), b0 = desc_sw64(su32(base + 4 * 128 * 64));
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0 && rank == 0) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        // A advances 32 bytes per step in both modes; B 32 (dense) or 64 (sparse) bytes
        mma<SP>(tmem, a0 + (uint64_t)((u * 128 * 64) >> 4), b0 + (uint64_t)((u * N * 64) >> 4), idesc, 1u, tmem + 256);
        mma<SP>(tmem, a0 + (uint64_t)((u * 128 * 64 + 32) >> 4),
                b0 + (uint64_t)((u * N * 64 + (SP ? 0 : 32)) >> 4), idesc, 1u, tmem + 256);
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

template <int SP, int N>
void run(int sms, int iters) {
  constexpr int CG = 1;
  const int smem = 4 * 128 * 64 + 4 * N * 64 + 1024;
  cudaFuncSetAttribute(rate_kernel<SP, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
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
  cudaLaunchKernelEx(&cfg, rate_kernel<SP, N>, iters / 10, cyc);  // warm-up
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, rate_kernel<SP, N>, iters, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[1024] = {0};
  cudaMemcpy(h, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const int K = SP ? 32 : 16;  // logical K per MMA
  const double macs = (double)sms * iters * 8 * 128.0 * N * K;
  const double mma_per_sm_cycle = (double)iters * 8 / mx;  // MMAs per issuing-CTA cycle
  printf("{\"sparse\": %d, \"M\": 128, \"N\": %d, \"K\": %d, \"ctas\": %d, \"err\": \"%s\", \"ms\": %.3f, "
         "\"logical_tflops\": %.1f, \"cycles_per_mma\": %.2f}\n",
         SP, N, K, sms, cudaGetErrorString(err), ms, 2 * macs / (ms * 1e-3) / 1e12, 1.0 / mma_per_sm_cycle);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  run<0, 128>(sms, iters);
  run<1, 128>(sms, iters);
  run<0, 256>(sms, iters);
  run<1, 256>(sms, iters);
  return 0;
}
