// FMA-pipe rate probe for the online filter's inner loop:
// warp-instruction throughput of fp32 FFMA (3 registers), FHFMA
// (fma.rn.f32.f16: fp16 x fp16 + fp32), FFMA2 (fma.rn.f32x2) and HFMA2, and
// of the shared-memory-staged K9 inner loop (entry broadcast by shuffle ->
// LDS.128 of 8 fp16 query values -> 8 FHFMA), on all SMs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fma_rate tools/fma_rate.cu
//   tools/fma_rate
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kIters = 4096;

__global__ void ffma_kernel(float* out, float a0, float b0) {
  float acc[16];
  float a = a0 + threadIdx.x, b = b0;
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = k;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[k]) : "f"(a), "f"(b));
    a += 1e-7f;
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void fhfma_kernel(float* out, float a0) {
  float acc[16];
  __half2 z = __floats2half2_rn(a0, a0 + 1);
  uint32_t zp = *reinterpret_cast<uint32_t*>(&z);
  uint16_t ah = __half_as_ushort(__float2half_rn(a0 + threadIdx.x));
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = k;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; k += 2)
      asm volatile(
          "{ .reg .f16 lo, hi, ah; mov.b32 {lo, hi}, %2; mov.b16 ah, %3;\n\t"
          "fma.rn.f32.f16 %0, ah, lo, %0; fma.rn.f32.f16 %1, ah, hi, %1; }"
          : "+f"(acc[k]), "+f"(acc[k + 1])
          : "r"(zp), "h"(ah));
    zp += 1;
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma2_kernel(float* out, float a0) {
  uint64_t acc[8];
  float2 av = make_float2(a0 + threadIdx.x, a0);
  uint64_t a = *reinterpret_cast<uint64_t*>(&av);
  uint64_t b = a ^ 0x1234;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = k;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[k]) : "l"(a), "l"(b));
    a += 3;
  }
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}

__global__ void hfma2_kernel(float* out, float a0) {
  uint32_t acc[16];
  __half2 z = __floats2half2_rn(a0, a0 + 1);
  uint32_t a = *reinterpret_cast<uint32_t*>(&z) + threadIdx.x, b = a ^ 7;
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = k;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) asm volatile("fma.rn.f16x2 %0, %1, %2, %0;" : "+r"(acc[k]) : "r"(a), "r"(b));
    a += 1;
  }
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}

// Staged K9 inner loop: each warp streams 32-entry chunks (col | fp16 u << 16)
// from global memory (next chunk prefetched), stages them in shared memory,
// reads them back two at a time (broadcast LDS.128), gathers each entry's
// 16-byte slice of a shared-memory Zh row (SROWS x 256 halves) and does 8
// FHFMA into the lane's 8 query accumulators.
template <int SROWS, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) staged_kernel(float* out, const uint32_t* ent, int nchunks) {
  extern __shared__ __align__(16) unsigned char zs[];
  __shared__ __align__(16) uint32_t ent_s[WARPS][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < SROWS * 128; i += blockDim.x) reinterpret_cast<uint32_t*>(zs)[i] = i * 2654435761u;
  __syncthreads();
  float acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.f;
  const uint32_t* src = ent + (size_t)(blockIdx.x * WARPS + warp) * 64 * 32;
  uint32_t nxt = src[lane];
  const unsigned char* zl = zs + lane * 16;
  for (int c = 0; c < nchunks; ++c) {
    const uint32_t cur = nxt;
    nxt = src[((c + 1) % 64) * 32 + lane];
    __syncwarp();
    ent_s[warp][lane] = cur;
    __syncwarp();
#pragma unroll 4
    for (int j = 0; j < 32; j += 4) {
      const uint4 e4 = *reinterpret_cast<const uint4*>(&ent_s[warp][j]);
      const uint32_t ee[4] = {e4.x, e4.y, e4.z, e4.w};
      uint4 t[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) t[g] = *reinterpret_cast<const uint4*>(zl + (ee[g] & 0xffffu) * 512);
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint16_t ah = (uint16_t)(ee[g] >> 16);
        asm("{ .reg .f16 lo, hi, ah; mov.b32 {lo, hi}, %2; mov.b16 ah, %3;\n\t"
            "fma.rn.f32.f16 %0, ah, lo, %0; fma.rn.f32.f16 %1, ah, hi, %1; }"
            : "+f"(acc[0]), "+f"(acc[1]) : "r"(t[g].x), "h"(ah));
        asm("{ .reg .f16 lo, hi, ah; mov.b32 {lo, hi}, %2; mov.b16 ah, %3;\n\t"
            "fma.rn.f32.f16 %0, ah, lo, %0; fma.rn.f32.f16 %1, ah, hi, %1; }"
            : "+f"(acc[2]), "+f"(acc[3]) : "r"(t[g].y), "h"(ah));
        asm("{ .reg .f16 lo, hi, ah; mov.b32 {lo, hi}, %2; mov.b16 ah, %3;\n\t"
            "fma.rn.f32.f16 %0, ah, lo, %0; fma.rn.f32.f16 %1, ah, hi, %1; }"
            : "+f"(acc[4]), "+f"(acc[5]) : "r"(t[g].z), "h"(ah));
        asm("{ .reg .f16 lo, hi, ah; mov.b32 {lo, hi}, %2; mov.b16 ah, %3;\n\t"
            "fma.rn.f32.f16 %0, ah, lo, %0; fma.rn.f32.f16 %1, ah, hi, %1; }"
            : "+f"(acc[6]), "+f"(acc[7]) : "r"(t[g].w), "h"(ah));
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float time_ms(F&& launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int threads = 256, per_sm = 8, grid = sms * per_sm;
  float* out;
  cudaMalloc(&out, (size_t)grid * threads * 4);
  const double warp_instr = (double)grid * threads / 32 * kIters * 16;  // per kernel (16 FMA-class instr per iter)
  struct R {
    const char* name;
    float ms;
    double instr;
    double macs_per_instr;
  } rs[5];
  rs[0] = {"FFMA (3 reg)", time_ms([&] { ffma_kernel<<<grid, threads>>>(out, 1.f, 1e-3f); }), warp_instr, 1};
  rs[1] = {"FHFMA fma.rn.f32.f16", time_ms([&] { fhfma_kernel<<<grid, threads>>>(out, 1.f); }), warp_instr, 1};
  rs[2] = {"FFMA2 fma.rn.f32x2", time_ms([&] { ffma2_kernel<<<grid, threads>>>(out, 1.f); }), warp_instr / 2, 2};
  rs[3] = {"HFMA2 fma.rn.f16x2", time_ms([&] { hfma2_kernel<<<grid, threads>>>(out, 1.f); }), warp_instr, 2};
  uint32_t* ent;
  const int nchunks = 256;
  const size_t nent = (size_t)sms * 32 * 64 * 32;
  cudaMalloc(&ent, nent * 4);
  uint32_t* h = new uint32_t[nent];
  uint32_t s = 12345;
  for (size_t i = 0; i < nent; ++i) {
    s = s * 1664525u + 1013904223u;
    h[i] = ((s >> 8) % 192) | (0x3c00u << 16);
  }
  cudaMemcpy(ent, h, nent * 4, cudaMemcpyHostToDevice);
  using KernT = void (*)(float*, const uint32_t*, int);
  auto run_staged = [&](KernT kern, int warps, int ctas_per_sm, int srows, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, srows * 512);
    const int g = sms * ctas_per_sm;
    void* args[] = {&out, &ent, (void*)&nchunks};
    float ms = time_ms([&] { cudaLaunchKernel((const void*)kern, dim3(g), dim3(32 * warps), args, srows * 512, 0); });
    cudaError_t err = cudaDeviceSynchronize();
    const double entries = (double)g * warps * nchunks * 32;  // warp-entries (256 queries x 1 entry each)
    printf("{\"op\": \"%s\", \"err\": \"%s\", \"ms\": %.4f, \"entry_x256q_per_clk_per_sm\": %.4f, "
           "\"ms_for_1e8_entries_x1024q\": %.3f}\n", name, cudaGetErrorString(err), ms,
           entries / (ms * 1e-3) / sms / (clk * 1e3), 4e8 / (entries / (ms * 1e-3)) * 1e3);
  };
  run_staged(staged_kernel<192, 8>, 8, 1, 192, "staged, 8 warps/SM, 96 KB");
  run_staged(staged_kernel<192, 8>, 8, 2, 192, "staged, 16 warps/SM (2 CTAs x 96 KB)");
  run_staged(staged_kernel<192, 16>, 16, 1, 192, "staged, 16 warps/SM (1 CTA x 96 KB)");
  run_staged(staged_kernel<96, 8>, 8, 3, 96, "staged, 24 warps/SM (3 CTAs x 48 KB)");
  run_staged(staged_kernel<96, 16>, 16, 2, 96, "staged, 32 warps/SM (2 CTAs x 48 KB)");
  for (int i = 0; i < 4; ++i) {
    const double per_smsp_clk = rs[i].instr / (rs[i].ms * 1e-3) / (sms * 4.0) / (clk * 1e3);
    printf("{\"op\": \"%s\", \"ms\": %.4f, \"warp_instr_per_smsp_clk\": %.3f, \"tmac_s\": %.2f}\n", rs[i].name,
           rs[i].ms, per_smsp_clk, rs[i].instr * 32 * rs[i].macs_per_instr / (rs[i].ms * 1e-3) / 1e12);
  }
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  return 0;
}
