// L2 -> SM read bandwidth probe for the K9 roofline (B200, sm_100a).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_bw tools/l2_bw.cu
//   tools/l2_bw            -> one JSON line
//
// stream: every warp reads consecutive 512-byte segments of a buffer of the
//   given size over and over (L2-resident below ~60 MB, DRAM above).
// gather: every warp reads whole 1 KB rows (32 lanes x 2 x float4) at
//   pseudo-random row indices of a (rows x 256 fp32) matrix -- K9's access
//   pattern (Zs rows gathered per nonzero of U~) without the arithmetic.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void stream_kernel(const float4* __restrict__ buf, int64_t n4, int iters, float* out) {
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    for (int64_t j = i; j < n4; j += nthreads) {
      const float4 v = __ldg(buf + j);
      acc += v.x + v.y + v.z + v.w;
    }
  }
  if (acc == 1.2345f) out[0] = acc;
}

__global__ void gather_kernel(const float4* __restrict__ buf, int64_t rows, int64_t per_warp, float* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint64_t s = 0x9E3779B97F4A7C15ull * (warp + 1);
  float acc = 0.f;
  for (int64_t k = 0; k < per_warp; k += 8) {
    float4 v[8][2];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      s ^= s << 13;
      s ^= s >> 7;
      s ^= s << 17;
      const int64_t row = (int64_t)(((s >> 32) * (uint64_t)rows) >> 32);
      const float4* p = buf + row * 64 + lane;  // 256 floats = 64 float4 per row
      v[g][0] = __ldg(p);
      v[g][1] = __ldg(p + 32);
    }
#pragma unroll
    for (int g = 0; g < 8; ++g) acc += v[g][0].x + v[g][1].y;
  }
  if (acc == 1.2345f) out[0] = acc;
}

// gather of short rows: LPR lanes x float4 per row (LPR = 8: 128-byte rows, 4
// random rows per warp access; LPR = 4: 64-byte rows, 8 per access) -- the K2
// slab kernel's access pattern (tools/k2_slab.cu) without its index stream.
template <int LPR, int DEPTH>
__global__ void gather_short_kernel(const float4* __restrict__ buf, int64_t rows, int64_t per_warp, float* out) {
  const int lane = threadIdx.x & 31, grp = lane / LPR, sl = lane % LPR;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint64_t s = 0x9E3779B97F4A7C15ull * (warp * (32 / LPR) + grp + 1);
  float acc = 0.f;
  for (int64_t k = 0; k < per_warp; k += DEPTH) {
    float4 v[DEPTH];
#pragma unroll
    for (int g = 0; g < DEPTH; ++g) {
      s ^= s << 13;
      s ^= s >> 7;
      s ^= s << 17;
      const int64_t row = (int64_t)(((s >> 32) * (uint64_t)rows) >> 32);
      v[g] = __ldg(buf + row * LPR + sl);
    }
#pragma unroll
    for (int g = 0; g < DEPTH; ++g) acc += v[g].x + v[g].w;
  }
  if (acc == 1.2345f) out[0] = acc;
}

template <int LPR, int DEPTH>
static void run_short(const char* name, int sms, float* out, cudaEvent_t e0, cudaEvent_t e1) {
  const int64_t mbs[] = {16, 32, 64};
  for (int64_t mb : mbs) {
    const int64_t bytes = mb << 20, rows = bytes / (16 * LPR);
    float4* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    const int grid = sms * 8;
    const int64_t per_warp = 8192;
    gather_short_kernel<LPR, DEPTH><<<grid, 256>>>(buf, rows, 64, out);
    cudaEventRecord(e0);
    gather_short_kernel<LPR, DEPTH><<<grid, 256>>>(buf, rows, per_warp, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double moved = (double)grid * 8 * per_warp * 512;
    printf(", \"%s_%lldMB_GBs\": %.1f", name, (long long)mb, moved / ms / 1e6);
    cudaFree(buf);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"sms\": %d", sms);
  const int64_t sizes_mb[] = {8, 16, 24, 32, 48, 64, 96, 8192};
  for (int64_t mb : sizes_mb) {
    const int64_t bytes = mb << 20;
    float4* buf;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
    cudaMemset(buf, 0, bytes);
    const int iters = mb >= 1024 ? 2 : (int)(16384 / mb);
    const int grid = sms * 8;
    stream_kernel<<<grid, 256>>>(buf, bytes / 16, 1, out);
    cudaEventRecord(e0);
    stream_kernel<<<grid, 256>>>(buf, bytes / 16, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf(", \"stream_%lldMB_GBs\": %.1f", (long long)mb, (double)bytes * iters / ms / 1e6);
    cudaFree(buf);
  }
  const int64_t rows_list[] = {5000, 20000, 60000};
  for (int64_t rows : rows_list) {
    const int64_t bytes = rows * 1024;
    float4* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    const int grid = sms * 8;
    const int64_t per_warp = 4096;
    gather_kernel<<<grid, 256>>>(buf, rows, 64, out);
    cudaEventRecord(e0);
    gather_kernel<<<grid, 256>>>(buf, rows, per_warp, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double moved = (double)grid * 8 * per_warp * 1024;
    printf(", \"gather_1KB_rows_%lldMB_GBs\": %.1f", (long long)(bytes >> 20), moved / ms / 1e6);
    cudaFree(buf);
  }
  run_short<8, 4>("gather_128B_rows_d4", sms, out, e0, e1);
  run_short<8, 8>("gather_128B_rows_d8", sms, out, e0, e1);
  run_short<4, 8>("gather_64B_rows_d8", sms, out, e0, e1);
  run_short<2, 8>("gather_32B_rows_d8", sms, out, e0, e1);
  printf("}\n");
  return 0;
}
