// Die-locality probe (B200 = two dies, L2 split between them).
//
// 1. classify: the CTA that lands on SM 0 times an L2-hit load (ld.global.cg,
//    after a warming read) of every 2 KB chunk of a 64 MB buffer; chunks slower
//    than the median are "far" from SM 0's die.
// 2. sm_die: every SM times loads of 64 near(SM0) and 64 far(SM0) chunks and
//    is assigned to SM 0's die if the near set is faster.
// 3. gather: every warp reads 1 KB rows (two 16-byte loads per lane) at
//    pseudo-random positions from a row list: (a) rows in chunks near its own
//    die, (b) rows in chunks far from it, (c) all rows.  Same footprint.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/die_probe tools/die_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
// clock read that waits for v (register dependency)
__device__ __forceinline__ long long clock_after(unsigned v) {
  long long t;
  asm volatile("{\n\t.reg .u32 d;\n\tmov.u32 d, %1;\n\tmov.u64 %0, %%clock64;\n\t}" : "=l"(t) : "r"(v) : "memory");
  return t;
}
__device__ __forceinline__ unsigned ld_cg(const unsigned* p) {
  unsigned v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void classify_kernel(const unsigned* buf, int64_t chunks, int target_sm, unsigned* lat, int* done) {
  if (smid() != (unsigned)target_sm || threadIdx.x != 0) return;
  if (atomicAdd(done, 1) != 0) return;
  unsigned sink = 0;
  for (int64_t c = 0; c < chunks; ++c) {
    const unsigned* p = buf + c * 512;
    unsigned v = ld_cg(p + (sink & 511));  // warm (may come from DRAM)
    const long long t0 = clock64();
#pragma unroll 1
    for (int rep = 0; rep < 32; ++rep) v = ld_cg(p + (v & 511));  // dependent chain of L2 hits
    sink += v;
    const long long t1 = clock_after(sink);
    lat[c] = (unsigned)((t1 - t0) / 32);
  }
  if (sink == 12345u) lat[0] = sink;
}

__global__ void sm_die_kernel(const unsigned* buf, const int* near_c, const int* far_c, int m, int* die_of_sm) {
  if (threadIdx.x != 0) return;
  const unsigned s = smid();
  unsigned sink = 0;
  long long tn = 0, tf = 0;
  for (int pass = 0; pass < 2; ++pass) {
    tn = tf = 0;
    for (int i = 0; i < m; ++i) {
      const unsigned* p = buf + (int64_t)near_c[i] * 512;
      unsigned v = sink & 511;
      long long t0 = clock64();
#pragma unroll 1
      for (int rep = 0; rep < 8; ++rep) v = ld_cg(p + (v & 511));
      sink += v;
      tn += clock_after(sink) - t0;
      const unsigned* q = buf + (int64_t)far_c[i] * 512;
      v = sink & 511;
      t0 = clock64();
#pragma unroll 1
      for (int rep = 0; rep < 8; ++rep) v = ld_cg(q + (v & 511));
      sink += v;
      tf += clock_after(sink) - t0;
    }
  }
  die_of_sm[s] = (tn < tf ? 0 : 1) + (sink == 12345u ? 2 : 0);
}

// rows: list per die (rows of 1 KB; row id -> byte offset row * 1024)
__global__ void gather_kernel(const float4* __restrict__ buf, const int* __restrict__ rows0, int n0,
                              const int* __restrict__ rows1, int n1, const int* __restrict__ die_of_sm, int mode,
                              int64_t per_warp, float* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int die = die_of_sm[smid()] & 1;
  // mode 0: own die's rows, 1: other die's rows, 2: both lists (uniform)
  const int* lst = (mode == 0) == (die == 0) ? rows0 : rows1;
  int nl = (mode == 0) == (die == 0) ? n0 : n1;
  uint64_t s = 0x9E3779B97F4A7C15ull * (warp + 1);
  float acc = 0.f;
  for (int64_t k = 0; k < per_warp; k += 8) {
    float4 v[8][2];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      s ^= s << 13;
      s ^= s >> 7;
      s ^= s << 17;
      int row;
      if (mode == 2) {
        const int64_t t = (int64_t)(((s >> 32) * (uint64_t)(n0 + n1)) >> 32);
        row = t < n0 ? __ldg(rows0 + t) : __ldg(rows1 + (t - n0));
      } else {
        row = __ldg(lst + (int64_t)(((s >> 32) * (uint64_t)nl) >> 32));
      }
      const float4* p = buf + (int64_t)row * 64 + lane;
      v[g][0] = __ldg(p);
      v[g][1] = __ldg(p + 32);
    }
#pragma unroll
    for (int g = 0; g < 8; ++g) acc += v[g][0].x + v[g][1].y;
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t bytes = 64ll << 20, chunks = bytes / 2048;
  unsigned* buf;
  unsigned *lat;
  int* done;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  cudaMalloc(&lat, chunks * 4);
  cudaMalloc(&done, 4);
  cudaMemset(done, 0, 4);
  classify_kernel<<<sms * 4, 32>>>(buf, chunks, 0, lat, done);
  std::vector<unsigned> h(chunks);
  cudaMemcpy(h.data(), lat, chunks * 4, cudaMemcpyDeviceToHost);
  std::vector<unsigned> srt = h;
  std::sort(srt.begin(), srt.end());
  const unsigned med = srt[chunks / 2];
  // histogram summary
  printf("{\"chunks\": %lld, \"lat_p10\": %u, \"lat_p25\": %u, \"lat_p50\": %u, \"lat_p75\": %u, \"lat_p90\": %u",
         (long long)chunks, srt[chunks / 10], srt[chunks / 4], med, srt[3 * chunks / 4], srt[9 * chunks / 10]);
  std::vector<int> nearc, farc;
  for (int64_t c = 0; c < chunks; ++c) (h[c] < med ? nearc : farc).push_back((int)c);
  printf(", \"near_chunks\": %zu, \"far_chunks\": %zu", nearc.size(), farc.size());
  const int m = 64;
  int *d_near, *d_far, *d_die;
  cudaMalloc(&d_near, m * 4);
  cudaMalloc(&d_far, m * 4);
  cudaMalloc(&d_die, 1024 * 4);
  cudaMemset(d_die, 0xff, 1024 * 4);
  std::vector<int> sn(nearc.begin(), nearc.begin() + m), sf(farc.begin(), farc.begin() + m);
  cudaMemcpy(d_near, sn.data(), m * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_far, sf.data(), m * 4, cudaMemcpyHostToDevice);
  sm_die_kernel<<<sms * 8, 32>>>(buf, d_near, d_far, m, d_die);
  std::vector<int> die(1024);
  cudaMemcpy(die.data(), d_die, 1024 * 4, cudaMemcpyDeviceToHost);
  int cnt0 = 0, cnt1 = 0, unk = 0;
  for (int s = 0; s < sms; ++s) {
    if (die[s] < 0) ++unk;
    else if ((die[s] & 1) == 0) ++cnt0;
    else ++cnt1;
  }
  printf(", \"sms_die0\": %d, \"sms_die1\": %d, \"sms_unknown\": %d", cnt0, cnt1, unk);
  printf(", \"sm_die\": \"");
  for (int s = 0; s < sms; ++s) printf("%d", die[s] < 0 ? 9 : (die[s] & 1));
  printf("\"");
  // gather footprint: the first `fp` MB of the buffer, rows of 1 KB (2 per chunk)
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int64_t fp_mb : {5ll, 20ll, 60ll}) {
    std::vector<int> r0, r1;
    const int64_t lim = (fp_mb << 20) / 2048;
    for (int64_t c = 0; c < lim; ++c) {
      auto& L = h[c] < med ? r0 : r1;
      L.push_back((int)(2 * c));
      L.push_back((int)(2 * c + 1));
    }
    int *d0, *d1;
    cudaMalloc(&d0, r0.size() * 4);
    cudaMalloc(&d1, r1.size() * 4);
    cudaMemcpy(d0, r0.data(), r0.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d1, r1.data(), r1.size() * 4, cudaMemcpyHostToDevice);
    const int64_t per_warp = 4096;
    const int grid = sms * 8;
    const char* names[] = {"near", "far", "all"};
    for (int mode = 0; mode < 3; ++mode) {
      gather_kernel<<<grid, 256>>>((const float4*)buf, d0, (int)r0.size(), d1, (int)r1.size(), d_die, mode, 64, out);
      cudaEventRecord(e0);
      gather_kernel<<<grid, 256>>>((const float4*)buf, d0, (int)r0.size(), d1, (int)r1.size(), d_die, mode,
                                   per_warp, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double gb = (double)grid * 8 * per_warp * 1024;
      printf(", \"gather_%s_%lldMB_GBs\": %.1f", names[mode], (long long)fp_mb, gb / ms / 1e6);
    }
    cudaFree(d0);
    cudaFree(d1);
  }
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
