// Standalone probe for the tcgen05 / TMA building blocks (not part of libfsr).
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2 tools/tc_debug.cu \
//        -Iinclude -lcublas -lcusolver -o tools/tc_debug && ./tools/tc_debug
// 1) TMA: load a 32 x 16 fp32 box with SWIZZLE_128B, dump smem, check the
//    128B-swizzle image (16B chunk c of row r lands at chunk c ^ (r % 8)).
// 2) MMA: place A (MN-major 128 x 8) and B (MN-major 256 x 8) in smem by hand
//    in the canonical SW128 layout, run one kind::tf32 MMA, dump TMEM.
// 3) tc_gram / tc_apply end to end vs a CPU reference.
#include "../paper_1703_06935_b200/csrc/fsr_ctx.cu"
#include "../paper_1703_06935_b200/csrc/tc_gemm.cu"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

using namespace fsr::tc;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__global__ void tma_dump_kernel(const __grid_constant__ CUtensorMap m, float* out, int bytes) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, bytes);
    tma_load_2d(smem, &m, &bar, 0, 0);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = ((float*)smem)[i];
}

// canonical SW128 MN-major placement of element (mn, k) for a block with
// `rows` K-rows per MN-block of 32: byte offset within the operand buffer.
__host__ __device__ inline int sw128_mn_offset(int mn, int k, int rows) {
  const int blk = mn / 32, e = mn % 32;
  const int row = k;                    // K row within the block
  const int chunk = (e * 4) / 16;       // 16B chunk within the 128B row
  const int within = (e * 4) % 16;
  const int sw = chunk ^ (row % 8);
  return blk * rows * 128 + row * 128 + sw * 16 + within;
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31]));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void mma_tf32_mask(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  uint32_t z = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(z), "r"(z), "r"(z), "r"(z)
      : "memory");
}

__host__ __device__ inline int sw128_k_offset(int mn, int k) {   // K-major SW128, K<=32 tf32
  const int chunk = (k * 4) / 16, within = (k * 4) % 16;
  return (mn / 8) * 1024 + (mn % 8) * 128 + ((chunk ^ (mn % 8)) * 16) + within;
}
__host__ __device__ inline int none_k_offset(int mn, int k) {    // K-major interleave: LBO=128 (K core), SBO=256 (M group)
  return (mn / 8) * 256 + (k / 4) * 128 + (mn % 8) * 16 + (k % 4) * 4;
}
__device__ __forceinline__ uint64_t desc_generic(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// mode: 0 plain form, 1 mask form, 2 st/ld roundtrip only (no MMA), 3 prefill 7.0 then MMA (accumulate=1)
__global__ void mma_probe_kernel(const float* A, const float* B, float* out, uint32_t idesc_override, int mode) {
  // A: 128 (M) x 8 (K) fp32, value A[m*8+k]; B: 256 (N) x 8 (K)
  extern __shared__ uint8_t raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = smem;            // 4 blocks * 8 rows * 128 B = 4 KB
  uint8_t* sb = smem + 16384;    // up to 32 KB (K-major SW128: 32 atoms of 1 KB)
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) ((float*)smem)[i] = 0.f;
  __syncthreads();
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) {
    const int m = i / 8, k = i % 8;
    const int off = mode == 4 ? sw128_k_offset(m, k) : mode == 5 ? none_k_offset(m, k) : sw128_mn_offset(m, k, 8);
    *(float*)(sa + off) = A[i];
  }
  for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) {
    const int n = i / 8, k = i % 8;
    const int off = mode == 4 ? sw128_k_offset(n, k) : mode == 5 ? none_k_offset(n, k) : sw128_mn_offset(n, k, 8);
    *(float*)(sb + off) = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (mode >= 2 && warp < 4) {
    float pre[32];
    for (int t = 0; t < 32; ++t) pre[t] = mode == 2 ? (float)(threadIdx.x * 1000 + t) : 7.0f;
    for (int cc = 0; cc < 8; ++cc) tmem_st32(tmem + ((uint32_t)(32 * warp) << 16) + cc * 32, pre);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_override ? idesc_override : idesc_tf32(128, 256, true, true);
    const uint64_t ad = smem_desc_sw128(smem_u32(sa), 8 * 128, 1024);
    const uint64_t bd = smem_desc_sw128(smem_u32(sb), 8 * 128, 1024);
    if (mode == 0) mma_tf32(tmem, ad, bd, idesc, 0);
    if (mode == 1) mma_tf32_mask(tmem, ad, bd, idesc, 0);
    if (mode == 3) mma_tf32(tmem, ad, bd, idesc, 1);
    if (mode == 4) {
      const uint32_t id = idesc_tf32(128, 256, false, false);
      mma_tf32(tmem, desc_generic(smem_u32(sa), 16, 1024, 2), desc_generic(smem_u32(sb), 16, 1024, 2), id, 0);
    }
    if (mode == 5) {
      const uint32_t id = idesc_tf32(128, 256, false, false);
      mma_tf32(tmem, desc_generic(smem_u32(sa), 128, 256, 0), desc_generic(smem_u32(sb), 128, 256, 0), id, 0);
    }
    if (mode == 6) {  // swap LBO/SBO meaning for MN-major
      mma_tf32(tmem, smem_desc_sw128(smem_u32(sa), 1024, 8 * 128), smem_desc_sw128(smem_u32(sb), 1024, 8 * 128),
               idesc, 0);
    }
    if (mode == 0 && blockIdx.x == 0) printf("idesc=0x%08x adesc=0x%016llx bdesc=0x%016llx tmem=0x%08x\n", idesc,
                                             (unsigned long long)ad, (unsigned long long)bd, tmem);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  // 4 warps read lanes 32w..32w+31
  if (warp < 4) {
    for (int cc = 0; cc < 8; ++cc) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + cc * 32, v);
      const int row = 32 * warp + (threadIdx.x & 31);
      for (int t = 0; t < 32; ++t) out[row * 256 + cc * 32 + t] = v[t];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

int main() {
  // ---------------- 3) tc_gram end to end
  {
    const int n = 1000, k = 40;
    std::vector<float> A(n * k);
    srand(1);
    for (auto& x : A) x = (float)rand() / RAND_MAX - 0.5f;
    float* dA;
    double* dG;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dG, k * k * 8));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    fsr_ctx* ctx;
    fsr_ctx_create(0, &ctx);
    for (int np : {1, 3}) {
      int st = fsr::tc_gram(ctx, n, k, dA, k, k, dA, k, dG, 0, np, 1);
      CK(cudaDeviceSynchronize());
      std::vector<double> G(k * k);
      CK(cudaMemcpy(G.data(), dG, G.size() * 8, cudaMemcpyDeviceToHost));
      double mx = 0, mref = 0;
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) {
          double ref = 0;
          for (int r = 0; r < n; ++r) ref += (double)A[r * k + i] * A[r * k + j];
          mx = fmax(mx, fabs(G[i * k + j] - ref));
          mref = fmax(mref, fabs(ref));
        }
      printf("[gram nprod=%d] status %d (%s) rel err %.3e  G[0]=%g\n", np, st, ctx->err.c_str(), mx / mref, G[0]);
    }
    // apply: Out = A * M (k x k)
    std::vector<double> M(k * k);
    for (auto& x : M) x = (double)rand() / RAND_MAX - 0.5;
    double* dM;
    float* dO;
    CK(cudaMalloc(&dM, M.size() * 8));
    CK(cudaMalloc(&dO, (size_t)n * k * 4));
    CK(cudaMemcpy(dM, M.data(), M.size() * 8, cudaMemcpyHostToDevice));
    int st = fsr::tc_apply(ctx, n, k, dA, k, k, dM, k, 0, dO, k);
    CK(cudaDeviceSynchronize());
    std::vector<float> O((size_t)n * k);
    CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
    double mx = 0, mref = 0;
    for (int r = 0; r < n; ++r)
      for (int j = 0; j < k; ++j) {
        double ref = 0;
        for (int i = 0; i < k; ++i) ref += (double)A[r * k + i] * M[i * k + j];
        mx = fmax(mx, fabs(O[r * k + j] - ref));
        mref = fmax(mref, fabs(ref));
      }
    printf("[apply] status %d rel err %.3e  O[0]=%g\n", st, mx / mref, O[0]);
    fsr_ctx_destroy(ctx);
  }
  // ---------------- 4) error growth with the reduction length
  {
    fsr_ctx* ctx;
    fsr_ctx_create(0, &ctx);
    for (int K : {32, 256, 2048, 8192}) {
      const int n = 512, N2 = 64;
      std::vector<float> A((size_t)n * K);
      std::vector<double> M((size_t)K * N2);
      srand(K);
      for (auto& x : A) x = (float)rand() / RAND_MAX;          // positive: worst case for biased rounding
      for (auto& x : M) x = (double)rand() / RAND_MAX;
      float *dA, *dO;
      double* dM;
      CK(cudaMalloc(&dA, A.size() * 4));
      CK(cudaMalloc(&dO, (size_t)n * N2 * 4));
      CK(cudaMalloc(&dM, M.size() * 8));
      CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dM, M.data(), M.size() * 8, cudaMemcpyHostToDevice));
      fsr::tc_apply(ctx, n, K, dA, K, N2, dM, N2, 0, dO, N2);
      CK(cudaDeviceSynchronize());
      std::vector<float> O((size_t)n * N2);
      CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
      double mx = 0, sgn = 0;
      for (int r = 0; r < 64; ++r)
        for (int j = 0; j < N2; ++j) {
          double ref = 0;
          for (int i = 0; i < K; ++i) ref += (double)A[(size_t)r * K + i] * M[(size_t)i * N2 + j];
          const double e = (O[r * N2 + j] - ref) / ref;
          mx = fmax(mx, fabs(e));
          sgn += e;
        }
      printf("[apply K=%5d] max rel err %.3e  mean signed rel err %.3e\n", K, mx, sgn / (64 * N2));
      // gram on the same positive data, n=K rows of 64 columns
      double* dG;
      CK(cudaMalloc(&dG, 64 * 64 * 8));
      for (int np : {1, 3}) {
        fsr::tc_gram(ctx, K, 64, dA, 64, 64, dA, 64, dG, 0, np, 1);
        CK(cudaDeviceSynchronize());
        std::vector<double> G(64 * 64);
        CK(cudaMemcpy(G.data(), dG, G.size() * 8, cudaMemcpyDeviceToHost));
        double gm = 0, gs = 0;
        for (int i = 0; i < 64; ++i)
          for (int j = 0; j < 64; ++j) {
            double ref = 0;
            for (int r = 0; r < K; ++r) ref += (double)A[(size_t)r * 64 + i] * A[(size_t)r * 64 + j];
            const double e = (G[i * 64 + j] - ref) / ref;
            gm = fmax(gm, fabs(e));
            gs += e;
          }
        printf("[gram  rows=%5d nprod=%d] max rel err %.3e  mean signed %.3e\n", K, np, gm, gs / 4096);
      }
      cudaFree(dA); cudaFree(dO); cudaFree(dM); cudaFree(dG);
    }
    fsr_ctx_destroy(ctx);
  }
  return 0;
}
