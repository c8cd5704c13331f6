// K9 Zs-layout probe: the production K9 kernel (spmm_rowpanel_T_kernel, NV=2,
// 256-column panels) on a synthetic C3-shaped U~ (n = 1e6, 100 sorted random
// columns per row out of r = 5000, b = 1024), with Zs
//   (a) row-major r x b (ld = b; one launch, panels strided by 1 KB), as shipped;
//   (b) row-major, one launch per panel;
//   (c) panel-contiguous [b/256][r][256] (one launch per panel, ld = 256).
// Prints ms per full product for each and the max |diff| between them.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -Iinclude tools/k9_layout.cu -o tools/k9_layout
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include "../paper_1703_06935_b200/csrc/spmm.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 1000000, r = 5000, b = 1024, per = 100, PW = 256;
  const int64_t tau = n * per;
  std::vector<int64_t> ip(n + 1);
  std::vector<int32_t> ci(tau);
  std::vector<float> va(tau);
  std::mt19937_64 g(1);
  for (int64_t i = 0; i <= n; ++i) ip[i] = i * per;
  const int64_t stride = r / per;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = 0; k < per; ++k) {
      ci[i * per + k] = (int32_t)(k * stride + g() % stride);
      va[i * per + k] = (float)((g() % 2001) - 1000) * 1e-3f;
    }
  std::vector<float> zs(r * b);
  for (auto& z : zs) z = (float)((g() % 2001) - 1000) * 1e-3f;
  std::vector<float> zp(r * b);  // panel-contiguous copy
  for (int64_t p = 0; p < b / PW; ++p)
    for (int64_t j = 0; j < r; ++j)
      for (int64_t c = 0; c < PW; ++c) zp[(p * r + j) * PW + c] = zs[j * b + p * PW + c];
  int64_t* d_ip; int32_t* d_ci; float *d_va, *d_zs, *d_zp, *d_y1, *d_y2, *d_y3;
  CK(cudaMalloc(&d_ip, (n + 1) * 8)); CK(cudaMalloc(&d_ci, tau * 4)); CK(cudaMalloc(&d_va, tau * 4));
  CK(cudaMalloc(&d_zs, r * b * 4)); CK(cudaMalloc(&d_zp, r * b * 4));
  CK(cudaMalloc(&d_y1, n * b * 4)); CK(cudaMalloc(&d_y2, n * b * 4)); CK(cudaMalloc(&d_y3, n * b * 4));
  CK(cudaMemcpy(d_ip, ip.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ci, ci.data(), tau * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_va, va.data(), tau * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_zs, zs.data(), r * b * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_zp, zp.data(), r * b * 4, cudaMemcpyHostToDevice));
  auto kern = fsr::spmm_rowpanel_T_kernel<float, 4, 2, fsr::kGatherDepth, 32>;
  const size_t smem = 32 * (PW + 1) * 4;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned gx = (unsigned)((n + 31) / 32);
  auto va_ = [&]() { kern<<<dim3(gx, b / PW), 256, smem>>>(n, d_ip, d_ci, d_va, b, d_zs, b, d_y1, n); };
  auto vb_ = [&]() {
    for (int64_t p = 0; p < b / PW; ++p)
      kern<<<dim3(gx, 1), 256, smem>>>(n, d_ip, d_ci, d_va, PW, d_zs + p * PW, b, d_y2 + p * PW * n, n);
  };
  auto vc_ = [&]() {
    for (int64_t p = 0; p < b / PW; ++p)
      kern<<<dim3(gx, 1), 256, smem>>>(n, d_ip, d_ci, d_va, PW, d_zp + p * r * PW, PW, d_y3 + p * PW * n, n);
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto f) {
    f(); f();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    return best;
  };
  for (int round = 0; round < 2; ++round) {
    const float ta = timeit(va_), tb = timeit(vb_), tc = timeit(vc_);
    printf("{\"n\": %lld, \"a_rowmajor_one_launch_ms\": %.3f, \"b_rowmajor_per_panel_ms\": %.3f, \"c_panel_contig_ms\": %.3f}\n",
           (long long)n, ta, tb, tc);
  }
  CK(cudaGetLastError());
  std::vector<float> y1(n * b), y3(n * b);
  CK(cudaMemcpy(y1.data(), d_y1, n * b * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(y3.data(), d_y3, n * b * 4, cudaMemcpyDeviceToHost));
  double md = 0;
  for (int64_t i = 0; i < n * b; ++i) md = std::max(md, (double)std::fabs(y1[i] - y3[i]));
  printf("{\"max_abs_diff_a_c\": %g}\n", md);
  return 0;
}
