// K11: connected components of an adjacency (reference graph.py:215-250
// connected_components, a host union-find).  Used by decompose_blockwise
// (spectral.py:312-390).
//
// Device: min-label hooking with pointer jumping.  comp[v] is a parent
// pointer that only ever decreases and always stays inside v's component;
// each round (1) hooks, for every stored entry (i, j), the larger of the two
// current roots under the smaller (atomicMin), (2) compresses every pointer
// to its root.  At the fixed point every vertex points at the smallest vertex
// index of its component -- the same root the reference's union-find (which
// always links the larger root under the smaller) ends with.  Every stored
// entry counts as an edge, whatever its value, as in the reference.
#include "fsr_common.cuh"

namespace {

__global__ void cc_init_kernel(int64_t n, unsigned long long* __restrict__ comp) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    comp[i] = (unsigned long long)i;
}

// warp per row: lanes over the row's entries
__global__ void cc_hook_kernel(int64_t n, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                               unsigned long long* comp, int* __restrict__ changed) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool any = false;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
    const unsigned long long ci = comp[i];
    for (int64_t e = indptr[i] + lane; e < indptr[i + 1]; e += 32) {
      const unsigned long long cj = comp[indices[e]];
      if (ci != cj) {
        const unsigned long long hi = ci > cj ? ci : cj, lo = ci > cj ? cj : ci;
        atomicMin(&comp[hi], lo);
        any = true;
      }
    }
  }
  if (__any_sync(0xffffffffu, any) && lane == 0) *changed = 1;
}

__global__ void cc_jump_kernel(int64_t n, unsigned long long* comp) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long c = comp[i];
    unsigned long long p = comp[c];
    while (p != c) {
      c = p;
      p = comp[c];
    }
    comp[i] = c;
  }
}

}  // namespace

extern "C" {

int fsr_connected_components(fsr_ctx* ctx, int64_t n, const int64_t* indptr, const int32_t* indices, int64_t* root,
                             int64_t* rounds_host) {
  FSR_REQUIRE(ctx, n >= 0 && indptr && root, "connected_components: bad args");
  if (!n) return FSR_OK;
  unsigned long long* comp = (unsigned long long*)root;
  int* flag = nullptr;
  FSR_TRY(fsr::scratch_aux(ctx, sizeof(int), (void**)&flag));
  cc_init_kernel<<<fsr::grid_for(n, 256, ctx, 8), 256, 0, ctx->stream>>>(n, comp);
  FSR_TRY(fsr::launched(ctx, "cc_init_kernel"));
  int64_t rounds = 0;
  for (;;) {
    FSR_CUDA(ctx, cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
    cc_hook_kernel<<<fsr::grid_for(n * 32, 256, ctx, 8), 256, 0, ctx->stream>>>(n, indptr, indices, comp, flag);
    FSR_TRY(fsr::launched(ctx, "cc_hook_kernel"));
    cc_jump_kernel<<<fsr::grid_for(n, 256, ctx, 8), 256, 0, ctx->stream>>>(n, comp);
    FSR_TRY(fsr::launched(ctx, "cc_jump_kernel"));
    int h = 0;
    FSR_CUDA(ctx, cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    ++rounds;
    if (!h) break;
    FSR_REQUIRE(ctx, rounds <= 4096, "connected_components: no convergence");
  }
  if (rounds_host) *rounds_host = rounds;
  return FSR_OK;
}

}  // extern "C"
