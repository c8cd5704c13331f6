// Shared internals of libfsr: the context, error plumbing, launch accounting.
#pragma once

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/fsr.h"

// Device-side bounds / capacity assertions, compiled only with
// -DFSR_DEBUG_CHECKS (build.py, FSR_DEBUG_CHECKS=1): a violated check traps
// the kernel and the next libfsr call reports the CUDA error.
#ifdef FSR_DEBUG_CHECKS
#include <cassert>
#define FSR_DCHECK(cond) assert(cond)
#else
#define FSR_DCHECK(cond) ((void)0)
#endif

struct fsr_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cublasHandle_t blas = nullptr;
  cusolverDnHandle_t solver = nullptr;
  // grow-only scratch arena, stream-ordered (all work runs on `stream`)
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  void* scratch_aux = nullptr;  // caller-level temporaries that outlive a scratch() user
  size_t scratch_aux_bytes = 0;
  int dense_path = 0;           // FSR_OPT_DENSE_PATH: 0 auto (tcgen05 for F32), 1 cuBLAS
  int spmm_panel_bytes = 0;     // FSR_OPT_SPMM_PANEL_BYTES: 0 wide row panels, else L2 panel width
  int topk_prune = 1;           // FSR_OPT_TOPK_PRUNE: certified fp16-pruned K9 for top-k-only fp32 batches
  int topk_segments = 0;        // FSR_OPT_TOPK_SEGMENTS: 0 auto, else segments per row when b < #SMs
  void* topk_state = nullptr;   // persistent, self-cleaning state of the few-row top-k (topk.cuh)
  int* dev_info = nullptr;
  double* host_stage = nullptr;  // pinned staging for small host reads
  size_t host_stage_bytes = 0;
  std::string err;
  uint64_t launches = 0;
  uint64_t library_calls = 0;
  // optional per-stage device timing (CUDA events on the context stream)
  bool timing = false;
  struct Pending {
    int stage;
    cudaEvent_t start, stop;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  double stage_ms[FSR_NUM_STAGES] = {};
  uint64_t stage_count[FSR_NUM_STAGES] = {};
};

namespace fsr {

inline int set_error(fsr_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  return code;
}

inline int cuda_status(fsr_ctx* ctx, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return FSR_OK;
  return set_error(ctx, e == cudaErrorMemoryAllocation ? FSR_ENOMEM : FSR_ECUDA, "%s: %s", what,
                   cudaGetErrorString(e));
}

inline int blas_status(fsr_ctx* ctx, cublasStatus_t s, const char* what) {
  ctx->library_calls++;
  if (s == CUBLAS_STATUS_SUCCESS) return FSR_OK;
  return set_error(ctx, FSR_ELIBRARY, "%s: cublas status %d", what, (int)s);
}

inline int solver_status(fsr_ctx* ctx, cusolverStatus_t s, const char* what) {
  ctx->library_calls++;
  if (s == CUSOLVER_STATUS_SUCCESS) return FSR_OK;
  return set_error(ctx, FSR_ELIBRARY, "%s: cusolver status %d", what, (int)s);
}

// Check the launch that was just issued and count it.
inline int launched(fsr_ctx* ctx, const char* name) {
  ctx->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ctx, FSR_ECUDA, "launch %s: %s", name, cudaGetErrorString(e));
  return FSR_OK;
}

// Scratch arena: returns a device pointer with at least `bytes` bytes.  Growing
// synchronises the stream first so in-flight kernels never see a freed buffer.
inline int scratch(fsr_ctx* ctx, size_t bytes, void** out) {
  if (bytes <= ctx->scratch_bytes) {
    *out = ctx->scratch;
    return FSR_OK;
  }
  cudaStreamSynchronize(ctx->stream);
  if (ctx->scratch) cudaFree(ctx->scratch);
  ctx->scratch = nullptr;
  ctx->scratch_bytes = 0;
  size_t want = bytes + bytes / 8 + 256;
  cudaError_t e = cudaMalloc(&ctx->scratch, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(ctx, FSR_ENOMEM, "scratch alloc of %zu bytes failed", want);
  }
  ctx->scratch_bytes = want;
  *out = ctx->scratch;
  return FSR_OK;
}

inline int scratch_aux(fsr_ctx* ctx, size_t bytes, void** out) {
  if (bytes <= ctx->scratch_aux_bytes) {
    *out = ctx->scratch_aux;
    return FSR_OK;
  }
  cudaStreamSynchronize(ctx->stream);
  if (ctx->scratch_aux) cudaFree(ctx->scratch_aux);
  ctx->scratch_aux = nullptr;
  ctx->scratch_aux_bytes = 0;
  cudaError_t e = cudaMalloc(&ctx->scratch_aux, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(ctx, FSR_ENOMEM, "aux scratch alloc of %zu bytes failed", bytes);
  }
  ctx->scratch_aux_bytes = bytes;
  *out = ctx->scratch_aux;
  return FSR_OK;
}

// tcgen05 kernels (tc_gemm.cu)
int tc_gram(fsr_ctx* ctx, int64_t n, int64_t ka, const float* A, int64_t lda, int64_t kb, const float* B,
            int64_t ldb, double* C, int accumulate, int levels, int symmetric);
int tc_apply(fsr_ctx* ctx, int64_t n, int64_t K, const float* A, int64_t lda, int64_t N2, const double* M,
             int64_t ldm, int m_col_major, float* Out, int64_t ldo, int m_slices = 4);

inline int host_stage(fsr_ctx* ctx, size_t bytes, void** out) {
  if (bytes > ctx->host_stage_bytes) {
    if (ctx->host_stage) cudaFreeHost(ctx->host_stage);
    ctx->host_stage = nullptr;
    ctx->host_stage_bytes = 0;
    cudaError_t e = cudaMallocHost((void**)&ctx->host_stage, bytes);
    if (e != cudaSuccess) return cuda_status(ctx, e, "pinned staging alloc");
    ctx->host_stage_bytes = bytes;
  }
  *out = ctx->host_stage;
  return FSR_OK;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the CURRENT
// device only, so the "already configured" state is kept per (kernel, device):
// a process driving two GPUs (one fsr_ctx each) configures each of them.
inline int ensure_smem(fsr_ctx* ctx, const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{kernel, ctx->device}];
  if (have >= bytes) return FSR_OK;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return cuda_status(ctx, e, "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
  have = bytes;
  return FSR_OK;
}

template <typename K>
inline int ensure_smem(fsr_ctx* ctx, K* kernel, size_t bytes) {
  return ensure_smem(ctx, reinterpret_cast<const void*>(kernel), bytes);
}

inline size_t dtype_size(int dtype) { return dtype == FSR_F64 ? 8 : 4; }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int grid_for(int64_t work, int block, fsr_ctx* ctx, int per_sm = 16) {
  int64_t g = ceil_div(work, block);
  int64_t cap = (int64_t)ctx->num_sms * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// Exact mul-then-add (no FMA contraction): bitwise equal to the sequential
// `y += a * x` of scipy's sparsetools in float64.
__device__ __forceinline__ double mul_add_rn(double acc, double a, double x) {
  return __dadd_rn(acc, __dmul_rn(a, x));
}
__device__ __forceinline__ float mul_add_rn(float acc, float a, float x) {
  return __fadd_rn(acc, __fmul_rn(a, x));
}

// Order key of |u| (sign cleared): monotone in |u| for finite values.
__device__ __forceinline__ uint64_t abs_key(float v) {
  return (uint64_t)(__float_as_uint(v) & 0x7fffffffu);
}
__device__ __forceinline__ uint64_t abs_key(double v) {
  return (uint64_t)__double_as_longlong(v) & 0x7fffffffffffffffull;
}

inline cudaEvent_t pooled_event(fsr_ctx* ctx) {
  if (!ctx->event_pool.empty()) {
    cudaEvent_t e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Brackets the device work issued in its scope with CUDA events when the
// context has timing enabled (fsr_ctx_enable_timing); no cost otherwise.
struct StageTimer {
  fsr_ctx* ctx;
  int stage;
  cudaEvent_t start = nullptr;
  StageTimer(fsr_ctx* c, int s) : ctx(c), stage(s) {
    if (ctx->timing) {
      start = pooled_event(ctx);
      cudaEventRecord(start, ctx->stream);
    }
  }
  ~StageTimer() {
    if (start) {
      cudaEvent_t stop = pooled_event(ctx);
      cudaEventRecord(stop, ctx->stream);
      ctx->pending.push_back({stage, start, stop});
    }
  }
};

}  // namespace fsr

#define FSR_TRY(expr)              \
  do {                             \
    int _st = (expr);              \
    if (_st != FSR_OK) return _st; \
  } while (0)

#define FSR_CUDA(ctx, expr) FSR_TRY(::fsr::cuda_status((ctx), (expr), #expr))
#define FSR_BLAS(ctx, expr) FSR_TRY(::fsr::blas_status((ctx), (expr), #expr))
#define FSR_SOLVER(ctx, expr) FSR_TRY(::fsr::solver_status((ctx), (expr), #expr))

#define FSR_REQUIRE(ctx, cond, ...)                                          \
  do {                                                                       \
    if (!(cond)) return ::fsr::set_error((ctx), FSR_EINVAL, __VA_ARGS__);    \
  } while (0)
