// Context lifecycle, error reporting and launch accounting for libfsr.
#include "fsr_common.cuh"

static void fold_pending(fsr_ctx* ctx);

extern "C" {

int fsr_abi_version(void) { return FSR_ABI_VERSION; }

int fsr_ctx_create(int device, fsr_ctx** out) {
  if (!out) return FSR_EINVAL;
  *out = nullptr;
  fsr_ctx* ctx = new fsr_ctx();
  ctx->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete ctx;
    return FSR_ECUDA;
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  ctx->stream = nullptr;  // legacy default stream until fsr_ctx_set_stream
  if (cublasCreate(&ctx->blas) != CUBLAS_STATUS_SUCCESS ||
      cusolverDnCreate(&ctx->solver) != CUSOLVER_STATUS_SUCCESS ||
      cudaMalloc(&ctx->dev_info, sizeof(int) * 4) != cudaSuccess) {
    fsr_ctx_destroy(ctx);
    return FSR_ELIBRARY;
  }
  // Pure FP32/FP64 arithmetic: never let cuBLAS substitute TF32 tensor ops.
  cublasSetMathMode(ctx->blas, CUBLAS_PEDANTIC_MATH);
  // The operator-level calls (fsr_ops.cu) take stream-ordered temporaries
  // from the device's default memory pool; keep freed blocks in the pool
  // instead of returning them at every synchronisation (re-mapping hundreds of
  // MB per call cost ~0.2 s per sparsify at C3).
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  *out = ctx;
  return FSR_OK;
}

void fsr_ctx_destroy(fsr_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  else cudaDeviceSynchronize();
  if (ctx->scratch) cudaFree(ctx->scratch);
  if (ctx->scratch_aux) cudaFree(ctx->scratch_aux);
  if (ctx->topk_state) cudaFree(ctx->topk_state);
  if (ctx->dev_info) cudaFree(ctx->dev_info);
  if (ctx->host_stage) cudaFreeHost(ctx->host_stage);
  fold_pending(ctx);
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  if (ctx->blas) cublasDestroy(ctx->blas);
  if (ctx->solver) cusolverDnDestroy(ctx->solver);
  delete ctx;
}

int fsr_ctx_set_stream(fsr_ctx* ctx, void* stream) {
  if (!ctx) return FSR_EINVAL;
  ctx->stream = (cudaStream_t)stream;
  FSR_BLAS(ctx, cublasSetStream(ctx->blas, ctx->stream));
  FSR_SOLVER(ctx, cusolverDnSetStream(ctx->solver, ctx->stream));
  return FSR_OK;
}

const char* fsr_last_error(const fsr_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

uint64_t fsr_launch_count(const fsr_ctx* ctx) { return ctx ? ctx->launches : 0; }

uint64_t fsr_library_calls(const fsr_ctx* ctx) { return ctx ? ctx->library_calls : 0; }

}  // extern "C"

static void fold_pending(fsr_ctx* ctx) {
  for (auto& p : ctx->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, p.start, p.stop) == cudaSuccess) {
      ctx->stage_ms[p.stage] += ms;
      ctx->stage_count[p.stage] += 1;
    }
    ctx->event_pool.push_back(p.start);
    ctx->event_pool.push_back(p.stop);
  }
  ctx->pending.clear();
  cudaGetLastError();
}

extern "C" {

int fsr_ctx_set_option(fsr_ctx* ctx, int option, int64_t value) {
  if (!ctx) return FSR_EINVAL;
  switch (option) {
    case FSR_OPT_DENSE_PATH:
      if (value < 0 || value > 1) return fsr::set_error(ctx, FSR_EINVAL, "dense path must be 0 or 1");
      ctx->dense_path = (int)value;
      return FSR_OK;
    case FSR_OPT_SPMM_PANEL_BYTES:
      if (value != 0 && value != 32 && value != 64 && value != 128)
        return fsr::set_error(ctx, FSR_EINVAL, "spmm panel must be 0, 32, 64 or 128 bytes");
      ctx->spmm_panel_bytes = (int)value;
      return FSR_OK;
    case FSR_OPT_TOPK_PRUNE:
      if (value < 0 || value > 1) return fsr::set_error(ctx, FSR_EINVAL, "topk prune must be 0 or 1");
      ctx->topk_prune = (int)value;
      return FSR_OK;
    case FSR_OPT_TOPK_SEGMENTS:
      if (value < 0 || value > 4096) return fsr::set_error(ctx, FSR_EINVAL, "topk segments must lie in [0, 4096]");
      ctx->topk_segments = (int)value;
      return FSR_OK;
    default:
      return fsr::set_error(ctx, FSR_EINVAL, "unknown option %d", option);
  }
}

int fsr_ctx_enable_timing(fsr_ctx* ctx, int on) {
  if (!ctx) return FSR_EINVAL;
  ctx->timing = on != 0;
  return FSR_OK;
}

int fsr_stage_time(fsr_ctx* ctx, int stage, double* ms, uint64_t* count) {
  if (!ctx || stage < 0 || stage >= FSR_NUM_STAGES) return FSR_EINVAL;
  FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  fold_pending(ctx);
  if (ms) *ms = ctx->stage_ms[stage];
  if (count) *count = ctx->stage_count[stage];
  return FSR_OK;
}

int fsr_stage_reset(fsr_ctx* ctx) {
  if (!ctx) return FSR_EINVAL;
  FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  fold_pending(ctx);
  for (int i = 0; i < FSR_NUM_STAGES; ++i) {
    ctx->stage_ms[i] = 0.0;
    ctx->stage_count[i] = 0;
  }
  return FSR_OK;
}

int fsr_synchronize(fsr_ctx* ctx) {
  if (!ctx) return FSR_EINVAL;
  FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FSR_OK;
}

}  // extern "C"
