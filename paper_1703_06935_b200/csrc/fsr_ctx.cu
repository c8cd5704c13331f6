// Context lifecycle, error reporting and launch accounting for libfsr.
#include "fsr_common.cuh"

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
  *out = ctx;
  return FSR_OK;
}

void fsr_ctx_destroy(fsr_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  else cudaDeviceSynchronize();
  if (ctx->scratch) cudaFree(ctx->scratch);
  if (ctx->dev_info) cudaFree(ctx->dev_info);
  if (ctx->host_stage) cudaFreeHost(ctx->host_stage);
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

int fsr_synchronize(fsr_ctx* ctx) {
  if (!ctx) return FSR_EINVAL;
  FSR_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return FSR_OK;
}

}  // extern "C"
