// C ABI of K2 (see spmm.cuh for the kernel).
#include "spmm.cuh"

extern "C" int fsr_csr_spmm(fsr_ctx* ctx, int dtype, int64_t n_rows, const int64_t* indptr,
                            const int32_t* indices, const void* values, int64_t ncols, const void* X,
                            int64_t ldx, void* Y, int64_t ldy) {
  FSR_REQUIRE(ctx, n_rows >= 0 && ncols >= 0 && ldx >= ncols && ldy >= ncols, "csr_spmm: bad shape");
  fsr::StageTimer timer(ctx, FSR_STAGE_SPMM);
  if (dtype == FSR_F64)
    return fsr::launch_spmm<double>(ctx, n_rows, indptr, indices, (const double*)values, ncols,
                                    (const double*)X, ldx, (double*)Y, ldy);
  return fsr::launch_spmm<float>(ctx, n_rows, indptr, indices, (const float*)values, ncols, (const float*)X,
                                 ldx, (float*)Y, ldy);
}
